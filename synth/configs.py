"""Model shapes and round parameters of BASELINE.json configs (shapes, not
arithmetic).  Qwen2.5 shapes follow the public Qwen2 configs (the paper only
says "Qwen2.5 family" -- P:1121).  The tiny decoder's KV heads and d_ff are
not given by BASELINE.json; SURVEY.md §8(d) C1 proposes KV=2, d_ff=1024.
"""

MODELS = {
    "tiny": dict(n_layers=2, d_model=256, n_heads=4, n_kv_heads=2, head_dim=64,
                 d_ff=1024, vocab=4096, eos_id=4095, rope_theta=1e6, rms_eps=1e-6,
                 qkv_bias=1),
    # the 14B attention shape (KV=8, g=5, hd=128) at tiny width: TP=2/4/8
    # parity in one process (single-GPU local groups)
    "tiny-kv8": dict(n_layers=2, d_model=512, n_heads=40, n_kv_heads=8, head_dim=128,
                     d_ff=2048, vocab=4096, eos_id=4095, rope_theta=1e6, rms_eps=1e-6,
                     qkv_bias=1),
    "qwen2.5-7b": dict(n_layers=28, d_model=3584, n_heads=28, n_kv_heads=4, head_dim=128,
                       d_ff=18944, vocab=152064, eos_id=151643, rope_theta=1e6, rms_eps=1e-6,
                       qkv_bias=1),
    "qwen2.5-14b": dict(n_layers=48, d_model=5120, n_heads=40, n_kv_heads=8, head_dim=128,
                        d_ff=13824, vocab=152064, eos_id=151643, rope_theta=1e6, rms_eps=1e-6,
                        qkv_bias=1),
    "qwen2.5-32b": dict(n_layers=64, d_model=5120, n_heads=40, n_kv_heads=8, head_dim=128,
                        d_ff=27648, vocab=152064, eos_id=151643, rope_theta=1e6, rms_eps=1e-6,
                        qkv_bias=1),
}


def model_config(name, n_layers=None):
    c = dict(MODELS[name])
    c["name"] = name
    if n_layers is not None:
        c["n_layers"] = n_layers
    return c


# Round parameters per BASELINE.json config.  n_submit is the
# per-GPU submitted prompt count of a short round, target its accepted count
# (floor(n_submit / eta), reading Z8), G responses per prompt.
ROUNDS = {
    "C1-tiny": dict(model="tiny", n_submit=8, target=6, G=4, short_cap=128, long_cap=512,
                    prompt_len=(8, 32), trace=dict(mu0=3.4, sigma_p=0.6, sigma_r=0.85, l_max=600)),
    "C2-7b": dict(model="qwen2.5-7b", n_submit=32, target=25, G=8, short_cap=8192, long_cap=8192,
                  prompt_len=(256, 768), trace=dict(mu0=6.0, sigma_p=0.6, sigma_r=0.85, l_max=16384)),
}

WEIGHT_SEED = 0
PROMPT_SEED = 1
TRACE_SEED = 2
SAMPLE_SEED = 3
