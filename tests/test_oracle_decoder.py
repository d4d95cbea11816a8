"""Pins of oracle/decoder.py: closed forms of each piece (SURVEY.md §8(c)
"What pins each part") and a library cross-check of the whole decoder
against transformers' Qwen2 on the tiny config."""
import numpy as np
import pytest

from oracle import decoder as D
from oracle.weights import Weights
from synth.configs import model_config


def test_softmax_closed_form():
    p = D.softmax(np.log(np.array([1.0, 2.0, 3.0])))
    assert np.allclose(p, [1 / 6, 1 / 3, 1 / 2], atol=1e-15)


def test_attention_single_position_returns_v():
    rng = np.random.default_rng(0)
    q = rng.normal(size=(2, 1, 8)); k = rng.normal(size=(1, 1, 8)); v = rng.normal(size=(1, 1, 8))
    out = D.attention(q, k, v)
    assert np.allclose(out[0, 0], v[0, 0]) and np.allclose(out[1, 0], v[0, 0])


def test_attention_equal_scores_mean_and_dominant():
    v = np.arange(12, dtype=np.float64).reshape(1, 3, 4)
    q = np.zeros((1, 1, 4)); k = np.ones((1, 3, 4))
    out = D.attention(q, k, v)                           # equal scores -> mean of v
    assert np.allclose(out[0, 0], v[0].mean(axis=0))
    k2 = np.zeros((1, 3, 4)); k2[0, 1] = 1e4
    q2 = np.ones((1, 1, 4))
    assert np.allclose(D.attention(q2, k2, v)[0, 0], v[0, 1])


def test_attention_causal_mask():
    rng = np.random.default_rng(1)
    q = rng.normal(size=(1, 3, 4)); k = rng.normal(size=(1, 3, 4)); v = rng.normal(size=(1, 3, 4))
    out = D.attention(q, k, v)
    assert np.allclose(out[0, 0], v[0, 0])               # first query sees only key 0


def test_rmsnorm_constant_vector():
    c, eps = 3.0, 1e-6
    out = D.rmsnorm(np.full((1, 16), c), np.full(16, 2.0), eps)
    assert np.allclose(out, 2.0 * c / np.sqrt(c * c + eps))


def test_rope_identity_norm_relative():
    rng = np.random.default_rng(2)
    x = rng.normal(size=(1, 1, 64))
    assert np.allclose(D.rope(x, [0], 1e6), x)
    y = D.rope(x, [12345], 1e6)
    assert np.isclose(np.linalg.norm(y), np.linalg.norm(x))
    q = rng.normal(size=(1, 1, 64)); k = rng.normal(size=(1, 1, 64))
    d1 = (D.rope(q, [7], 1e4) * D.rope(k, [3], 1e4)).sum()
    d2 = (D.rope(q, [104], 1e4) * D.rope(k, [100], 1e4)).sum()
    assert np.isclose(d1, d2)


def test_silu():
    assert D.silu(np.array(0.0)) == 0.0
    assert np.isclose(D.silu(np.array(1.0)), 1 / (1 + np.exp(-1)))


def test_kv_decoder_equals_full_forward():
    cfg = model_config("tiny")
    w = Weights(cfg, 0)
    toks = np.array([5, 17, 99, 3, 1000, 4000, 7])
    full = D.logits(w, toks)
    dec = D.KVDecoder(w)
    a = dec.step(toks[:4])
    b = [dec.step(toks[i:i + 1]) for i in range(4, 7)]
    inc = np.concatenate([a] + b)
    assert np.allclose(inc, full, atol=1e-10)


def test_kv_decoder_fork_and_hidden():
    """fork(): siblings continuing one prompt prefix equal full forwards of
    their own sequences; head=False returns the final-norm hidden rows."""
    cfg = model_config("tiny")
    w = Weights(cfg, 0)
    prompt = np.array([5, 17, 99, 3, 1000])
    dec = D.KVDecoder(w)
    dec.step(prompt, head=False)
    for cont in ([7, 8, 9], [4000, 1]):
        h = dec.fork().step(cont, head=False)
        full = D.hidden(w, np.concatenate([prompt, cont]))
        assert np.allclose(h, full[len(prompt):], atol=1e-12)
    assert dec.n == len(prompt)


# tiny (g=2, hd=64), the 14B attention shape at tiny width (g=5, hd=128) and
# ONE full-width Qwen2.5-7B layer (d=3584, g=7, hd=128, d_ff=18944; vocab cut
# to 4096 to keep the LM head small -- it does not touch the layer arithmetic)
XCHECK = [("tiny", {}), ("tiny-kv8", {}), ("qwen2.5-7b", dict(n_layers=1, vocab=4096, eos_id=4095))]


@pytest.mark.parametrize("name,over", XCHECK, ids=[x[0] for x in XCHECK])
def test_cross_check_transformers_qwen2(name, over):
    """Library cross-check (the whole decoder): the oracle's logits equal
    transformers' Qwen2ForCausalLM in float64 with the same weights."""
    torch = pytest.importorskip("torch")
    tr = pytest.importorskip("transformers")
    cfg = dict(model_config(name), **over)
    w = Weights(cfg, 0, use_c=cfg["d_model"] > 1024)
    hc = tr.Qwen2Config(vocab_size=cfg["vocab"], hidden_size=cfg["d_model"],
                        intermediate_size=cfg["d_ff"], num_hidden_layers=cfg["n_layers"],
                        num_attention_heads=cfg["n_heads"], num_key_value_heads=cfg["n_kv_heads"],
                        head_dim=cfg["head_dim"], rope_theta=cfg["rope_theta"], rms_norm_eps=cfg["rms_eps"],
                        tie_word_embeddings=False, max_position_embeddings=4096, use_sliding_window=False)
    hc._attn_implementation = "eager"
    m = tr.Qwen2ForCausalLM(hc).to(torch.float64).eval()
    from oracle.weights import tensor, tensor_c, TID_EMBED
    T = lambda a: torch.from_numpy(np.asarray(a, np.float64))
    gen_t = tensor_c if w.use_c else tensor
    with torch.no_grad():
        m.model.embed_tokens.weight.copy_(T(gen_t(0, TID_EMBED, (cfg["vocab"], cfg["d_model"]))))
        m.lm_head.weight.copy_(T(w.lm_head()))
        for l, layer in enumerate(m.model.layers):
            lw = w.layer(l)
            a = layer.self_attn
            a.q_proj.weight.copy_(T(lw["q"])); a.q_proj.bias.copy_(T(lw["bq"]))
            a.k_proj.weight.copy_(T(lw["k"])); a.k_proj.bias.copy_(T(lw["bk"]))
            a.v_proj.weight.copy_(T(lw["v"])); a.v_proj.bias.copy_(T(lw["bv"]))
            a.o_proj.weight.copy_(T(lw["o"]))
            layer.mlp.gate_proj.weight.copy_(T(lw["gate"]))
            layer.mlp.up_proj.weight.copy_(T(lw["up"]))
            layer.mlp.down_proj.weight.copy_(T(lw["down"]))
    toks = np.array([1, 2, 3, 400, 4000, 17, 9, 9, 9, 2048])
    with torch.no_grad():
        ref = m(torch.from_numpy(toks)[None]).logits[0].numpy()
    ours = D.logits(w, toks)
    # transformers runs RMSNorm and the RoPE frequencies in fp32 even for a
    # float64 model, so agreement is ~1e-7; a dropped term, wrong sign or
    # transposed operand moves logits by >= 1e-3.
    assert np.max(np.abs(ours - ref)) < 1e-5
