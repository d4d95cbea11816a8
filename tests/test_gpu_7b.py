"""Full-size parity (BASELINE.json configs[1], Qwen2.5-7B-shaped) in the launch
configuration bench.py times: 32 prompts x G=8 = 256 sequences per GPU,
prompt lengths 256-768, cap 8192, CUDA graphs of 16 decode steps.

* the first short round of the bench workload reproduces the oracle schedule
  bit-exactly at every step (live lists, acceptance, done), the accepted set
  and its order, the retained lengths and the FIFO -- properties that hold at
  any size, checked here at the full one;
* teacher-forced logits of the full-width 28-layer decoder on a short prompt
  agree with the fp64 oracle within the north-star max-abs 2e-2 (the oracle
  streams its weights layer by layer: ~85 s of host time).
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def bench_engine():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    from paper_2509_21009_b200 import rp
    import bench
    W = bench.Workload("C2-7b", 1)
    lo, hi = W.R["prompt_len"]
    eng = rp.Engine(W.model, max_seqs=W.n_submit * W.G, max_prompts=W.n_submit, max_prompt_len=hi,
                    max_prompt_tokens=W.n_submit * hi, max_cap=max(W.R["short_cap"], W.R["long_cap"]),
                    graph_steps=16, kv_fraction=0.85)
    yield W, eng
    eng.close()


def test_7b_short_round_schedule_bit_exact(bench_engine):
    from oracle import sched
    W, eng = bench_engine
    kind, ids, target, cap, L = W.plan()
    assert kind == "short"
    ref = sched.closed_form(L, cap, target, sched.SHORT, with_steps=True)
    eng.debug_trace_enable(ref.t_end + 32)
    eng.submit([W.prompts[i] for i in ids], W.G, cap, target, trace=L, round_id=0)
    st = eng.run()
    got = eng.debug_trace(ref.t_end + 32)
    assert st.t == ref.t_end and len(got) == ref.t_end
    for a, b in zip(got, ref.steps):
        assert np.array_equal(a["live"], b["live"]), a["t"]
        assert a["accepted"] == b["accepted"] and a["done"] == b["done"], a["t"]
    res = eng.collect()
    eos = W.model["eos_id"]
    acc = list(dict.fromkeys(r["prompt_id"] for r in res))
    assert acc == [ids[i] for i in ref.accepted]
    for r in res:
        i = ids.index(r["prompt_id"])
        assert r["len"] == L[i, r["j"]] == ref.retained_len[i, r["j"]]
        assert r["tokens"][-1] == eos and not np.any(r["tokens"][:-1] == eos)
    assert eng.long_queue() == [ids[i] for i in ref.deferred]


def test_7b_teacher_forced_logits(bench_engine):
    from oracle import decoder, weights
    from synth import configs, gen
    W, eng = bench_engine
    cfg = W.model
    toks = gen.prompts(1, 0, cfg["eos_id"], (8, 8), 5)[0]["tokens"]
    got = eng.debug_logits(toks)                               # [8, V] fp32 from the GPU path
    weights.build_c()
    w = weights.Weights(cfg, configs.WEIGHT_SEED, use_c=True)
    x = np.asarray(w.embed_rows(toks), np.float64)
    pos = np.arange(len(toks))
    for layer in range(cfg["n_layers"]):                       # stream the layers: ~1 GB of host memory each
        x = decoder.layer_forward(x, w.layer(layer), cfg, pos)
        w.drop_layer(layer)
    h = decoder.rmsnorm(x, w.final_norm(), cfg["rms_eps"])
    lm = w.lm_head()
    worst = 0.0
    for v0 in range(0, cfg["vocab"], 16384):                   # fp64 LM head in vocab chunks
        ref = h @ np.asarray(lm[v0:v0 + 16384], np.float64).T
        worst = max(worst, float(np.max(np.abs(got[:, v0:v0 + 16384] - ref))))
    print("7b teacher-forced logits max-abs vs fp64 oracle: %.4g" % worst)
    assert worst <= 2e-2, worst
