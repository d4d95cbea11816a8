"""Full-size parity (BASELINE.json configs[1], Qwen2.5-7B-shaped) in the launch
configuration bench.py times: 32 prompts x G=8 = 256 sequences per GPU,
prompt lengths 256-768, cap 8192, CUDA graphs of 16 decode steps.

* the first short round of the bench workload reproduces the oracle schedule
  bit-exactly at every step (live lists, acceptance, done), the accepted set
  and its order, the retained lengths and the FIFO -- properties that hold at
  any size, checked here at the full one;
* teacher-forced logits of the full-width 28-layer decoder -- prefill of a
  short prompt and a graphed decode step at 16 live rows -- agree with the
  fp64 oracle within the north-star max-abs 2e-2, and the sampled tokens
  follow the gap rule (the oracle streams its weights layer by layer).
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
    """All 28 layers at full width, against the fp64 oracle streamed layer by
    layer (one weight generation for every check):
    * prefill logits of an 8-token prompt (rp_debug_logits);
    * decode-step logits of the bench engine's timed path (CUDA graph of 16
      steps, split-K / cooperative GEMMs with the fused RoPE epilogue, the
      folded norm over 28 partials, decode attention) for 2 responses at step
      17 of a 16-row round, teacher-forced on the GPU's own tokens (6 rows);
    * the sampled tokens of steps 1-17 of those responses (gap rule)."""
    from oracle import decoder, sampler, weights
    from synth import configs, gen
    W, eng = bench_engine
    cfg = W.model
    toks = gen.prompts(1, 0, cfg["eos_id"], (8, 8), 5)[0]["tokens"]
    got = eng.debug_logits(toks)                               # [8, V] fp32 from the GPU path
    # a 16-row long round: 2 prompts x G = 8, trace length 20
    ps = gen.prompts(2, 0, cfg["eos_id"], (40, 56), 6, first_id=500)
    L = np.full((2, 8), 20, np.int32)
    eng.debug_trace_enable(64)
    eng.submit(ps, 8, 32, 2, long_round=True, trace=L, round_id=9)
    st = eng.step(1)                                           # one graph: steps 2..17
    lg, slots = eng.debug_last_logits()
    assert st.t == 17 and len(slots) == 16
    eng.run()
    res = {(r["prompt_id"], r["j"]): r["tokens"] for r in eng.collect()}
    pick = [(0, 2), (0, 5), (0, 7), (1, 0), (1, 3), (1, 7)]    # (prompt, j)
    seqs = [np.asarray(toks)] + [np.concatenate([ps[p]["tokens"], res[(ps[p]["prompt_id"], j)][:16]])
                                 for p, j in pick]
    weights.build_c()
    w = weights.Weights(cfg, configs.WEIGHT_SEED, use_c=True)
    xs = [np.asarray(w.embed_rows(s), np.float64) for s in seqs]
    for layer in range(cfg["n_layers"]):                       # stream the layers: ~1 GB of host memory each
        lw = w.layer(layer)
        xs = [decoder.layer_forward(x, lw, cfg, np.arange(len(x))) for x in xs]
        w.drop_layer(layer)
    hs = [decoder.rmsnorm(x, w.final_norm(), cfg["rms_eps"]) for x in xs]
    # rows: the 8 prompt rows; per picked response the rows of tokens 1..17
    rows = [hs[0]] + [h[len(ps[p]["tokens"]) - 1:] for h, (p, j) in zip(hs[1:], pick)]
    H = np.concatenate(rows)
    lm = w.lm_head()
    ref = np.empty((H.shape[0], cfg["vocab"]))
    for v0 in range(0, cfg["vocab"], 16384):                   # fp64 LM head in vocab chunks
        ref[:, v0:v0 + 16384] = H @ np.asarray(lm[v0:v0 + 16384], np.float64).T
    worst = float(np.max(np.abs(got - ref[:8])))
    print("7b teacher-forced prefill logits max-abs vs fp64 oracle: %.4g" % worst)
    assert worst <= 2e-2, worst
    o, dworst, mism = 8, 0.0, 0
    for p, j in pick:
        r17 = ref[o + 16]                                      # logits of token 17
        row = list(slots).index(p * 8 + j)
        dworst = max(dworst, float(np.max(np.abs(lg[row] - r17))))
        pid = ps[p]["prompt_id"]
        for t in range(1, 18):
            tok, gap = sampler.sample(ref[o + t - 1], t, pid * 8 + j, 9, configs.SAMPLE_SEED,
                                      eos_id=cfg["eos_id"], trace_len=20)
            if tok != res[(pid, j)][t - 1]:
                assert gap <= 1e-2, (p, j, t, gap)
                mism += 1
        o += 17
    print("7b decode-step (graph, step 17, 16 rows) logits max-abs vs fp64 oracle: %.4g over %d rows; %d in-gap "
          "token mismatches of %d" % (dworst, len(pick), mism, 17 * len(pick)))
    assert dworst <= 2e-2, dworst
    assert mism <= 2
