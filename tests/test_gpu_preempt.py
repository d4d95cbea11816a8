"""KV-pressure preemption with recompute (
reading Z26) on the GPU against the oracle `sched.kv_step_loop`, through the
C ABI (RP_PREEMPT):

* the per-step live lists (survivors, then the re-admitted responses), the
  acceptance count and t_end are bit-exact for LONG and SHORT rounds, with
  CUDA graphs and eagerly, and under DP (a single-GPU local group of 2);
* the number of preempted prompts equals the oracle's;
* every response of a LONG round is retained with its trace length, and the
  tokens of the preempted-and-recomputed responses are the oracle's Gumbel
  argmax teacher-forced on the GPU's history (gap rule) -- the recomputed KV
  is the KV the response would have had;
* a pool too small for the last live prompt fails with RP_ENOMEM_KV.
"""
import numpy as np
import pytest

from oracle import decoder, sampler, sched, weights
from synth import configs, gen

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def tiny():
    return configs.model_config("tiny")


def page_bytes(cfg):
    return cfg["n_layers"] * cfg["n_kv_heads"] * 2 * 64 * cfg["head_dim"] * 2


def tight_pool(L, plen, cap, target, kind, world=1, want=2):
    """The largest pool (pages per rank) below the no-pressure size at which the
    oracle preempts at least `want` prompts without exhausting."""
    free = sched.kv_step_loop(L, plen, cap, target, kind, 10 ** 6, world=world)
    base = max(sum(sched._pages(p) for p in plen[lo:hi]) + L.shape[1] * (hi - lo) for lo, hi in
               sched.partition(len(plen), world))
    for pool in range(base + 60, base, -1):
        try:
            r = sched.kv_step_loop(L, plen, cap, target, kind, pool, world=world, with_steps=True)
        except sched.KVExhausted:
            continue
        if min(r.preemptions) >= want and r.t_end > free.t_end:
            return pool, r
    pytest.skip("no pool size preempts this trace")


def engine(cfg, pool, graph_steps, **kw):
    from paper_2509_21009_b200 import rp
    return rp.Engine(cfg, max_seqs=64, max_prompts=16, max_prompt_len=128, max_prompt_tokens=1024, max_cap=512,
                     kv_pool_bytes=pool * page_bytes(cfg), graph_steps=graph_steps,
                     sample_seed=configs.SAMPLE_SEED, **kw)


def check_trace(got, ref_steps, rank=0):
    """The device's per-step trace (steps with live rows on this rank) against
    the oracle's steps: slots decoded, accepted count, done."""
    k = 0
    for st in ref_steps:
        live = st["live"][rank]
        if not len(live):
            continue
        a = got[k]
        assert a["t"] == st["t"], (a["t"], st["t"])
        assert np.array_equal(a["live"], live), (st["t"], a["live"], live)
        assert a["accepted"] == st["accepted"] and a["done"] == st["done"], st["t"]
        k += 1
    assert k == len(got)


def _trace(n, G, seed, lo=60, hi=260):
    rng = np.random.default_rng(seed)
    return rng.integers(lo, hi, size=(n, G)).astype(np.int64)


@pytest.mark.parametrize("graph_steps", [0, 4])
def test_long_round_preemption_bit_exact(tiny, graph_steps):
    n, G, cap = 6, 3, 400
    ps = gen.prompts(n, 0, tiny["eos_id"], (5, 80), 31)
    plen = np.array([len(p["tokens"]) for p in ps])
    L = _trace(n, G, 5)
    pool, ref = tight_pool(L, plen, cap, n, sched.LONG)
    eng = engine(tiny, pool, graph_steps)
    eng.debug_trace_enable(ref.t_end + 8)
    eng.submit(ps, G, cap, n, long_round=True, trace=L, round_id=7, preempt=True)
    st = eng.run()
    got = eng.debug_trace(ref.t_end + 8)
    res = eng.collect()
    eng.close()
    assert st.t == ref.t_end and st.preemptions == ref.preemptions[0] > 0
    check_trace(got, ref.steps)
    assert len(res) == n * G
    for r in res:
        assert r["len"] == L[r["prompt_id"], r["j"]]
    # tokens of every response vs the oracle (gap rule): the preempted ones were recomputed
    w = weights.Weights(tiny, configs.WEIGHT_SEED)
    checked = mism = 0
    for r in res:
        p = ps[r["prompt_id"]]["tokens"]
        seq = np.concatenate([p, r["tokens"]])
        lg = decoder.logits(w, seq[:-1], rows=np.arange(len(p) - 1, len(seq) - 1))
        for t in range(1, r["len"] + 1):
            tok, gap = sampler.sample(lg[t - 1], t, r["prompt_id"] * G + r["j"], 7, configs.SAMPLE_SEED,
                                      eos_id=tiny["eos_id"], trace_len=L[r["prompt_id"], r["j"]])
            checked += 1
            if tok != r["tokens"][t - 1]:
                assert gap <= 1e-2, (r["prompt_id"], r["j"], t, gap)
                mism += 1
    assert checked > 1000 and mism <= checked // 50


def test_short_round_preemption_bit_exact(tiny):
    n, G, cap, target = 8, 3, 250, 6
    ps = gen.prompts(n, 0, tiny["eos_id"], (5, 100), 41)
    plen = np.array([len(p["tokens"]) for p in ps])
    L = _trace(n, G, 9, 40, 300)
    pool, ref = tight_pool(L, plen, cap, target, sched.SHORT, want=1)
    eng = engine(tiny, pool, 4)
    eng.debug_trace_enable(ref.t_end + 8)
    eng.submit(ps, G, cap, target, trace=L, round_id=3, preempt=True)
    st = eng.run()
    got = eng.debug_trace(ref.t_end + 8)
    res = eng.collect()
    q = eng.long_queue()
    eng.close()
    assert st.t == ref.t_end and st.accepted == len(ref.accepted) and st.preemptions == ref.preemptions[0]
    check_trace(got, ref.steps)
    assert list(dict.fromkeys(r["prompt_id"] for r in res)) == ref.accepted
    assert q == ref.deferred


def test_preemption_dp_local_group(tiny):
    """DP = 2 in a single-GPU local group: rank-local pools, global cutoff and
    a global pause whenever some rank re-admits."""
    import threading
    from paper_2509_21009_b200 import rp
    n, G, cap = 8, 3, 400
    ps = gen.prompts(n, 0, tiny["eos_id"], (5, 80), 51)
    plen = np.array([len(p["tokens"]) for p in ps])
    L = _trace(n, G, 13)
    pool, ref = tight_pool(L, plen, cap, n, sched.LONG, world=2, want=1)
    g = rp.LocalGroup(2, 1)
    out, errs = [None, None], []
    bar = threading.Barrier(2)

    def th(r):
        import torch
        torch.cuda.set_device(0)
        e = None
        try:
            e = engine(tiny, pool, 4, rank=r, world=2, local_group=g)
            e.debug_trace_enable(ref.t_end + 8)
            bar.wait(300)
            e.submit(ps, G, cap, n, long_round=True, trace=L, round_id=2, preempt=True)
            st = e.run()
            out[r] = (st.t, st.preemptions, e.debug_trace(ref.t_end + 8), e.collect())
            bar.wait(300)
        except BaseException as ex:
            errs.append(repr(ex))
            bar.abort()
        finally:
            if e is not None:
                e.close()

    ts = [threading.Thread(target=th, args=(r,), daemon=True) for r in range(2)]
    for t in ts:
        t.start()
    for t in ts:
        t.join(600)
    g.close()
    assert not errs, errs
    for r in range(2):
        t_end, pre, got, res = out[r]
        assert t_end == ref.t_end and pre == ref.preemptions[r]
        check_trace(got, ref.steps, rank=r)
        lo, hi = sched.partition(n, 2)[r]
        assert sorted((x["prompt_id"], x["j"]) for x in res) == [(i, j) for i in range(lo, hi) for j in range(G)]


def test_exhaustion_is_an_error(tiny):
    from paper_2509_21009_b200 import rp
    ps = gen.prompts(2, 0, tiny["eos_id"], (64, 64), 5)
    L = np.array([[130], [130]])
    # the hand-worked oracle case: 5 pages finish (t_end 195), 4 pages cannot
    ref = sched.kv_step_loop(L, [64, 64], 1000, 2, sched.LONG, 5, with_steps=True)
    eng = engine(tiny, 5, 4)
    eng.debug_trace_enable(210)
    eng.submit(ps, 1, 300, 2, long_round=True, trace=L, round_id=1, preempt=True)
    st = eng.run()
    assert st.t == ref.t_end == 195 and st.preemptions == 1
    check_trace(eng.debug_trace(210), ref.steps)
    eng.collect()
    eng.close()
    eng = engine(tiny, 4, 4)
    eng.submit(ps, 1, 300, 2, long_round=True, trace=L, round_id=1, preempt=True)
    with pytest.raises(rp.RPError) as e:
        eng.run()
    assert e.value.code == rp.RP_ENOMEM_KV
    eng.close()
