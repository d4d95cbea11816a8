"""Multi-rank parity on ONE GPU: a single-GPU local
group runs every rank of a data-parallel (DP), tensor-parallel (TP) or DP x TP
job as a context of this process, one thread per rank, exchanging through
device memory (k_comm.cu) the same messages the NCCL path exchanges:

* DP short rounds (rows a11, a13): the per-step cutoff exchange and the round
  membership.  Per-rank live lists, t_end, the accepted set and every rank's
  (global) long-prompt queue equal the single-rank oracle schedule bit-exactly
  (the C3 protocol of SURVEY §8(e)), with and without
  response-level speculation and continuous issuance; long rounds are planned
  by the library (rp_plan_round) and pop the global queue on every rank.
* TP long rounds (rows a7, a14) at TP = 2, 4, 8 on the 14B attention shape
  (KV = 8, g = 5, hd = 128): teacher-forced logits gathered over the vocab
  shards within 2e-2 of the fp64 oracle, the long-round schedule bit-exact,
  identical tokens on every rank, sampled tokens equal to the oracle's
  Gumbel argmax wherever its top-2 gap exceeds 1e-2.  Decode all-reduces go
  through the peer-push path (GEMM epilogue stores into every rank's receive
  slot + tp_norm), prefill and the argmax through the device collectives.
* DP x TP (BASELINE configs[3]'s "DP=2 x TP=4" short rounds, here 2 x 2 and
  2 x 4): the DP exchange between replicas, TP inside each.
"""
import threading
import traceback

import numpy as np
import pytest

from oracle import decoder, sampler, sched, weights
from synth import configs, gen

pytestmark = pytest.mark.gpu


def run_group(world, tp, cfg, body, timeout=900, **kw):
    """Create world x tp engines of one local group, one thread each, run
    body(engine, rank, tp_rank, barrier) in every thread and return the
    per-context results (index rank * tp + tp_rank).  Assertions belong in the
    caller: a rank that stopped early would leave its peers waiting."""
    import torch
    from paper_2509_21009_b200 import rp
    g = rp.LocalGroup(world, tp)
    n = world * tp
    bar = threading.Barrier(n)
    out, errs = [None] * n, []
    args = dict(max_seqs=64, max_prompts=16, max_prompt_len=128, max_prompt_tokens=1024, max_cap=512,
                kv_pool_bytes=64 << 20, graph_steps=4)
    args.update(kw)

    def th(idx):
        r, q = divmod(idx, tp)
        eng = None
        try:
            torch.cuda.set_device(0)
            eng = rp.Engine(cfg, rank=r, world=world, tp=tp, tp_rank=q, local_group=g, **args)
            eng.debug_trace_enable(700)          # before any collective: it frees / allocates
            bar.wait(timeout)
            out[idx] = body(eng, r, q, bar)
            bar.wait(timeout)
        except BaseException:
            errs.append((idx, traceback.format_exc()))
            bar.abort()
        finally:
            if eng is not None:
                eng.close()

    ths = [threading.Thread(target=th, args=(i,), daemon=True) for i in range(n)]
    for t in ths:
        t.start()
    for t in ths:
        t.join(timeout)
    alive = [t for t in ths if t.is_alive()]
    assert not alive, "local group threads still running"
    g.close()
    assert not errs, errs[0][1]
    return out


def _slice_live(step_live, lo, hi, G):
    """This rank's live list = the global live slots of its prompt range,
    renumbered to local slots."""
    a = np.asarray(step_live)
    return a[(a >= lo * G) & (a < hi * G)] - lo * G


def _check_rank_trace(trace, steps, lo, hi, G):
    """A rank's per-step trace against its slice of the oracle's global
    steps.  The trace ends at the rank's last step with live rows (it keeps
    stepping with none until the round is done everywhere)."""
    exp = [_slice_live(b["live"], lo, hi, G) for b in steps]
    k = sum(1 for e in exp if len(e))
    assert len(trace) == k and all(len(e) == 0 for e in exp[k:]), (len(trace), k)
    for a, e, b in zip(trace, exp, steps):
        assert np.array_equal(a["live"], e), a["t"]
        assert a["accepted"] == b["accepted"] and a["done"] == b["done"], a["t"]


# ------------------------------------------------------------------ DP
@pytest.mark.parametrize("world", [2, 4])
def test_local_dp_rounds(world):
    cfg = configs.model_config("tiny")
    n, G, cap, target = 13, 4, 128, 10
    rounds = []
    for seed in range(4):
        Gs, keep = (G, None) if seed < 3 else (5, 4)
        ps = gen.prompts(n, 0, cfg["eos_id"], (1, 100), 40 + seed, first_id=100 * seed)
        tr = gen.length_trace(n, Gs, 3.4, 0.6, 0.85, 600, seed)
        rounds.append((ps, tr, Gs, keep))

    def body(eng, r, q, bar):
        res = []
        for ps, tr, Gs, keep in rounds:
            eng.submit(ps, Gs, cap, target, trace=tr[:, 0, :], trace_retry=tr[:, 1, :], round_id=len(res),
                       keep=keep or 0)
            st = eng.run()
            trace = eng.debug_trace()
            out = eng.collect()
            res.append(dict(t=st.t, accepted=st.accepted, trace=trace, out=out, queue=eng.long_queue()))
        # the library plans the next round: the queue holds >= P0 = 8 -> LONG,
        # popped from the global queue on every rank
        kind, m = eng.plan(8, 1.25)
        long_res = None
        if kind == "long":
            eng.submit(None, G, 200, m, long_round=True, round_id=77, trace_mode=True)
            st = eng.run()
            long_res = dict(t=st.t, trace=eng.debug_trace(), out=eng.collect(), queue=eng.long_queue())
        return dict(rounds=res, plan=(kind, m), long=long_res)

    got = run_group(world, 1, cfg, body)
    fifo = []
    for k, (ps, tr, Gs, keep) in enumerate(rounds):
        L = tr[:, 0, :]
        ref = sched.closed_form(L, cap, target, sched.SHORT, with_steps=True, keep=keep)
        fifo += [ps[i]["prompt_id"] for i in ref.deferred]
        acc = []
        for r in range(world):
            x = got[r]["rounds"][k]
            lo, hi = sched.partition(n, world)[r]
            assert x["t"] == ref.t_end and x["accepted"] == len(ref.accepted), (r, k)
            # this rank's live list at every step = its slice of the oracle's
            _check_rank_trace(x["trace"], ref.steps, lo, hi, Gs)
            for o in x["out"]:
                i = o["prompt_id"] - ps[0]["prompt_id"]
                assert lo <= i < hi and o["len"] == L[i, o["j"]] == ref.retained_len[i, o["j"]]
            acc += list(dict.fromkeys(o["prompt_id"] for o in x["out"]))
            assert x["queue"] == fifo, (r, k)           # every rank holds the global queue
        assert sorted(acc) == sorted(ps[i]["prompt_id"] for i in ref.accepted)
    # the long round over the head of the global queue, re-rolled (attempt 1)
    assert len(fifo) >= 8
    for r in range(world):
        assert got[r]["plan"] == ("long", 8)
    head = fifo[:8]
    by_id = {p["prompt_id"]: (k, i) for k, (ps, _, _, _) in enumerate(rounds) for i, p in enumerate(ps)}
    L2 = np.array([rounds[by_id[pid][0]][1][by_id[pid][1], 1, :G] for pid in head])
    ref2 = sched.closed_form(L2, 200, 8, sched.LONG, with_steps=True)
    for r in range(world):
        x = got[r]["long"]
        lo, hi = sched.partition(8, world)[r]
        assert x["t"] == ref2.t_end
        _check_rank_trace(x["trace"], ref2.steps, lo, hi, G)
        assert sorted(o["prompt_id"] for o in x["out"]) == sorted(head[i] for i in range(lo, hi) for _ in range(G))
        for o in x["out"]:
            assert o["len"] == min(L2[head.index(o["prompt_id"]), o["j"]], 200)
        assert x["queue"] == fifo[8:]


@pytest.mark.parametrize("world", [2, 3])
def test_local_dp_continuous_issuance(world):
    """NEXT-4 under DP: rank-local issue caps, the global cutoff exchange
    (oracle sched.issue_dp_protocol); never-issued prompts are returned, not
    deferred, and the deferred ones reach every rank's queue."""
    cfg = configs.model_config("tiny")
    n, G, cap = 13, 4, 128
    cases = [(5, 3, 7), (6, 2, 5), (7, 2, 4)]
    data = [(gen.prompts(n, 0, cfg["eos_id"], (2, 100), 40 + s, first_id=1000 * s),
             gen.length_trace(n, G, 3.4, 0.6, 0.85, 300, s)[:, 0, :], A, tg) for s, A, tg in cases]

    def body(eng, r, q, bar):
        res = []
        for ps, L, A, tg in data:
            eng.issue_cap(A)
            eng.submit(ps, G, cap, tg, trace=L, round_id=len(res))
            st = eng.run()
            out = eng.collect()
            res.append(dict(t=st.t, out=out, queue=eng.long_queue(), un=eng.unissued()))
        eng.issue_cap(0)
        return res

    got = run_group(world, 1, cfg, body)
    fifo = []
    for k, (ps, L, A, tg) in enumerate(data):
        t_end, r_acc, r_def, r_un = sched.issue_dp_protocol(L, cap, tg, sched.SHORT, world, A)
        fifo += [ps[i]["prompt_id"] for i in r_def]
        acc = []
        for r in range(world):
            x = got[r][k]
            lo, hi = sched.partition(n, world)[r]
            assert x["t"] == t_end and x["queue"] == fifo, (r, k)
            assert x["un"] == [ps[i]["prompt_id"] for i in r_un if lo <= i < hi]
            for o in x["out"]:
                assert o["len"] == L[o["prompt_id"] - ps[0]["prompt_id"], o["j"]]
            acc += list(dict.fromkeys(o["prompt_id"] for o in x["out"]))
        assert sorted(acc) == sorted(ps[i]["prompt_id"] for i in r_acc)


# ------------------------------------------------------------------ TP
def _check_tokens(cfg, w, res, prompts_by_id, G, L_by_id, round_id, limit=None):
    checked = mism = 0
    bad = []
    for r in res[:limit]:
        p = prompts_by_id[r["prompt_id"]]
        seq = np.concatenate([p, r["tokens"]])
        lg = decoder.logits(w, seq[:-1], rows=np.arange(len(p) - 1, len(seq) - 1))
        for t in range(1, r["len"] + 1):
            tok, gap = sampler.sample(lg[t - 1], t, r["prompt_id"] * G + r["j"], round_id, configs.SAMPLE_SEED,
                                      eos_id=cfg["eos_id"], trace_len=L_by_id[r["prompt_id"]][r["j"]])
            checked += 1
            if tok != r["tokens"][t - 1]:
                mism += 1
                if gap > 1e-2:
                    bad.append((r["prompt_id"], r["j"], t, gap))
    return checked, mism, bad


@pytest.mark.parametrize("tp", [2, 4, 8])
def test_local_tp_long_round(tp):
    cfg = configs.model_config("tiny-kv8")
    w = weights.Weights(cfg, configs.WEIGHT_SEED)
    toks = gen.prompts(1, 0, cfg["eos_id"], (70, 70), 9)[0]["tokens"]
    n, G = 6, 3
    ps = gen.prompts(n, 0, cfg["eos_id"], (5, 80), 21)
    L = np.minimum(gen.length_trace(n, G, 3.4, 0.6, 0.85, 600, 7)[:, 1, :], 150)

    def body(eng, r, q, bar):
        part = eng.debug_logits(toks)
        eng.submit(ps, G, 120, n, long_round=True, trace=L, round_id=11)
        st = eng.run()
        return dict(part=part, t=st.t, trace=eng.debug_trace(), out=eng.collect(), peer=eng.tp_peer)

    got = run_group(1, tp, cfg, body, sample_seed=configs.SAMPLE_SEED)
    assert all(x["peer"] for x in got)
    full = np.concatenate([x["part"] for x in got], axis=1)
    err = float(np.max(np.abs(full - decoder.logits(w, toks))))
    assert err <= 2e-2, err
    ref = sched.closed_form(L, 120, n, sched.LONG, with_steps=True)
    for x in got:
        assert x["t"] == ref.t_end and len(x["trace"]) == ref.t_end
        for a, b in zip(x["trace"], ref.steps):
            assert np.array_equal(a["live"], b["live"]) and a["accepted"] == b["accepted"]
        key = [(o["prompt_id"], o["j"], o["tokens"].tolist()) for o in x["out"]]
        assert key == [(o["prompt_id"], o["j"], o["tokens"].tolist()) for o in got[0]["out"]]
        assert len(x["out"]) == n * G
    checked, mism, bad = _check_tokens(cfg, w, got[0]["out"], {p["prompt_id"]: p["tokens"] for p in ps}, G,
                                       {p["prompt_id"]: L[i] for i, p in enumerate(ps)}, 11)
    assert not bad and checked > 100 and mism <= checked // 50, (checked, mism, bad[:3])


@pytest.mark.parametrize("world,tp", [(2, 2), (2, 4)])
def test_local_dp_x_tp(world, tp):
    """DP x TP: a short round sharded over `world` replicas of `tp` ranks
    (the C4 short-round layout), then the planned long round over the global
    queue; identical tokens inside each replica, schedule bit-exact."""
    cfg = configs.model_config("tiny-kv8")
    w = weights.Weights(cfg, configs.WEIGHT_SEED)
    n, G, cap, target = 10, 3, 96, 7
    ps = gen.prompts(n, 0, cfg["eos_id"], (4, 60), 61)
    tr = gen.length_trace(n, G, 3.4, 0.6, 0.85, 300, 12)
    L = tr[:, 0, :]

    def body(eng, r, q, bar):
        eng.submit(ps, G, cap, target, trace=L, trace_retry=tr[:, 1, :], round_id=5)
        st = eng.run()
        trace = eng.debug_trace()
        out = eng.collect()
        queue = eng.long_queue()
        kind, m = eng.plan(len(queue), 1.25) if queue else ("short", 0)
        long_out = None
        if kind == "long":
            eng.submit(None, G, cap, m, long_round=True, round_id=6, trace_mode=True)
            st2 = eng.run()
            long_out = dict(t=st2.t, out=eng.collect())
        return dict(t=st.t, trace=trace, out=out, queue=queue, long=long_out)

    got = run_group(world, tp, cfg, body, sample_seed=configs.SAMPLE_SEED)
    ref = sched.closed_form(L, cap, target, sched.SHORT, with_steps=True)
    acc = []
    for r in range(world):
        lo, hi = sched.partition(n, world)[r]
        for q in range(tp):
            x = got[r * tp + q]
            assert x["t"] == ref.t_end
            _check_rank_trace(x["trace"], ref.steps, lo, hi, G)
            assert x["queue"] == [ps[i]["prompt_id"] for i in ref.deferred]
            key = [(o["prompt_id"], o["j"], o["tokens"].tolist()) for o in x["out"]]
            assert key == [(o["prompt_id"], o["j"], o["tokens"].tolist()) for o in got[r * tp]["out"]]
        acc += list(dict.fromkeys(o["prompt_id"] for o in got[r * tp]["out"]))
    assert sorted(acc) == sorted(ps[i]["prompt_id"] for i in ref.accepted)
    # the long round re-rolls the deferred prompts (attempt 1) on every replica slice
    dq = [ps[i]["prompt_id"] for i in ref.deferred]
    if dq:
        L2 = tr[ref.deferred, 1, :]
        ref2 = sched.closed_form(L2, cap, len(dq), sched.LONG)
        for x in got:
            assert x["long"]["t"] == ref2.t_end
        outs = [o for r in range(world) for o in got[r * tp]["long"]["out"]]
        assert sorted((o["prompt_id"], o["j"]) for o in outs) == sorted((p, j) for p in dq for j in range(G))
        by_id = {p["prompt_id"]: p["tokens"] for p in ps}
        checked, mism, bad = _check_tokens(cfg, w, outs, by_id, G, {pid: L2[k] for k, pid in enumerate(dq)}, 6,
                                           limit=6)
        assert not bad and mism <= max(1, checked // 50)
    # tokens of the short round vs the oracle (a few responses)
    outs = [o for r in range(world) for o in got[r * tp]["out"]]
    checked, mism, bad = _check_tokens(cfg, w, outs, {p["prompt_id"]: p["tokens"] for p in ps}, G,
                                       {p["prompt_id"]: L[i] for i, p in enumerate(ps)}, 5, limit=6)
    assert not bad and mism <= max(1, checked // 50)
