"""Migration of an in-flight round by recompute (PAPER P:921-925,
P:965-972; reading Z27), through the C ABI (rp_round_export / rp_round_import):

* a round stepped to some step t on one engine, exported, and imported into a
  fresh engine (on the same GPU, or on a second GPU) continues with the
  oracle's schedule: the per-step live lists, acceptance counts and done flags
  of every step after t and t_end are bit-exact (sched.closed_form), SHORT and
  LONG rounds, CUDA graphs and eager;
* the collected responses are the oracle's (accepted prompts in order,
  lengths = the trace) and every token -- sampled before the migration on the
  first engine or after it on the second, whose KV was recomputed -- equals
  the oracle's Gumbel argmax teacher-forced on the GPU's history (gap rule);
* unsupported or mismatched imports fail with RP_EINVAL, exports without an
  active round with RP_ESTATE.
"""
import numpy as np
import pytest

from oracle import decoder, sampler, sched, weights
from synth import configs, gen

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def tiny():
    return configs.model_config("tiny")


def engine(cfg, graph_steps, **kw):
    from paper_2509_21009_b200 import rp
    return rp.Engine(cfg, max_seqs=64, max_prompts=16, max_prompt_len=128, max_prompt_tokens=1024, max_cap=512,
                     kv_pool_bytes=64 << 20, graph_steps=graph_steps, sample_seed=configs.SAMPLE_SEED, **kw)


def _trace(n, G, seed, lo=20, hi=300):
    return np.random.default_rng(seed).integers(lo, hi, size=(n, G)).astype(np.int64)


def _check_tokens(cfg, res, ps, L, G, round_id):
    w = weights.Weights(cfg, configs.WEIGHT_SEED)
    checked = mism = 0
    for r in res:
        p = ps[r["prompt_id"] - ps[0]["prompt_id"]]["tokens"]
        seq = np.concatenate([p, r["tokens"]])
        lg = decoder.logits(w, seq[:-1], rows=np.arange(len(p) - 1, len(seq) - 1))
        i = r["prompt_id"] - ps[0]["prompt_id"]
        for t in range(1, r["len"] + 1):
            tok, gap = sampler.sample(lg[t - 1], t, r["prompt_id"] * G + r["j"], round_id, configs.SAMPLE_SEED,
                                      eos_id=cfg["eos_id"], trace_len=L[i, r["j"]])
            checked += 1
            if tok != r["tokens"][t - 1]:
                assert gap <= 1e-2, (r["prompt_id"], r["j"], t, gap)
                mism += 1
    return checked, mism


def _migrate(cfg, kind, graph_steps, t_cut, dev_b=0, n=8, G=3, seed=21):
    import torch
    ps = gen.prompts(n, 0, cfg["eos_id"], (5, 100), 61 + seed)
    L = _trace(n, G, seed)
    long_round = kind == "long"
    cap, target = (400, n) if long_round else (250, 6)
    ref = sched.closed_form(L, cap, target, sched.LONG if long_round else sched.SHORT, with_steps=True)
    assert ref.t_end > t_cut + 10
    round_id = 9
    torch.cuda.set_device(0)
    a = engine(cfg, graph_steps)
    a.submit(ps, G, cap, target, long_round=long_round, trace=L, round_id=round_id)
    st = a.step(t_cut - 1)
    t_exp = st.t                       # graphs step in whole graphs: the actual cut
    state = a.export_round()
    a.close()
    torch.cuda.set_device(dev_b)
    b = engine(cfg, graph_steps)
    b.debug_trace_enable(ref.t_end + 8)
    b.import_round(state, ps, G, cap, target, long_round=long_round, trace=L, round_id=round_id)
    st2 = b.run()
    got = b.debug_trace(ref.t_end + 8, start=t_exp + 1)
    res = b.collect()
    b.close()
    torch.cuda.set_device(0)
    assert st2.t == ref.t_end and st2.accepted == len(ref.accepted)
    assert len(got) == ref.t_end - t_exp
    for g in got:
        want = ref.steps[g["t"] - 1]
        assert np.array_equal(g["live"], want["live"]), g["t"]
        assert g["accepted"] == want["accepted"] and g["done"] == want["done"], g["t"]
    assert list(dict.fromkeys(r["prompt_id"] for r in res)) == [ps[i]["prompt_id"] for i in ref.accepted]
    for r in res:
        i = r["prompt_id"] - ps[0]["prompt_id"]
        assert r["len"] == min(L[i, r["j"]], cap)
    checked, mism = _check_tokens(cfg, res, ps, L, G, round_id)
    assert checked > 500 and mism <= checked // 50
    return t_exp


@pytest.mark.parametrize("kind,graph_steps,t_cut", [("short", 4, 37), ("short", 0, 90), ("long", 0, 61),
                                                    ("long", 4, 150)])
def test_migrate_round_bit_exact(tiny, kind, graph_steps, t_cut):
    _migrate(tiny, kind, graph_steps, t_cut)


def test_migrate_round_to_second_gpu(tiny):
    import torch
    if torch.cuda.device_count() < 2:
        pytest.skip("needs 2 GPUs")
    _migrate(tiny, "long", 4, 101, dev_b=1)


def test_migrate_errors(tiny):
    from paper_2509_21009_b200 import rp
    ps = gen.prompts(3, 0, tiny["eos_id"], (5, 40), 3)
    L = _trace(3, 2, 4)
    a = engine(tiny, 0)
    with pytest.raises(rp.RPError) as e:
        a.export_round()                               # no active round
    assert e.value.code == rp.RP_ESTATE
    a.submit(ps, 2, 300, 3, long_round=True, trace=L, round_id=1)
    a.step(5)
    state = a.export_round()
    a.close()
    b = engine(tiny, 0)
    with pytest.raises(rp.RPError) as e:
        b.import_round(state, ps, 3, 300, 3, long_round=True, trace=np.repeat(L, 2, axis=1)[:, :3], round_id=1)
    assert e.value.code == rp.RP_EINVAL               # G differs from the exported round
    with pytest.raises(rp.RPError) as e:
        b.import_round(state[:-8], ps, 2, 300, 3, long_round=True, trace=L, round_id=1)
    assert e.value.code == rp.RP_EINVAL               # truncated state
    b.import_round(state, ps, 2, 300, 3, long_round=True, trace=L, round_id=1)
    st = b.run()
    assert st.done
    b.collect()
    b.close()


def test_migrate_dp_round_local_group(tiny):
    """DP = 2 in a single-GPU local group: both ranks export their slices at the
    same step and a second local group of two fresh contexts imports them; the
    per-rank live counts of every later step, t_end and the acceptance follow
    the oracle's DP protocol (sched.dp_protocol)."""
    import threading
    from paper_2509_21009_b200 import rp
    n, G, cap, target, rid = 8, 3, 250, 6, 4
    ps = gen.prompts(n, 0, tiny["eos_id"], (5, 100), 71)
    L = _trace(n, G, 33)
    t_end, accepted, live_counts = sched.dp_protocol(L, cap, target, sched.SHORT, 2)
    states, cut, errs = [None, None], [0, 0], []
    out = [None, None]

    def run_group(fn):
        g = rp.LocalGroup(2, 1)
        bar = threading.Barrier(2)

        def th(r):
            import torch
            torch.cuda.set_device(0)
            e = None
            try:
                e = engine(tiny, 4, rank=r, world=2, local_group=g)
                bar.wait(300)
                fn(e, r)
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

    def first(e, r):
        e.submit(ps, G, cap, target, trace=L, round_id=rid)
        st = e.step(40)
        cut[r] = st.t
        states[r] = e.export_round()

    def second(e, r):
        e.debug_trace_enable(t_end + 8)
        e.import_round(states[r], ps, G, cap, target, trace=L, round_id=rid)
        st = e.run()
        out[r] = (st.t, st.accepted, e.debug_trace(t_end + 8, start=cut[r] + 1), e.collect())

    run_group(first)
    assert cut[0] == cut[1] and cut[0] < t_end - 10
    run_group(second)
    res_all = []
    for r in range(2):
        t2, acc, got, res = out[r]
        assert t2 == t_end and acc == len(accepted)
        for x in got:
            assert len(x["live"]) == live_counts[x["t"] - 1][r], (r, x["t"])
        res_all += res
        for x in res:
            i = x["prompt_id"] - ps[0]["prompt_id"]
            assert x["len"] == L[i, x["j"]]
    assert sorted(set(x["prompt_id"] - ps[0]["prompt_id"] for x in res_all)) == sorted(accepted)


@pytest.mark.parametrize("w_from,w_to", [(2, 1), (1, 2)])
def test_migrate_dp_reshard(tiny, w_from, w_to):
    """The rollout GPU set shrinks (DP 2 -> 1) or grows (1 -> 2) mid-round: the
    ranks' exported states are re-sharded (rp_round_reshard) and imported into
    contexts of the new world (single-GPU local groups); the schedule after
    the cut is the oracle's (world-invariant, Z1): per-rank live counts from
    sched.dp_protocol at the new world, t_end, the accepted set, lengths, and
    the tokens vs the oracle's Gumbel argmax (gap rule)."""
    import threading
    from paper_2509_21009_b200 import rp
    n, G, cap, target, rid = 8, 3, 250, 6, 5
    ps = gen.prompts(n, 0, tiny["eos_id"], (5, 100), 81)
    L = _trace(n, G, 44)
    t_end, accepted, live_new = sched.dp_protocol(L, cap, target, sched.SHORT, w_to)
    ref = sched.closed_form(L, cap, target, sched.SHORT, with_steps=True)
    assert ref.t_end == t_end and sorted(ref.accepted) == sorted(accepted)
    errs = []

    def run_group(world, fn):
        g = rp.LocalGroup(world, 1) if world > 1 else None
        bar = threading.Barrier(world)

        def th(r):
            import torch
            torch.cuda.set_device(0)
            e = None
            try:
                kw = dict(rank=r, world=world, local_group=g) if world > 1 else {}
                e = engine(tiny, 4, **kw)
                bar.wait(300)
                fn(e, r)
                bar.wait(300)
            except BaseException as ex:
                errs.append(repr(ex))
                bar.abort()
            finally:
                if e is not None:
                    e.close()

        ts = [threading.Thread(target=th, args=(r,), daemon=True) for r in range(world)]
        for t in ts:
            t.start()
        for t in ts:
            t.join(600)
        if g is not None:
            g.close()
        assert not errs, errs

    states, cut = [None] * w_from, [0] * w_from

    def first(e, r):
        e.submit(ps, G, cap, target, trace=L, round_id=rid)
        cut[r] = e.step(40).t
        states[r] = e.export_round()

    run_group(w_from, first)
    assert len(set(cut)) == 1 and cut[0] < t_end - 10
    new_states = rp.reshard_round_states(states, n, w_to)
    out = [None] * w_to

    def second(e, r):
        e.debug_trace_enable(t_end + 8)
        e.import_round(new_states[r], ps, G, cap, target, trace=L, round_id=rid)
        st = e.run()
        out[r] = (st.t, st.accepted, e.debug_trace(t_end + 8, start=cut[0] + 1), e.collect())

    run_group(w_to, second)
    res_all = []
    for r in range(w_to):
        t2, acc, got, res = out[r]
        assert t2 == t_end and acc == len(accepted)
        assert len(got) == t_end - cut[0]
        for x in got:
            assert len(x["live"]) == live_new[x["t"] - 1][r], (r, x["t"])
            if w_to == 1:
                assert np.array_equal(x["live"], ref.steps[x["t"] - 1]["live"]), x["t"]
        res_all += res
        for x in res:
            i = x["prompt_id"] - ps[0]["prompt_id"]
            assert x["len"] == L[i, x["j"]]
    got_acc = [x["prompt_id"] - ps[0]["prompt_id"] for x in res_all]
    assert sorted(set(got_acc)) == sorted(accepted)
    if w_to == 1:
        assert list(dict.fromkeys(got_acc)) == ref.accepted       # acceptance order restored
    checked, mism = _check_tokens(tiny, res_all, ps, L, G, rid)
    assert checked > 300 and mism <= max(1, checked // 50)


def test_migrate_tp_local_group():
    """A TP=2 long round (the 14B attention shape at tiny width, single-GPU
    local group) exported at step ~40 by both TP ranks and imported into a
    fresh TP=2 group: the recompute runs through the TP prefill (all-reduced
    partials); schedule after the cut, identical tokens on both ranks and the
    tokens vs the oracle (gap rule)."""
    from test_gpu_local import run_group
    cfg = configs.model_config("tiny-kv8")
    n, G, cap, rid = 6, 3, 200, 12
    ps = gen.prompts(n, 0, cfg["eos_id"], (5, 80), 23)
    L = _trace(n, G, 57, 60, 190)
    ref = sched.closed_form(L, cap, n, sched.LONG, with_steps=True)

    def first(eng, r, q, bar):
        eng.submit(ps, G, cap, n, long_round=True, trace=L, round_id=rid)
        st = eng.step(39)
        return dict(t=st.t, state=eng.export_round())

    got1 = run_group(1, 2, cfg, first, sample_seed=configs.SAMPLE_SEED)
    cut = got1[0]["t"]
    assert got1[1]["t"] == cut and cut < ref.t_end - 10
    assert len(got1[0]["state"]) == len(got1[1]["state"])    # (unused tails of the buffers differ by rank)

    def second(eng, r, q, bar):
        eng.debug_trace_enable(ref.t_end + 8)
        eng.import_round(got1[q]["state"], ps, G, cap, n, long_round=True, trace=L, round_id=rid)
        st = eng.run()
        return dict(t=st.t, trace=eng.debug_trace(ref.t_end + 8, start=cut + 1), out=eng.collect())

    got2 = run_group(1, 2, cfg, second, sample_seed=configs.SAMPLE_SEED)
    for x in got2:
        assert x["t"] == ref.t_end and len(x["trace"]) == ref.t_end - cut
        for a in x["trace"]:
            assert np.array_equal(a["live"], ref.steps[a["t"] - 1]["live"]), a["t"]
        assert [(o["prompt_id"], o["j"], o["tokens"].tolist()) for o in x["out"]] == \
            [(o["prompt_id"], o["j"], o["tokens"].tolist()) for o in got2[0]["out"]]
    res = got2[0]["out"]
    assert len(res) == n * G
    checked, mism = _check_tokens(cfg, res, ps, L, G, rid)
    assert checked > 500 and mism <= checked // 50


def test_migrate_with_waiting_preempted_prompts(tiny):
    """KV pressure (RP_PREEMPT, NEXT-2) and migration together: a LONG round on
    a pool too small for its contexts is exported at a step where preempted
    prompts wait for re-admission; the importing engine (same pool size)
    re-admits and recomputes them itself.  Live lists after the cut, t_end and
    the preemption count follow the oracle's kv_step_loop; every response keeps
    its trace length; tokens vs the oracle (gap rule)."""
    import ctypes
    from paper_2509_21009_b200 import rp
    from test_gpu_preempt import tight_pool, page_bytes
    from test_reshard_host import Ctl
    n, G, cap = 6, 3, 400
    ps = gen.prompts(n, 0, tiny["eos_id"], (5, 80), 31)
    plen = np.array([len(p["tokens"]) for p in ps])
    L = np.random.default_rng(5).integers(60, 260, size=(n, G)).astype(np.int64)
    pool, ref = tight_pool(L, plen, cap, n, sched.LONG)
    mk = lambda: rp.Engine(tiny, max_seqs=64, max_prompts=16, max_prompt_len=128, max_prompt_tokens=1024,
                           max_cap=512, kv_pool_bytes=pool * page_bytes(tiny), graph_steps=0,
                           sample_seed=configs.SAMPLE_SEED)
    a = mk()
    a.submit(ps, G, cap, n, long_round=True, trace=L, round_id=7, preempt=True)
    state, cut = None, 0
    while True:
        st = a.step(1)
        assert not st.done, "no step with waiting prompts"
        try:
            s = a.export_round()
        except rp.RPError:
            continue                                   # a re-admission paused this step
        c = Ctl.from_buffer_copy(s[13 * 8:13 * 8 + ctypes.sizeof(Ctl)])
        if c.wait_tail > c.wait_head:
            state, cut = s, st.t
            break
    a.close()
    b = mk()
    b.debug_trace_enable(ref.t_end + 8)
    b.import_round(state, ps, G, cap, n, long_round=True, trace=L, round_id=7, preempt=True)
    st = b.run()
    got = b.debug_trace(ref.t_end + 8, start=cut + 1)
    res = b.collect()
    b.close()
    assert st.t == ref.t_end and st.preemptions == ref.preemptions[0] > 0
    steps = [x for x in ref.steps if x["t"] > cut and len(x["live"][0])]
    assert len(got) == len(steps)
    for g_, w_ in zip(got, steps):
        assert g_["t"] == w_["t"] and np.array_equal(g_["live"], w_["live"][0]), w_["t"]
        assert g_["accepted"] == w_["accepted"] and g_["done"] == w_["done"]
    assert len(res) == n * G
    for r in res:
        assert r["len"] == L[r["prompt_id"] - ps[0]["prompt_id"], r["j"]]
    checked, mism = _check_tokens(tiny, res, ps, L, G, 7)
    assert checked > 1000 and mism <= checked // 50
