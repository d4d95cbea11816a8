"""GPU parity of the CUDA path (through the C ABI) against the oracle.

Bars (BASELINE.json north_star): schedules / compaction / membership
bit-exact given a recorded length trace; teacher-forced logits within
max-abs 2e-2; sampled tokens equal to the oracle's Gumbel argmax wherever the
oracle's top-2 perturbed gap exceeds 1e-2."""
import numpy as np
import pytest

from oracle import decoder, sampler, sched, weights
from synth import configs, gen

pytestmark = pytest.mark.gpu

LOGIT_TOL = 2e-2
GAP = 1e-2


@pytest.fixture(scope="module")
def torch():
    import torch as t
    t.cuda.set_device(0)
    return t


@pytest.fixture(scope="module")
def tiny():
    return configs.model_config("tiny")


@pytest.fixture(scope="module")
def oracle_w(tiny):
    return weights.Weights(tiny, configs.WEIGHT_SEED)


def make_engine(cfg, graph_steps=4, max_seqs=64, max_prompts=16, max_prompt_len=128, max_prompt_tokens=1024,
                max_cap=512, kv_pool_bytes=64 << 20, **kw):
    from paper_2509_21009_b200 import rp
    return rp.Engine(cfg, max_seqs=max_seqs, max_prompts=max_prompts, max_prompt_len=max_prompt_len,
                     max_prompt_tokens=max_prompt_tokens, max_cap=max_cap, kv_pool_bytes=kv_pool_bytes,
                     graph_steps=graph_steps, **kw)


# ------------------------------------------------------------------ GEMM
@pytest.mark.parametrize("M,K", [(128, 64), (512, 256), (256, 1024), (4608, 3584), (2048, 256)])
@pytest.mark.parametrize("N", [1, 7, 16, 100, 256, 300, 513])
def test_gemm_tcgen05_vs_fp32(torch, tiny, M, K, N):
    eng = _shared_engine(tiny)
    g = torch.Generator(device="cuda").manual_seed(M * 7 + K * 3 + N)
    W = (torch.randn(M, K, device="cuda", generator=g) * 0.05).to(torch.float16)
    X = (torch.randn(max(N, 1) + 40, K, device="cuda", generator=g)).to(torch.float16)
    ref = X[:N].float() @ W.float().T
    for splits, tiled in ((1, False), (3, False), (1, True), (3, True)):
        Y = eng.debug_gemm(W, X, N, splits=splits, tiled=tiled)
        torch.cuda.synchronize()
        err = (Y - ref).abs().max().item() if N else 0.0
        assert err <= 1e-3 * max(1.0, ref.abs().max().item()), (splits, tiled, err)


@pytest.mark.parametrize("M,K", [(256, 1024), (4608, 3584), (1024, 18944)])
@pytest.mark.parametrize("N", [1, 16, 50, 100, 128, 129, 256, 300])
def test_gemm_split_precision_vs_fp64(torch, tiny, M, K, N):
    """Split-precision activations (reading Z22): with X = X_hi + X_lo (fp16
    values and their fp16 rounding residuals) the GEMM equals W X^T for the
    fp32 X to ~1e-6 of sum |x||w| (fp32 accumulation over K up to 18944) --
    the fp16-only product is >= 5x further off --
    at chunk widths 1..300 (128-column chunks, hi and lo rows in one MMA),
    with and without split-K."""
    eng = _shared_engine(tiny)
    g = torch.Generator(device="cuda").manual_seed(M + K + N)
    W = (torch.randn(M, K, device="cuda", generator=g) * 0.02).to(torch.float16)
    X32 = torch.randn(max(N, 1) + 8, K, device="cuda", generator=g)
    Xh = X32.to(torch.float16)
    Xl = (X32 - Xh.float()).to(torch.float16)
    ref = (X32[:N].double() @ W.double().T)
    scale = (X32[:N].double().abs() @ W.double().abs().T).max().item()
    for splits, tiled in ((1, True), (4, True), (1, False)):
        Y = eng.debug_gemm(W, Xh, N, splits=splits, tiled=tiled, X_lo=Xl).double()
        err = (Y - ref).abs().max().item() / scale
        Y0 = eng.debug_gemm(W, Xh, N, splits=splits, tiled=tiled).double()
        err0 = (Y0 - ref).abs().max().item() / scale
        assert err <= 2e-6 and err < err0 / 5, (splits, tiled, err, err0)


_ENG = {}


def _shared_engine(cfg):
    if "tiny" not in _ENG:
        _ENG["tiny"] = make_engine(cfg)
    return _ENG["tiny"]


# ------------------------------------------------------ teacher-forced logits
@pytest.mark.parametrize("n", [1, 2, 17, 63, 64, 65, 128])
def test_teacher_forced_logits(tiny, oracle_w, n):
    eng = _shared_engine(tiny)
    rng = np.random.default_rng(n)
    toks = rng.integers(0, tiny["eos_id"], size=n).astype(np.int32)
    got = eng.debug_logits(toks)
    want = decoder.logits(oracle_w, toks)
    err = np.max(np.abs(got - want))
    assert err <= LOGIT_TOL, err


# ----------------------------------------------------------- schedules
def _trace(n, G, seed, l_max=600, mu0=3.4):
    return gen.length_trace(n, G, mu0, 0.6, 0.85, l_max, seed)


def _check_round_trace(eng, L, cap, target, kind, keep=None):
    ref = sched.closed_form(L, cap, target, kind, with_steps=True, keep=keep)
    got = eng.debug_trace(ref.t_end + 2)
    assert len(got) == ref.t_end
    for a, b in zip(got, ref.steps):
        assert np.array_equal(a["live"], b["live"]), a["t"]
        assert a["accepted"] == b["accepted"], a["t"]
        assert a["done"] == b["done"], a["t"]
    return ref


@pytest.mark.parametrize("seed", [0, 1, 2])
@pytest.mark.parametrize("graph_steps", [0, 4])
def test_short_round_schedule_bit_exact(tiny, seed, graph_steps):
    eng = make_engine(tiny, graph_steps=graph_steps)
    R = configs.ROUNDS["C1-tiny"]
    n, G = 12, 4
    ps = gen.prompts(n, 0, tiny["eos_id"], (1, 100), 10 + seed)
    L = _trace(n, G, seed)[:, 0, :]
    cap, target = R["short_cap"], 9
    eng.debug_trace_enable(700)
    eng.submit(ps, G, cap, target, trace=L, round_id=seed)
    st = eng.run()
    ref = _check_round_trace(eng, L, cap, target, sched.SHORT)
    assert st.t == ref.t_end and st.accepted == len(ref.accepted) and bool(st.underfilled) == ref.underfilled
    # device histogram of live rows per decode step (bench round_roofline) = the oracle's live counts
    # of steps 2..t_end (step 1 samples from the prefill logits)
    hist = eng.rows_histogram()
    want = np.bincount([len(x["live"]) for x in ref.steps[1:]], minlength=len(hist))
    assert np.array_equal(hist, want[:len(hist)])
    # KV tokens the decode steps' attention read (measurement counters of the roofline): every row's
    # context incl. the appended token, and with each prompt's shared full pages counted once per step
    plen = np.array([len(p["tokens"]) for p in ps])
    sh = (plen // 64) * 64
    per_row = unique = 0
    for x in ref.steps[1:]:
        live = np.asarray(x["live"])
        ctx = plen[live // G] + x["t"] - 1
        per_row += int(ctx.sum())
        unique += int((ctx - sh[live // G]).sum()) + int(sh[np.unique(live // G)].sum())
    assert st.kv_tokens_read == per_row and st.kv_tokens_unique == unique, (st.kv_tokens_read, per_row,
                                                                            st.kv_tokens_unique, unique)
    res = eng.collect()
    acc = list(dict.fromkeys(r["prompt_id"] for r in res))
    assert acc == [ps[i]["prompt_id"] for i in ref.accepted]
    for r in res:
        i = r["prompt_id"] - ps[0]["prompt_id"]
        assert r["len"] == L[i, r["j"]] and r["tokens"][-1] == tiny["eos_id"]
        assert np.all(r["tokens"][:-1] != tiny["eos_id"])
    assert eng.long_queue() == [ps[i]["prompt_id"] for i in ref.deferred]
    # long round over the queue: every response retained, truncated at the cap
    q = eng.long_queue()
    L2 = _trace(n, G, seed)[:, 1, :][[i - ps[0]["prompt_id"] for i in q]]
    eng.debug_trace_enable(700)
    eng.submit([ps[i - ps[0]["prompt_id"]] for i in q], G, 200, len(q), long_round=True, trace=L2, round_id=100 + seed)
    st = eng.run()
    ref2 = _check_round_trace(eng, L2, 200, len(q), sched.LONG)
    res2 = eng.collect()
    assert len(res2) == len(q) * G
    for r in res2:
        k = q.index(r["prompt_id"])
        assert r["len"] == min(L2[k, r["j"]], 200)
    eng.close()


@pytest.mark.parametrize("seed,graph_steps", [(0, 0), (1, 4), (2, 4)])
def test_response_speculation_schedule_bit_exact(tiny, seed, graph_steps):
    """NEXT-1: G = ceil(1.25 R0) = 5 responses
    launched per prompt, the first R0 = 4 to finish kept, siblings aborted at
    once.  Per-step live lists, acceptance, the retained set and the queue
    match the oracle; the long round re-runs R0 responses without
    speculation."""
    eng = make_engine(tiny, graph_steps=graph_steps, max_seqs=80)
    n, G, R0 = 14, 5, 4
    ps = gen.prompts(n, 0, tiny["eos_id"], (1, 100), 50 + seed)
    full = _trace(n, G, 60 + seed)
    L = full[:, 0, :]
    cap, target = 128, 10
    eng.debug_trace_enable(700)
    eng.submit(ps, G, cap, target, trace=L, round_id=seed, keep=R0)
    st = eng.run()
    ref = _check_round_trace(eng, L, cap, target, sched.SHORT, keep=R0)
    assert st.t == ref.t_end and st.accepted == len(ref.accepted) and bool(st.underfilled) == ref.underfilled
    assert st.decoded_tokens == sum(len(x["live"]) for x in ref.steps)
    res = eng.collect()
    assert len(res) == len(ref.accepted) * R0
    got = [(r["prompt_id"] - ps[0]["prompt_id"], r["j"], r["len"]) for r in res]
    want = [(i, j, int(ref.retained_len[i, j])) for i in ref.accepted for j in range(G) if ref.retained_len[i, j]]
    assert got == want
    for r in res:
        assert r["tokens"][-1] == tiny["eos_id"] and r["finish"] == 1
    assert eng.long_queue() == [ps[i]["prompt_id"] for i in ref.deferred]
    q = eng.long_queue()
    if len(q) >= 2:
        L2 = full[:, 1, :R0][[i - ps[0]["prompt_id"] for i in q]]
        eng.debug_trace_enable(700)
        eng.submit([ps[i - ps[0]["prompt_id"]] for i in q], R0, cap, len(q), long_round=True, trace=L2,
                   round_id=100 + seed)
        eng.run()
        _check_round_trace(eng, L2, cap, len(q), sched.LONG)
        assert len(eng.collect()) == len(q) * R0
    eng.close()


def test_response_speculation_ties_and_sampling(tiny, oracle_w):
    """Hand-worked ties (oracle test_speculation_keeps_first_finishers...):
    G=4, keep=2; prompt 0 keeps j=1,3 (both end at 3), prompt 1 keeps j=0
    and j=1 (j=2 ends at the same step 7 and is dropped).  The kept tokens
    are the oracle's Gumbel argmax with uid = prompt_id * G + j."""
    eng = make_engine(tiny, graph_steps=2)
    ps = gen.prompts(2, 0, tiny["eos_id"], (10, 30), 77)
    L = np.array([[5, 3, 9, 3], [2, 7, 7, 20]])
    eng.debug_trace_enable(64)
    eng.submit(ps, 4, 100, 2, trace=L, round_id=4, keep=2)
    st = eng.run()
    _check_round_trace(eng, L, 100, 2, sched.SHORT, keep=2)
    assert st.t == 7
    res = eng.collect()
    assert [(r["prompt_id"] - ps[0]["prompt_id"], r["j"], r["len"]) for r in res] == [
        (0, 1, 3), (0, 3, 3), (1, 0, 2), (1, 1, 7)]
    by_id = {p["prompt_id"]: p["tokens"] for p in ps}
    tr = {p["prompt_id"]: L[i] for i, p in enumerate(ps)}
    checked, mism = _check_sampled(tiny, oracle_w, res, by_id, 4, 4, 3, trace=tr)
    assert checked == 15 and mism <= 1
    # keep = G is the non-speculative schedule
    eng.debug_trace_enable(64)
    eng.submit(ps, 4, 100, 2, trace=L, round_id=4, keep=4)
    st = eng.run()
    _check_round_trace(eng, L, 100, 2, sched.SHORT)
    assert st.t == 20 and len(eng.collect()) == 8
    eng.close()


def _check_issue_trace(eng, L, cap, target, kind, A, keep=None):
    ref = sched.issue_step_loop(L, cap, target, kind, A, with_steps=True, keep=keep)
    got = eng.debug_trace(ref.t_end + 2)
    assert len(got) == ref.t_end
    for a, b in zip(got, ref.steps):
        assert np.array_equal(a["live"], b["live"]), a["t"]
        assert a["accepted"] == b["accepted"] and a["done"] == b["done"], a["t"]
    return ref


@pytest.mark.parametrize("seed,graph_steps,A,keep", [(0, 0, 3, None), (1, 4, 5, None), (2, 4, 4, 3),
                                                     (3, 0, 1, None), (4, 4, 12, None)])
def test_continuous_issuance_schedule_bit_exact(tiny, seed, graph_steps, A, keep):
    """NEXT-4: at most A prompts active, new ones issued after every
    step in index order.  Per-step live lists (incl. the rows issued into the
    batch), acceptance, the retained set, the queue and the unissued prompts
    match the oracle's step loop; A >= n is the plain round."""
    eng = make_engine(tiny, graph_steps=graph_steps)
    n, G = 12, 4
    ps = gen.prompts(n, 0, tiny["eos_id"], (2, 100), 90 + seed)
    L = _trace(n, G, 70 + seed, l_max=120)[:, 0, :]
    cap, target = 96, 8
    eng.issue_cap(A)
    eng.debug_trace_enable(900)
    eng.submit(ps, G, cap, target, trace=L, round_id=seed, keep=keep or 0)
    st = eng.run()
    ref = _check_issue_trace(eng, L, cap, target, sched.SHORT, A, keep=keep)
    assert st.t == ref.t_end and st.accepted == len(ref.accepted) and bool(st.underfilled) == ref.underfilled
    assert st.decoded_tokens == sum(len(x["live"]) for x in ref.steps)
    hist = eng.rows_histogram()
    want = np.bincount([len(x["live"]) for x in ref.steps[1:]], minlength=len(hist))
    assert np.array_equal(hist, want[:len(hist)])
    res = eng.collect()
    got = [(r["prompt_id"] - ps[0]["prompt_id"], r["j"], r["len"]) for r in res]
    want = [(i, j, int(ref.retained_len[i, j])) for i in ref.accepted for j in range(G) if ref.retained_len[i, j]]
    assert got == want
    for r in res:
        assert r["tokens"][-1] == tiny["eos_id"] and np.all(r["tokens"][:-1] != tiny["eos_id"])
    assert eng.long_queue() == [ps[i]["prompt_id"] for i in ref.deferred]
    assert eng.unissued() == [ps[i]["prompt_id"] for i in ref.unissued]
    if A >= n:
        assert ref.unissued == [] and ref.t_end == sched.closed_form(L, cap, target, sched.SHORT, keep=keep).t_end
    # issuance off again: the plain schedule
    eng.issue_cap(0)
    eng.debug_trace_enable(900)
    eng.submit(ps, G, cap, target, trace=L, round_id=seed, keep=keep or 0)
    eng.run()
    _check_round_trace(eng, L, cap, target, sched.SHORT, keep=keep)
    eng.collect()
    eng.close()


def test_continuous_issuance_sampling_and_long_round(tiny, oracle_w):
    """Late-issued prompts decode their last prompt token as their first step;
    their tokens are still the oracle's Gumbel argmax at token index k (the
    counter does not depend on the issue step).  Long round, A = 2 of 6."""
    eng = make_engine(tiny, graph_steps=4)
    n, G = 6, 3
    ps = gen.prompts(n, 0, tiny["eos_id"], (2, 70), 23)
    ps[3]["tokens"] = np.repeat(ps[3]["tokens"][:1], 65)   # 64 prefilled tokens: the first step opens a page
    L = np.minimum(_trace(n, G, 9)[:, 0, :], 30)
    eng.issue_cap(2)
    eng.debug_trace_enable(400)
    eng.submit(ps, G, 24, n, long_round=True, trace=L, round_id=6)
    st = eng.run()
    ref = _check_issue_trace(eng, L, 24, n, sched.LONG, 2)
    assert st.t == ref.t_end and eng.unissued() == []
    res = eng.collect()
    assert len(res) == n * G
    by_id = {p["prompt_id"]: np.asarray(p["tokens"]) for p in ps}
    tr = {p["prompt_id"]: L[i] for i, p in enumerate(ps)}
    checked, mism = _check_sampled(tiny, oracle_w, res, by_id, G, 6, 3, trace=tr)
    assert checked > 100 and mism <= checked // 50
    eng.close()


def test_streaming_collect(tiny):
    """NEXT-3: responses streamed between rp_step calls are final
    (identical to the closing collect, same order) and only ever cover prompts
    accepted by the current step, in the oracle's acceptance order."""
    eng = make_engine(tiny, graph_steps=0)
    n, G, R0 = 12, 5, 4
    ps = gen.prompts(n, 0, tiny["eos_id"], (1, 100), 91)
    L = _trace(n, G, 92)[:, 0, :]
    eng.submit(ps, G, 128, 9, trace=L, round_id=3, keep=R0)
    ref = sched.closed_form(L, 128, 9, sched.SHORT, keep=R0)
    streamed, first, calls = [], 0, 0
    while True:
        st = eng.step(7)
        got, first_new = eng.collect_ready(first)
        assert len(got) == (first_new - first) * R0
        # every streamed prompt completed no later than the current step
        for r in got:
            i = r["prompt_id"] - ps[0]["prompt_id"]
            assert ref.retained_len[i, r["j"]] == r["len"] <= st.t
        streamed += got
        first, calls = first_new, calls + 1
        if st.done:
            break
    final = eng.collect()
    key = lambda rs: [(r["prompt_id"], r["j"], r["len"], r["tokens"].tolist()) for r in rs]
    assert key(streamed) == key(final) and calls > 3
    assert list(dict.fromkeys(r["prompt_id"] - ps[0]["prompt_id"] for r in final)) == ref.accepted
    eng.close()


def test_underfilled_and_edge_rounds(tiny):
    eng = make_engine(tiny, graph_steps=3)
    ps = gen.prompts(3, 0, tiny["eos_id"], (64, 64), 5)          # page-aligned prompts
    L = np.array([[5, 200], [300, 3], [4, 4]])
    eng.debug_trace_enable(200)
    eng.submit(ps, 2, 100, 2, trace=L)
    st = eng.run()
    ref = _check_round_trace(eng, L, 100, 2, sched.SHORT)
    assert st.underfilled == 1 and ref.underfilled
    eng.collect()
    # all lengths 1: done at step 1 (the prefill step)
    L1 = np.ones((3, 2), np.int32)
    eng.submit(ps, 2, 100, 3, trace=L1)
    st = eng.run()
    assert st.done and st.t == 1 and st.accepted == 3
    res = eng.collect()
    assert all(r["len"] == 1 and r["tokens"][0] == tiny["eos_id"] for r in res)
    eng.close()


# ------------------------------------------------------------- sampling
def _check_sampled(cfg, w, res, prompts_by_id, G, round_id, seed, trace=None):
    checked = mism = 0
    for r in res:
        p = prompts_by_id[r["prompt_id"]]
        seq = np.concatenate([p, r["tokens"]])
        lg = decoder.logits(w, seq[:-1], rows=np.arange(len(p) - 1, len(seq) - 1))
        uid = r["prompt_id"] * G + r["j"]
        L = None if trace is None else trace[r["prompt_id"]][r["j"]]
        for t in range(1, r["len"] + 1):
            tok, gap = sampler.sample(lg[t - 1], t, uid, round_id, seed, eos_id=cfg["eos_id"], trace_len=L)
            checked += 1
            if tok != r["tokens"][t - 1]:
                assert gap <= GAP, (r["prompt_id"], r["j"], t, tok, r["tokens"][t - 1], gap)
                mism += 1
    return checked, mism


def test_sampled_tokens_trace_mode(tiny, oracle_w):
    eng = make_engine(tiny, graph_steps=4)
    n, G = 6, 3
    ps = gen.prompts(n, 0, tiny["eos_id"], (5, 40), 21)
    L = np.minimum(_trace(n, G, 7)[:, 0, :], 40)
    eng.submit(ps, G, 128, n, long_round=True, trace=L, round_id=5)
    eng.run()
    res = eng.collect()
    by_id = {p["prompt_id"]: p["tokens"] for p in ps}
    tr = {p["prompt_id"]: L[i] for i, p in enumerate(ps)}
    checked, mism = _check_sampled(tiny, oracle_w, res, by_id, G, 5, 3, trace=tr)
    assert checked > 100 and mism <= checked // 50
    eng.close()


def test_sampled_tokens_natural_eos(tiny, oracle_w):
    """Natural mode: EOS is sampled, never forced; responses end at EOS or the
    cap.  Every token is checked against the oracle's argmax (gap rule)."""
    eng = make_engine(tiny, graph_steps=2)
    n, G = 4, 2
    ps = gen.prompts(n, 0, tiny["eos_id"], (5, 30), 31)
    eng.submit(ps, G, 48, n, long_round=True, round_id=9)
    eng.run()
    res = eng.collect()
    assert len(res) == n * G
    by_id = {p["prompt_id"]: p["tokens"] for p in ps}
    checked, mism = _check_sampled(tiny, oracle_w, res, by_id, G, 9, 3)
    assert checked >= n * G and mism <= max(1, checked // 50)
    eng.close()


def test_decode_step_logits(tiny, oracle_w):
    """Logits of eager decode steps (paged decode attention, split-K GEMMs)
    against the oracle teacher-forced on the GPU's own history."""
    eng = make_engine(tiny, graph_steps=0)
    n, G = 3, 2
    ps = gen.prompts(n, 0, tiny["eos_id"], (60, 70), 41)           # crosses a page boundary
    L = np.full((n, G), 30, np.int32)
    eng.debug_trace_enable(64)
    eng.submit(ps, G, 64, n, long_round=True, trace=L, round_id=1)
    hist = {}
    worst = 0.0
    for step in range(8):
        st = eng.step(1)
        lg, slots = eng.debug_last_logits()
        # tokens generated so far come from the trace of decoded lists + collect later;
        # rebuild them from the final collect instead: store logits now
        hist[st.t] = (lg.copy(), slots.copy())
    eng.run()
    res = eng.collect()
    toks = {(r["prompt_id"] - ps[0]["prompt_id"], r["j"]): r["tokens"] for r in res}
    for t, (lg, slots) in hist.items():
        for row, s in enumerate(slots):
            p, j = divmod(int(s), G)
            seq = np.concatenate([ps[p]["tokens"], toks[(p, j)][:t - 1]])
            want = decoder.logits(oracle_w, seq, rows=[len(seq) - 1])[0]
            worst = max(worst, float(np.max(np.abs(lg[row] - want))))
    assert worst <= LOGIT_TOL, worst
    eng.close()


def test_decode_step_logits_fused_qkv(tiny, oracle_w, monkeypatch):
    """The optional fused path (RP_FUSE_QKV=1, profiles/r02_fused_qkv_ab.txt):
    the decode attention sums the QKV GEMM's split partials, applies the
    folded norm, bias and RoPE and appends k / v itself."""
    monkeypatch.setenv("RP_FUSE_QKV", "1")
    test_decode_step_logits(tiny, oracle_w)
    test_sampled_tokens_trace_mode(tiny, oracle_w)


def test_invalid_arguments(tiny):
    from paper_2509_21009_b200 import rp
    eng = make_engine(tiny, graph_steps=0)
    ps = gen.prompts(2, 0, tiny["eos_id"], (4, 8), 1)
    with pytest.raises(rp.RPError) as e:
        eng.submit(ps, 0, 10, 1)
    assert e.value.code == rp.RP_EINVAL
    with pytest.raises(rp.RPError):
        eng.submit(ps, 2, 10, 3)
    with pytest.raises(rp.RPError):
        eng.submit(ps, 2, 10, 1, long_round=True)
    with pytest.raises(rp.RPError):
        eng.submit(ps, 2, 10, 1, keep=3)                         # keep > G
    with pytest.raises(rp.RPError):
        eng.submit(ps, 2, 10, 2, long_round=True, keep=1)        # no speculation in a long round
    with pytest.raises(rp.RPError) as e:
        eng.step()
    assert e.value.code == rp.RP_ESTATE
    eng.submit(ps, 2, 10, 1)
    with pytest.raises(rp.RPError) as e:
        eng.submit(ps, 2, 10, 1)
    assert e.value.code == rp.RP_EBUSY
    eng.run()
    eng.collect()
    eng.close()


def test_decode_long_context_split_kv(tiny, oracle_w):
    """Contexts of ~650 tokens: 11 KV pages per work item and 512-token
    key splits (kv_lo > 0) merged by attn_merge; logits of the decode step vs
    the oracle teacher-forced on the GPU's own history."""
    eng = make_engine(tiny, graph_steps=0, max_cap=640)
    n, G = 2, 3
    ps = gen.prompts(n, 0, tiny["eos_id"], (100, 110), 77)
    L = np.full((n, G), 600, np.int32)
    eng.debug_trace_enable(700)
    eng.submit(ps, G, 640, n, long_round=True, trace=L, round_id=3)
    eng.step(540)
    lg, slots = eng.debug_last_logits()
    st = eng.step(1)
    t_lg = st.t - 1
    eng.run()
    res = eng.collect()
    toks = {(r["prompt_id"] - ps[0]["prompt_id"], r["j"]): r["tokens"] for r in res}
    worst = 0.0
    for row, s in enumerate(slots):
        p, j = divmod(int(s), G)
        seq = np.concatenate([ps[p]["tokens"], toks[(p, j)][:t_lg - 1]])
        want = decoder.logits(oracle_w, seq, rows=[len(seq) - 1])[0]
        worst = max(worst, float(np.max(np.abs(lg[row] - want))))
    assert len(seq) > 600 and worst <= LOGIT_TOL, (len(seq), worst)
    eng.close()


@pytest.mark.parametrize("model", ["tiny", "tiny-kv8"])
@pytest.mark.parametrize("G", [1, 3, 8, 10])
@pytest.mark.parametrize("mode", ["auto", "group", "single", "split", "rows"])
def test_decode_attention_sibling_groups(model, G, mode, monkeypatch):
    """Decode attention over sibling groups (k_attn_group.cu, RP_ATTN_GROUP:
    1 'auto', 2 forced sibling groups, 3 forced single rows, 4 shared pages
    in group units and private pages in per-row units merged per row; by default it
    runs only above 200 live rows) and the per-row kernel (0, k_attn.cu):
    logits of eager decode steps vs
    the oracle teacher-forced on the GPU's own history, for groups of 1-8
    members (rep 4 / 2 / 1 warps per member pair), a G = 10 prompt split into
    groups of 8 and 2, siblings dying mid-round (groups shrink), head_dim 64
    (g = 2) and 128 (g = 5), and ~650-token contexts cut into many page
    splits merged per member."""
    monkeypatch.setenv("RP_ATTN_GROUP", {"auto": "1", "group": "2", "single": "3", "split": "4", "rows": "0"}[mode])
    monkeypatch.setenv("RP_ATTN_GROUP_MIN", "0")          # the group kernel at every live batch
    cfg = configs.model_config(model)
    w = weights.Weights(cfg, configs.WEIGHT_SEED)
    eng = make_engine(cfg, graph_steps=0, max_cap=640, max_seqs=32, max_prompt_len=160, kv_pool_bytes=256 << 20)
    n = 2
    ps = gen.prompts(n, 0, cfg["eos_id"], (100, 130), 91 + G)
    L = np.full((n, G), 600, np.int32)
    L[:, : G // 2] = 40 + 7 * np.arange(G // 2)          # the first half of the siblings end early
    eng.debug_trace_enable(700)
    eng.submit(ps, G, 640, n, long_round=True, trace=L, round_id=5)
    caps, cur = {}, 1                                     # rp_submit_round decodes step 1
    for t_stop in (3, 45, 560):
        st = eng.step(t_stop - cur)
        cur = st.t
        lg, slots = eng.debug_last_logits()
        caps[st.t] = (lg.copy(), slots.copy())
    eng.run()
    res = eng.collect()
    eng.close()
    toks = {(r["prompt_id"] - ps[0]["prompt_id"], r["j"]): r["tokens"] for r in res}
    worst, rows = 0.0, 0
    for t, (lg, slots) in caps.items():
        for row, s in enumerate(slots):
            p, j = divmod(int(s), G)
            if j % 3 and row % 2:                         # a sample of the rows keeps the oracle cheap
                continue
            seq = np.concatenate([ps[p]["tokens"], toks[(p, j)][:t - 1]])
            want = decoder.logits(w, seq, rows=[len(seq) - 1])[0]
            worst = max(worst, float(np.max(np.abs(lg[row] - want))))
            rows += 1
    assert max(caps) >= 560 and rows >= 4 and worst <= LOGIT_TOL, (caps.keys(), rows, worst)


def test_gemm_dsm_split_k_subprocess():
    """The optional DSMEM split-K reduction (RP_GEMM_DSM=1, off by default:
    profiles/r02_gemm_dsm_ab.txt): the GEMM sweep and the decode-step logits
    in a fresh process (the switch is read once per process)."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, RP_GEMM_DSM="1")
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", os.path.join(root, "tests", "test_gpu_parity.py"),
                        "-k", "gemm_tcgen05_vs_fp32 or decode_step_logits and not fused"],
                       cwd=root, env=env, capture_output=True, text=True, timeout=1200)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]
