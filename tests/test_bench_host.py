"""Host logic of bench.py (no GPU): the workload stream and planner state for
the three schedules, checked against the oracle's round outcomes."""
import numpy as np

import bench
from oracle import sched


def _run(W, n_rounds, A=None):
    """Drive the workload with oracle rounds (what the engines return)."""
    kinds = []
    for _ in range(n_rounds):
        kind, ids, target, cap, L = W.plan()
        kinds.append(kind)
        if kind == "long":
            r = sched.closed_form(L, cap, len(ids), sched.LONG)
            W.commit(kind, ids, [ids[i] for i in r.accepted])
        elif A:
            r = sched.issue_step_loop(L, cap, target, sched.SHORT, A)
            W.commit(kind, ids, [ids[i] for i in r.accepted], [ids[i] for i in r.unissued])
        else:
            r = sched.closed_form(L, cap, target, sched.SHORT)
            W.commit(kind, ids, [ids[i] for i in r.accepted])
    return kinds


def test_tail_schedule_matches_oracle_simulate():
    W = bench.Workload("C1-tiny", 1)
    kinds = _run(W, 6)
    ref = sched.simulate(W.trace, 6, W.P0, 1.25, W.G, W.R["short_cap"], W.R["long_cap"],
                         n_launch_override=W.n_submit)
    assert kinds == [x["kind"] for x in ref]
    assert W.queue.ids == ref[-1]["queue_after"]


def test_sync_schedule_takes_fresh_prompts():
    W = bench.Workload("C1-tiny", 2, "sync")
    seen = []
    for _ in range(3):
        kind, ids, target, cap, L = W.plan()
        assert kind == "long" and target == W.P0 and cap == W.R["long_cap"]
        assert np.array_equal(L, W.trace[ids, 0, :])
        seen += ids
        W.commit(kind, ids, ids)
    assert seen == list(range(3 * W.P0)) and len(W.queue) == 0


def test_issue_schedule_returns_unissued_prompts():
    W = bench.Workload("C1-tiny", 1, "issue")
    A = 2
    stream = []
    for _ in range(8):
        kind, ids, target, cap, L = W.plan()
        if kind == "short":
            stream.append(list(ids))
            r = sched.issue_step_loop(L, cap, target, sched.SHORT, A)
            un = [ids[i] for i in r.unissued]
            W.commit(kind, ids, [ids[i] for i in r.accepted], un)
            assert W.returned == un
            nxt, _, _, _, _ = W.plan()
            if nxt == "short":
                assert W.plan()[1][:len(un)] == un            # back at the front of the stream
        else:
            r = sched.closed_form(L, cap, len(ids), sched.LONG)
            W.commit(kind, ids, [ids[i] for i in r.accepted])
    # every fresh id enters a short round in order, none skipped
    firsts = sorted(set(i for s in stream for i in s))
    assert firsts == list(range(len(firsts)))


def test_grid_interpolation():
    grid = {"points": [dict(tp=1, B=8, ctx=1024, ms_per_step=3.0), dict(tp=1, B=256, ctx=1024, ms_per_step=8.0),
                       dict(tp=1, B=8, ctx=4096, ms_per_step=4.0), dict(tp=2, B=256, ctx=4096, ms_per_step=5.0)]}
    assert bench.grid_step_ms(grid, 1, 256, 2000) == 8.0                 # nearest context 1024 (log space)
    assert abs(bench.grid_step_ms(grid, 1, 132, 1024) - 5.5) < 1e-9      # linear in B
    assert abs(bench.grid_step_ms(grid, 1, 504, 1024) - 13.0) < 1e-9     # extrapolated past the last batch
    assert bench.grid_step_ms(grid, 1, 8, 8192) == 4.0                    # single point of that context
    assert bench.grid_step_ms(grid, 2, 8, 100) == 5.0
    assert bench.grid_step_ms(grid, 4, 8, 100) is None


def test_whole_round_roofline_accounting():
    """bench.roofline over a synthetic whole-round profile: algorithmic bytes
    summed over every launch at its live batch; the dominant class is the
    largest measured time; below the ridge the bound is HBM."""
    from synth import configs
    cfg = configs.model_config("qwen2.5-7b")
    L = cfg["n_layers"]
    hist = [0] * 257
    hist[16], hist[256] = 90, 10                     # 100 decode steps
    gu16, _ = bench.launch_work(cfg, 1, "gemm_gu", 16)
    gu256, f256 = bench.launch_work(cfg, 1, "gemm_gu", 256)
    assert gu16 == 2 * cfg["d_ff"] * cfg["d_model"] * 2 + 16 * cfg["d_model"] * 2 + 16 * cfg["d_ff"] * 2
    assert f256 == 2.0 * 256 * 2 * cfg["d_ff"] * cfg["d_model"]
    ms = {"gemm_gu": 100.0, "gemm_down": 50.0, "attention": 40.0}
    prof = dict(kind="short", hist=hist, kv_tokens=1000 * 100, tp=1, ms=ms,
                launches={"gemm_gu": 100 * L, "gemm_down": 100 * L, "attention": 100 * L}, rows=0, ctx=0, steps=100)
    roof, detail = bench.roofline([prof], cfg)
    assert roof["kernel"] == "gemm_gu" and roof["bound"] == "hbm" and roof["unit"] == "GB/s"
    want = (90 * gu16 + 10 * gu256) * L / 0.1 / 1e9
    assert abs(roof["achieved"] - want) < 0.1 and abs(roof["frac"] - want / roof["peak"]) < 1e-4
    assert detail["gemm_gu"]["share"] == round(100 / 190, 4)
