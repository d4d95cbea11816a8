"""Pins of oracle/sched.py: brute force (the literal step loop) against the
closed form on every tiny trace, SPEC worked examples, special
cases, invariants and DP-split invariance."""
import itertools

import numpy as np
import pytest

from oracle import sched as X
from oracle import sched
from synth.gen import length_trace


def _cmp(a, b):
    assert a.t_end == b.t_end
    assert a.accepted == b.accepted
    assert a.deferred == b.deferred
    assert a.underfilled == b.underfilled
    assert np.array_equal(a.outcome, b.outcome)
    assert np.array_equal(a.retained_len, b.retained_len)


def test_brute_force_equals_closed_form_all_tiny_traces():
    """3 prompts x G=2 x lengths 1..4 (4^6 traces), every target and cap."""
    n, G = 3, 2
    for flat in itertools.product(range(1, 5), repeat=n * G):
        L = np.array(flat).reshape(n, G)
        for cap in range(1, 5):
            _cmp(X.step_loop(L, cap, n, X.LONG), X.closed_form(L, cap, n, X.LONG))
            for target in range(1, n + 1):
                _cmp(X.step_loop(L, cap, target, X.SHORT), X.closed_form(L, cap, target, X.SHORT))


def test_brute_force_speculation_all_tiny_traces():
    """Response-level speculation: 2 prompts x G=3 x
    lengths 1..4 (4^6 traces), every keep < G, cap and target."""
    n, G = 2, 3
    for flat in itertools.product(range(1, 5), repeat=n * G):
        L = np.array(flat).reshape(n, G)
        for keep in (1, 2):
            for cap in (2, 4):
                for target in (1, 2):
                    _cmp(X.step_loop(L, cap, target, X.SHORT, keep=keep),
                         X.closed_form(L, cap, target, X.SHORT, keep=keep))


def test_speculation_keeps_first_finishers_and_aborts_siblings():
    """Hand-worked case: G=4, keep=2.  Prompt 0 lengths (5,3,9,3): the two
    3s finish first -> T_0 = 3, j=1,3 kept, j=0,2 aborted after step 3.
    Prompt 1 (2,7,7,20): T_1 = 7, tie at 7 goes to j=1 (lower index), j=2
    finishes at 7 but is not retained, j=3 aborted."""
    L = np.array([[5, 3, 9, 3], [2, 7, 7, 20]])
    r = X.closed_form(L, 100, 2, X.SHORT, keep=2)
    assert r.accepted == [0, 1] and r.t_end == 7
    assert r.retained_len.tolist() == [[0, 3, 0, 3], [2, 7, 0, 0]]
    assert r.outcome.tolist() == [[X.ABORTED, X.FINISHED, X.ABORTED, X.FINISHED],
                                  [X.FINISHED, X.FINISHED, X.FINISHED, X.ABORTED]]
    # keep = G reproduces the non-speculative schedule
    for keep in (None, 4):
        r = X.closed_form(L, 100, 2, X.SHORT, keep=keep)
        assert r.accepted == [0, 1] and r.t_end == 20


def test_speculation_decodes_fewer_tokens():
    """With keep < G every prompt completes no later and fewer tokens are
    decoded than with keep = G on the same trace (monotonicity)."""
    tr = length_trace(40, 8, 4.0, 0.5, 0.8, 2000, 11)[:, 0, :]
    full = X.closed_form(tr, 1024, 30, X.SHORT, with_steps=True)
    spec = X.closed_form(tr, 1024, 30, X.SHORT, with_steps=True, keep=6)
    assert spec.t_end <= full.t_end
    assert sum(len(s["live"]) for s in spec.steps) < sum(len(s["live"]) for s in full.steps)
    assert all(int(np.count_nonzero(spec.retained_len[i])) == 6 for i in spec.accepted)


def test_per_step_records_match():
    rng = np.random.default_rng(5)
    for it in range(40):
        L = rng.integers(1, 40, size=(6, 4))
        keep = None if it % 2 == 0 else 1 + it % 3
        for kind, target in ((X.SHORT, 4), (X.LONG, 6)):
            a = X.step_loop(L, 30, target, kind, with_steps=True, keep=keep)
            b = X.closed_form(L, 30, target, kind, with_steps=True, keep=keep)
            assert len(a.steps) == len(b.steps) == a.t_end
            for sa, sb in zip(a.steps, b.steps):
                assert np.array_equal(sa["live"], sb["live"])
                assert np.array_equal(np.sort(sa["ending"]), sb["ending"])
                assert np.array_equal(sa["counts"], sb["counts"])
                assert sa["accepted"] == sb["accepted"] and sa["done"] == sb["done"]


def test_spec_plan_round_examples():
    assert X.plan_round(0, 128, 1.25) == ("short", 160, 128)
    assert X.n_launch(8, 1.25) == 10                                   # S:277 responses
    assert X.plan_round(128, 128, 1.25) == ("long", 128, 128)
    assert X.plan_round(0, 128, 1.25, tail_batching=False) == ("baseline", 128, 128)
    assert X.n_launch(25, 1.25) == 32


def test_spec_acceptance_defers_32_of_160():
    rng = np.random.default_rng(0)
    L = rng.integers(1, 1000, size=(160, 8))
    r = X.closed_form(L, 100000, 128, X.SHORT)
    assert len(r.accepted) == 128 and len(r.deferred) == 32


def test_uniform_lengths_accept_lowest_indices():
    L = np.full((10, 3), 7)
    r = X.closed_form(L, 100, 8, X.SHORT)
    assert r.accepted == list(range(8)) and r.deferred == [8, 9]       # S:296 (ties -> index)
    assert r.t_end == 7


def test_eta_one_no_deferrals():
    rng = np.random.default_rng(1)
    L = rng.integers(1, 50, size=(12, 4))
    r = X.closed_form(L, 100, 12, X.SHORT)
    assert r.deferred == [] and r.t_end == L.max()


def test_target_all_is_plain_sync_rollout():
    rng = np.random.default_rng(2)
    L = rng.integers(1, 50, size=(8, 4))
    r = X.closed_form(L, 10_000, 8, X.SHORT)
    assert r.t_end == L.max()


def test_G1_reduces_to_order_statistic():
    L = np.array([[9], [3], [7], [3], [12]])
    r = X.closed_form(L, 100, 3, X.SHORT)
    assert r.accepted == [1, 3, 2] and r.t_end == 7


def test_underfilled_round():
    L = np.array([[5, 200], [300, 3], [4, 4]])
    r = X.closed_form(L, 100, 2, X.SHORT)
    assert r.underfilled and r.accepted == [2] and r.t_end == 100


def test_long_round_truncates_and_retains():
    L = np.array([[5, 700], [10, 20]])
    r = X.closed_form(L, 512, 2, X.LONG)
    assert r.accepted == [1, 0] and r.t_end == 512
    assert r.retained_len.tolist() == [[5, 512], [10, 20]]
    assert r.outcome[0, 1] == X.CAPPED


def test_no_short_response_exceeds_cap_and_retained_count_exact():
    tr = length_trace(400, 8, 5.0, 0.6, 0.85, 4000, 9)
    for res in X.simulate(tr, 10, 25, 1.25, 8, 600, 4000):
        r = res["round"]
        if res["kind"] == "short":
            assert r.retained_len.max() <= 600
            if not r.underfilled:
                assert (r.retained_len > 0).sum() == 25 * 8
        assert np.all(r.retained_len[r.outcome == X.ABORTED] == 0)


def test_periodicity_four_short_one_long():
    """P:572-574 / S:685: with 32 deferrals per short round (P0=128, eta=1.25)
    a long round follows every four short rounds."""
    tr = length_trace(160 * 20, 8, 6.0, 0.6, 0.85, 16384, 2)
    out = X.simulate(tr, 20, 128, 1.25, 8, 8192, 8192)
    kinds = "".join(o["kind"][0].upper() for o in out)
    assert all(len(o["round"].deferred) == 32 for o in out if o["kind"] == "short")
    assert kinds == "SSSSL" * 4


def test_coverage_no_starvation_and_no_resubmission():
    tr = length_trace(2000, 4, 4.0, 0.6, 0.85, 2000, 11)
    out = X.simulate(tr, 40, 16, 1.25, 4, 256, 2000)
    seen_short, trained = set(), []
    for o in out:
        if o["kind"] == "short":
            assert not (set(o["ids"]) & seen_short)                      # never resubmitted
            seen_short |= set(o["ids"])
        r = o["round"]
        trained += [o["ids"][i] for i in r.accepted]
    queue = set(out[-1]["queue_after"])
    # every submitted prompt is either trained once or still queued
    assert sorted(trained + sorted(queue)) == sorted(seen_short)
    assert len(set(trained)) == len(trained)


@pytest.mark.parametrize("world", [1, 2, 3, 4, 8])
def test_dp_protocol_matches_single_rank(world):
    rng = np.random.default_rng(world)
    for _ in range(20):
        n = int(rng.integers(world, 40))
        L = rng.integers(1, 60, size=(n, 4))
        target = int(rng.integers(1, n + 1))
        for keep in (None, 3, 1):               # also under response-level speculation (keep < G)
            ref = X.closed_form(L, 50, target, X.SHORT, keep=keep)
            t_end, acc, _ = X.dp_protocol(L, 50, target, X.SHORT, world, keep=keep)
            assert t_end == ref.t_end and acc == ref.accepted


def test_partition_contiguous():
    assert X.partition(10, 4) == [(0, 3), (3, 6), (6, 8), (8, 10)]


# ---------------------------------------------------------------- NEXT-4 continuous issuance

def _issue_equal(a, b, steps=True):
    assert a.t_end == b.t_end and a.accepted == b.accepted and a.deferred == b.deferred
    assert a.unissued == b.unissued and a.underfilled == b.underfilled
    assert np.array_equal(a.issue_step, b.issue_step)
    assert np.array_equal(a.outcome, b.outcome) and np.array_equal(a.retained_len, b.retained_len)
    if steps:
        assert len(a.steps) == len(b.steps)
        for x, y in zip(a.steps, b.steps):
            assert np.array_equal(x["live"], y["live"]) and x["accepted"] == y["accepted"] and x["done"] == y["done"]


def test_issue_hand_worked():
    # G = 1, at most 2 active, lengths 3 1 2 4, target 3.  Steps 1: {0, 1}; 1 ends -> 2 issued at 2;
    # step 3: 0 and 2 end, 3 accepted -> done; prompt 3 (tau would be 4) is never issued.
    L = np.array([[3], [1], [2], [4]])
    for r in (sched.issue_step_loop(L, 8, 3, sched.SHORT, 2, with_steps=True),
              sched.issue_closed_form(L, 8, 3, sched.SHORT, 2, with_steps=True)):
        assert r.t_end == 3 and r.accepted == [1, 0, 2] and r.deferred == [] and r.unissued == [3]
        assert list(r.issue_step) == [1, 1, 2, 0]
        assert [list(s["live"]) for s in r.steps] == [[0, 1], [0, 2], [0, 2]]
    # a prompt that can never complete (capped response) holds its slot until its last response ends
    L = np.array([[9, 1], [1, 1], [2, 2]])
    r = sched.issue_step_loop(L, 4, 2, sched.SHORT, 1)
    # prompt 0 holds the only slot for 4 steps (capped at 4), 1 runs at step 5, 2 at 6-7
    assert list(r.issue_step) == [1, 5, 6] and r.accepted == [1, 2] and r.t_end == 7 and r.deferred == [0]


def test_issue_reduces_to_plain_round():
    """max_active >= n issues everything at step 1: the plain round."""
    rng = np.random.default_rng(11)
    for _ in range(300):
        n, G = int(rng.integers(1, 8)), int(rng.integers(1, 4))
        L = rng.integers(1, 10, (n, G))
        cap = int(rng.integers(1, 10))
        kind = int(rng.integers(0, 2))
        target = int(rng.integers(1, n + 1)) if kind == sched.SHORT else n
        keep = int(rng.integers(1, G + 1)) if kind == sched.SHORT else None
        a = sched.issue_step_loop(L, cap, target, kind, n + int(rng.integers(0, 3)), keep=keep)
        b = sched.closed_form(L, cap, target, kind, keep=keep)
        assert a.t_end == b.t_end and a.accepted == b.accepted and a.deferred == b.deferred and a.unissued == []
        assert np.array_equal(a.outcome, b.outcome) and np.array_equal(a.retained_len, b.retained_len)


def test_issue_step_loop_vs_list_scheduling_exhaustive():
    """Two formulations -- the literal step loop and list scheduling of the
    prompts' (issue-independent) active durations -- agree on every n <= 3,
    G <= 2 trace of lengths 1..3 for every cap, max_active, target and keep."""
    import itertools
    for G in (1, 2):
        for n in (1, 2, 3):
            for Ls in itertools.product(range(1, 4), repeat=n * G):
                L = np.array(Ls).reshape(n, G)
                for cap in (1, 2, 3):
                    for A in range(1, n + 1):
                        for kind in (sched.SHORT, sched.LONG):
                            for target in (range(1, n + 1) if kind == sched.SHORT else [n]):
                                for keep in (range(1, G + 1) if kind == sched.SHORT else [None]):
                                    _issue_equal(sched.issue_step_loop(L, cap, target, kind, A, True, keep),
                                                 sched.issue_closed_form(L, cap, target, kind, A, keep, True))


def test_issue_invariants_random():
    rng = np.random.default_rng(12)
    for _ in range(400):
        n, G = int(rng.integers(1, 10)), int(rng.integers(1, 5))
        L = rng.integers(1, 14, (n, G))
        cap = int(rng.integers(1, 14))
        A = int(rng.integers(1, n + 1))
        target = int(rng.integers(1, n + 1))
        keep = int(rng.integers(1, G + 1))
        r = sched.issue_step_loop(L, cap, target, sched.SHORT, A, True, keep)
        _issue_equal(r, sched.issue_closed_form(L, cap, target, sched.SHORT, A, keep, True))
        tau = r.issue_step
        issued = [i for i in range(n) if tau[i] > 0]
        assert issued == list(range(len(issued)))                          # index order
        assert r.unissued == list(range(len(issued), n))
        assert sorted(r.accepted + r.deferred + r.unissued) == list(range(n))
        for s in r.steps:
            active = set(int(x) // G for x in s["live"])
            assert len(active) <= A
            # work conserving: a free slot is never left idle while prompts wait
            waiting = [i for i in range(n) if tau[i] == 0 or tau[i] > s["t"]]
            if len(active) < A and waiting and s["t"] < r.t_end:
                assert all(tau[i] == 0 or tau[i] > s["t"] for i in waiting)
                nxt = s["t"] + 1
                assert any(tau[i] == nxt for i in range(n)) or not waiting or r.t_end == s["t"]


def test_issue_dp_protocol_single_rank_and_plain():
    """world = 1 is the single-instance round; max_active >= slice size is
    the plain dp_protocol."""
    rng = np.random.default_rng(13)
    for _ in range(300):
        n, G = int(rng.integers(1, 12)), int(rng.integers(1, 4))
        L = rng.integers(1, 12, (n, G))
        cap = int(rng.integers(1, 12))
        target = int(rng.integers(1, n + 1))
        keep = int(rng.integers(1, G + 1))
        A = int(rng.integers(1, n + 1))
        r = sched.issue_step_loop(L, cap, target, sched.SHORT, A, keep=keep)
        t, acc, dfr, un = sched.issue_dp_protocol(L, cap, target, sched.SHORT, 1, A, keep=keep)
        assert (t, acc, dfr, un) == (r.t_end, r.accepted, r.deferred, r.unissued)
        world = int(rng.integers(1, 4))
        t2, acc2, _ = sched.dp_protocol(L, cap, target, sched.SHORT, world, keep=keep)
        t3, acc3, _, un3 = sched.issue_dp_protocol(L, cap, target, sched.SHORT, world, n, keep=keep)
        assert (t2, acc2) == (t3, acc3) and un3 == []
