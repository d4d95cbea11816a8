"""Pins of the KV-pressure oracle (NEXT-2: recompute preemption, re-admission,
the TP heuristic; oracle/sched.py, readings DESIGN.md Z26) against what the
paper and the arithmetic fix:

* with a pool large enough for every response the schedule IS the plain round
  (`step_loop`, already pinned by brute force / SPEC examples), per-step live
  lists included, for SHORT / LONG, speculation, and the DP protocol;
* a hand-worked two-prompt LONG round with a 5-page pool (LIFO victim,
  re-admission once the survivor finishes, t_end 195 instead of 130);
* page conservation: at the end of a LONG round every private page is back
  (free = pool - prompt pages); a preempted prompt is never decoded while
  waiting; every prompt of a LONG round still gets its G responses with the
  trace lengths; preemption only delays completions;
* the planner heuristic of P:741-746 on worked sequences.
"""
import numpy as np
import pytest

from oracle import sched


def _rand(seed, n, G, lmax=300, mu=3.5):
    rng = np.random.default_rng(seed)
    L = np.clip(np.rint(np.exp(rng.normal(mu, 0.9, size=(n, G)))), 1, lmax).astype(np.int64)
    plen = rng.integers(1, 200, size=n)
    return L, plen


@pytest.mark.parametrize("seed", range(6))
@pytest.mark.parametrize("kind,keep", [(sched.SHORT, None), (sched.LONG, None), (sched.SHORT, 2)])
def test_ample_pool_is_the_plain_round(seed, kind, keep):
    n, G = 7, 3
    L, plen = _rand(seed, n, G)
    cap, target = 150, 5
    ref = sched.step_loop(L, cap, target, kind, with_steps=True, keep=keep)
    got = sched.kv_step_loop(L, plen, cap, target, kind, 10 ** 6, with_steps=True, keep=keep)
    assert got.t_end == ref.t_end and got.accepted == ref.accepted and got.deferred == ref.deferred
    assert np.array_equal(got.retained_len, ref.retained_len) and got.preemptions == [0]
    for a, b in zip(got.steps, ref.steps):
        assert np.array_equal(a["live"][0], b["live"]) and a["accepted"] == b["accepted"] and a["done"] == b["done"]


@pytest.mark.parametrize("world", [2, 3])
def test_ample_pool_dp_is_dp_protocol(world):
    for seed in range(4):
        L, plen = _rand(10 + seed, 11, 3)
        t, acc, _ = sched.dp_protocol(L, 150, 8, sched.SHORT, world)
        got = sched.kv_step_loop(L, plen, 150, 8, sched.SHORT, 10 ** 6, world=world)
        assert got.t_end == t and got.accepted == acc


def test_hand_worked_two_prompts():
    """plen = 64 (one prompt page each, no partial page), G = 1, L = 130, pool
    5 pages (3 free after the prompt pages).  Step 1 allocates one page each
    (free 1).  At step 65 both responses have written 128 positions and need a
    third page: 2 > 1, so prompt 1 (the later admission) is preempted, freeing
    its page (free 2 -> 1 after prompt 0's page).  Re-admission needs
    ceil((64 + 65) / 64) - 1 = 2 pages: it waits until prompt 0 finishes at
    step 130 (freeing 3 pages), then prompt 1 continues at token 66 from step
    131 and finishes at step 195."""
    L = np.array([[130], [130]])
    r = sched.kv_step_loop(L, [64, 64], 1000, 2, sched.LONG, 5, with_steps=True)
    assert r.t_end == 195 and r.accepted == [0, 1] and r.preemptions == [1]
    live = {s["t"]: list(s["live"][0]) for s in r.steps}
    assert live[65] == [0, 1] and live[66] == [0] and live[130] == [0] and live[131] == [1] and live[195] == [1]
    assert np.array_equal(r.retained_len, [[130], [130]])
    # one page less: prompt 0 alone cannot finish while prompt 1 holds its prompt page
    with pytest.raises(sched.KVExhausted):
        sched.kv_step_loop(L, [64, 64], 1000, 2, sched.LONG, 4)


class Audit(sched.KVRank):
    """KVRank with the page ledger re-derived from scratch after every step."""

    def pressure(self):
        super().pressure()
        G = self.G
        held = sum(sched._pages(p) for p in self.plen)
        for s in self.live:
            i, j = divmod(s, G)
            nxt = self.kv[i, j] + (1 if True else 0)
            held += sched._pages(nxt) - self.own0[i]       # pages through the next append
        assert held + self.free == self.pool, (held, self.free, self.pool)
        for v in self.wait:
            assert all(s // G != v for s in self.live)


@pytest.mark.parametrize("seed", range(8))
def test_pressure_invariants_long_round(seed):
    n, G = 6, 3
    L, plen = _rand(100 + seed, n, G, lmax=400, mu=4.8)
    pool = sum(sched._pages(p) for p in plen) + G * n + 12
    r = sched.KVRank(L, plen, 10 ** 6, sched.LONG, pool, G)
    r.pool = pool
    audit = Audit.__new__(Audit)
    audit.__dict__.update(r.__dict__)
    t, comp_at = 0, {}
    try:
        while audit.live:
            t += 1
            dec, comp = audit.step(t)
            for i in comp:
                comp_at[i] = t
            for v in audit.wait:                         # waiting prompts are not decoded
                assert all(s // G != v for s in dec)
            audit.pressure()
    except sched.KVExhausted:
        pytest.skip("pool too small for this trace")
    assert sorted(comp_at) == list(range(n))             # every prompt completes (LONG)
    assert np.array_equal(audit.g, L)                    # with its trace lengths
    assert audit.free == pool - sum(sched._pages(p) for p in plen)   # every private page returned
    plain = sched.step_loop(L, 10 ** 6, n, sched.LONG)
    assert t >= plain.t_end                              # pressure only delays



def test_pressure_preempts_under_tight_pool():
    rng = np.random.default_rng(7)
    L, plen = rng.integers(100, 400, size=(8, 4)), rng.integers(1, 200, size=8)
    plain = sched.kv_step_loop(L, plen, 10 ** 6, 8, sched.LONG, 10 ** 6)
    tight_pool = sum(sched._pages(p) for p in plen) + 4 * 8 + 10
    tight = sched.kv_step_loop(L, plen, 10 ** 6, 8, sched.LONG, tight_pool)
    assert tight.preemptions[0] > 0 and tight.t_end > plain.t_end
    assert sorted(tight.accepted) == list(range(8))


def test_plan_tp_heuristic():
    """> 1.05x rise doubles (capped at the server), four zero
    rounds halve, anything else keeps the size."""
    assert sched.plan_tp(1, 8, 100, 106, 0) == (2, 0)     # 1.06x
    assert sched.plan_tp(2, 8, 100, 105, 0) == (2, 0)     # 1.05x is not > 1.05x
    assert sched.plan_tp(8, 8, 10, 20, 0) == (8, 0)       # already the whole server
    assert sched.plan_tp(4, 8, 0, 1, 0) == (8, 0)         # from zero: any preemption is a rise
    tp, z = 4, 0
    for _ in range(3):
        tp, z = sched.plan_tp(tp, 8, 0, 0, z)
    assert (tp, z) == (4, 3)
    assert sched.plan_tp(tp, 8, 0, 0, z) == (2, 0)        # the fourth zero round halves
    assert sched.plan_tp(1, 8, 0, 0, 3) == (1, 0)         # never below 1
