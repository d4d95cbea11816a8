"""Tail-batching round schedule.  TEST INFRASTRUCTURE
ONLY (see oracle/__init__.py).  Integer-only; compared bit-exactly.

Paper: a short round "launches more than P0 prompts but retains only the
first P0 that finish"; prompts aborted during the
speculative short round go to a FIFO long-prompt queue and "once the queue
reaches size P0" they run in a long round "where speculative execution is
disabled", "capped at the same maximum".
SPEC: plan_round / on_prompt_accepted / run_long_round.

Readings: time is the logical decode step (Z1); a prompt
completes when all G responses finished (Z2); reaching the cap without EOS
aborts the response in a short round and truncates-and-retains it in a long
round (Z3); a round with fewer than `target` completable prompts ends when
no sequence is live (Z4); deferred prompts are re-rolled from scratch in the
long round, trace attempt 1 (Z5); the queue is FIFO and deferrals enter in
submission order (Z7); n_submit = ceil(eta * P0) (Z8).

Sequence s = (prompt i, response j) has slot i*G + j; its trace length
L[i][j] >= 1 counts the EOS token (Z16); token 1 is sampled from the prefill
logits; e_s = min(L_s, cap).
"""
from dataclasses import dataclass, field
from fractions import Fraction
from collections import deque
import math
import numpy as np

SHORT, LONG = 0, 1
FINISHED, CAPPED, ABORTED = 1, 2, 3


@dataclass
class Round:
    kind: int
    t_end: int
    accepted: list            # prompt indices, acceptance order
    deferred: list            # prompt indices, submission order
    underfilled: bool
    outcome: np.ndarray       # [n, G] FINISHED / CAPPED / ABORTED
    retained_len: np.ndarray  # [n, G] length of retained responses, 0 if dropped
    steps: list = field(default_factory=list)   # per-step records (optional)


def _e(L, cap):
    return np.minimum(np.asarray(L, np.int64), cap)


def _kept(L, cap, keep):
    """Response-level speculation: the first `keep` of
    a prompt's responses to finish (EOS within the cap) are retained; ties at
    the same step go to the lower response index j.  Returns the boolean mask
    and T_i = the step of the keep-th finish (inf if fewer finish)."""
    L = np.asarray(L, np.int64)
    n, G = L.shape
    kept = np.zeros((n, G), bool)
    T = np.full(n, np.iinfo(np.int64).max)
    for i in range(n):
        fin = [(L[i, j], j) for j in range(G) if L[i, j] <= cap]
        fin.sort()
        if len(fin) >= keep:
            for _, j in fin[:keep]:
                kept[i, j] = True
            T[i] = fin[keep - 1][0]
    return kept, T


def closed_form(L, cap, target, kind, with_steps=False, keep=None):
    """The schedule written out directly from the definition.

    SHORT: T_i = the keep-th smallest finished length of prompt i (keep = G:
    max_j L_ij if every L_ij <= cap), inf if fewer than keep finish within the
    cap; pi = prompts sorted by (T_i, i); A = first min(target, #finite) of
    pi; t_end = T_pi[target-1] if #finite >= target else the last step any
    sequence is live.  With keep < G a prompt's remaining siblings are aborted
    right after step T_i.  LONG (no speculation, keep = G): every prompt
    accepted, in (max_j e_ij, i) order; t_end = max e."""
    L = np.asarray(L, np.int64)
    n, G = L.shape
    keep = G if keep is None else keep
    e = _e(L, cap)
    if kind == SHORT:
        kept, T = _kept(L, cap, keep)
        # a sequence stops at its own end or when its prompt completes
        e = np.minimum(e, np.minimum(T, np.iinfo(np.int64).max)[:, None])
    else:
        kept = np.ones((n, G), bool)
        T = e.max(axis=1)
    order = sorted(range(n), key=lambda i: (T[i], i))
    n_fin = int(np.sum(T < np.iinfo(np.int64).max))
    if kind == LONG:
        target = n
    n_acc = min(target, n_fin)
    accepted = order[:n_acc]
    underfilled = n_fin < target
    t_end = int(T[order[target - 1]]) if not underfilled else int(e.max())
    deferred = sorted(set(range(n)) - set(accepted))
    e0 = _e(L, cap)
    outcome = np.where(L <= cap, FINISHED, CAPPED)
    outcome = np.where((e0 > t_end) | ((e0 > e) & (kind == SHORT)), ABORTED, outcome)
    retained = np.zeros_like(L)
    for i in accepted:
        retained[i] = np.where(kept[i], e0[i], 0)
    r = Round(kind, t_end, accepted, deferred, bool(underfilled), outcome.astype(np.int32), retained)
    if with_steps:
        r.steps = closed_form_steps(L, cap, target, kind, t_end, T, order, e, keep)
    return r


def closed_form_steps(L, cap, target, kind, t_end, T, order, e_eff=None, keep=None):
    """Per-step records for t = 1..t_end: live slots decoded at step t
    (e_s >= t, stable slot order), slots finishing at t, c_i(t), accepted(t),
    done(t)."""
    L = np.asarray(L, np.int64)
    n, G = L.shape
    e0 = _e(L, cap).reshape(-1)
    e = (e0 if e_eff is None else np.asarray(e_eff)).reshape(-1)
    fin_ok = (L.reshape(-1) <= cap) | (kind == LONG)
    rank = {p: k for k, p in enumerate(order)}
    if kind == LONG:
        target = n
    steps = []
    for t in range(1, t_end + 1):
        live = np.nonzero(e >= t)[0].astype(np.int32)
        ending = np.nonzero((e == t) & (e == e0))[0].astype(np.int32)   # EOS or cap, not a sibling abort
        Lf = np.minimum(np.asarray(L, np.int64).reshape(-1), cap)
        c = np.sum(((Lf <= t) & (e >= Lf) & fin_ok).reshape(n, G), axis=1)
        c = np.minimum(c, G if keep is None or kind == LONG else keep).astype(np.int32)
        acc = min(target, sum(1 for p in range(n) if T[p] <= t and rank[p] < target))
        steps.append(dict(t=t, live=live, ending=ending, counts=c, accepted=acc,
                          done=int(acc == target or t == int(e.max()))))
    return steps


def step_loop(L, cap, target, kind, with_steps=False, keep=None):
    """Literal step-by-step simulation of the round (the brute-force pin of
    `closed_form`): every live sequence emits token t; it ends on EOS (t == L)
    or at the cap; a prompt completes when `keep` of its responses finished
    (its other live responses are aborted after that step); completed prompts
    are admitted in index order until `target` are accepted or nothing is
    live."""
    L = np.asarray(L, np.int64)
    n, G = L.shape
    keep = G if (keep is None or kind == LONG) else keep
    kept = np.zeros((n, G), bool)
    done_p = [False] * n
    if kind == LONG:
        target = n
    live = list(range(n * G))
    cnt = [0] * n
    accepted, steps = [], []
    outcome = np.zeros((n, G), np.int32)
    t = 0
    while True:
        t += 1
        decoded = list(live)
        ending, completed = [], []
        for s in decoded:                          # slot order: lower j first
            i, j = divmod(s, G)
            if t == L[i, j]:                       # token t is EOS
                outcome[i, j] = FINISHED
                ending.append(s)
                if not done_p[i] and cnt[i] < keep:
                    cnt[i] += 1
                    kept[i, j] = True
                    if cnt[i] == keep:
                        completed.append(i)
            elif t == cap:                         # length cap reached
                outcome[i, j] = CAPPED
                ending.append(s)
                if kind == LONG:
                    cnt[i] += 1
                    kept[i, j] = True
                    if cnt[i] == G:
                        completed.append(i)
        for i in completed:
            done_p[i] = True
        for i in sorted(completed):
            if len(accepted) < target:
                accepted.append(i)
        # siblings of a prompt that completed at t are aborted after step t
        aborted_now = [s for s in decoded if s not in set(ending) and done_p[s // G]]
        for s in aborted_now:
            outcome[s // G, s % G] = ABORTED
        live = [s for s in decoded if s not in set(ending) and not done_p[s // G]]
        done = len(accepted) == target or not live
        if with_steps:
            steps.append(dict(t=t, live=np.array(decoded, np.int32), ending=np.array(ending, np.int32),
                              counts=np.array(cnt, np.int32), accepted=len(accepted), done=int(done)))
        if done:
            break
    for s in live:
        outcome[s // G, s % G] = ABORTED
    deferred = [i for i in range(n) if i not in accepted]
    retained = np.zeros((n, G), np.int64)
    for i in accepted:
        retained[i] = np.where(kept[i], np.minimum(L[i], cap), 0)
    r = Round(kind, t, accepted, deferred, len(accepted) < target, outcome, retained, steps)
    return r


# ------------------------------------------- continuous issuance (NEXT-4)
#
# P:1386 (DAPO integration): "we set a maximum number of active requests for
# each LLM instance and continuously issue new requests ... other unfinished
# prompts are retained in the queue".  Readings (Z21): a request is
# a prompt with its G responses; a prompt is active from its issue step tau
# until none of its responses is live; after each step the lowest-index
# unissued prompts are issued while fewer than `max_active` are active; a
# prompt issued at tau emits its k-th token at step tau + k - 1 (tau = 1 for
# the first min(max_active, n)); acceptance, the cutoff and the keep rule are
# those of the plain round; prompts never issued before the round ends are
# returned unissued (neither accepted nor deferred).

UNISSUED = 0


@dataclass
class IssueRound(Round):
    issue_step: np.ndarray = None   # [n] tau_i, 0 if never issued
    unissued: list = field(default_factory=list)


def issue_step_loop(L, cap, target, kind, max_active, with_steps=False, keep=None):
    """Literal step loop of a round with continuous issuance: each step every
    live response emits its next token; endings, completions, acceptance and
    sibling aborts as in `step_loop`; then prompts are issued in index order
    while fewer than `max_active` prompts have a live response."""
    L = np.asarray(L, np.int64)
    n, G = L.shape
    keep = G if (keep is None or kind == LONG) else keep
    if kind == LONG:
        target = n
    tau = np.zeros(n, np.int64)
    kept = np.zeros((n, G), bool)
    done_p = [False] * n
    cnt = [0] * n
    outcome = np.zeros((n, G), np.int32)
    nxt = min(max_active, n)
    tau[:nxt] = 1
    live = list(range(nxt * G))
    accepted, steps = [], []
    t = 0
    while True:
        t += 1
        decoded = list(live)
        ending, completed = [], []
        for s in decoded:
            i, j = divmod(s, G)
            k = t - tau[i] + 1                     # local token index
            if k == L[i, j]:
                outcome[i, j] = FINISHED
                ending.append(s)
                if not done_p[i] and cnt[i] < keep:
                    cnt[i] += 1
                    kept[i, j] = True
                    if cnt[i] == keep:
                        completed.append(i)
            elif k == cap:
                outcome[i, j] = CAPPED
                ending.append(s)
                if kind == LONG:
                    cnt[i] += 1
                    kept[i, j] = True
                    if cnt[i] == G:
                        completed.append(i)
        for i in completed:
            done_p[i] = True
        for i in sorted(completed):
            if len(accepted) < target:
                accepted.append(i)
        for s in decoded:
            if s not in ending and done_p[s // G]:
                outcome[s // G, s % G] = ABORTED
        live = [s for s in decoded if s not in set(ending) and not done_p[s // G]]
        active = len(set(s // G for s in live))
        done = len(accepted) == target
        while not done and active < max_active and nxt < n:      # issue after step t
            tau[nxt] = t + 1
            live.extend(range(nxt * G, nxt * G + G))
            nxt += 1
            active += 1
        done = done or not live
        if with_steps:
            steps.append(dict(t=t, live=np.array(decoded, np.int32), ending=np.array(ending, np.int32),
                              counts=np.array(cnt, np.int32), accepted=len(accepted), done=int(done)))
        if done:
            break
    for s in live:
        if tau[s // G] <= t:
            outcome[s // G, s % G] = ABORTED
    unissued = [i for i in range(n) if tau[i] == 0 or tau[i] > t]
    tau[unissued] = 0
    deferred = [i for i in range(n) if i not in accepted and i not in unissued]
    retained = np.zeros((n, G), np.int64)
    for i in accepted:
        retained[i] = np.where(kept[i], np.minimum(L[i], cap), 0)
    return IssueRound(kind, t, accepted, deferred, len(accepted) < target, outcome, retained, steps,
                      issue_step=tau, unissued=unissued)


def _issue_schedule(L, cap, kind, max_active, keep=None):
    """List scheduling of one instance's prompts: returns tau (issue step),
    C (completion step, inf if the prompt cannot complete), d (steps active),
    e0 = min(L, cap), e (steps each response decodes) and the keep mask."""
    import heapq
    L = np.asarray(L, np.int64)
    n, G = L.shape
    keep = G if (keep is None or kind == LONG) else keep
    INF = np.iinfo(np.int64).max
    e0 = _e(L, cap)
    if kind == SHORT:
        kept, T = _kept(L, cap, keep)
        e = np.minimum(e0, T[:, None])
    else:
        kept = np.ones((n, G), bool)
        T = e0.max(axis=1)
        e = e0
    d = e.max(axis=1)                                   # steps a prompt stays active
    tau = np.zeros(n, np.int64)
    slots = []
    for i in range(n):
        if i < max_active:
            tau[i] = 1
        else:
            tau[i] = heapq.heappop(slots) + 1
        heapq.heappush(slots, int(tau[i] + d[i] - 1))
    C = np.where(T < INF, tau + np.where(T < INF, T, 0) - 1, INF)
    return tau, C, d, e0, e, kept


def issue_dp_protocol(L, cap, target, kind, world, max_active, keep=None):
    """Continuous issuance under DP: each rank issues its own contiguous
    slice with its own cap of `max_active` ("for each LLM instance"),
    and the per-step cutoff exchange of `dp_protocol` admits completions
    globally.  Returns (t_end, accepted in acceptance order, deferred,
    unissued), prompt indices."""
    L = np.asarray(L, np.int64)
    n, G = L.shape
    if kind == LONG:
        target = n
    INF = np.iinfo(np.int64).max
    parts = partition(n, world)
    tau, C, last = np.zeros(n, np.int64), np.full(n, INF), 0
    for lo, hi in parts:
        if hi > lo:
            ta, Ca, d, _, _, _ = _issue_schedule(L[lo:hi], cap, kind, max_active, keep)
            tau[lo:hi], C[lo:hi] = ta, Ca
            last = max(last, int(np.max(ta + d - 1)))
    acc, accepted, t = 0, [], 0
    while True:
        t += 1
        before = acc
        total = 0
        for lo, hi in parts:
            comp = [i for i in range(lo, hi) if C[i] == t]
            take = min(len(comp), max(0, target - before - total))
            accepted.extend(comp[:take])
            total += take
        acc += total
        if acc == target or t >= last:
            break
    unissued = [i for i in range(n) if tau[i] > t]
    deferred = [i for i in range(n) if i not in set(accepted) and i not in set(unissued)]
    return t, accepted, deferred, unissued


def issue_closed_form(L, cap, target, kind, max_active, keep=None, with_steps=False):
    """The same round from its definition as list scheduling: prompt i is
    active for d_i steps (T_i if it completes, else its longest response,
    e = min(L, cap)), independent of when it is issued; prompts take the
    earliest-freed of `max_active` slots in index order (tau_i = 1 + the
    step the slot freed); prompt i completes at C_i = tau_i + T_i - 1; the
    first `target` by (C_i, i) are accepted and t_end is the target-th
    completion (else the last active step); prompts with tau_i > t_end are
    unissued."""
    L = np.asarray(L, np.int64)
    n, G = L.shape
    INF = np.iinfo(np.int64).max
    if kind == LONG:
        target = n
    tau, C, d, e0, e, kept = _issue_schedule(L, cap, kind, max_active, keep)
    order = sorted(range(n), key=lambda i: (C[i], i))
    n_fin = int(np.sum(C < INF))
    n_acc = min(target, n_fin)
    accepted = order[:n_acc]
    underfilled = n_fin < target
    t_end = int(C[order[target - 1]]) if not underfilled else int(np.max(tau + d - 1))
    unissued = [i for i in range(n) if tau[i] > t_end]
    deferred = [i for i in range(n) if i not in set(accepted) and i not in set(unissued)]
    end_abs = tau[:, None] + e - 1                      # last step each response decodes
    outcome = np.where(L <= cap, FINISHED, CAPPED)
    outcome = np.where((tau[:, None] + e0 - 1 > t_end) | ((e0 > e) & (kind == SHORT)), ABORTED, outcome)
    outcome[unissued] = UNISSUED
    retained = np.zeros_like(L)
    for i in accepted:
        retained[i] = np.where(kept[i], e0[i], 0)
    tau_out = tau.copy()
    tau_out[unissued] = 0
    r = IssueRound(kind, t_end, accepted, deferred, bool(underfilled), outcome.astype(np.int32), retained,
                   issue_step=tau_out, unissued=unissued)
    if with_steps:
        tflat, endf = np.repeat(tau, G), end_abs.reshape(-1)
        for t in range(1, t_end + 1):
            live = np.nonzero((tflat <= t) & (endf >= t))[0].astype(np.int32)
            acc = sum(1 for p in order[:n_acc] if C[p] <= t)
            r.steps.append(dict(t=t, live=live, accepted=acc,
                                done=int(acc == target or t == t_end)))
    return r


# ---------------------------------------------------------------- DP (C3)

def partition(n, world):
    """Contiguous ranges of global prompt indices per rank (first n % world
    ranks get one more)."""
    base, extra = divmod(n, world)
    out, lo = [], 0
    for r in range(world):
        hi = lo + base + (1 if r < extra else 0)
        out.append((lo, hi))
        lo = hi
    return out


def dp_protocol(L, cap, target, kind, world, keep=None):
    """The per-step DP cutoff exchange: each rank counts
    k_r(t), the prompts of its range completing at step t; after an
    all-gather rank r admits min(k_r, max(0, target - acc - sum_{r'<r} k_r'))
    of them, lowest index first.  Returns (t_end, accepted in acceptance
    order, per-rank live counts per step)."""
    L = np.asarray(L, np.int64)
    n, G = L.shape
    if kind == LONG:
        target = n
    e = _e(L, cap)
    if kind == SHORT:
        _, T = _kept(L, cap, G if keep is None else keep)
        e = np.minimum(e, T[:, None])
    else:
        T = e.max(axis=1)
    parts = partition(n, world)
    acc, accepted, t = 0, [], 0
    emax = int(e.max())
    live_counts = []
    while True:
        t += 1
        ks, comp = [], []
        for lo, hi in parts:
            c = [i for i in range(lo, hi) if T[i] == t]
            comp.append(c)
            ks.append(len(c))
        live_counts.append([int(np.sum(e[lo:hi] >= t)) for lo, hi in parts])
        before = acc
        for r in range(world):
            take = min(ks[r], max(0, target - before - sum(ks[:r])))
            accepted.extend(comp[r][:take])
            acc += take
        if acc == target or t >= emax:
            return t, accepted, live_counts


# ---------------------------------------------------------------- planner

def n_launch(P0, eta):
    """ceil(eta * P0) in exact rational arithmetic."""
    return math.ceil(Fraction(eta).limit_denominator(1000) * P0)


def plan_round(queue_len, P0, eta, tail_batching=True):
    """LONG over the first P0 queued prompts when |Q| >= P0, else a
    SHORT round launching ceil(eta*P0) fresh prompts with target P0;
    BASELINE (plain synchronous rollout) when tail batching is off.
    Returns (kind_name, n_prompts, target)."""
    if not tail_batching:
        return ("baseline", P0, P0)
    if queue_len >= P0:
        return ("long", P0, P0)
    return ("short", n_launch(P0, eta), P0)


def simulate(trace, n_rounds, P0, eta, G, short_cap, long_cap, tail_batching=True, n_launch_override=None):
    """Run `n_rounds` RL steps.  trace [n_prompts_total, 2, G] (attempt 0:
    first submission, attempt 1: long-round re-roll).  Returns a list of
    dicts {kind, ids, round: Round, queue_after}."""
    queue, nxt, out = deque(), 0, []
    for _ in range(n_rounds):
        kind, n, target = plan_round(len(queue), P0, eta, tail_batching)
        if kind == "short" and n_launch_override:
            n = n_launch_override
        if kind == "long":
            ids = [queue.popleft() for _ in range(P0)]
            r = closed_form(trace[ids, 1, :G], long_cap, target, LONG)
        elif kind == "baseline":
            ids = list(range(nxt, nxt + n)); nxt += n
            r = closed_form(trace[ids, 0, :G], long_cap, n, LONG)
        else:
            ids = list(range(nxt, nxt + n)); nxt += n
            r = closed_form(trace[ids, 0, :G], short_cap, target, SHORT)
            queue.extend(ids[i] for i in r.deferred)
        out.append(dict(kind=kind, ids=ids, round=r, queue_after=list(queue)))
    return out


# ------------------------------------------ KV pressure (NEXT-2)
#
# short rounds raise memory pressure and serving engines "alleviate
# memory pressure by preempting ongoing requests"; the planner
# "keeps track of the preemption counts and adapts the TP sizes ... a sudden
# rise in preemptions (e.g., >1.05x) triggers an increase in TP (doubling the
# size), while sustained zero preemptions across four steps trigger a
# decrease (halving the size)".  Readings (Z26):
#   * the KV pool holds n_pages pages of PAGE tokens; a prompt of plen tokens
#     holds ceil(plen / PAGE) prompt pages for the whole round (its G
#     responses share the floor(plen / PAGE) full ones) and each response a
#     private copy of the partial last prompt page, then private pages for
#     its generated tokens; a response that generated g tokens has written
#     kv = plen + g - 1 positions (token g is its next input) and holds
#     ceil(kv / PAGE) - floor(plen / PAGE) private pages;
#   * after the step's endings free their pages, the survivors need one page
#     each whose kv is a multiple of PAGE; while that exceeds the free pages
#     the most recently admitted prompt with a live response is preempted
#     (LIFO, whole prompt: all its live responses, their private pages
#     freed) and joins the back of a FIFO wait queue -- never the last live
#     prompt: if it alone does not fit, the pool is exhausted;
#   * preemption is by recompute: a step that preempts nothing re-admits
#     wait-queue prompts from the head while their pages fit --
#     sum over their preempted responses of ceil((plen + g) / PAGE) -
#     floor(plen / PAGE) (the recomputed prefix and the next append) -- after
#     the survivors' needs; a re-admitted response continues at token g + 1
#     in the next step (its KV for positions plen .. plen + g - 2 recomputed
#     between the two steps) and its prompt becomes the most recent admission;
#   * the next step's rows: the survivors in their order, then the
#     re-admitted responses (re-admission order, j ascending);
#   * a round whose live set is empty ends (plain rule) unless re-admission
#     refills it; no live row and a wait-queue head that does not fit, or a
#     single live prompt that does not fit, is KV exhaustion.

PAGE = 64
PREEMPTED = 5


class KVExhausted(Exception):
    pass


def _pages(x):
    return -(-int(x) // PAGE)


class KVRank:
    """One rank's round state under KV pressure (the per-rank part of
    `kv_step_loop`; the DP cutoff couples ranks only through `done`)."""

    def __init__(self, L, plen, cap, kind, n_pages, keep, first_prompt=0):
        self.L = np.asarray(L, np.int64)
        self.n, self.G = self.L.shape
        self.plen = [int(x) for x in plen]
        self.cap, self.kind, self.keep = cap, kind, keep
        self.own0 = [p // PAGE for p in self.plen]
        used = sum(_pages(p) for p in self.plen) + sum(self.G * (p % PAGE != 0) for p in self.plen)
        if used > n_pages:
            raise KVExhausted("prompt pages do not fit at submit")
        self.free = n_pages - used
        self.g = np.zeros((self.n, self.G), np.int64)
        self.kv = np.array([[p] * self.G for p in self.plen], np.int64)
        self.status = np.zeros((self.n, self.G), np.int32)           # 0 live / FINISHED / CAPPED / ABORTED / PREEMPTED
        self.kept = np.zeros((self.n, self.G), bool)
        self.cnt = [0] * self.n
        self.done_p = [False] * self.n
        self.adm = list(range(self.n))                                # admission order (oldest first)
        self.wait = []                                                # FIFO of preempted prompts
        self.live = [i * self.G + j for i in range(self.n) for j in range(self.G)]
        self.preemptions = 0
        self.first = first_prompt

    def step(self, t):
        """Decode step t on this rank.  Returns (decoded slots, prompts
        completed at t (local indices, ascending))."""
        G = self.G
        decoded = list(self.live)
        ending, completed = [], []
        for s in decoded:
            i, j = divmod(s, G)
            self.g[i, j] += 1
            if t >= 2:
                self.kv[i, j] += 1                     # the input token's KV was appended
            k = self.g[i, j]
            if k == self.L[i, j]:
                self.status[i, j] = FINISHED
                ending.append(s)
                if not self.done_p[i] and self.cnt[i] < self.keep:
                    self.cnt[i] += 1
                    self.kept[i, j] = True
                    if self.cnt[i] == self.keep:
                        completed.append(i)
            elif k == self.cap:
                self.status[i, j] = CAPPED
                ending.append(s)
                if self.kind == LONG:
                    self.cnt[i] += 1
                    self.kept[i, j] = True
                    if self.cnt[i] == G:
                        completed.append(i)
        for i in completed:
            self.done_p[i] = True
        ended = set(ending)
        for s in decoded:
            if s not in ended and self.done_p[s // G]:
                self.status[s // G, s % G] = ABORTED
                ended.add(s)
        for s in ended:
            i, j = divmod(s, G)
            self.free += _pages(self.kv[i, j]) - self.own0[i]
        self.survivors = [s for s in decoded if s not in ended]
        return decoded, sorted(completed)

    def pressure(self):
        """Preemption (LIFO whole prompts) until the survivors' next-step
        pages fit, then (if nothing was preempted) re-admission from the head
        of the wait queue.  Sets the next step's live list."""
        G = self.G
        need = lambda rows: sum(1 for s in rows if self.kv[s // G, s % G] % PAGE == 0)
        rows = list(self.survivors)
        preempted = False
        while need(rows) > self.free:
            live_p = set(s // G for s in rows)
            if len(live_p) <= 1:
                raise KVExhausted("the last live prompt does not fit")
            v = max(live_p, key=lambda i: self.adm.index(i))
            for s in [s for s in rows if s // G == v]:
                j = s % G
                self.free += _pages(self.kv[v, j]) - self.own0[v]
                self.status[v, j] = PREEMPTED
            rows = [s for s in rows if s // G != v]
            self.wait.append(v)
            self.preemptions += 1
            preempted = True
        avail = self.free - need(rows)
        self.free = avail
        if not preempted:
            while self.wait:
                v = self.wait[0]
                js = [j for j in range(G) if self.status[v, j] == PREEMPTED]
                req = sum(_pages(self.plen[v] + self.g[v, j]) - self.own0[v] for j in js)
                if req > self.free:
                    break
                self.wait.pop(0)
                self.free -= req
                for j in js:
                    self.status[v, j] = 0
                    self.kv[v, j] = self.plen[v] + self.g[v, j] - 1
                    rows.append(v * G + j)
                self.adm.remove(v)
                self.adm.append(v)
        if not rows and self.wait:
            v = self.wait[0]
            req = sum(_pages(self.plen[v] + self.g[v, j]) - self.own0[v] for j in range(G)
                      if self.status[v, j] == PREEMPTED)
            if req > self.free:
                raise KVExhausted("the wait-queue head can never fit")
        self.live = rows


def kv_step_loop(L, plen, cap, target, kind, n_pages, world=1, with_steps=False, keep=None):
    """Literal step loop of a round under KV pressure (readings above),
    sharded over `world` DP ranks (contiguous prompt ranges, `n_pages` pages
    per rank) with the per-step cutoff exchange of `dp_protocol`.  With
    enough pages it is `step_loop` / `dp_protocol` (a test).  Returns a Round
    whose steps carry each rank's decoded slots (local), plus `preemptions`
    (per rank) and `order` (each rank's final admission order)."""
    L = np.asarray(L, np.int64)
    n, G = L.shape
    keep = G if (keep is None or kind == LONG) else keep
    if kind == LONG:
        target = n
    parts = partition(n, world)
    ranks = [KVRank(L[lo:hi], plen[lo:hi], cap, kind, n_pages, keep, lo) for lo, hi in parts]
    accepted, steps = [], []
    t = 0
    while True:
        t += 1
        dec, comps = [], []
        for r in ranks:
            d, c = r.step(t)
            dec.append(d)
            comps.append(c)
        before = len(accepted)
        for (lo, hi), c in zip(parts, comps):          # rank order = prompt-index order
            take = min(len(c), max(0, target - len(accepted)))
            accepted.extend(lo + i for i in c[:take])
        for r in ranks:
            r.pressure()
        done = len(accepted) >= target or all(not r.live for r in ranks)
        if with_steps:
            steps.append(dict(t=t, live=[np.array(d, np.int32) for d in dec], accepted=len(accepted),
                              done=int(done)))
        if done:
            break
    outcome = np.zeros((n, G), np.int32)
    retained = np.zeros((n, G), np.int64)
    acc = set(accepted)
    for (lo, hi), r in zip(parts, ranks):
        st = r.status.copy()
        st[(st == 0) | (st == PREEMPTED)] = ABORTED
        outcome[lo:hi] = st
        for i in range(lo, hi):
            if i in acc:
                retained[i] = np.where(r.kept[i - lo], np.minimum(L[i], cap), 0)
    deferred = [i for i in range(n) if i not in accepted]
    rnd = Round(kind, t, accepted, deferred, len(accepted) < target, outcome, retained, steps)
    rnd.preemptions = [r.preemptions for r in ranks]
    return rnd


def plan_tp(tp, tp_max, prev_preemptions, preemptions, zero_streak):
    """The parallelism planner's heuristic: a sudden rise in
    preemptions (> 1.05x the previous round of the same kind) doubles the TP
    size (up to the GPUs of one server, tp_max); four consecutive rounds with
    zero preemptions halve it.  Returns (next tp, next zero streak)."""
    streak = zero_streak + 1 if preemptions == 0 else 0
    if preemptions > 0 and preemptions > 1.05 * prev_preemptions:
        return min(2 * tp, tp_max), 0
    if streak >= 4:
        return max(tp // 2, 1), 0
    return tp, streak
