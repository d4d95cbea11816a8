"""World-size-2 (gloo, CPU) tests of the multi-rank host path: the contiguous
partition rule, the per-step cutoff exchange done with a real collective
(all_gather of {k_r, rows still live} every step, exactly the message the
CUDA graph all-gathers over NCCL), membership all-gather and the replicated
long-prompt FIFO -- compared with the single-rank oracle schedule."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import sched
from paper_2509_21009_b200 import dp
from synth import gen


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def rank_round(L, cap, target, kind, rank, world):
    """One round on this rank's slice with the per-step exchange over
    torch.distributed (mirror of ctl phase A -> all_gather -> phase B)."""
    n, G = L.shape
    lo, hi = dp.partition(n, world)[rank]
    Lr = np.asarray(L[lo:hi], np.int64)
    e = np.minimum(Lr, cap)
    fin_ok = (Lr <= cap) | (kind == sched.LONG)
    if kind == sched.LONG:
        target = n
    acc, accepted, t = 0, [], 0
    done_mask = np.zeros(hi - lo, bool)
    while True:
        t += 1
        comp = [i for i in range(hi - lo) if not done_mask[i] and np.all(fin_ok[i]) and int(e[i].max()) == t]
        for i in comp:
            done_mask[i] = True
        live_next = int(np.sum(e > t))
        msg = torch.tensor([len(comp), live_next], dtype=torch.int64)
        allm = [torch.zeros(2, dtype=torch.int64) for _ in range(world)]
        dist.all_gather(allm, msg)
        ks = [int(m[0]) for m in allm]
        total = 0
        for r in range(world):
            take = min(ks[r], max(0, target - acc - total))
            if r == rank:
                accepted += [lo + i for i in comp[:take]]
            total += take
        acc += total
        if acc >= target or sum(int(m[1]) for m in allm) == 0:
            return t, accepted


def worker(rank, world, port, out_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        tr = gen.length_trace(200, 4, 3.5, 0.6, 0.85, 400, 17)
        P0, n_sub = 10, 13
        q = dp.GlobalQueue()
        nxt, log = 0, []
        for rnd in range(12):
            if len(q) >= P0:
                ids = q.pop(P0)
                t, acc = rank_round(tr[ids, 1, :], 300, P0, sched.LONG, rank, world)
                kind = "long"
            else:
                ids = list(range(nxt, nxt + n_sub))
                nxt += n_sub
                t, acc_local = rank_round(tr[ids, 0, :], 64, P0, sched.SHORT, rank, world)
                acc = acc_local
                kind = "short"
            acc_ids = dp.all_gather_ids([ids[i] for i in acc])
            if kind == "short":
                q.defer(ids, acc_ids)
            log.append((kind, t, sorted(acc_ids), list(q.ids)))
        out_q.put((rank, log))
    finally:
        dist.destroy_process_group()


def reference_log():
    tr = gen.length_trace(200, 4, 3.5, 0.6, 0.85, 400, 17)
    out = sched.simulate(tr, 12, 10, 1.25, 4, 64, 300, n_launch_override=13)
    log = []
    for o in out:
        r = o["round"]
        log.append((o["kind"], r.t_end, sorted(o["ids"][i] for i in r.accepted), list(o["queue_after"])))
    return log


def test_partition_matches_library_rule():
    # engine.cu: lo = r*base + min(r, extra); n_loc = base + (r < extra)
    for n in range(1, 40):
        for w in range(1, 9):
            base, extra = divmod(n, w)
            got = dp.partition(n, w)
            for r in range(w):
                lo = r * base + min(r, extra)
                assert got[r] == (lo, lo + base + (1 if r < extra else 0))


@pytest.mark.parametrize("world", [2])
def test_dp_rounds_match_single_rank_oracle(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    logs = dict(q.get(timeout=240) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    ref = reference_log()
    for r in range(world):
        assert logs[r] == ref
    kinds = [x[0] for x in ref]
    assert "long" in kinds and "short" in kinds
