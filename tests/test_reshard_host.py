"""Host logic of rp_round_reshard (NEXT-3 migration across DP world sizes,
reading Z27), on the CPU: synthetic exported rank states -- built here with
the layout include/rollpacker.h documents (header words, control block, then
the step-state sections) -- re-sharded to another world size.  Checks that
every prompt's per-response and per-prompt state lands in the right slot of
the right new rank, that the next step's inputs are rebuilt from the live
responses in slot order (last token, position, page-table row, one attention
item per row), that the local acceptance order is (completion step, index),
that the global counters are kept and the measurement counters summed onto
the new rank 0, and that mismatched inputs are rejected."""
import ctypes

import numpy as np
import pytest

from paper_2509_21009_b200 import rp

ST_LIVE, ST_FINISHED, ST_CAPPED = 0, 1, 2
PS_RUNNING, PS_ACCEPTED, PS_COMPLETE = 0, 1, 2
MAGIC = 0x3153525052


class Ctl(ctypes.Structure):          # kernels.h CtlBlock
    _fields_ = [(n, ctypes.c_int) for n in ("n_live", "t", "acc", "acc_local", "done", "err", "n_final", "t_end",
                                             "underfilled", "k_step", "n_next", "n_items", "free_top", "need_pages")] + \
               [("decoded", ctypes.c_longlong), ("ctx_sum", ctypes.c_longlong), ("kv_read", ctypes.c_longlong)] + \
               [(n, ctypes.c_int) for n in ("n_issued", "issue_n", "preemptions", "wait_head", "wait_tail", "adm_ctr",
                                             "readmit_n", "readmit_rows", "readmit_pages", "pause", "n_live_saved",
                                             "n_items_saved", "n_gitems", "n_gitems_saved", "n_rejobs")] + \
               [("kv_read_unique", ctypes.c_longlong)]


ITEM, GITEM = 32, 192                 # sizeof(AttnItem), sizeof(AttnGroupItem)
S, P, CAP, U = 16, 6, 40, 6
MI = S + U                            # max_items_dec; the group list holds S + MI


def sizes():
    return [ctypes.sizeof(Ctl), S * 4, S * 4, S * 4, S * 4, MI * ITEM, (S + MI) * GITEM, S * 4, S * 4, S * 4, S * 4,
            S * CAP * 4, P * 4, P * 4, P * 4, (S + 1) * 8, P * 4, P * 4, P * 4]


def part(n, world, r):
    base, extra = n // world, n % world
    return r * base + min(r, extra), base + (1 if r < extra else 0)


def make_world(n, G, world, plen, gen, status, pstate, t, acc):
    """Exported states of `world` ranks from global per-response arrays."""
    states = []
    for r in range(world):
        lo, nl = part(n, world, r)
        secs = [bytearray(x) for x in sizes()]
        c = Ctl(t=t, acc=acc, n_issued=nl, decoded=100 + r, kv_read=1000 + r)
        kv = np.zeros(S, np.int32); gn = np.zeros(S, np.int32); st = np.full(S, 3, np.int32)
        tok = np.zeros((S, CAP), np.int32)
        for li in range(nl):
            for j in range(G):
                s, gs = li * G + j, (lo + li) * G + j
                gn[s] = gen[gs]; st[s] = status[gs]; kv[s] = plen[lo + li] + gen[gs] - 1
                tok[s, :gen[gs]] = 7000 + 100 * gs + np.arange(gen[gs])
        secs[7][:] = kv.tobytes(); secs[8][:] = gn.tobytes(); secs[9][:] = st.tobytes(); secs[11][:] = tok.tobytes()
        secs[12][:] = np.array([pstate[lo + li] if li < nl else 0 for li in range(P)], np.int32).tobytes()
        hist = np.zeros(S + 1, np.uint64); hist[3] = 10 + r
        secs[15][:] = hist.tobytes()
        c.acc_local = sum(1 for li in range(nl) if pstate[lo + li] == PS_ACCEPTED)
        secs[0][:] = bytes(c)
        hdr = np.array([MAGIC, S, P, CAP, MI, ctypes.sizeof(Ctl), G, nl, 0, G, world, 1, r], np.int64)
        states.append(hdr.tobytes() + b"".join(bytes(x) for x in secs))
    return states


def split(blob):
    off, out = 13 * 8, []
    for x in sizes():
        out.append(blob[off:off + x])
        off += x
    return np.frombuffer(blob[:13 * 8], np.int64), out


def test_reshard_two_ranks_to_one_and_three():
    n, G = 5, 2
    plen = [70, 10, 130, 64, 5]
    # prompt 0 accepted at step 9 (lengths 9, 4), prompt 1 complete-not-accepted, prompt 2 accepted at
    # step 6 (6, 6), prompts 3-4 running (prompt 4: one response finished, one live)
    gen = [4, 9, 12, 12, 6, 6, 12, 12, 3, 12]
    status = [ST_FINISHED, ST_FINISHED, ST_FINISHED, ST_FINISHED, ST_FINISHED, ST_FINISHED,
              ST_LIVE, ST_LIVE, ST_FINISHED, ST_LIVE]
    pstate = [PS_ACCEPTED, PS_COMPLETE, PS_ACCEPTED, PS_RUNNING, PS_RUNNING]
    t = 13
    states = make_world(n, G, 2, plen, gen, status, pstate, t, acc=2)
    out = rp.reshard_round_states(states, n, 1)
    assert len(out) == 1
    hdr, sec = split(out[0])
    assert list(hdr) == [MAGIC, S, P, CAP, MI, ctypes.sizeof(Ctl), G, n, 0, G, 1, 1, 0]
    c = Ctl.from_buffer_copy(sec[0])
    assert c.t == t and c.acc == 2 and c.acc_local == 2 and c.decoded == 201 and c.kv_read == 2001
    gn = np.frombuffer(sec[8], np.int32); st = np.frombuffer(sec[9], np.int32)
    kv = np.frombuffer(sec[7], np.int32); tok = np.frombuffer(sec[11], np.int32).reshape(S, CAP)
    assert list(gn[:n * G]) == gen and list(st[:n * G]) == status
    assert list(kv[:n * G]) == [plen[s // G] + gen[s] - 1 for s in range(n * G)]
    assert all(tok[s, gen[s] - 1] == 7000 + 100 * s + gen[s] - 1 for s in range(n * G))
    assert list(np.frombuffer(sec[12], np.int32)[:n]) == pstate
    # live responses in slot order: 6, 7, 9; their last token, position, page-table row
    live = [6, 7, 9]
    assert c.n_live == 3 and c.n_items == 3 and c.n_gitems == 0
    assert list(np.frombuffer(sec[1], np.int32)[:3]) == live
    assert list(np.frombuffer(sec[2], np.int32)[:3]) == [7000 + 100 * s + gen[s] - 1 for s in live]
    assert list(np.frombuffer(sec[3], np.int32)[:3]) == [kv[s] for s in live]
    assert list(np.frombuffer(sec[4], np.int32)[:3]) == live
    assert c.ctx_sum == sum(int(kv[s]) + 1 for s in live)
    it = np.frombuffer(sec[5], np.int32).reshape(MI, 8)[:3]
    for k, s in enumerate(live):                  # q_row0, n_qtok, pos0, pt_row, kv_lo, kv_hi, nsplit, item0
        assert list(it[k]) == [k, 1, kv[s], s, 0, kv[s] + 1, 1, k]
    # acceptance order by completion step: prompt 2 (step 6) before prompt 0 (step 9)
    assert list(np.frombuffer(sec[14], np.int32)[:2]) == [2, 0]
    assert np.frombuffer(sec[15], np.uint64)[3] == 21
    # and to three ranks: slices [0, 2), [2, 4), [4, 5)
    out3 = rp.reshard_round_states(states, n, 3)
    for r, blob in enumerate(out3):
        hdr, sec = split(blob)
        lo, nl = part(n, 3, r)
        assert hdr[7] == nl and hdr[10] == 3 and hdr[12] == r
        c = Ctl.from_buffer_copy(sec[0])
        gn = np.frombuffer(sec[8], np.int32)
        assert list(gn[:nl * G]) == gen[lo * G:(lo + nl) * G]
        want_live = [s - lo * G for s in (6, 7, 9) if lo * G <= s < (lo + nl) * G]
        assert c.n_live == len(want_live)
        assert list(np.frombuffer(sec[1], np.int32)[:c.n_live]) == want_live
        assert c.decoded == (201 if r == 0 else 0)
    # rank 0 of the 3-way split holds prompts 0 and 1: only prompt 0 is accepted there
    c0 = Ctl.from_buffer_copy(split(out3[0])[1][0])
    assert c0.acc_local == 1


def test_reshard_rejects_bad_inputs():
    n, G = 4, 2
    gen = [3] * 8
    status = [ST_LIVE] * 8
    states = make_world(n, G, 2, [20, 20, 20, 20], gen, status, [PS_RUNNING] * 4, 4, 0)
    with pytest.raises(rp.RPError):
        rp.reshard_round_states(states[:1], n, 1)               # not every old rank
    with pytest.raises(rp.RPError):
        rp.reshard_round_states([states[1], states[0]], n, 1)   # rank order
    with pytest.raises(rp.RPError):
        rp.reshard_round_states(states, n + 1, 1)               # slices do not match n_prompts
    bad = bytearray(states[0])
    bad[0] ^= 1
    with pytest.raises(rp.RPError):
        rp.reshard_round_states([bytes(bad), states[1]], n, 1)  # not a round state
    with pytest.raises(rp.RPError):
        rp.reshard_round_states(states, n, 0)                   # new world
