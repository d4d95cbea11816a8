"""Multi-GPU (DP) parity: run under torchrun with 2+ GPUs (gpurun --gpus 2):
    python -m torch.distributed.run --nproc-per-node 2 --master-addr 127.0.0.1 tests/test_gpu_dp.py
Every rank submits the same prompt list and decodes its contiguous slice; the
per-step cutoff is exchanged with an NCCL all-gather inside the CUDA graph.
The schedule (t_end, accepted set, FIFO) must equal the single-rank oracle
schedule bit-exactly, and every rank must report the same global status."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch
    import torch.distributed as dist
    from oracle import sched
    from paper_2509_21009_b200 import dp, rp
    from synth import configs, gen
    world = int(os.environ["WORLD_SIZE"]); rank = int(os.environ["RANK"]); local = int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dist.init_process_group("gloo")
    obj = [rp.nccl_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    cfg = configs.model_config("tiny")
    n, G, cap = 13, 4, 128
    eng = rp.Engine(cfg, max_seqs=64, max_prompts=16, max_prompt_len=128, max_prompt_tokens=1024, max_cap=512,
                    kv_pool_bytes=64 << 20, graph_steps=4, rank=rank, world=world, nccl_id=obj[0])
    ok = True
    fifo = []
    for seed in range(5):
        # seeds 3, 4: response-level speculation, G = 5 launched, R0 = 4 kept
        Gs, keep = (G, None) if seed < 3 else (5, 4)
        ps = gen.prompts(n, 0, cfg["eos_id"], (1, 100), 40 + seed)
        L = gen.length_trace(n, Gs, 3.4, 0.6, 0.85, 600, seed)[:, 0, :]
        target = 10
        eng.submit(ps, Gs, cap, target, trace=L, round_id=seed, keep=keep or 0)
        st = eng.run()
        res = eng.collect()
        acc_local = list(dict.fromkeys(r["prompt_id"] for r in res))
        acc = dp.all_gather_ids(acc_local)
        ref = sched.closed_form(L, cap, target, sched.SHORT, keep=keep)
        lo, hi = dp.partition(n, world)[rank]
        fifo += [ps[i]["prompt_id"] for i in ref.deferred]   # the global queue, identical on every rank
        good = (st.t == ref.t_end and sorted(acc) == sorted(ps[i]["prompt_id"] for i in ref.accepted)
                and st.accepted == len(ref.accepted)
                and all(lo <= r["prompt_id"] - ps[0]["prompt_id"] < hi for r in res)
                and eng.long_queue() == fifo)
        for r in res:
            i = r["prompt_id"] - ps[0]["prompt_id"]
            good = good and r["len"] == L[i, r["j"]] and ref.retained_len[i, r["j"]] == r["len"]
        good = good and len(res) == sum(int(np.count_nonzero(ref.retained_len[i])) for i in range(lo, hi))
        print("rank %d seed %d t_end %d/%d accepted %d/%d ok=%s" % (rank, seed, st.t, ref.t_end, st.accepted,
                                                                  len(ref.accepted), good), flush=True)
        ok = ok and good
    # continuous issuance (NEXT-4): at most A prompts active per rank, issued
    # rank-locally; the cutoff exchange is unchanged
    for seed, A, tg in ((5, 3, 7), (6, 2, 5), (7, 2, 4)):
        ps = gen.prompts(n, 0, cfg["eos_id"], (2, 100), 40 + seed)
        L = gen.length_trace(n, G, 3.4, 0.6, 0.85, 300, seed)[:, 0, :]
        eng.issue_cap(A)
        eng.submit(ps, G, cap, tg, trace=L, round_id=seed)
        st = eng.run()
        res = eng.collect()
        acc = dp.all_gather_ids(list(dict.fromkeys(r["prompt_id"] for r in res)))
        t_end, r_acc, r_def, r_un = sched.issue_dp_protocol(L, cap, tg, sched.SHORT, world, A)
        lo, hi = dp.partition(n, world)[rank]
        fifo += [ps[i]["prompt_id"] for i in r_def]
        good = (st.t == t_end and sorted(acc) == sorted(ps[i]["prompt_id"] for i in r_acc)
                and eng.long_queue() == fifo
                and eng.unissued() == [ps[i]["prompt_id"] for i in r_un if lo <= i < hi])
        for r in res:
            good = good and r["len"] == L[r["prompt_id"] - ps[0]["prompt_id"], r["j"]]
        print("rank %d issue seed %d t_end %d/%d accepted %d unissued %d ok=%s" % (
            rank, seed, st.t, t_end, len(acc), len(r_un), good), flush=True)
        ok = ok and good
    eng.issue_cap(0)
    eng.close()
    # full size, in the launch configuration bench.py times at N GPUs: the
    # first short round of the C2-7b workload (32 prompts x G=8 per GPU,
    # graphs of 16 steps, data-parallel over the world) against the
    # single-rank oracle schedule
    import bench
    W = bench.Workload("C2-7b", world)
    lo, hi = W.R["prompt_len"]
    n_loc = -(-W.n_submit // world)
    obj = [rp.nccl_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    eng = rp.Engine(W.model, max_seqs=n_loc * W.G, max_prompts=n_loc, max_prompt_len=hi,
                    max_prompt_tokens=n_loc * hi, max_cap=W.R["short_cap"], graph_steps=16, rank=rank,
                    world=world, nccl_id=obj[0], kv_fraction=0.85)
    kind, ids, target, cap, L = W.plan()
    eng.submit([W.prompts[i] for i in ids], W.G, cap, target, trace=L, round_id=0)
    st = eng.run()
    res = eng.collect()
    ref = sched.closed_form(L, cap, target, sched.SHORT)
    acc = dp.all_gather_ids(list(dict.fromkeys(r["prompt_id"] for r in res)))
    lo_r, hi_r = dp.partition(len(ids), world)[rank]
    good = (st.t == ref.t_end and sorted(acc) == sorted(ids[i] for i in ref.accepted) and
            all(lo_r <= ids.index(r["prompt_id"]) < hi_r and r["len"] == L[ids.index(r["prompt_id"]), r["j"]]
                for r in res))
    print("rank %d full-size 7B short round: t_end %d/%d accepted %d/%d ok=%s" % (
        rank, st.t, ref.t_end, st.accepted, len(ref.accepted), good), flush=True)
    ok = ok and good
    eng.close()
    flag = torch.tensor([1 if ok else 0])
    dist.all_reduce(flag, op=dist.ReduceOp.MIN)
    dist.destroy_process_group()
    if rank == 0:
        print("DP PARITY", "PASS" if flag.item() == 1 else "FAIL")
    sys.exit(0 if flag.item() == 1 else 1)


if __name__ == "__main__":
    main()
