"""DP x TP with real NCCL communicators (one process per GPU): run under
torchrun on 4 GPUs (gpurun --gpus 4) as 2 replicas x TP 2:
    python -m torch.distributed.run --nproc-per-node 4 --master-addr 127.0.0.1 tests/test_gpu_dpxtp.py
Rank g is replica g // tp, tp rank g % tp; the DP group (nccl_id) joins the
ranks with the same tp rank, the TP group (tp_nccl_id) the ranks of a
replica.  A short round on the KV = 8 tiny variant: per-rank schedule vs the
single-rank oracle, identical tokens inside each replica, the global queue
on every rank, then the planned LONG round popped from it."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch
    import torch.distributed as dist
    from oracle import sched
    from paper_2509_21009_b200 import rp
    from synth import configs, gen
    world_all = int(os.environ["WORLD_SIZE"]); g = int(os.environ["RANK"]); local = int(os.environ["LOCAL_RANK"])
    tp = int(os.environ.get("RP_TEST_TP", "2"))
    dp = world_all // tp
    r, q = divmod(g, tp)
    torch.cuda.set_device(local)
    dist.init_process_group("gloo")
    ids = [[rp.nccl_unique_id() for _ in range(tp)], [rp.nccl_unique_id() for _ in range(dp)]] if g == 0 else None
    obj = [ids]
    dist.broadcast_object_list(obj, src=0)
    dp_ids, tp_ids = obj[0]
    cfg = configs.model_config("tiny-kv8")
    eng = rp.Engine(cfg, max_seqs=64, max_prompts=16, max_prompt_len=128, max_prompt_tokens=1024, max_cap=512,
                    kv_pool_bytes=256 << 20, graph_steps=4, rank=r, world=dp, nccl_id=dp_ids[q], tp=tp, tp_rank=q,
                    tp_nccl_id=tp_ids[r], tp_peer=False, sample_seed=configs.SAMPLE_SEED)
    n, G, cap, target = 10, 3, 96, 7
    ps = gen.prompts(n, 0, cfg["eos_id"], (4, 60), 61)
    tr = gen.length_trace(n, G, 3.4, 0.6, 0.85, 300, 12)
    L = tr[:, 0, :]
    eng.submit(ps, G, cap, target, trace=L, trace_retry=tr[:, 1, :], round_id=5)
    st = eng.run()
    res = eng.collect()
    ref = sched.closed_form(L, cap, target, sched.SHORT)
    lo, hi = sched.partition(n, dp)[r]
    ok = st.t == ref.t_end and eng.long_queue() == [ps[i]["prompt_id"] for i in ref.deferred]
    ok = ok and all(lo <= x["prompt_id"] < hi and x["len"] == L[x["prompt_id"], x["j"]] for x in res)
    key = [(x["prompt_id"], x["j"], x["tokens"].tolist()) for x in res]
    allk = [None] * world_all
    dist.all_gather_object(allk, key)
    ok = ok and allk[g] == allk[r * tp]                     # identical tokens inside the replica
    acc = sorted(set(p for k in allk[::tp] for p, _, _ in k))
    ok = ok and acc == sorted(ps[i]["prompt_id"] for i in ref.accepted)
    kind, m = eng.plan(len(eng.long_queue()), 1.25) if eng.long_queue() else ("short", 0)
    if kind == "long":
        eng.submit(None, G, cap, m, long_round=True, round_id=6, trace_mode=True)
        st2 = eng.run()
        res2 = eng.collect()
        L2 = tr[ref.deferred, 1, :]
        ok = ok and st2.t == sched.closed_form(L2, cap, m, sched.LONG).t_end and eng.long_queue() == []
        lo2, hi2 = sched.partition(m, dp)[r]
        ok = ok and len(res2) == (hi2 - lo2) * G
    print("rank %d (replica %d, tp %d): t_end %d/%d ok=%s" % (g, r, q, st.t, ref.t_end, ok), flush=True)
    eng.close()
    flag = torch.tensor([1 if ok else 0])
    dist.all_reduce(flag, op=dist.ReduceOp.MIN)
    dist.destroy_process_group()
    if g == 0:
        print("DPxTP PARITY", "PASS" if flag.item() == 1 else "FAIL")
    sys.exit(0 if flag.item() == 1 else 1)


if __name__ == "__main__":
    main()
