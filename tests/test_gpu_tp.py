"""Tensor-parallel (long-round) parity, run under torchrun on 2 GPUs:
    python -m torch.distributed.run --nproc-per-node 2 --master-addr 127.0.0.1 tests/test_gpu_tp.py
Checks (BASELINE.json north_star bars): teacher-forced logits gathered over
the vocab shards within 2e-2 of the fp64 oracle; a TP long round reproduces
the oracle schedule bit-exactly; both ranks produce identical tokens; sampled
tokens equal the oracle's Gumbel argmax wherever the top-2 gap > 1e-2."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch
    import torch.distributed as dist
    from oracle import decoder, sampler, sched, weights
    from paper_2509_21009_b200 import rp
    from synth import configs, gen
    world = int(os.environ["WORLD_SIZE"]); rank = int(os.environ["RANK"]); local = int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dist.init_process_group("gloo")
    obj = [rp.nccl_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    cfg = configs.model_config("tiny")
    w = weights.Weights(cfg, configs.WEIGHT_SEED)
    ok = True
    # decode all-reduce over NVLink peer memory (default), then the NCCL path
    for peer in (True, False):
        ok &= run_checks(rp, gen, sched, decoder, sampler, dist, cfg, w, world, rank, obj[0], peer)
    flag = torch.tensor([1 if ok else 0])
    dist.all_reduce(flag, op=dist.ReduceOp.MIN)
    dist.destroy_process_group()
    if rank == 0:
        print("TP PARITY", "PASS" if flag.item() == 1 else "FAIL")
    sys.exit(0 if flag.item() == 1 else 1)


def run_checks(rp, gen, sched, decoder, sampler, dist, cfg, w, world, rank, nccl_id, peer):
    if not peer:
        obj = [rp.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        nccl_id = obj[0]
    eng = rp.Engine(cfg, max_seqs=64, max_prompts=16, max_prompt_len=128, max_prompt_tokens=1024, max_cap=512,
                    kv_pool_bytes=64 << 20, graph_steps=4, tp=world, tp_rank=rank, nccl_id=nccl_id, tp_peer=peer)
    ok = eng.tp_peer == peer
    print("rank %d decode all-reduce: %s" % (rank, "NVLink peer push" if eng.tp_peer else "NCCL"), flush=True)
    # 1. teacher-forced logits, gathered over the vocab shards
    toks = gen.prompts(1, 0, cfg["eos_id"], (70, 70), 9)[0]["tokens"]
    part = eng.debug_logits(toks)
    parts = [None] * world
    dist.all_gather_object(parts, part)
    full = np.concatenate(parts, axis=1)
    err = float(np.max(np.abs(full - decoder.logits(w, toks))))
    print("rank %d tp logits max-abs %.3g" % (rank, err), flush=True)
    ok &= err <= 2e-2
    # 2. a long round in trace mode
    n, G = 6, 3
    ps = gen.prompts(n, 0, cfg["eos_id"], (5, 80), 21)
    L = np.minimum(gen.length_trace(n, G, 3.4, 0.6, 0.85, 600, 7)[:, 1, :], 150)
    eng.debug_trace_enable(300)
    eng.submit(ps, G, 120, n, long_round=True, trace=L, round_id=11)
    st = eng.run()
    ref = sched.closed_form(L, 120, n, sched.LONG, with_steps=True)
    got = eng.debug_trace(ref.t_end + 2)
    sched_ok = st.t == ref.t_end and len(got) == ref.t_end and all(
        np.array_equal(a["live"], b["live"]) and a["accepted"] == b["accepted"] for a, b in zip(got, ref.steps))
    res = eng.collect()
    all_res = [None] * world
    dist.all_gather_object(all_res, [(r["prompt_id"], r["j"], r["tokens"].tolist()) for r in res])
    same = all(a == all_res[0] for a in all_res)
    # 3. sampled tokens vs oracle (gap rule)
    checked = mism = 0
    gap_ok = True
    by_id = {p["prompt_id"]: (i, p["tokens"]) for i, p in enumerate(ps)}
    for r in res:
        i, p = by_id[r["prompt_id"]]
        seq = np.concatenate([p, r["tokens"]])
        lg = decoder.logits(w, seq[:-1], rows=np.arange(len(p) - 1, len(seq) - 1))
        for t in range(1, r["len"] + 1):
            tok, gap = sampler.sample(lg[t - 1], t, r["prompt_id"] * G + r["j"], 11, 3, eos_id=cfg["eos_id"],
                                      trace_len=L[i, r["j"]])
            checked += 1
            if tok != r["tokens"][t - 1]:
                mism += 1
                gap_ok &= gap <= 1e-2
    print("rank %d schedule %s identical-across-ranks %s sampled %d mismatches %d gap_ok %s" % (
        rank, sched_ok, same, checked, mism, gap_ok), flush=True)
    ok &= sched_ok and same and gap_ok and len(res) == n * G
    eng.close()
    return ok


if __name__ == "__main__":
    main()
