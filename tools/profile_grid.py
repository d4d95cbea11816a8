"""Offline throughput profile ("benchmark
prefill/decode throughput vs TP, batch and sequence length"): decode-step time
of one model on a TP group of the launching size, over a grid of live batch B
and context length.  Run with plain python for TP = 1, under torchrun for
TP = 2 / 4:

  python -m torch.distributed.run --nproc-per-node 2 --master-addr 127.0.0.1 \
      tools/profile_grid.py --out gpurun_out/grid_tp2.json

Each point: B / G prompts of exactly `ctx` tokens (G = 8 siblings share the
prefix), a long round in trace mode with every response forced to length 64;
the graph-replayed decode steps 17..48 are timed with CUDA events (max over
ranks).  Points whose KV would not fit the pool are skipped.  The planner in
bench.py (--long-tp profile) reads the merged table.
"""
import argparse
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def workspace(rp, cfg, tp, rank, max_b, ctx, max_tok):
    """Workspace bytes of an engine with these capacities (rp_query_sizes, host only)."""
    import ctypes
    md, rd, sz = rp.model_desc(cfg, 0), rp.RuntimeDesc(), rp.Sizes()
    rd.rank, rd.world, rd.tp, rd.tp_rank = 0, 1, tp, rank
    rd.max_seqs, rd.max_prompts, rd.max_prompt_len = max_b, max(1, max_b // 8), ctx
    rd.max_prompt_tokens, rd.max_cap, rd.graph_steps, rd.kv_pool_bytes = max_tok, 64, 16, 1 << 30
    rd.sample_seed, rd.temperature = 3, 1.0
    dummy = ctypes.create_string_buffer(128)           # validate() wants an id for tp > 1
    rd.nccl_id = ctypes.cast(dummy, ctypes.c_void_p)
    if rp.lib().rp_query_sizes(ctypes.byref(md), ctypes.byref(rd), ctypes.byref(sz)):
        return float("inf")
    return sz.workspace_bytes


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--model", default="qwen2.5-7b")
    ap.add_argument("--batches", default="8,32,128,256")
    ap.add_argument("--ctx", default="1024,4096,16384")
    ap.add_argument("--out", default="")
    a = ap.parse_args()
    import torch
    import torch.distributed as dist
    from paper_2509_21009_b200 import rp
    from synth import configs, gen
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", "0")))
    if world > 1:
        dist.init_process_group("gloo")
    cfg = configs.model_config(a.model)
    G, steps_cap = 8, 64
    batches = [int(x) for x in a.batches.split(",")]
    ctxs = [int(x) for x in a.ctx.split(",")]
    max_b = max(batches)
    free = torch.cuda.mem_get_info()[0]
    rows = []
    for ctx in ctxs:
        # one engine per context length: the prefill workspace grows with
        # max_prompt_len x max_prompt_tokens, so take the largest prompt-token
        # budget of this row whose workspace leaves half the memory for KV
        cands = sorted({max(1, b // G) * ctx for b in batches}, reverse=True)
        max_tok = next((m for m in cands if workspace(rp, cfg, world, rank, max_b, ctx, m) < 0.55 * free), None)
        if max_tok is None:
            continue
        nccl_id = None
        if world > 1:
            obj = [rp.nccl_unique_id() if rank == 0 else None]
            dist.broadcast_object_list(obj, src=0)
            nccl_id = obj[0]
        eng = rp.Engine(cfg, max_seqs=max_b, max_prompts=max(1, max_b // G), max_prompt_len=ctx,
                        max_prompt_tokens=max_tok, max_cap=steps_cap, graph_steps=16, tp=world, tp_rank=rank,
                        nccl_id=nccl_id, sample_seed=configs.SAMPLE_SEED, kv_fraction=0.85)
        kv_tok_bytes = 2 * cfg["n_layers"] * (cfg["n_kv_heads"] // world) * cfg["head_dim"] * 2
        pool = eng.kv_pool.numel()
        if rank == 0:
            print("tp %d ctx %d: KV pool %.1f GB, max prompt tokens %d" % (world, ctx, pool / 1e9, max_tok), flush=True)
        for B in batches:
            n_p = max(1, B // G)
            need = n_p * G * (ctx + steps_cap + 64) * kv_tok_bytes
            if n_p * ctx > max_tok or need > 0.95 * pool:
                if rank == 0:
                    print("skip B=%d ctx=%d: KV %.1f GB / prompt tokens %d do not fit" % (B, ctx, need / 1e9, n_p * ctx),
                          flush=True)
                continue
            ps = gen.prompts(n_p, 0, cfg["eos_id"], (ctx, ctx), 1000 + ctx)
            L = np.full((n_p, G), steps_cap, np.int64)
            eng.submit(ps, G, steps_cap, n_p, long_round=True, trace=L, round_id=ctx + B)
            eng.step(16)                     # graph capture + warm-up
            if world > 1:
                dist.barrier()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(eng.stream)
            eng.step(32)
            e1.record(eng.stream)
            torch.cuda.synchronize()
            t = torch.tensor([e0.elapsed_time(e1) / 32.0], dtype=torch.float64)
            if world > 1:
                dist.all_reduce(t, op=dist.ReduceOp.MAX)
            eng.run()
            eng.collect()
            rows.append(dict(tp=world, B=n_p * G, ctx=ctx, ms_per_step=round(float(t.item()), 4),
                             tokens_per_s=round(n_p * G * 1e3 / float(t.item()), 1)))
            if rank == 0:
                print(json.dumps(rows[-1]), flush=True)
        eng.close()
        del eng
        torch.cuda.empty_cache()
    if rank == 0 and a.out:
        json.dump(dict(model=a.model, tp=world, G=G, points=rows,
                       method="decode steps 17..48 of a trace-mode long round, graph replay, CUDA events, "
                              "max over ranks"), open(a.out, "w"), indent=1)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
