"""a Qwen2.5-14B-shaped long round under tensor
parallelism (row a14, elastic TP); --model qwen2.5-32b gives the C4 long round.  Run under torchrun on N GPUs (N = 2 or 4):

  python -m torch.distributed.run --nproc-per-node 2 --master-addr 127.0.0.1 \
      tools/c3_long_round.py [--p0 32] [--cap 32768] [--out gpurun_out/c3_tp2.json]

Long-prompt queue recipe: the C2 trace generator (mu0 6.0,
sigma_p 0.6, sigma_r 0.85) with L_max = 32768, run through the C-1 oracle's
tail-batching planner (sched.simulate: eta = 1.25, P0 prompts per RL step,
short cap 8192) until its first LONG round; that round's P0 queued prompts
(default 128, the paper's batch) are decoded as re-rolls (trace
attempt 1, reading Z5) with speculation disabled, every response retained and
truncated at the cap.  --preempt runs the round under
KV pressure with recompute preemption (NEXT-2, RP_PREEMPT, reading Z26) and
checks t_end, the preemption count and the per-step live-row histogram
against the oracle sched.kv_step_loop at the engine's pool size (--kv-gb
caps the pool).  Rank 0 prints one JSON line.
"""
import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--p0", type=int, default=128)
    ap.add_argument("--preempt", action="store_true", help="KV-pressure recompute preemption (RP_PREEMPT)")
    ap.add_argument("--kv-gb", type=float, default=0.0, help="KV pool per GPU in GB (0: 85%% of free memory)")
    ap.add_argument("--model", default="qwen2.5-14b", help="qwen2.5-14b (C3) or qwen2.5-32b (C4 long round)")
    ap.add_argument("--cap", type=int, default=32768)
    ap.add_argument("--short-cap", type=int, default=8192)
    ap.add_argument("--out", default="")
    ap.add_argument("--profile-steps", type=int, default=0,
                    help="after 1000 graph steps, time this many eager steps per kernel class (not timed run)")
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
    G = 8
    lo, hi = 256, 768
    from oracle import sched
    n_pool = 4000
    tr = gen.length_trace(n_pool, G, 6.0, 0.6, 0.85, 32768, configs.TRACE_SEED)
    plan = sched.simulate(tr, 12, a.p0, 1.25, G, a.short_cap, a.cap)
    first_long = next(x for x in plan if x["kind"] == "long")
    queue = list(first_long["ids"])
    ps_all = gen.prompts(n_pool, 0, cfg["eos_id"], (lo, hi), configs.PROMPT_SEED)
    prompts = [ps_all[i] for i in queue]
    L = tr[queue, 1, :]
    nccl_id = None
    if world > 1:
        obj = [rp.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        nccl_id = obj[0]
    kw = dict(kv_pool_bytes=int(a.kv_gb * 1e9)) if a.kv_gb else dict(kv_fraction=0.85)
    eng = rp.Engine(cfg, max_seqs=a.p0 * G, max_prompts=a.p0, max_prompt_len=hi, max_prompt_tokens=a.p0 * hi,
                    max_cap=a.cap, graph_steps=16, tp=world, tp_rank=rank, nccl_id=nccl_id,
                    sample_seed=configs.SAMPLE_SEED, **kw)
    # warm-up: a short long-round of 2 prompts (graph capture, NCCL setup)
    eng.submit(prompts[:2], G, 64, 2, long_round=True, trace=np.minimum(L[:2], 64), round_id=999)
    eng.run()
    eng.collect()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    w0 = time.perf_counter()
    e0.record(eng.stream)
    eng.submit(prompts, G, a.cap, len(prompts), long_round=True, trace=L, round_id=1, preempt=a.preempt)
    prof = None
    if a.profile_steps:
        st = eng.step(1000)
        eng.debug_profile_arm(a.profile_steps)
        st = eng.step(a.profile_steps)
        prof = eng.debug_profile_read()
        eng.debug_profile_arm(-1)
    st = eng.run()
    res = eng.collect()
    e1.record(eng.stream)
    torch.cuda.synchronize()
    wall = time.perf_counter() - w0
    dev = e0.elapsed_time(e1) / 1e3
    t = torch.tensor([dev, wall], dtype=torch.float64)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    dev, wall = t.tolist()
    ok = (len(res) == len(prompts) * G and
          all(r["len"] == min(int(L[queue.index(r["prompt_id"])][r["j"]]), a.cap) for r in res))
    hist = eng.rows_histogram()
    oracle_check = None
    if a.preempt and rank == 0:
        plen = [len(p["tokens"]) for p in prompts]
        t0 = time.perf_counter()
        ref = sched.kv_step_loop(L, plen, a.cap, len(prompts), sched.LONG, eng.n_pages, with_steps=True)
        want = np.bincount([len(x["live"][0]) for x in ref.steps[1:]], minlength=len(hist))
        oracle_check = dict(t_end=ref.t_end, preemptions=ref.preemptions[0], pool_pages=int(eng.n_pages),
                            t_end_equal=ref.t_end == st.t, preemptions_equal=ref.preemptions[0] == st.preemptions,
                            live_rows_histogram_equal=bool(np.array_equal(hist, want[:len(hist)])),
                            oracle_s=round(time.perf_counter() - t0, 1))
    if rank == 0:
        line = dict(config="%s %s-shaped long round" % ("C3" if "14b" in a.model else "C4", a.model), tp=world, p0=len(prompts), G=G, cap=a.cap,
                    steps=st.t, decoded_tokens=st.decoded_tokens, retained=sum(r["len"] for r in res),
                    kv_tokens_read=st.kv_tokens_read, dev_s=round(dev, 3), wall_s=round(wall, 3),
                    tokens_per_s=round(st.decoded_tokens / dev, 1), ms_per_step=round(1e3 * dev / st.t, 3),
                    lengths_match_trace=bool(ok), max_len=int(min(L.max(), a.cap)),
                    preempt=a.preempt, preemptions=st.preemptions, oracle=oracle_check,
                    queue_recipe="the first LONG round of the C-1 oracle planner (sched.simulate, eta 1.25, P0 %d, "
                                 "short cap %d) on the C2 trace recipe with L_max 32768" % (len(prompts), a.short_cap))
        if prof:
            n = max(1, prof["steps"])
            line["profile"] = dict(rows=round(prof["rows"] / n, 1), ctx=round(prof["ctx"] / max(1, prof["rows"]), 0),
                                   ms_per_step={k: round(v / n, 3) for k, v in prof["ms"].items() if v > 0})
            line["note"] = "profiled run: eager steps inside the round, dev_s not a clean timing"
        print(json.dumps(line), flush=True)
        if a.out:
            json.dump(line, open(a.out, "w"), indent=1)
    eng.close()
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
