"""Decode-step A/B tool: graph-replayed 7B decode-step time (CUDA events on
the engine stream, steps 17..48 of a long round) and the per-kernel-class
eager profile (events around every launch, gated) at several live batches.
Each point: B / 8 prompts of `ctx` tokens x G = 8 (siblings share the prompt
pages), responses forced to length 64 (trace mode).  Env switches of the
library (RP_*) select the variant; prints one JSON line per point.

  python tools/step_ab.py --batches 16,64,256 --ctx 1024 [--tag name]
"""
import argparse
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--model", default="qwen2.5-7b")
    ap.add_argument("--batches", default="16,64,256")
    ap.add_argument("--ctx", type=int, default=1024)
    ap.add_argument("--tag", default="")
    ap.add_argument("--layers", type=int, default=0)
    ap.add_argument("--G", type=int, default=8, help="responses per prompt (1: no sibling sharing)")
    a = ap.parse_args()
    import torch
    from paper_2509_21009_b200 import rp
    from synth import configs, gen
    torch.cuda.set_device(0)
    cfg = configs.model_config(a.model, n_layers=a.layers or None)
    batches = [int(x) for x in a.batches.split(",")]
    G, cap = a.G, 64
    maxb = max(batches)
    eng = rp.Engine(cfg, max_seqs=maxb, max_prompts=maxb // G, max_prompt_len=a.ctx,
                    max_prompt_tokens=maxb // G * a.ctx, max_cap=cap, graph_steps=16, kv_fraction=0.5)
    for B in batches:
        n = B // G
        ps = gen.prompts(n, 0, cfg["eos_id"], (a.ctx, a.ctx), 11)
        L = np.full((n, G), cap, np.int32)
        eng.submit(ps, G, cap, n, long_round=True, trace=L, round_id=1)
        eng.step(16)                                     # steps 2..17 (graph capture + warm)
        s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s0.record(eng.stream)
        st = eng.step(32)                                # steps 18..49
        s1.record(eng.stream)
        s1.synchronize()
        graph_ms = s0.elapsed_time(s1) / 32
        eng.debug_profile_arm(8)
        eng.step(8)
        p = eng.debug_profile_read()
        eng.debug_profile_arm(-1)
        eng.run()
        eng.collect()
        tot = sum(p["ms"].values())
        row = dict(tag=a.tag, B=B, G=G, ctx=a.ctx, graph_step_ms=round(graph_ms, 4), eager_step_ms=round(tot / p["steps"], 4),
                   cls={k: round(v / p["steps"] * 1e3 / max(1, p["launches"][k] / p["steps"]), 2)
                        for k, v in p["ms"].items() if v > 0})
        print(json.dumps(row), flush=True)
    eng.close()


if __name__ == "__main__":
    main()
