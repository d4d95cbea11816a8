"""Whole-round per-kernel-class profile of the bench workload (C2-7b, one
GPU): the first short round and the first long round are decoded eagerly with
CUDA events around every launch (rp_debug_profile), the other short rounds
in graph mode.  Prints one JSON object per profiled round: ms per class
summed over the round, share, mean live rows and mean context per row.

  python tools/round_profile.py [--out gpurun_out/round_profile.json]
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default="")
    ap.add_argument("--rounds", type=int, default=5)
    a = ap.parse_args()
    import torch
    from paper_2509_21009_b200 import rp
    import bench
    W = bench.Workload("C2-7b", 1)
    lo, hi = W.R["prompt_len"]
    eng = rp.Engine(W.model, max_seqs=W.n_submit * W.G, max_prompts=W.n_submit, max_prompt_len=hi,
                    max_prompt_tokens=W.n_submit * hi, max_cap=max(W.R["short_cap"], W.R["long_cap"]),
                    graph_steps=16)
    out, seen = [], set()
    for rnd in range(a.rounds):
        kind, ids, target, cap, L = W.plan()
        eng.submit([W.prompts[i] for i in ids], W.G, cap, target, long_round=(kind == "long"), trace=L,
                   round_id=rnd)
        prof = kind not in seen
        seen.add(kind)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        if prof:
            eng.debug_profile_arm(1 << 30)
        st = eng.run()
        torch.cuda.synchronize()
        wall = time.perf_counter() - t0
        res = eng.collect()
        W.commit(kind, ids, list(dict.fromkeys(r["prompt_id"] for r in res)))
        if prof:
            p = eng.debug_profile_read()
            eng.debug_profile_arm(-1)
            tot = sum(p["ms"].values())
            row = dict(kind=kind, t_end=st.t, decoded=st.decoded_tokens, eager_wall_s=round(wall, 2),
                       kernel_ms=round(tot, 1), mean_rows=round(p["rows"] / max(1, p["steps"]), 1),
                       mean_ctx=round(p["ctx"] / max(1, p["rows"]), 0),
                       classes={k: dict(ms=round(v, 1), share=round(v / tot, 4)) for k, v in
                                sorted(p["ms"].items(), key=lambda kv: -kv[1]) if v > 0})
            print(json.dumps(row), flush=True)
            out.append(row)
        else:
            print(json.dumps(dict(kind=kind, t_end=st.t, decoded=st.decoded_tokens, graph_wall_s=round(wall, 2))),
                  flush=True)
    eng.close()
    if a.out:
        json.dump(out, open(a.out, "w"), indent=1)


if __name__ == "__main__":
    main()
