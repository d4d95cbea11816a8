"""BASELINE.json configs[4] analogue: tail batching vs plain synchronous
rollout on the same prompt stream and length trace (Qwen2.5-7B-shaped, one
GPU, 32 prompts x G=8 submitted per short round, P0 = 25).

  tail batching  -- the planner of S:271-279: short rounds of ceil(1.25 P0)
                    prompts (cap 8192) accepting the first P0, long rounds of
                    P0 queued prompts (attempt-1 lengths, cap 8192);
  plain sync     -- every RL step decodes P0 fresh prompts to completion
                    ("rollout must complete before training begins";
                    the veRL baseline), i.e. a long round on fresh prompts;
  tail + resp.   -- tail batching with response-level speculation as well
                    (eta = 1.25 for P and R): short
                    rounds launch ceil(1.25 R0) = 10 responses per prompt and
                    keep the first R0 = 8; long rounds run R0 without
                    speculation.

Both retain exactly P0 x G responses per RL step.  Reports rollout
seconds per RL step and tokens/s for each mode and median:max ratio.
All modes read the same 10-response trace (8-response modes use j < 8).
Usage: python tools/sweep_c5.py [--steps 5] [--ratios 25,28,32] [--modes tail,sync,tailpr] [--out f.json]
"""
import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

SIGMA_R = {25: 0.83, 28: 0.86, 32: 0.9}     # per-prompt sigma giving the batch median:max ratio


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--ratios", default="25,32")
    ap.add_argument("--out", default="")
    ap.add_argument("--modes", default="tail,sync,tailpr")
    a = ap.parse_args()
    import torch
    from paper_2509_21009_b200 import rp
    from synth import configs, gen
    cfg = configs.model_config("qwen2.5-7b")
    n_sub, P0, G, cap = 32, 25, 8, 8192
    G_spec = 10                                   # ceil(1.25 * R0)
    eng = rp.Engine(cfg, max_seqs=n_sub * G_spec, max_prompts=n_sub, max_prompt_len=768, max_prompt_tokens=n_sub * 768,
                    max_cap=cap, graph_steps=16)
    out = []
    for ratio in [int(x) for x in a.ratios.split(",")]:
        total = n_sub * (a.steps + 2) * 2
        ps = gen.prompts(total, 0, cfg["eos_id"], (256, 768), configs.PROMPT_SEED)
        tr = gen.length_trace(total, G_spec, 6.0, 0.6, SIGMA_R.get(ratio, 0.85), 16384, configs.TRACE_SEED)
        big = gen.length_trace(128 * 40, G, 6.0, 0.6, SIGMA_R.get(ratio, 0.85), 16384, 99)[:, 0, :]
        meas = float(np.median([b.max() / np.median(b) for b in big.reshape(-1, 128 * G)]))
        for mode in a.modes.split(","):
            queue, nxt, times, toks, kinds = [], 0, [], 0, []
            for step in range(a.steps):
                Gr, keep = G, 0
                if mode == "sync":
                    ids = list(range(nxt, nxt + P0)); nxt += P0
                    L = tr[ids, 0, :G]
                    kind, target, long_round = "baseline", P0, True
                elif len(queue) >= P0:
                    ids, queue = queue[:P0], queue[P0:]
                    L = tr[ids, 1, :G]
                    kind, target, long_round = "long", P0, True
                else:
                    ids = list(range(nxt, nxt + n_sub)); nxt += n_sub
                    if mode == "tailpr":
                        Gr, keep = G_spec, G
                    L = tr[ids, 0, :Gr]
                    kind, target, long_round = "short", P0, False
                torch.cuda.synchronize()
                t0 = time.perf_counter()
                eng.submit([ps[i] for i in ids], Gr, cap, target, long_round=long_round, trace=L, round_id=step,
                           keep=keep)
                st = eng.run()
                res = eng.collect()
                torch.cuda.synchronize()
                times.append(time.perf_counter() - t0)
                toks += st.decoded_tokens
                kinds.append(kind)
                if kind == "short":
                    acc = set(r["prompt_id"] for r in res)
                    queue += [i for i in ids if i not in acc]
            row = dict(ratio=ratio, measured_median_max=round(meas, 1), mode=mode, steps=a.steps, kinds="".join(
                k[0].upper() for k in kinds), s_per_rl_step=round(float(np.mean(times)), 3),
                max_round_s=round(float(np.max(times)), 3), decoded_tokens_per_s=round(toks / sum(times), 1))
            print(json.dumps(row), flush=True)
            out.append(row)
    eng.close()
    if a.out:
        json.dump(out, open(a.out, "w"), indent=1)


if __name__ == "__main__":
    main()
