"""Run the bench workload's first 7B round for a bounded number of eager
decode steps (no graphs: one launch per kernel, so ncu can select them) and
exit.  Used under ncu:  python tools/ncu_step.py --steps 3"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--skip", type=int, default=0, help="decode steps to run (graphs) before the eager ones")
    ap.add_argument("--config", default="C2-7b")
    ap.add_argument("--graph-steps", type=int, default=0)
    ap.add_argument("--kv-fraction", type=float, default=0.5)
    a = ap.parse_args()
    import torch
    from paper_2509_21009_b200 import rp
    import bench
    W = bench.Workload(a.config, 1)
    lo, hi = W.R["prompt_len"]
    eng = rp.Engine(W.model, max_seqs=W.n_submit * W.G, max_prompts=W.n_submit, max_prompt_len=hi,
                    max_prompt_tokens=W.n_submit * hi, max_cap=W.R["short_cap"], graph_steps=a.graph_steps,
                    kv_fraction=a.kv_fraction)
    kind, ids, target, cap, L = W.plan()
    eng.submit([W.prompts[i] for i in ids], W.G, cap, target, trace=L, round_id=0)
    if a.skip:
        done = 0
        while done < a.skip:
            st = eng.step(100)
            done += 100
            print("t=%d live=%d done=%d" % (st.t, st.n_live, st.done), flush=True)
            if st.done:
                break
    st = eng.step(a.steps)
    torch.cuda.synchronize()
    print("ok t=%d live=%d" % (st.t, st.n_live), flush=True)
    eng.close()


if __name__ == "__main__":
    main()
