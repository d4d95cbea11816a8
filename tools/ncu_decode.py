"""Decode steps of the bench workload's first round under profiler start/stop:
  python tools/ncu_decode.py SKIP STEPS   (graph steps to skip, then eager steps profiled)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch
    from paper_2509_21009_b200 import rp
    import bench
    skip = int(sys.argv[1]) if len(sys.argv) > 1 else 0
    steps = int(sys.argv[2]) if len(sys.argv) > 2 else 1
    W = bench.Workload("C2-7b", 1)
    lo, hi = W.R["prompt_len"]
    eng = rp.Engine(W.model, max_seqs=W.n_submit * W.G, max_prompts=W.n_submit, max_prompt_len=hi,
                    max_prompt_tokens=W.n_submit * hi, max_cap=W.R["short_cap"], graph_steps=16, kv_fraction=0.5)
    kind, ids, target, cap, L = W.plan()
    eng.submit([W.prompts[i] for i in ids], W.G, cap, target, trace=L, round_id=0)
    if skip:
        eng.step(skip)
    torch.cuda.synchronize()
    eng.debug_profile_arm(steps)
    torch.cuda.profiler.start()
    st = eng.step(steps)
    torch.cuda.synchronize()
    torch.cuda.profiler.stop()
    print("ok t=%d live=%d" % (st.t, st.n_live))
    eng.close()


if __name__ == "__main__":
    main()
