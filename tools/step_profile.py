"""Per-kernel-class profile of eager decode steps at several live-batch sizes
during one bench round (first short round of the C2-7b workload)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch
    from paper_2509_21009_b200 import rp
    import bench
    W = bench.Workload("C2-7b", 1)
    lo, hi = W.R["prompt_len"]
    eng = rp.Engine(W.model, max_seqs=W.n_submit * W.G, max_prompts=W.n_submit, max_prompt_len=hi,
                    max_prompt_tokens=W.n_submit * hi, max_cap=W.R["short_cap"], graph_steps=16)
    kind, ids, target, cap, L = W.plan()
    eng.submit([W.prompts[i] for i in ids], W.G, cap, target, trace=L, round_id=0)
    marks = [int(x) for x in (sys.argv[1:] or ["256", "128", "64", "32", "16"])]
    st = eng.step(0)
    for b in marks:
        while not st.done and st.n_live > b:
            st = eng.step(16)
        if st.done:
            break
        import time
        torch.cuda.synchronize()
        n0, t0 = st.t, time.perf_counter()
        st = eng.step(64)
        torch.cuda.synchronize()
        gms = (time.perf_counter() - t0) * 1e3 / max(1, st.t - n0)
        if st.done:
            break
        eng.debug_profile_arm(16)
        st = eng.step(16)
        p = eng.debug_profile_read()
        tot = sum(p["ms"].values())
        print("B~%d rows/step=%.1f ctx/row=%.0f eager_step_ms=%.3f graph_step_ms=%.3f" % (
            b, p["rows"] / p["steps"], p["ctx"] / max(1, p["rows"]), tot / p["steps"], gms))
        print("   " + "  ".join("%s=%.3f" % (k, v / p["steps"]) for k, v in p["ms"].items() if v > 0))
    eng.close()


if __name__ == "__main__":
    main()
