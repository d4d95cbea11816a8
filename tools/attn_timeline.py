"""Attention CTA timeline (RP_ATTN_TIMELINE) inside graph replays at several
live-batch sizes of the bench workload's first round."""
import os
import sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ.setdefault("RP_ATTN_TIMELINE", "1")


def main():
    from paper_2509_21009_b200 import rp
    import bench
    W = bench.Workload("C2-7b", 1)
    lo, hi = W.R["prompt_len"]
    eng = rp.Engine(W.model, max_seqs=W.n_submit * W.G, max_prompts=W.n_submit, max_prompt_len=hi,
                    max_prompt_tokens=W.n_submit * hi, max_cap=W.R["short_cap"], graph_steps=16)
    kind, ids, target, cap, L = W.plan()
    eng.submit([W.prompts[i] for i in ids], W.G, cap, target, trace=L, round_id=0)
    st = eng.step(0)
    for b in [int(x) for x in (sys.argv[1:] or ["256", "64", "16"])]:
        while not st.done and st.n_live > b:
            st = eng.step(16)
        if st.done:
            break
        sys.stderr.write("==== MARK B<=%d n_live=%d\n" % (b, st.n_live))
        st = eng.step(16)
        sys.stderr.write("==== END\n")
    eng.close()


if __name__ == "__main__":
    main()
