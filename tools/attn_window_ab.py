"""Decode attention on the bench's own live sets: the first 7B short round of
bench.py (32 prompts x G = 8, trace mode) stepped with graphs, and at a series
of steps a window of 4 eager profiled steps (CUDA events around every launch)
reports the attention us per launch, the live rows and the mean context.
Run twice with the library switch to compare kernels on identical windows:
  RP_ATTN_GROUP=0 python tools/attn_window_ab.py --tag rows
  RP_ATTN_GROUP_MIN=0 python tools/attn_window_ab.py --tag group
One JSON line per window."""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--tag", default="")
    ap.add_argument("--at", default="2,30,80,150,250,400,600,900,1300,1800,2300")
    a = ap.parse_args()
    import torch
    from paper_2509_21009_b200 import rp
    from synth import configs, gen
    torch.cuda.set_device(0)
    cfg = configs.model_config("qwen2.5-7b")
    R = configs.ROUNDS["C2-7b"]
    tr = R["trace"]
    n, G, cap, target = 32, 8, R["short_cap"], 25
    ps = gen.prompts(n, 0, cfg["eos_id"], R["prompt_len"], configs.PROMPT_SEED)
    L = gen.length_trace(n, G, tr["mu0"], tr["sigma_p"], tr["sigma_r"], tr["l_max"], configs.TRACE_SEED)[:, 0, :]
    eng = rp.Engine(cfg, max_seqs=256, max_prompts=32, max_prompt_len=768, max_prompt_tokens=32 * 768,
                    max_cap=cap, graph_steps=16, kv_fraction=0.5, sample_seed=configs.SAMPLE_SEED)
    eng.submit(ps, G, cap, target, trace=L, round_id=3)
    t = 1
    for at in [int(x) for x in a.at.split(",")]:
        if at > t:
            st = eng.step(at - t)
            t = st.t
            if st.done:
                break
        eng.debug_profile_arm(4)
        st = eng.step(4)
        p = eng.debug_profile_read()
        eng.debug_profile_arm(-1)
        t = st.t
        att = p["ms"]["attention"] / max(1, p["launches"]["attention"]) * 1e3
        print(json.dumps(dict(tag=a.tag, t=t, rows=p["rows"] / max(1, p["steps"]), ctx=p["ctx"] / max(1, p["rows"]),
                              attention_us=round(att, 2))), flush=True)
        if st.done:
            break
    eng.run()
    eng.collect()
    eng.close()


if __name__ == "__main__":
    main()
