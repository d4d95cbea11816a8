"""Reach a small-batch, long-context decode state (16 sequences, ~3K tokens of
context), then run eager decode steps inside cudaProfilerStart/Stop so that
`ncu --profile-from-start off` captures only those steps."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import numpy as np
    import torch
    from paper_2509_21009_b200 import rp
    from synth import configs, gen
    steps = int(sys.argv[1]) if len(sys.argv) > 1 else 1
    warm = int(sys.argv[2]) if len(sys.argv) > 2 else 2200
    cfg = configs.model_config("qwen2.5-7b")
    eng = rp.Engine(cfg, max_seqs=64, max_prompts=8, max_prompt_len=768, max_prompt_tokens=2048, max_cap=8192,
                    graph_steps=16, kv_fraction=0.5)
    ps = gen.prompts(2, 0, cfg["eos_id"], (700, 768), 5)
    L = np.full((2, 8), 8000, np.int32)
    eng.submit(ps, 8, 8192, 2, long_round=True, trace=L)
    eng.step(warm)
    torch.cuda.synchronize()
    eng.debug_profile_arm(steps)       # eager launches for the profiled steps
    torch.cuda.profiler.start()
    st = eng.step(steps)
    torch.cuda.synchronize()
    torch.cuda.profiler.stop()
    p = eng.debug_profile_read()
    print("t=%d live=%d ctx/row=%.0f" % (st.t, st.n_live, p["ctx"] / max(1, p["rows"])))
    print("  ".join("%s=%.3f" % (k, v / max(1, p["steps"])) for k, v in p["ms"].items() if v > 0))
    eng.close()


if __name__ == "__main__":
    main()
