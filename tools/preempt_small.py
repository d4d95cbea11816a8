"""A small KV-pressure round on the tiny model (RP_PREEMPT, graphs of 4
steps) checked against the oracle's schedule; a driver for compute-sanitizer
runs (tools/gpu_sanitize.sh)."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch
    from paper_2509_21009_b200 import rp
    from oracle import sched
    from synth import configs, gen
    torch.cuda.set_device(0)
    cfg = configs.model_config("tiny")
    ps = gen.prompts(2, 0, cfg["eos_id"], (64, 64), 5)
    L = np.array([[130], [130]])
    page = cfg["n_layers"] * cfg["n_kv_heads"] * 2 * 64 * cfg["head_dim"] * 2
    eng = rp.Engine(cfg, max_seqs=16, max_prompts=4, max_prompt_len=128, max_prompt_tokens=256, max_cap=256,
                    kv_pool_bytes=5 * page, graph_steps=4)
    eng.submit(ps, 1, 200, 2, long_round=True, trace=L, round_id=1, preempt=True)
    st = eng.run()
    res = eng.collect()
    ref = sched.kv_step_loop(L, [64, 64], 200, 2, sched.LONG, 5)
    assert st.t == ref.t_end and st.preemptions == ref.preemptions[0] and len(res) == 2, (st.t, st.preemptions)
    eng.close()
    print("preempt_small ok: t_end %d preemptions %d" % (st.t, st.preemptions))


if __name__ == "__main__":
    main()
