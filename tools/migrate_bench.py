"""Cost of migrating an in-flight 7B round (NEXT-3, rp_round_export /
rp_round_import): the bench's first short round (32 prompts of 256-768 tokens
x G = 8, trace mode) is decoded to step t on one engine, exported, the engine
freed, and imported into a fresh engine, which recomputes the live responses'
KV; then both the import time and the time the first engine spent reaching
step t are reported (what a restart from scratch would repeat), and the
import engine finishes the round.  One JSON line.

  python tools/migrate_bench.py --t 200 400
"""
import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--t", type=int, nargs="+", default=[200])
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
    kw = dict(max_seqs=256, max_prompts=32, max_prompt_len=768, max_prompt_tokens=32 * 768, max_cap=cap,
              graph_steps=16, kv_fraction=0.5, sample_seed=configs.SAMPLE_SEED)
    out = []
    for t_cut in a.t:
        e1 = rp.Engine(cfg, **kw)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        e1.submit(ps, G, cap, target, trace=L, round_id=3)
        st = e1.step(t_cut - 1)
        torch.cuda.synchronize()
        reach_s = time.perf_counter() - t0
        t1 = time.perf_counter()
        state = e1.export_round()
        export_s = time.perf_counter() - t1
        live = st.n_live
        e1.close()
        del e1
        torch.cuda.empty_cache()
        e2 = rp.Engine(cfg, **kw)
        torch.cuda.synchronize()
        t2 = time.perf_counter()
        e2.import_round(state, ps, G, cap, target, trace=L, round_id=3)
        torch.cuda.synchronize()
        import_s = time.perf_counter() - t2
        st2 = e2.run()
        res = e2.collect()
        e2.close()
        del e2
        torch.cuda.empty_cache()
        out.append(dict(t_cut=st.t, live_rows=live, state_bytes=len(state), export_s=round(export_s, 4),
                        import_s=round(import_s, 4), reach_s=round(reach_s, 3), t_end=st2.t,
                        accepted=st2.accepted, retained=len(res)))
        print(json.dumps(out[-1]), flush=True)


if __name__ == "__main__":
    main()
