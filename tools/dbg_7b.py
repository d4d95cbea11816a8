import os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import torch
from paper_2509_21009_b200 import rp
from synth import configs, gen
cfg = configs.model_config("qwen2.5-7b", n_layers=int(os.environ.get("NL", "2")))
stage = sys.argv[1]
eng = rp.Engine(cfg, max_seqs=64, max_prompts=8, max_prompt_len=768, max_prompt_tokens=4096, max_cap=256,
                kv_pool_bytes=int(os.environ.get("KVB", str(8 << 30))), graph_steps=0)
print("init ok", flush=True)
n = int(os.environ.get("NT", "100"))
toks = np.arange(1, n + 1, dtype=np.int32)
if stage == "logits":
    t = time.time(); lg = eng.debug_logits(toks); print("logits ok", lg.shape, np.abs(lg).max(), time.time() - t, flush=True)
else:
    ps = gen.prompts(8, 0, cfg["eos_id"], (n, n), 1)
    L = np.full((8, 8), 40, np.int32)
    eng.submit(ps, 8, 64, 6, trace=L); print("submit ok", flush=True)
    st = eng.step(5); print("step ok", st.t, flush=True)
    st = eng.run(); print("run ok", st.t, flush=True)
