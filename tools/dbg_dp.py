import os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import torch
import torch.distributed as dist
world = int(os.environ["WORLD_SIZE"]); rank = int(os.environ["RANK"]); local = int(os.environ["LOCAL_RANK"])
def log(*a):
    print("[r%d %.1f]" % (rank, time.time() % 1000), *a, flush=True)
torch.cuda.set_device(local)
dist.init_process_group("gloo")
log("pg ok")
from paper_2509_21009_b200 import rp
from synth import configs, gen
obj = [rp.nccl_unique_id() if rank == 0 else None]
dist.broadcast_object_list(obj, src=0)
log("id ok")
cfg = configs.model_config("tiny")
gs = int(os.environ.get("GS", "0"))
eng = rp.Engine(cfg, max_seqs=64, max_prompts=16, max_prompt_len=128, max_prompt_tokens=1024, max_cap=512,
                kv_pool_bytes=64 << 20, graph_steps=gs, rank=rank, world=world, nccl_id=obj[0])
log("engine ok")
ps = gen.prompts(13, 0, cfg["eos_id"], (1, 100), 40)
L = gen.length_trace(13, 4, 3.4, 0.6, 0.85, 600, 0)[:, 0, :]
eng.submit(ps, 4, 128, 10, trace=L, round_id=0)
log("submit ok")
st = eng.step(1); log("step1", st.t, st.n_live, st.accepted)
st = eng.run(); log("run", st.t, st.accepted)
res = eng.collect(); log("collect", len(res))
eng.close()
dist.destroy_process_group()
log("done")
