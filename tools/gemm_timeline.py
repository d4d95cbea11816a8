import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ["RP_GEMM_TIMELINE"] = "1"
import torch
from paper_2509_21009_b200 import rp
from synth.configs import model_config
torch.cuda.set_device(0)
eng = rp.Engine(model_config("tiny"), max_seqs=256, max_prompts=16, max_prompt_len=64, max_prompt_tokens=512,
                max_cap=64, kv_pool_bytes=64 << 20, graph_steps=0)
for M, K in [(37888, 3584), (4608, 3584), (3584, 18944), (152064, 3584)]:
    W = (torch.randn(M, K, device="cuda") * 0.02).to(torch.bfloat16)
    X = torch.randn(512, K, device="cuda").to(torch.bfloat16)
    for N in (16, 256):
        _, ms = eng.debug_gemm(W, X, N, splits=0, iters=10, timed=True)
        print("M=%d K=%d N=%d: %.1f us" % (M, K, N, ms * 1e3), flush=True)
    del W, X
