"""Per-CTA phase timeline (RP_GEMM_TIMELINE) of single GEMM launches with L2
flushed before each, at the decode shapes of the 7B model."""
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
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
shapes = [(4608, 3584), (3584, 3584), (37888, 3584), (3584, 18944)]
for M, K in shapes:
    W = (torch.randn(M, K, device="cuda") * 0.02).to(torch.float16)
    X = torch.randn(512, K, device="cuda").to(torch.float16)
    for N in [int(x) for x in (sys.argv[1:] or ["16", "32", "64"])]:
        for sp in (0,):
            flush.fill_(1)
            torch.cuda.synchronize()
            _, ms = eng.debug_gemm(W, X, N, splits=sp, iters=10, timed=True)
            print("M=%d K=%d N=%d: %.1f us (10 back-to-back, L2-warm if W fits)" % (M, K, N, ms * 1e3), flush=True)
    del W, X
