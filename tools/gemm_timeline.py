"""Per-CTA phase timeline (RP_GEMM_TIMELINE, printed by the library to stderr)
of single GEMM launches at the 7B decode shapes, weights in the model's tiled
layout and split-precision activations (X_lo) as in the decode step; L2
flushed before each.  Then the mean time of 10 back-to-back launches.

  python tools/gemm_timeline.py 16 32 64
"""
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
shapes = [(4608, 3584, "qkv"), (3584, 3584, "o"), (37888, 3584, "gate/up"), (3584, 18944, "down")]
for M, K, name in shapes:
    W = (torch.randn(M, K, device="cuda") * 0.02).to(torch.float16)
    X32 = torch.randn(512, K, device="cuda")
    X = X32.to(torch.float16)
    X_lo = (X32 - X.float()).to(torch.float16)
    for N in [int(x) for x in (sys.argv[1:] or ["16", "32", "64"])]:
        flush.fill_(1)
        torch.cuda.synchronize()
        print("%s M=%d K=%d N=%d:" % (name, M, K, N), flush=True)
        _, ms = eng.debug_gemm(W, X, N, splits=0, iters=10, timed=True, tiled=True, X_lo=X_lo)
        torch.cuda.synchronize()
        print("  %.1f us per launch (10 back-to-back)" % (ms * 1e3), flush=True)
    del W, X, X_lo, X32
