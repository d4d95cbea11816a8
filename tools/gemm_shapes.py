"""Time single GEMM launches (rp_debug_gemm) at given shapes and split-K
factors: python tools/gemm_shapes.py M,K,N [M,K,N ...] [--splits 0,1,2]"""
import os
import sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
from paper_2509_21009_b200 import rp
from synth.configs import model_config
torch.cuda.set_device(0)
eng = rp.Engine(model_config("tiny"), max_seqs=256, max_prompts=16, max_prompt_len=64, max_prompt_tokens=512,
                max_cap=64, kv_pool_bytes=64 << 20, graph_steps=0)
args = sys.argv[1:]
splits = [0, 1, 2]
if "--splits" in args:
    i = args.index("--splits")
    splits = [int(x) for x in args[i + 1].split(",")]
    args = args[:i] + args[i + 2:]
for spec in args:
    M, K, N = (int(x) for x in spec.split(","))
    W = (torch.randn(M, K, device="cuda") * 0.02).to(torch.float16)
    X = torch.randn(512, K, device="cuda").to(torch.float16)
    for sp in splits:
        _, ms = eng.debug_gemm(W, X, N, splits=sp, iters=5, timed=True)
        us = ms * 1e3
        print("M=%d K=%d N=%d splits=%s: %.1f us  %.2f TB/s  %.0f TFLOP/s" % (
            M, K, N, sp or "auto", us, M * K * 2 / us / 1e6, 2.0 * M * N * K / us / 1e6), flush=True)
    del W, X
