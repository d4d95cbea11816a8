"""Does the GEMM's speed depend on the activation magnitude (tensor-core
power under the power cap)?  Same shapes, X scaled by 1 and by 50."""
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
for M, K, N in [(37888, 3584, 256), (4608, 3584, 256), (37888, 3584, 64)]:
    W = (torch.rand(M, K, device="cuda") * 0.0693 - 0.0346).to(torch.float16)
    for scale in (1.0, 50.0, 1.0, 50.0):
        X = (torch.randn(512, K, device="cuda") * scale).to(torch.float16)
        _, ms = eng.debug_gemm(W, X, N, splits=0, iters=50, timed=True)
        print("M=%d K=%d N=%d |X| x%.0f: %.1f us" % (M, K, N, scale, ms * 1e3), flush=True)
