"""One timed launch set of the gate/up-shaped GEMM at N=256 (for ncu)."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
from paper_2509_21009_b200 import rp
from synth.configs import model_config
torch.cuda.set_device(0)
eng = rp.Engine(model_config("tiny"), max_seqs=256, max_prompts=16, max_prompt_len=64, max_prompt_tokens=512,
                max_cap=64, kv_pool_bytes=64 << 20, graph_steps=0)
M, K, N = 37888, 3584, int(sys.argv[1]) if len(sys.argv) > 1 else 256
W = (torch.rand(M, K, device="cuda") * 0.0693 - 0.0346).to(torch.float16)
X = torch.randn(512, K, device="cuda").to(torch.float16)
_, ms = eng.debug_gemm(W, X, N, splits=1, iters=3, timed=True)
print("us", ms * 1e3)
