"""Time the tcgen05 GEMM alone on the decode shapes (back-to-back launches,
CUDA events) at several live-batch sizes; prints GB/s and TFLOP/s."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch
    from paper_2509_21009_b200 import rp
    from synth.configs import model_config
    torch.cuda.set_device(0)
    eng = rp.Engine(model_config("tiny"), max_seqs=256, max_prompts=16, max_prompt_len=64, max_prompt_tokens=512,
                    max_cap=64, kv_pool_bytes=64 << 20, graph_steps=0)
    shapes = {"qkv": (4608, 3584), "o": (3584, 3584), "gu": (37888, 3584), "down": (3584, 18944),
              "lm": (152064, 3584)}
    only = sys.argv[1:] or list(shapes)
    for name in only:
        M, K = shapes[name]
        W = (torch.randn(M, K, device="cuda") * 0.02).to(torch.float16)
        X = torch.randn(512, K, device="cuda").to(torch.float16)
        for N in (16, 64, 128, 256):
            for sp in (0, 1, 2, 4, 8):
                try:
                    _, ms = eng.debug_gemm(W, X, N, splits=sp, iters=20, timed=True)
                except rp.RPError as e:
                    continue
                by = M * K * 2 + N * K * 2 + N * M * 4
                print("%-5s N=%3d splits=%s  %8.1f us  %7.0f GB/s  %6.0f TFLOP/s" % (
                    name, N, sp or "auto", ms * 1e3, by / ms / 1e6, 2 * M * N * K / ms / 1e9))
        del W, X
    eng.close()


if __name__ == "__main__":
    main()
