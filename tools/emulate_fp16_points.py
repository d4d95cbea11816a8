"""Which fp16 rounding points of the decode path matter at full depth (run by hand, ~15 min of CPU):

    python tests/emulate_activation_precision.py

The fp64 oracle decoder with its activations rounded at the GPU path's
rounding points (GEMM inputs h / attention output / SwiGLU output, q/k/v and
the KV cache, the attention probabilities P) to bf16 or fp16; teacher-forced
logits of an 8-token prompt on the full 28-layer 7B shape against plain fp64.
Measured: all bf16 0.1251, all fp16 0.0160, bf16 with any single point kept
exact 0.10-0.14 (no point dominates).  Test infrastructure only (oracle/).
"""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import time, numpy as np
from oracle import weights, decoder
from synth import configs, gen
cfg = configs.model_config("qwen2.5-7b")
weights.build_c()
def bf(x):
    x32 = np.asarray(x, np.float32)
    u = x32.view(np.uint32).astype(np.uint64)
    r = ((u + 0x7FFF + ((u >> 16) & 1)) >> 16) << 16
    return r.astype(np.uint32).view(np.float32).astype(np.float64)
def f16(x):
    return np.asarray(x, np.float64).astype(np.float16).astype(np.float64)
H, KV, hd, eps, d = cfg["n_heads"], cfg["n_kv_heads"], cfg["head_dim"], cfg["rms_eps"], cfg["d_model"]
ident = lambda a: a
def layer_bf(x, w, pos, R):
    f = lambda a: np.asarray(a, np.float64)
    r = 1.0 / np.sqrt(np.mean(x * x, -1, keepdims=True) + eps)
    hb = R["h"](x) ; sc = r
    q = (hb @ f(w["q"]).T) * sc + f(w["bq"]); k = (hb @ f(w["k"]).T) * sc + f(w["bk"]); v = (hb @ f(w["v"]).T) * sc + f(w["bv"])
    T = x.shape[0]
    q = decoder.rope(q.reshape(T, H, hd).transpose(1, 0, 2), pos, cfg["rope_theta"])
    k = decoder.rope(k.reshape(T, KV, hd).transpose(1, 0, 2), pos, cfg["rope_theta"])
    v = v.reshape(T, KV, hd).transpose(1, 0, 2)
    q, k, v = R["q"](q), R["k"](k), R["v"](v)
    g = H // KV
    out = np.empty((H, T, hd))
    for h in range(H):
        s = q[h] @ k[h // g].T / np.sqrt(hd)
        s = s + np.triu(np.full((T, T), -np.inf), 1)
        m = s.max(-1, keepdims=True); p = np.exp(s - m); l = p.sum(-1, keepdims=True)
        out[h] = (R["p"](p) @ v[h // g]) / l
    a = R["a"](out.transpose(1, 0, 2).reshape(T, H * hd))
    x = x + a @ f(w["o"]).T
    r2 = 1.0 / np.sqrt(np.mean(x * x, -1, keepdims=True) + eps)
    h2 = R["h2"](x)   # second layer norm (gate/up input)
    gt = (h2 @ f(w["gate"]).T) * r2; up = (h2 @ f(w["up"]).T) * r2
    mid = R["mid"](decoder.silu(gt) * up)
    return x + mid @ f(w["down"]).T
pts = ["h", "h2", "hf", "q", "k", "v", "p", "a", "mid"]   # h: first norm (QKV input), h2: second norm (gate/up), hf: final
def mk(exact):
    return {p: (ident if p in exact else f16) for p in pts}
combos = {"all_fp16": [], "q+a+mid": ["q", "a", "mid"], "q+h+a+mid": ["q", "h", "a", "mid"],
          "q+h2+a+mid": ["q", "h2", "a", "mid"], "q+h2+mid": ["q", "h2", "mid"]}
variants = {m: mk(ex) for m, ex in combos.items()}
w = weights.Weights(cfg, configs.WEIGHT_SEED, use_c=True)
toks = gen.prompts(1, 0, cfg["eos_id"], (56, 56), 6)[0]["tokens"]
pos = np.arange(56)
x64 = np.asarray(w.embed_rows(toks), np.float64)
xs = {m: x64.copy() for m in variants}
for l in range(cfg["n_layers"]):
    wl = w.layer(l)
    x64 = decoder.layer_forward(x64, wl, cfg, pos)
    for m, R in variants.items(): xs[m] = layer_bf(xs[m], wl, pos, R)
    w.drop_layer(l)
lm = w.lm_head()
h64 = decoder.rmsnorm(x64, w.final_norm(), eps)
for m, R in variants.items():
    r = 1.0 / np.sqrt(np.mean(xs[m]**2, -1, keepdims=True) + eps)
    hb = R["hf"](xs[m]) * r
    worst = 0.0
    for v0 in range(0, cfg["vocab"], 16384):
        W = np.asarray(lm[v0:v0+16384], np.float64)
        worst = max(worst, float(np.max(np.abs(hb @ W.T - h64 @ W.T))))
    print(m, "logits max-abs vs fp64: %.4f" % worst, flush=True)
