"""Plain fp64 Qwen2-shaped decoder.  TEST
INFRASTRUCTURE ONLY (see oracle/__init__.py).

The paper's actor is "the Qwen2.5 family" decoded by vLLM;
it prints no architecture, so the structure follows the public Qwen2 model
(reading Z13/§2):

    h   = RMSNorm(x) * g1                         (eps = rms_eps)
    q,k,v = h Wq^T + bq, h Wk^T + bk, h Wv^T + bv
    q,k = RoPE(q,k; pos)                          (rotate-half, theta)
    a   = softmax(q k^T / sqrt(hd) + causal) v    (GQA: head h reads kv head h // g)
    x   = x + a Wo^T
    h2  = RMSNorm(x) * g2
    x   = x + (silu(h2 Wg^T) * (h2 Wu^T)) Wd^T
    logits = RMSNorm(x) * gf  W_lm^T              (untied, no bias)

Positions: the prompt occupies 0..n-1 and response token t is fed at
position n+t-1 (reading Z16).  Everything is computed in float64 from the
exact bf16 weight values; no blocking, fusion or reordering.
"""
import numpy as np


def rmsnorm(x, g, eps):
    """x / sqrt(mean(x^2) + eps) * g, row-wise."""
    x = np.asarray(x, np.float64)
    return x / np.sqrt(np.mean(x * x, axis=-1, keepdims=True) + eps) * np.asarray(g, np.float64)


def rope(x, pos, theta):
    """Rotate-half RoPE.  x [..., T, hd], pos [T].  Frequencies
    inv_freq_i = theta^(-2i/hd), i < hd/2; angle = pos * inv_freq."""
    hd = x.shape[-1]
    inv = theta ** (-np.arange(0, hd, 2, dtype=np.float64) / hd)
    ang = np.asarray(pos, np.float64)[:, None] * inv[None, :]          # [T, hd/2]
    cos = np.concatenate([np.cos(ang), np.cos(ang)], axis=-1)
    sin = np.concatenate([np.sin(ang), np.sin(ang)], axis=-1)
    x1, x2 = x[..., : hd // 2], x[..., hd // 2:]
    rot = np.concatenate([-x2, x1], axis=-1)
    return x * cos + rot * sin


def softmax(s, axis=-1):
    m = np.max(s, axis=axis, keepdims=True)
    e = np.exp(s - m)
    return e / np.sum(e, axis=axis, keepdims=True)


def silu(x):
    return x / (1.0 + np.exp(-x))


def attention(q, k, v, causal=True):
    """q [H, T, hd], k/v [KV, S, hd]; query i attends to keys j <= i + (S - T)."""
    H, T, hd = q.shape
    KV, S, _ = k.shape
    g = H // KV
    out = np.empty((H, T, hd), np.float64)
    for h in range(H):
        s = q[h] @ k[h // g].T / np.sqrt(hd)                              # [T, S]
        if causal:
            i = np.arange(T)[:, None] + (S - T)
            j = np.arange(S)[None, :]
            s = np.where(j <= i, s, -np.inf)
        out[h] = softmax(s) @ v[h // g]
    return out


def layer_forward(x, w, cfg, pos):
    """One decoder layer over a full sequence x [T, d] at positions pos."""
    H, KV, hd, eps = cfg["n_heads"], cfg["n_kv_heads"], cfg["head_dim"], cfg["rms_eps"]
    f64 = lambda a: np.asarray(a, np.float64)
    h = rmsnorm(x, w["ln1"], eps)
    q = h @ f64(w["q"]).T
    k = h @ f64(w["k"]).T
    v = h @ f64(w["v"]).T
    if "bq" in w:
        q, k, v = q + f64(w["bq"]), k + f64(w["bk"]), v + f64(w["bv"])
    T = x.shape[0]
    q = q.reshape(T, H, hd).transpose(1, 0, 2)
    k = k.reshape(T, KV, hd).transpose(1, 0, 2)
    v = v.reshape(T, KV, hd).transpose(1, 0, 2)
    q = rope(q, pos, cfg["rope_theta"])
    k = rope(k, pos, cfg["rope_theta"])
    a = attention(q, k, v, causal=True).transpose(1, 0, 2).reshape(T, H * hd)
    x = x + a @ f64(w["o"]).T
    h2 = rmsnorm(x, w["ln2"], eps)
    x = x + (silu(h2 @ f64(w["gate"]).T) * (h2 @ f64(w["up"]).T)) @ f64(w["down"]).T
    return x


def hidden(weights, tokens):
    """Final-norm hidden states [T, d] of a full token sequence."""
    cfg = weights.cfg
    tokens = np.asarray(tokens, np.int64)
    x = np.asarray(weights.embed_rows(tokens), np.float64)
    pos = np.arange(len(tokens))
    for l in range(cfg["n_layers"]):
        x = layer_forward(x, weights.layer(l), cfg, pos)
    return rmsnorm(x, weights.final_norm(), cfg["rms_eps"])


def logits(weights, tokens, rows=None):
    """Teacher-forced logits [T, V] (float64) of the sequence `tokens`;
    row i is the distribution of token i+1.  `rows` selects output rows."""
    h = hidden(weights, tokens)
    if rows is not None:
        h = h[np.asarray(rows)]
    return h @ np.asarray(weights.lm_head(), np.float64).T


class KVDecoder:
    """Incremental decode with a per-layer K/V cache -- the same arithmetic
    as `logits` (used for the CPU-baseline timing of decode steps; its
    equality with `logits` is a test)."""

    def __init__(self, weights):
        self.w, self.cfg = weights, weights.cfg
        self.k = [None] * self.cfg["n_layers"]
        self.v = [None] * self.cfg["n_layers"]
        self.n = 0

    def fork(self):
        """An independent decoder with the same cache (the G responses of a
        prompt continue one shared prompt prefix; `step` never writes the
        cached arrays in place, so sharing them is safe)."""
        d = KVDecoder(self.w)
        d.k, d.v, d.n = list(self.k), list(self.v), self.n
        return d

    def step(self, tokens, head=True):
        """Feed tokens [T] at positions n..n+T-1; returns logits [T, V], or
        with head=False the final-norm hidden states [T, d] (the caller
        applies the LM head, e.g. in vocab chunks)."""
        cfg = self.cfg
        H, KV, hd, eps = cfg["n_heads"], cfg["n_kv_heads"], cfg["head_dim"], cfg["rms_eps"]
        f64 = lambda a: np.asarray(a, np.float64)
        tokens = np.asarray(tokens, np.int64)
        T = len(tokens)
        pos = np.arange(self.n, self.n + T)
        x = np.asarray(self.w.embed_rows(tokens), np.float64)
        for l in range(cfg["n_layers"]):
            w = self.w.layer(l)
            h = rmsnorm(x, w["ln1"], eps)
            q, k, v = h @ f64(w["q"]).T, h @ f64(w["k"]).T, h @ f64(w["v"]).T
            if "bq" in w:
                q, k, v = q + f64(w["bq"]), k + f64(w["bk"]), v + f64(w["bv"])
            q = rope(q.reshape(T, H, hd).transpose(1, 0, 2), pos, cfg["rope_theta"])
            k = rope(k.reshape(T, KV, hd).transpose(1, 0, 2), pos, cfg["rope_theta"])
            v = v.reshape(T, KV, hd).transpose(1, 0, 2)
            self.k[l] = k if self.k[l] is None else np.concatenate([self.k[l], k], axis=1)
            self.v[l] = v if self.v[l] is None else np.concatenate([self.v[l], v], axis=1)
            a = attention(q, self.k[l], self.v[l], causal=True).transpose(1, 0, 2).reshape(T, H * hd)
            x = x + a @ f64(w["o"]).T
            h2 = rmsnorm(x, w["ln2"], eps)
            x = x + (silu(h2 @ f64(w["gate"]).T) * (h2 @ f64(w["up"]).T)) @ f64(w["down"]).T
        self.n += T
        h = rmsnorm(x, self.w.final_norm(), eps)
        if not head:
            return h
        return h @ np.asarray(self.w.lm_head(), np.float64).T
