"""Random-init weights of the Qwen2-shaped decoder (reading Z12).
TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

The paper trains real Qwen2.5 checkpoints; we have none, so every
weight is a formula of (weight_seed, tensor id, element index):

    x   = word (i & 3) of Philox4x32-10(ctr=(i >> 2, tid, 0, 0x57454947),
                                        key=(seed_lo, seed_hi))
    u   = ((x >> 9) + 0.5) * 2^-23                 exact in fp32, in (0,1)
    w32 = fl32(a * (2u - 1)),  a = fl32(0.02*sqrt(3))   (2u-1 is exact)
    w   = bf16_rne(w32)

i is the row-major index of the PyTorch-layout tensor [out, in] (or [n] for a
bias).  RMSNorm gains are exactly 1.  The sigma 0.02 follows Qwen2's
initializer_range.  Every value is returned as float32 holding the bf16
value exactly (widening is exact).

Tensor ids (DESIGN.md §3 Z12 table):
    embed 0x10000000, lm_head 0x10000001,
    layer l: 0x100*(l+1) + {q:0, k:1, v:2, bq:3, bk:4, bv:5, o:6, gate:7, up:8, down:9}
"""
import ctypes
import os

import numpy as np

from .philox import stream_words, philox4x32

_CLIB = os.path.join(os.path.dirname(os.path.abspath(__file__)), "c", "liboracle_weights.so")


def build_c():
    """Compile oracle/c/weights.c (gcc -O2 -fopenmp; -ffp-contract=off keeps
    the single fp32 rounding of the formula)."""
    import subprocess
    src = os.path.join(os.path.dirname(_CLIB), "weights.c")
    if os.path.exists(_CLIB) and os.path.getmtime(_CLIB) >= os.path.getmtime(src):
        return _CLIB
    subprocess.run(["gcc", "-O2", "-fopenmp", "-ffp-contract=off", "-shared", "-fPIC", src, "-o", _CLIB],
                   check=True)
    return _CLIB


def tensor_c(seed, tid, shape):
    """Same values as `tensor`, from the plain-C generator (large tensors)."""
    build_c()
    lib = ctypes.CDLL(_CLIB)
    n = int(np.prod(shape))
    out = np.empty(n, np.float32)
    lib.oracle_weights(out.ctypes.data_as(ctypes.c_void_p), ctypes.c_int64(0), ctypes.c_int64(n),
                       ctypes.c_uint32(tid), ctypes.c_uint64(seed))
    return out.reshape(shape)

WEIGHT_TAG = 0x57454947          # 'WEIG'
A_SCALE = np.float32(0.02 * np.sqrt(3.0))
TID_EMBED = 0x10000000
TID_LM_HEAD = 0x10000001
KIND = dict(q=0, k=1, v=2, bq=3, bk=4, bv=5, o=6, gate=7, up=8, down=9)


def layer_tid(layer, kind):
    return 0x100 * (layer + 1) + KIND[kind]


def bf16_rne(x32):
    """Round float32 -> bf16 (round to nearest even), returned as float32."""
    b = np.asarray(x32, dtype=np.float32).view(np.uint32).astype(np.uint64)
    r = (b + np.uint64(0x7FFF) + ((b >> np.uint64(16)) & np.uint64(1))) >> np.uint64(16)
    return (r.astype(np.uint32) << np.uint32(16)).view(np.float32)


def words_to_weights(x):
    u2m1 = ((x >> np.uint32(9)).astype(np.float32) + np.float32(0.5)) * np.float32(2.0 ** -22) - np.float32(1.0)
    return bf16_rne(A_SCALE * u2m1)


def tensor(seed, tid, shape):
    """The whole tensor `tid` of the given (PyTorch-layout) shape."""
    n = int(np.prod(shape))
    k0, k1 = seed & 0xFFFFFFFF, (seed >> 32) & 0xFFFFFFFF
    x = stream_words(n, tid, 0, WEIGHT_TAG, k0, k1)
    return words_to_weights(x).reshape(shape)


def rows(seed, tid, in_features, row_ids):
    """Selected rows of a [out, in] tensor (e.g. the embedding rows of the
    tokens actually used), without materialising the rest."""
    row_ids = np.asarray(row_ids, dtype=np.uint64)
    i = row_ids[:, None] * np.uint64(in_features) + np.arange(in_features, dtype=np.uint64)[None, :]
    k0, k1 = seed & 0xFFFFFFFF, (seed >> 32) & 0xFFFFFFFF
    x = philox4x32(i >> np.uint64(2), tid, 0, WEIGHT_TAG, k0, k1)
    word = (i & np.uint64(3)).astype(np.int64)
    xs = np.choose(word, x)
    return words_to_weights(xs.astype(np.uint32))


class Weights:
    """Lazily generated weights of a model config (dict with the keys of
    synth.configs).  Caches tensors as float32 (= the bf16 values)."""

    def __init__(self, cfg, seed, use_c=False):
        self.cfg, self.seed, self._c, self.use_c = cfg, seed, {}, use_c

    def _get(self, key, tid, shape):
        if key not in self._c:
            self._c[key] = (tensor_c if self.use_c else tensor)(self.seed, tid, shape)
        return self._c[key]

    def layer(self, l):
        c = self.cfg
        d, hd, H, KV, F = c["d_model"], c["head_dim"], c["n_heads"], c["n_kv_heads"], c["d_ff"]
        w = dict(
            q=self._get(("q", l), layer_tid(l, "q"), (H * hd, d)),
            k=self._get(("k", l), layer_tid(l, "k"), (KV * hd, d)),
            v=self._get(("v", l), layer_tid(l, "v"), (KV * hd, d)),
            o=self._get(("o", l), layer_tid(l, "o"), (d, H * hd)),
            gate=self._get(("gate", l), layer_tid(l, "gate"), (F, d)),
            up=self._get(("up", l), layer_tid(l, "up"), (F, d)),
            down=self._get(("down", l), layer_tid(l, "down"), (d, F)),
            ln1=np.ones(d, np.float32), ln2=np.ones(d, np.float32),
        )
        if c.get("qkv_bias", 1):
            w["bq"] = self._get(("bq", l), layer_tid(l, "bq"), (H * hd,))
            w["bk"] = self._get(("bk", l), layer_tid(l, "bk"), (KV * hd,))
            w["bv"] = self._get(("bv", l), layer_tid(l, "bv"), (KV * hd,))
        return w

    def lm_head(self):
        c = self.cfg
        return self._get("lm", TID_LM_HEAD, (c["vocab"], c["d_model"]))

    def final_norm(self):
        return np.ones(self.cfg["d_model"], np.float32)

    def embed_rows(self, tokens):
        return rows(self.seed, TID_EMBED, self.cfg["d_model"], tokens)

    def drop_layer(self, l):
        for k in list(self._c):
            if isinstance(k, tuple) and k[1] == l:
                del self._c[k]
