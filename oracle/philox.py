"""Philox4x32-10 (Salmon et al., SC'11 "Parallel random numbers: as easy as
1, 2, 3"), written out in NumPy.  TEST INFRASTRUCTURE ONLY (see
oracle/__init__.py).

The paper is silent on the RNG (reading Z10); we fix Philox4x32-10
because it is counter based, so every (token, vocab entry) draws an
independent stream that does not depend on batching or DP sharding.

Round function (one of 10), with multipliers M0, M1 and Weyl constants
W0, W1:
    (hi0, lo0) = M0 * c0 ;  (hi1, lo1) = M1 * c2
    c' = (hi1 ^ c1 ^ k0,  lo1,  hi0 ^ c3 ^ k1,  lo0)
    k  = (k0 + W0, k1 + W1)            (between rounds)
Pinned by the Random123 known-answer tests in tests/test_oracle_philox.py.
"""
import numpy as np

M0 = np.uint64(0xD2511F53)
M1 = np.uint64(0xCD9E8D57)
W0 = 0x9E3779B9
W1 = 0xBB67AE85
MASK32 = np.uint64(0xFFFFFFFF)


def philox4x32(c0, c1, c2, c3, k0, k1, rounds=10):
    """Vectorised Philox4x32-R.  Inputs are array-likes of uint32 values
    (broadcast together); keys are python ints or arrays.  Returns four
    uint32 arrays (x0, x1, x2, x3)."""
    c0, c1, c2, c3 = (np.asarray(c, dtype=np.uint64) & MASK32 for c in (c0, c1, c2, c3))
    c0, c1, c2, c3 = np.broadcast_arrays(c0, c1, c2, c3)
    k0 = np.uint64(int(k0) & 0xFFFFFFFF) if np.isscalar(k0) else np.asarray(k0, np.uint64)
    k1 = np.uint64(int(k1) & 0xFFFFFFFF) if np.isscalar(k1) else np.asarray(k1, np.uint64)
    for r in range(rounds):
        if r > 0:
            k0 = (k0 + np.uint64(W0)) & MASK32
            k1 = (k1 + np.uint64(W1)) & MASK32
        p0 = M0 * c0                       # < 2^64, exact in uint64
        p1 = M1 * c2
        hi0, lo0 = p0 >> np.uint64(32), p0 & MASK32
        hi1, lo1 = p1 >> np.uint64(32), p1 & MASK32
        c0, c1, c2, c3 = (hi1 ^ c1 ^ k0), lo1, (hi0 ^ c3 ^ k1), lo0
    return tuple(np.asarray(c, dtype=np.uint32) for c in (c0, c1, c2, c3))


def uniform_open01_f32(x):
    """u = ((x >> 9) + 0.5) * 2^-23 (Z10).  Exact in fp32, lies
    strictly inside (0, 1).  Returned as float32."""
    x = np.asarray(x, dtype=np.uint32)
    return ((x >> np.uint32(9)).astype(np.float32) + np.float32(0.5)) * np.float32(2.0 ** -23)


def stream_words(n, c1, c2, c3, k0, k1):
    """Words w[i] for i in [0, n): word (i & 3) of Philox(ctr=(i>>2, c1, c2, c3))."""
    i = np.arange(n, dtype=np.uint64)
    blocks = (n + 3) // 4
    x = philox4x32(np.arange(blocks, dtype=np.uint64), c1, c2, c3, k0, k1)
    w = np.stack(x, axis=1).reshape(-1)[:n]
    del i
    return w
