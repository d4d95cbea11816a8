"""Gumbel-max sampling with Philox noise (readings Z9-Z11).
TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

The paper samples G responses per prompt with vLLM and is
silent on temperature and the RNG; we read plain T=1 categorical sampling
(Z9) drawn as a Gumbel-max:

    (x0..x3) = Philox4x32-10(ctr=(v >> 2, t, uid, round_id), key=(seed_lo, seed_hi))
    u_v      = ((x_{v&3} >> 9) + 0.5) * 2^-23              exact in fp32
    g_v      = -ln(-ln u_v)
    token    = argmax_v (logit_v / T + g_v), ties -> lowest v
with uid = prompt_id * G + j.  Trace mode (Z15/Z16): logit[eos] = -inf for
t < L and token = eos at t = L.

Gumbel-max equals categorical sampling from softmax(logit / T) (the textbook
result pinned by a chi-square test in tests/test_oracle_sampler.py).
"""
import numpy as np

from .philox import philox4x32, uniform_open01_f32


def gumbel(V, t, uid, round_id, seed):
    """Gumbel noise g_v, v in [0, V), float64 computed from the exact fp32 u."""
    k0, k1 = seed & 0xFFFFFFFF, (seed >> 32) & 0xFFFFFFFF
    blocks = np.arange((V + 3) // 4, dtype=np.uint64)
    x = philox4x32(blocks, t, uid, round_id, k0, k1)
    w = np.stack(x, axis=1).reshape(-1)[:V]
    u = uniform_open01_f32(w).astype(np.float64)
    return -np.log(-np.log(u))


def perturbed(logits, t, uid, round_id, seed, temperature=1.0, eos_id=None, trace_len=None):
    """logit/T + g with the trace-mode EOS mask applied (float64)."""
    z = np.asarray(logits, np.float64) / temperature + gumbel(len(logits), t, uid, round_id, seed)
    if trace_len is not None and t < trace_len:
        z[eos_id] = -np.inf
    return z


def sample(logits, t, uid, round_id, seed, temperature=1.0, eos_id=None, trace_len=None):
    """Returns (token, top-2 gap of the perturbed scores)."""
    if trace_len is not None and t == trace_len:
        return int(eos_id), np.inf
    z = perturbed(logits, t, uid, round_id, seed, temperature, eos_id, trace_len)
    order = np.argsort(-z, kind="stable")           # stable -> ties to lowest v
    return int(order[0]), float(z[order[0]] - z[order[1]])
