"""Seeded generators of prompts and response-length traces.

Prompts (reading Z14): token ids uniform in [0, eos), lengths uniform in a
per-config range.  Traces (reading Z15): prompt-level lognormal,
    mu_i ~ N(mu0, sigma_p),  L ~ LogNormal(mu_i, sigma_r),
rounded and clamped to [1, l_max]; one independent draw of G lengths per
(prompt, attempt), sharing mu_i across attempts (prompt-level length
persistence).  Calibrated against P:69-72 (max/median 25-32x)
and P:308-310 (P75 755-1.1k at a 16k cap).
"""
import numpy as np


def prompts(n, vocab_lo, eos_id, len_range, seed, first_id=0):
    """n prompts: list of dicts {prompt_id, tokens(int32 array)}."""
    rng = np.random.default_rng([seed, 0x50524F4D])
    lo, hi = len_range
    out = []
    for i in range(n):
        ln = int(rng.integers(lo, hi + 1))
        toks = rng.integers(vocab_lo, eos_id, size=ln, dtype=np.int64).astype(np.int32)
        out.append(dict(prompt_id=first_id + i, tokens=toks))
    return out


def prompt_stream(n, cfg_model, len_range, seed):
    return prompts(n, 0, cfg_model["eos_id"], len_range, seed)


def length_trace(n_prompts, G, mu0, sigma_p, sigma_r, l_max, seed, n_attempts=2):
    """int32 array [n_prompts, n_attempts, G] of response lengths >= 1."""
    rng = np.random.default_rng([seed, 0x4C454E53])
    mu = rng.normal(mu0, sigma_p, size=n_prompts)
    z = rng.normal(0.0, 1.0, size=(n_prompts, n_attempts, G))
    L = np.exp(mu[:, None, None] + sigma_r * z)
    L = np.clip(np.rint(L), 1, l_max).astype(np.int32)
    return L


def trace_for_round(trace, prompt_ids, attempt):
    """[n, G] lengths of the given prompts at the given attempt."""
    return np.ascontiguousarray(trace[np.asarray(prompt_ids), attempt, :])
