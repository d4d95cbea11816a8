"""The synthetic input recipe matches the paper's workload statistics
(P:69-72 max/median 25-32x; P:308-310 P75 755-1.1k at a 16k cap) and is
deterministic per seed."""
import numpy as np

from synth import gen
from synth.configs import ROUNDS, MODELS


def test_trace_calibration_c2():
    p = ROUNDS["C2-7b"]["trace"]
    L = gen.length_trace(128 * 60, 8, p["mu0"], p["sigma_p"], p["sigma_r"], p["l_max"], 2)[:, 0, :]
    ratios, p75 = [], []
    for b in range(0, L.shape[0], 128):
        x = L[b:b + 128].reshape(-1)
        ratios.append(x.max() / np.median(x)); p75.append(np.percentile(x, 75))
    assert 25 <= np.median(ratios) <= 32
    assert 755 <= np.median(p75) <= 1100
    assert L.max() <= 16384 and L.min() >= 1


def test_prompts_deterministic_and_in_range():
    m = MODELS["tiny"]
    a = gen.prompts(8, 0, m["eos_id"], (8, 32), 1)
    b = gen.prompts(8, 0, m["eos_id"], (8, 32), 1)
    assert all(np.array_equal(x["tokens"], y["tokens"]) for x, y in zip(a, b))
    for p in a:
        assert 8 <= len(p["tokens"]) <= 32
        assert p["tokens"].max() < m["eos_id"] and p["tokens"].min() >= 0
