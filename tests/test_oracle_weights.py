"""Pins of oracle/weights.py (reading Z12): bf16 round-to-nearest-
even on hand-worked bit patterns, the range/moments the formula implies, and
agreement of the row-gather path with the whole-tensor path."""
import numpy as np

from oracle import weights as W


def _f(bits):
    return np.array([bits], np.uint32).view(np.float32)


def test_bf16_rne_hand_cases():
    # exactly representable: unchanged
    assert W.bf16_rne(_f(0x3F800000)).view(np.uint32)[0] == 0x3F800000
    # halfway, even lower half -> round down
    assert W.bf16_rne(_f(0x3F808000)).view(np.uint32)[0] == 0x3F800000
    # halfway, odd lower half -> round up to even
    assert W.bf16_rne(_f(0x3F818000)).view(np.uint32)[0] == 0x3F820000
    # just above half -> up
    assert W.bf16_rne(_f(0x3F808001)).view(np.uint32)[0] == 0x3F810000
    # negative
    assert W.bf16_rne(_f(0xBF80C000)).view(np.uint32)[0] == 0xBF810000


def test_scale_constant():
    assert W.A_SCALE == np.float32(0.034641016151377546)


def test_range_and_moments():
    w = W.tensor(0, W.layer_tid(0, "q"), (512, 512)).astype(np.float64)
    a = float(W.A_SCALE)
    assert np.all(np.abs(w) <= a * (1 + 2 ** -8))
    assert abs(w.mean()) < 3 * 0.02 / np.sqrt(w.size)
    assert abs(w.std() - 0.02) < 0.02 * 0.01
    # values are bf16 (low 16 bits zero)
    assert np.all((w.astype(np.float32).view(np.uint32) & 0xFFFF) == 0)


def test_rows_equal_tensor_rows():
    t = W.tensor(7, W.TID_EMBED, (64, 48))
    r = W.rows(7, W.TID_EMBED, 48, [0, 5, 63, 5])
    assert np.array_equal(r, t[[0, 5, 63, 5]])


def test_tensor_ids_distinct_streams():
    a = W.tensor(0, W.layer_tid(0, "k"), (8, 8))
    b = W.tensor(0, W.layer_tid(0, "v"), (8, 8))
    c = W.tensor(1, W.layer_tid(0, "k"), (8, 8))
    assert not np.array_equal(a, b) and not np.array_equal(a, c)


def test_first_element_by_hand():
    # element 0 of tid=0x100 (layer 0 q), seed 0: word 0 of Philox(ctr=(0,0x100,0,TAG), key=0)
    from oracle.philox import philox4x32
    x = int(philox4x32(0, 0x100, 0, W.WEIGHT_TAG, 0, 0)[0])
    u2m1 = ((x >> 9) + 0.5) * 2.0 ** -22 - 1.0            # exact in fp64 and fp32
    w32 = np.float32(np.float32(W.A_SCALE) * np.float32(u2m1))
    want = W.bf16_rne(np.array([w32], np.float32))[0]
    got = W.tensor(0, 0x100, (1, 1))[0, 0]
    assert got == want


def test_c_generator_equals_numpy():
    """oracle/c/weights.c (used for 7B-shaped baselines) equals the NumPy
    formula element for element."""
    for tid, shape, seed in [(W.TID_EMBED, (37, 64), 0), (W.layer_tid(3, "down"), (256, 129), 12345678901)]:
        assert np.array_equal(W.tensor_c(seed, tid, shape), W.tensor(seed, tid, shape))
