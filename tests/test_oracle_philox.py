"""Pins of oracle/philox.py against the Random123 known-answer tests
(Salmon et al. SC'11, kat_vectors "philox4x32 10"), not against itself."""
import numpy as np

from oracle.philox import philox4x32, uniform_open01_f32, stream_words

KAT = [
    ((0, 0, 0, 0), (0, 0), (0x6627E8D5, 0xE169C58D, 0xBC57AC4C, 0x9B00DBD8)),
    ((0xFFFFFFFF,) * 4, (0xFFFFFFFF,) * 2, (0x408F276D, 0x41C83B0E, 0xA20BC7C6, 0x6D5451FD)),
    ((0x243F6A88, 0x85A308D3, 0x13198A2E, 0x03707344), (0xA4093822, 0x299F31D0),
     (0xD16CFE09, 0x94FDCCEB, 0x5001E420, 0x24126EA1)),
]


def test_known_answers():
    for ctr, key, want in KAT:
        got = philox4x32(*ctr, *key)
        assert tuple(int(g) for g in got) == want


def test_vectorised_equals_scalar():
    c0 = np.arange(17, dtype=np.uint64) * 0x9E3779B1
    vec = philox4x32(c0, 5, 6, 7, 11, 12)
    for i in range(17):
        sc = philox4x32(int(c0[i]) & 0xFFFFFFFF, 5, 6, 7, 11, 12)
        assert all(int(v[i]) == int(s) for v, s in zip(vec, sc))


def test_uniform_mapping_open_interval_and_exact():
    x = np.array([0, 1, 511, 512, 0xFFFFFFFF, 0x80000000], dtype=np.uint32)
    u = uniform_open01_f32(x)
    assert u.dtype == np.float32
    assert np.all(u > 0) and np.all(u < 1)
    # exactness: u * 2^24 is an odd integer (2*(x>>9)+1)
    assert np.all((u.astype(np.float64) * 2.0 ** 24) == (2 * (x.astype(np.int64) >> 9) + 1))
    assert u[0] == np.float32(2.0 ** -24)
    assert float(u[4]) == 1.0 - 2.0 ** -24


def test_stream_words_layout():
    w = stream_words(10, 3, 4, 5, 6, 7)
    b1 = philox4x32(1, 3, 4, 5, 6, 7)
    assert int(w[5]) == int(b1[1]) and int(w[4]) == int(b1[0])
