"""Seeded input generator pins (CPU): SplitMix64 against its published reference outputs and the
G13 key/uniform recipe."""
import numpy as np

import lbminputs as LI


def test_splitmix64_reference_sequence():
    # SplitMix64 (Steele, Lea, Flood, OOPSLA 2014; Vigna's splitmix64.c) with state 0 yields
    # 0xe220a8397b1dcdaf, 0x6e789e6aa1b965f4, 0x06c45d188009454f: the k-th output is the
    # finaliser applied to k * 0x9E3779B97F4A7C15 (our hash adds one gamma to the key).
    G = 0x9E3779B97F4A7C15
    keys = np.array([(k * G) % 2 ** 64 for k in range(3)], dtype=np.uint64)
    out = [int(v) for v in LI.splitmix64(keys)]
    assert out == [0xE220A8397B1DCDAF, 0x6E789E6AA1B965F4, 0x06C45D188009454F]


def test_uniform_range_and_key_layout():
    ig = LI.global_index(8, 4, 0, 4).ravel()
    r = LI.uniform01(0, ig, 1)
    assert r.min() >= 0 and r.max() < 1 and abs(r.mean() - 0.5) < 0.1
    # 53-bit grid
    assert np.all(r * 2 ** 53 == np.floor(r * 2 ** 53))
    # key = (seed << 40) ^ (4 i + k): component k of cell i equals component 0 of key 4i+k
    a = LI.uniform01(3, np.array([5], np.uint64), 2)
    key = (3 << 40) ^ (4 * 5 + 2)
    b = (int(LI.splitmix64(np.array([key], np.uint64))[0]) >> 11) * 2.0 ** -53
    assert a[0] == b


def test_random_fields_decomposition_invariant():
    rho, u = LI.random_fields(0, 6, 5, 8, 1e-3, 0.01)
    rho2, u2 = LI.random_fields(0, 6, 5, 8, 1e-3, 0.01, z0=4, nz=4)
    np.testing.assert_array_equal(rho[4:], rho2)
    np.testing.assert_array_equal(u[:, 4:], u2)
    assert np.abs(rho - 1).max() <= 1e-3 and np.abs(u).max() <= 0.01


def test_geometries():
    fl = LI.cavity_flags(8)
    assert (fl == 0).sum() == 6 ** 3
    assert (fl == LI.UBB).sum() == 6 * 6  # lid interior; edges/corners are no-slip (G9)
    ch = LI.channel_flags(4, 10, 3)
    assert (ch == 0).sum() == 4 * 8 * 3
