"""Host-side check of the flat-row launch indexing arithmetic (csrc/kernels.cuh box_cell, csrc/runtime.cu
lbm_create): y = i / nx by one 32-bit multiply-high with magic = 2^32 / nx + 1 and a one-step
correction, for every in-plane index the runtime admits (nx ny < 2^30). Integer work: exact."""
import numpy as np
import pytest


def flat_xy(i, nx, magic):
    """The kernel's arithmetic on uint32 values, written with Python integers."""
    r = (i * magic) >> 32          # __umulhi(i, magic)
    if ((r * nx) & 0xFFFFFFFF) > i:  # r * nx in 32 bits
        r -= 1
    return i - r * nx, r


@pytest.mark.parametrize("nx", [2, 3, 19, 21, 44, 300, 301, 1000, 4097, 65535, 1 << 20, (1 << 29) - 1])
def test_flat_row_division_exact(nx):
    magic = (1 << 32) // nx + 1
    assert magic < 1 << 32
    rng = np.random.default_rng(nx)
    hi = (1 << 30) - 1
    samples = set(int(v) for v in rng.integers(0, hi, 2000))
    for k in range(0, hi // nx + 1, max(1, (hi // nx) // 50)):  # row starts and row ends
        samples.update(v for v in (k * nx - 1, k * nx, k * nx + 1, k * nx + nx - 1) if 0 <= v <= hi)
    samples.update((0, 1, hi - 1, hi))
    for i in samples:
        q = (i * magic) >> 32
        assert q - i // nx in (0, 1)          # the estimate is exact or one too large
        assert q * nx < 1 << 32               # its product fits the kernel's 32-bit compare
        assert flat_xy(i, nx, magic) == (i % nx, i // nx)


def test_flat_rows_cover_the_box_once():
    """Thread indices flat_start + t over ceil((flat_hi - flat_start) / 256) blocks of 256 hit every cell of the
    rows [y0, y1) exactly once and nothing else (flat_start = flat_lo rounded down to a multiple of 32)."""
    for nx, ny, y0, y1 in [(300, 100, 1, 99), (44, 11, 1, 10), (19, 7, 0, 7), (33, 5, 2, 3)]:
        lo, hi = y0 * nx, y1 * nx
        start = lo // 32 * 32
        nblocks = (hi - start + 255) // 256
        magic = (1 << 32) // nx + 1
        seen = np.zeros((ny, nx), int)
        for t in range(nblocks * 256):
            i = start + t
            if i < lo or i >= hi:
                continue
            x, y = flat_xy(i, nx, magic)
            seen[y, x] += 1
        assert (seen[y0:y1] == 1).all() and seen[:y0].sum() == 0 and seen[y1:].sum() == 0
