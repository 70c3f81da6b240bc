"""Seeded synthetic inputs shared by the oracle side and the CUDA side of the tests.

This module holds NONE of the method's arithmetic (no equilibrium, collision or streaming):
only the counter-based random fields, the shear-wave initial profile of config 2
and the flag-field geometries of the BASELINE configs (G9). Both the oracle and the GPU path
consume what it returns; the GPU's own ``lbm_init_random`` implements the same counter-based
generator independently in CUDA (tests compare the two).

G13: U(a, b) = a + (b - a) * r, r = top 53 bits of SplitMix64(key) * 2^-53,
key = (seed << 40) XOR (4 * i_global + k), i_global = x + nx * (y + ny * z),
k in {0: rho, 1: u_x, 2: u_y, 3: u_z}.
"""
from __future__ import annotations

import numpy as np

FLUID, NOSLIP, UBB = 0, 1, 2

_G = np.uint64(0x9E3779B97F4A7C15)
_M1 = np.uint64(0xBF58476D1CE4E5B9)
_M2 = np.uint64(0x94D049BB133111EB)


def splitmix64(key: np.ndarray) -> np.ndarray:
    """SplitMix64 finaliser applied to key + golden gamma (Steele, Lea, Flood 2014)."""
    with np.errstate(over="ignore"):
        z = np.asarray(key, dtype=np.uint64) + _G
        z = (z ^ (z >> np.uint64(30))) * _M1
        z = (z ^ (z >> np.uint64(27))) * _M2
        return z ^ (z >> np.uint64(31))


def uniform01(seed: int, i_global: np.ndarray, k: int) -> np.ndarray:
    key = (np.uint64(seed) << np.uint64(40)) ^ (np.uint64(4) * np.asarray(i_global, np.uint64) + np.uint64(k))
    return (splitmix64(key) >> np.uint64(11)).astype(np.float64) * (2.0 ** -53)


def uniform(seed: int, i_global: np.ndarray, k: int, a: float, b: float) -> np.ndarray:
    return a + (b - a) * uniform01(seed, i_global, k)


def global_index(nx: int, ny: int, z0: int, nz: int) -> np.ndarray:
    z, y, x = np.meshgrid(np.arange(z0, z0 + nz, dtype=np.uint64), np.arange(ny, dtype=np.uint64),
                          np.arange(nx, dtype=np.uint64), indexing="ij")
    return x + np.uint64(nx) * (y + np.uint64(ny) * z)


PROFILE_NONE, PROFILE_SHEAR_WAVE = 0, 1


def random_fields(seed: int, nx: int, ny: int, nz_global: int, rho_amp: float, u_amp: float,
                  profile: int = PROFILE_NONE, profile_amp: float = 0.0, z0: int = 0, nz: int | None = None):
    """(rho, u) for cells z in [z0, z0+nz) of an nx*ny*nz_global lattice.

    rho = 1 + U(-rho_amp, rho_amp); u_i = U(-u_amp, u_amp) (+ profile_amp*sin(2 pi z/nz_global)
    on u_x for the shear-wave profile of config 2)."""
    nz = nz_global - z0 if nz is None else nz
    ig = global_index(nx, ny, z0, nz)
    rho = 1.0 + uniform(seed, ig, 0, -rho_amp, rho_amp) if rho_amp != 0 else np.ones(ig.shape)
    u = np.stack([uniform(seed, ig, k, -u_amp, u_amp) if u_amp != 0 else np.zeros(ig.shape) for k in (1, 2, 3)])
    if profile == PROFILE_SHEAR_WAVE:
        z = np.arange(z0, z0 + nz, dtype=np.float64)[:, None, None]
        u[0] = profile_amp * np.sin(2.0 * np.pi * z / nz_global) + u[0]
    return rho, u


# ------------------------------------------------------------------------------------------
# Geometries (G9): walls are flagged cells inside the stated domain.
# ------------------------------------------------------------------------------------------
def channel_flags(nx: int, ny: int, nz: int) -> np.ndarray:
    """Config 1: no-slip walls at y = 0 and y = ny-1, periodic x/z. Shape (nz, ny, nx)."""
    fl = np.zeros((nz, ny, nx), np.uint8)
    fl[:, 0, :] = NOSLIP
    fl[:, ny - 1, :] = NOSLIP
    return fl


def cavity_flags(n: int) -> np.ndarray:
    """Config 3: cells with x in {0,n-1}, y in {0,n-1} or z = 0 are no-slip; remaining z = n-1
    cells are the moving lid (UBB)."""
    fl = np.zeros((n, n, n), np.uint8)
    fl[n - 1, :, :] = UBB
    fl[:, :, 0] = NOSLIP
    fl[:, :, n - 1] = NOSLIP
    fl[:, 0, :] = NOSLIP
    fl[:, n - 1, :] = NOSLIP
    fl[0, :, :] = NOSLIP
    return fl


def couette_flags(nx: int, H: int, nz: int) -> np.ndarray:
    """No-slip at y = 0, UBB at y = H+1, fluid y = 1..H (UBB sign/placement pin)."""
    fl = np.zeros((nz, H + 2, nx), np.uint8)
    fl[:, 0, :] = NOSLIP
    fl[:, H + 1, :] = UBB
    return fl


def random_obstacles(seed: int, nx: int, ny: int, nz: int, frac: float = 0.1, ubb_frac: float = 0.3) -> np.ndarray:
    """Random sprinkle of wall cells (NOSLIP / UBB) for data-movement tests."""
    ig = global_index(nx, ny, 0, nz)
    r = uniform01(seed + 7, ig, 0)
    s = uniform01(seed + 7, ig, 1)
    fl = np.zeros((nz, ny, nx), np.uint8)
    fl[r < frac] = NOSLIP
    fl[(r < frac) & (s < ubb_frac)] = UBB
    return fl


def fields_at(seed: int, nx: int, ny: int, nz: int, xs, ys, zs, rho_amp: float, u_amp: float,
              profile: int = PROFILE_NONE, profile_amp: float = 0.0):
    """(rho, u) at arbitrary (wrapped) global coordinates; arrays xs, ys, zs broadcast together.
    Same values as random_fields() at those cells."""
    xs, ys, zs = (np.asarray(v, np.int64) for v in np.broadcast_arrays(xs, ys, zs))
    xs, ys, zs = xs % nx, ys % ny, zs % nz
    ig = (xs + nx * (ys + ny * zs)).astype(np.uint64)
    rho = 1.0 + uniform(seed, ig, 0, -rho_amp, rho_amp) if rho_amp != 0 else np.ones(ig.shape)
    u = np.stack([uniform(seed, ig, k, -u_amp, u_amp) if u_amp != 0 else np.zeros(ig.shape) for k in (1, 2, 3)])
    if profile == PROFILE_SHEAR_WAVE:
        u[0] = profile_amp * np.sin(2.0 * np.pi * zs.astype(np.float64) / nz) + u[0]
    return rho, u
