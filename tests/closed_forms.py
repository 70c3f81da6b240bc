"""Closed-form flow solutions the tests hold both the oracle and the CUDA path to (no LB arithmetic
here: these are the continuum solutions the lattice method must approach).

* Start-up Poiseuille flow between half-way walls (config 1; SURVEY §8(c) "TRT + Guo" pin): a fluid at
  rest at t = 0 driven by a body force F along x between no-slip walls a distance H apart,
  u(eta, t) = u_s(eta) - sum_{k odd} 4 F H^2 / (nu k^3 pi^3) sin(k pi eta) exp(-k^2 pi^2 nu t / H^2),
  u_s = F H^2 / (2 nu) eta (1 - eta), eta = (y - 1/2) / H for lattice rows y = 1..H.
* Shear-wave decay (config 2; the viscosity pin of north_star): u_x = A(t) sin(2 pi z / L) with
  A(t) = A(0) exp(-nu k^2 t), k = 2 pi / L, nu = (1/omega_shear - 1/2) / 3.
"""
from __future__ import annotations

import numpy as np


def lattice_viscosity(omega_shear: float) -> float:
    """nu = c_s^2 (1/omega - 1/2) with c_s^2 = 1/3 (lattice units; the Chapman-Enskog relation)."""
    return (1.0 / omega_shear - 0.5) / 3.0


def poiseuille_startup(y: np.ndarray, H: int, F: float, nu: float, t: float, kmax: int = 2000) -> np.ndarray:
    """u_x(y, t) of the start-up channel flow for fluid rows y (1..H) between half-way walls."""
    eta = (np.asarray(y, np.float64) - 0.5) / H
    u = F * H ** 2 / (2 * nu) * eta * (1 - eta)
    for k in range(1, kmax, 2):
        u = u - 4 * F * H ** 2 / (nu * k ** 3 * np.pi ** 3) * np.sin(k * np.pi * eta) * np.exp(
            -k * k * np.pi ** 2 * nu * t / H ** 2)
    return u


def shear_wave_amplitude(ux_of_z: np.ndarray) -> float:
    """Projection of a z-profile of u_x (averaged over x, y) onto sin(2 pi z / L): A = (2/L) sum u sin."""
    L = ux_of_z.shape[0]
    z = np.arange(L)
    return float(2.0 / L * np.sum(ux_of_z * np.sin(2 * np.pi * z / L)))


def fitted_viscosity(A0: float, A1: float, t0: float, t1: float, L: int) -> float:
    """nu from two amplitudes of the decaying shear wave: A1 / A0 = exp(-nu k^2 (t1 - t0))."""
    k = 2 * np.pi / L
    return float(np.log(A0 / A1) / (k * k * (t1 - t0)))
