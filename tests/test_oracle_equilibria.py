"""Pins of the oracle's equilibrium variants (CPU, no GPU).

* incompressible Eq. (3) with rho0 = 1: closed-form moments, rho = 1 reduces to the
  compressible form, collisions conserve mass and j;
* moment-matched equilibrium: for D3Q27 it IS Eq. (3) (paper statement P:372-373);
  for D3Q19 its 19 basis moments (Eq. 5, summed directly over the populations) equal the raw moments
  of the continuous Maxwellian Eq. (7)-(8) obtained by Gauss-Hermite quadrature and truncated at 2nd
  order in u by exact polynomial interpolation in a velocity scale t — a route that shares nothing
  with the oracle's factorised-product formula and M^-1;
* every kind is a fixed point of SRT/TRT/MRT built on it, and collisions conserve mass/momentum.
"""
from itertools import product

import numpy as np
import pytest

import oracle as O
from oracle import methods

CS2 = 1.0 / 3.0


def _moment(c, f, e):
    return float((f * np.prod(c.astype(float) ** np.array(e), axis=1)).sum())


def _maxwellian_moment_quadrature(e, rho, u):
    """E[xi^e] of rho N(u, cs2 I) by 1-D Gauss-Hermite (probabilists') quadrature per axis (exact
    for polynomials of degree <= 2*20-1), then truncated at 2nd order in u: m(t) = moment at velocity
    t*u is a polynomial of degree <= 6 in t; interpolate it at 7 nodes and keep t^0..t^2 at t = 1."""
    x, wq = np.polynomial.hermite_e.hermegauss(20)
    wq = wq / wq.sum()
    ts = np.linspace(-1.5, 1.5, 7)
    vals = []
    for t in ts:
        m = rho
        for d in range(3):
            xi = t * u[d] + np.sqrt(CS2) * x
            m *= float((wq * xi ** e[d]).sum())
        vals.append(m)
    coef = np.linalg.solve(np.vander(ts, 7, increasing=True), np.array(vals))
    return float(coef[0] + coef[1] + coef[2])


def test_moment_matched_d3q27_is_eq3_paper():
    """for the Cartesian product stencil D3Q27 moment matching yields exactly Eq. (3)."""
    rng = np.random.default_rng(3)
    m = O.Method(Q=27, op="srt", rates=(1.8,), equilibrium="moment_matched")
    for _ in range(10):
        rho, u = 1 + rng.uniform(-0.1, 0.1), rng.uniform(-0.08, 0.08, 3)
        np.testing.assert_allclose(O.equilibrium_kind_cell(m, rho, u), O.equilibrium_cell(27, rho, u), rtol=0, atol=2e-16)


def test_moment_matched_d3q19_matches_maxwellian_by_quadrature():
    c, _, _ = O.stencil_arrays(19)
    m = O.Method(Q=19, op="srt", rates=(1.8,), equilibrium="moment_matched")
    basis = [next(iter(p)) for p in methods.monomial_basis("D3Q19")]
    rng = np.random.default_rng(4)
    for _ in range(5):
        rho, u = 1 + rng.uniform(-0.1, 0.1), rng.uniform(-0.08, 0.08, 3)
        f = O.equilibrium_kind_cell(m, rho, u)
        for e in basis:
            assert abs(_moment(c, f, e) - _maxwellian_moment_quadrature(e, rho, u)) < 2e-15, e
        # ... and differs from Eq. (3), in the x^2 y^2 family only
        f3 = O.equilibrium_cell(19, rho, u)
        for e in basis:
            d = _moment(c, f, e) - _moment(c, f3, e)
            if sorted(e) == [0, 2, 2]:
                zero_axis = e.index(0)
                assert abs(d - rho * u[zero_axis] ** 2 / 6) < 1e-15, e
            else:
                assert abs(d) < 1e-15, e


@pytest.mark.parametrize("Q", [19, 27])
def test_incompressible_moments_closed_form(Q):
    """Eq. (3) with rho0 = 1: sum f = rho, sum c f = u, sum c c f = rho cs2 I + u u."""
    c, w, _ = O.stencil_arrays(Q)
    m = O.Method(Q=Q, op="srt", rates=(1.8,), equilibrium="incompressible")
    rng = np.random.default_rng(5)
    for _ in range(10):
        rho, u = 1 + rng.uniform(-0.1, 0.1), rng.uniform(-0.1, 0.1, 3)
        f = O.equilibrium_kind_cell(m, rho, u)
        assert abs(f.sum() - rho) < 1e-15
        np.testing.assert_allclose(c.T @ f, u, atol=1e-16)
        Pi = np.einsum("qa,qb,q->ab", c, c, f)
        np.testing.assert_allclose(Pi, rho * CS2 * np.eye(3) + np.outer(u, u), atol=2e-16)
    u = rng.uniform(-0.1, 0.1, 3)
    np.testing.assert_allclose(O.equilibrium_kind_cell(m, 1.0, u), O.equilibrium_cell(Q, 1.0, u), rtol=0, atol=1e-16)


CASES = [(Q, op, rates, eq) for eq in ("incompressible", "moment_matched")
         for Q, op, rates in [(19, "srt", (1.8,)), (19, "trt", (1.6, 0.5)), (27, "trt", (1.3, 0.9)),
                              (19, "mrt", (1.9, 1.3, 1.1, 0.8))]]


@pytest.mark.parametrize("Q,op,rates,eq", CASES)
def test_equilibrium_kind_fixed_point_and_conservation(Q, op, rates, eq):
    c, w, _ = O.stencil_arrays(Q)
    m = O.Method(Q=Q, op=op, rates=rates, equilibrium=eq)
    rng = np.random.default_rng(6)
    rho, u = 1.02, np.array([0.03, -0.02, 0.04])
    feq = O.equilibrium_kind_cell(m, rho, u)
    np.testing.assert_allclose(O.collide_cell(m, feq), feq, rtol=0, atol=4e-16)
    f = feq * (1 + 0.05 * rng.uniform(-1, 1, Q))
    out = O.collide_cell(m, f)
    assert abs(out.sum() - f.sum()) < 1e-15
    np.testing.assert_allclose(c.T @ out, c.T @ f, atol=1e-16)


def test_incompressible_guo_momentum_gain():
    """With rho0 = 1 the Guo-forced TRT collision still adds exactly F to the momentum (G4)."""
    c, _, _ = O.stencil_arrays(19)
    F = np.array([1e-4, -2e-4, 5e-5])
    m = O.Method(Q=19, op="trt", rates=(1.6, 0.5), force=F, equilibrium="incompressible")
    rng = np.random.default_rng(7)
    f = O.equilibrium_kind_cell(m, 1.01, [0.02, 0.01, -0.03]) * (1 + 0.03 * rng.uniform(-1, 1, 19))
    out = O.collide_cell(m, f)
    np.testing.assert_allclose(c.T @ out - c.T @ f, F, rtol=0, atol=1e-16)
    assert abs(out.sum() - f.sum()) < 1e-15
