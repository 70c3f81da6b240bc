"""Oracle pins for the locally-varying relaxation rates of P:539-643 (CPU, no GPU).

Smagorinsky (Eqs. 11-14): the closed-form omega must satisfy Eq. (14) with |S| of Eq. (12)
evaluated at that same omega (the two-equation system the paper solves with sympy), reduce to SRT
for C_S = 0, and leave equilibrium fixed.
KBC (Eqs. 15-19): Delta_s is rebuilt independently from the closed-form weighted shear projector
(9/2) w_q c c : dev(Pi^neq) (G6), Delta_h = f - f_eq - Delta_s; the oracle's post-collision state
must equal f - w_s Delta_s - w_h Delta_h with w_h from Eq. (19), satisfy the linearised entropy
condition sum_q Delta_h f'/f_eq = 0 exactly, and give f_eq for w_s = 1.
"""
import numpy as np
import pytest

import oracle as O

RNG = np.random.default_rng(77)


def _state(Q, amp):
    rho = 1 + RNG.uniform(-0.05, 0.05)
    u = RNG.uniform(-0.05, 0.05, 3)
    _, w, _ = O.stencil_arrays(Q)
    return O.equilibrium_cell(Q, rho, u) + amp * w * RNG.uniform(-1, 1, Q)


def _pi_neq(Q, f):
    c, _, _ = O.stencil_arrays(Q)
    rho = f.sum()
    u = c.T @ f / rho
    feq = O.equilibrium_cell(Q, rho, u)
    return rho, feq, np.einsum("qa,qb,q->ab", c, c, f - feq)


@pytest.mark.parametrize("Q", [19, 27])
def test_smagorinsky_omega_solves_eq14(Q):
    omega0, cs = 1.9, 0.17
    m = O.Method(Q=Q, op="smagorinsky", rates=(omega0, cs))
    nu0 = (1 / omega0 - 0.5) / 3
    for amp in (1e-3, 0.05, 0.3):
        f = _state(Q, amp)
        w = O.smagorinsky_omega_cell(m, f)
        rho, feq, Pi = _pi_neq(Q, f)
        S = -3 * w / (2 * rho) * Pi                        # Eq. (12)
        Snorm = np.sqrt(2 * np.sum(S * S))                 # |S| = sqrt(2 S_ij S_ij)
        assert abs(w - 2 / (6 * cs * cs * Snorm + 6 * nu0 + 1)) < 1e-14   # Eq. (14)
        assert w < omega0                                  # the eddy viscosity only adds
        out = O.collide_cell(m, f)
        np.testing.assert_allclose(out, w * feq + (1 - w) * f, rtol=0, atol=1e-15)


def test_smagorinsky_limits():
    f = _state(19, 0.1)
    a = O.collide_cell(O.Method(Q=19, op="smagorinsky", rates=(1.7, 0.0)), f)
    b = O.collide_cell(O.Method(Q=19, op="srt", rates=(1.7,)), f)
    np.testing.assert_allclose(a, b, rtol=0, atol=1e-16)
    feq = O.equilibrium_cell(19, 1.01, np.array([0.02, -0.01, 0.03]))
    m = O.Method(Q=19, op="smagorinsky", rates=(1.7, 0.2))
    assert abs(O.smagorinsky_omega_cell(m, feq) - 1.7) < 1e-12
    np.testing.assert_allclose(O.collide_cell(m, feq), feq, rtol=0, atol=1e-15)


def _kbc_reference(f, ws, Q=19):
    c, w, _ = O.stencil_arrays(Q)
    rho, feq, Pi = _pi_neq(Q, f)
    dev = Pi - np.trace(Pi) / 3 * np.eye(3)
    ds = 4.5 * w * np.einsum("qa,qb,ab->q", c, c, dev)   # weighted shear projection (G6)
    dh = (f - feq) - ds
    wh = 1 + (1 - ws) * np.sum(ds * dh / feq) / np.sum(dh * dh / feq)   # Eq. (19)
    return feq, ds, dh, wh


@pytest.mark.parametrize("Q", [19, 27])
@pytest.mark.parametrize("ws", [1.99, 1.7, 1.2])
def test_kbc_matches_eq19_and_entropy_condition(ws, Q):
    """D3Q27: the same reading G17 on the D3Q27 weighted basis; the shear
    projector (9/2) w c c : dev(Pi) holds there too (4th-order isotropy of both weight sets)."""
    m = O.Method(Q=Q, op="kbc", rates=(ws,))
    c, _, _ = O.stencil_arrays(Q)
    for amp in (1e-3, 0.05, 0.2):
        f = _state(Q, amp)
        feq, ds, dh, wh = _kbc_reference(f, ws, Q)
        out = O.collide_cell(m, f)
        np.testing.assert_allclose(out, f - ws * ds - wh * dh, rtol=0, atol=1e-15)
        # linearised optimum (exact up to the rounding of sum(f - f_eq), ~1e-16)
        assert abs(np.sum(dh * out / feq)) < 1e-14
        assert abs(out.sum() - f.sum()) < 1e-15
        np.testing.assert_allclose(c.T @ out, c.T @ f, atol=1e-16)


@pytest.mark.parametrize("Q", [19, 27])
def test_kbc_limits(Q):
    f = _state(Q, 0.1)
    feq, _, _, _ = _kbc_reference(f, 1.0, Q)
    np.testing.assert_allclose(O.collide_cell(O.Method(Q=Q, op="kbc", rates=(1.0,)), f), feq, rtol=0, atol=1e-15)
    e = O.equilibrium_cell(Q, 0.99, np.array([0.01, 0.02, -0.03]))
    np.testing.assert_allclose(O.collide_cell(O.Method(Q=Q, op="kbc", rates=(1.8,)), e), e, rtol=0, atol=1e-15)


def test_kbc_entropy_not_below_linearised_neighbours():
    """The linearised w_h is near the true entropy maximiser for near-equilibrium states: the exact
    entropy S(w) = -sum f'(w) ln(f'(w)/f_eq) is within O(amp^3) of its maximum over w."""
    ws = 1.9
    f = _state(19, 0.01)
    feq, ds, dh, wh = _kbc_reference(f, ws)

    def S(w):
        fp = f - ws * ds - w * dh
        return -np.sum(fp * np.log(fp / feq))
    ws_grid = wh + np.linspace(-0.5, 0.5, 2001)
    best = ws_grid[np.argmax([S(w) for w in ws_grid])]
    assert abs(best - wh) < 0.05


# ---- KBC with the exact entropy maximum (Newton's method) ----

def _exact_entropy_wh(f, ws, feq, ds, dh):
    """Maximiser of S(w) = -sum f'(w) ln(f'(w)/f_eq) (Eq. 17) by bounded Brent search
    (scipy), an iteration that shares nothing with the oracle's Newton loop."""
    from scipy.optimize import minimize_scalar

    def negS(w):
        fp = f - ws * ds - w * dh
        if np.any(fp <= 0):
            return np.inf
        return float(np.sum(fp * np.log(fp / feq)))
    wh = 1 + (1 - ws) * np.sum(ds * dh / feq) / np.sum(dh * dh / feq)
    r = minimize_scalar(negS, bounds=(wh - 1.5, wh + 1.5), method="bounded",
                        options={"xatol": 1e-12, "maxiter": 2000})
    return r.x


@pytest.mark.parametrize("Q", [19, 27])
@pytest.mark.parametrize("ws", [1.99, 1.6])
def test_kbc_exact_maximises_entropy(ws, Q):
    m = O.Method(Q=Q, op="kbc_exact", rates=(ws,))
    c, _, _ = O.stencil_arrays(Q)
    for amp in (1e-3, 0.05, 0.4):
        f = _state(Q, amp)
        feq, ds, dh, wh_lin = _kbc_reference(f, ws, Q)
        out = O.collide_cell(m, f)
        # the update is still of the form of Eq. (16) with the same Delta_s
        w_star = np.dot(f - ws * ds - out, dh) / np.dot(dh, dh)
        np.testing.assert_allclose(out, f - ws * ds - w_star * dh, rtol=0, atol=1e-15)
        # optimality condition of P:620-623 holds to rounding
        g = np.sum(dh * (np.log(out / feq) + 1))
        assert abs(g) < 1e-13 * max(1.0, np.sum(np.abs(dh))), g
        # and it is the maximum found by an unrelated search (S is too flat near equilibrium for a
        # value-based search to locate w better than ~sqrt(eps / S''), so only the larger amplitudes)
        if amp >= 0.05:
            assert abs(w_star - _exact_entropy_wh(f, ws, feq, ds, dh)) < 1e-6
        # near equilibrium the linearisation of P:627-629 is accurate
        if amp <= 1e-3:
            assert abs(w_star - wh_lin) < 5e-3
        assert abs(out.sum() - f.sum()) < 1e-15
        np.testing.assert_allclose(c.T @ out, c.T @ f, atol=1e-16)
    # far from equilibrium the exact and linearised rates differ (the variant is not a relabel)
    f = _state(Q, 0.4)
    feq, ds, dh, wh_lin = _kbc_reference(f, ws, Q)
    out = O.collide_cell(m, f)
    assert abs(np.dot(f - ws * ds - out, dh) / np.dot(dh, dh) - wh_lin) > 1e-4


@pytest.mark.parametrize("Q", [19, 27])
def test_kbc_exact_limits(Q):
    """w_s = 1: f' = f_eq + (1 - w) Dh, whose entropy is maximal at w = 1 (sum Dh = 0) -> f_eq;
    equilibrium is a fixed point (Dh = 0)."""
    f = _state(Q, 0.1)
    feq, _, _, _ = _kbc_reference(f, 1.0, Q)
    np.testing.assert_allclose(O.collide_cell(O.Method(Q=Q, op="kbc_exact", rates=(1.0,)), f), feq,
                               rtol=0, atol=1e-15)
    e = O.equilibrium_cell(Q, 0.99, np.array([0.01, 0.02, -0.03]))
    np.testing.assert_allclose(O.collide_cell(O.Method(Q=Q, op="kbc_exact", rates=(1.8,)), e), e,
                               rtol=0, atol=1e-15)
