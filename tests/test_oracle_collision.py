"""Oracle pins: collision operators (CPU, no GPU).

Pins per SURVEY §8(c): conservation, equilibrium fixed points, degeneration SRT = TRT = MRT,
the closed form of weighted MRT at config-2 rates, and for the cumulant operator the
generating-function definition Eq. (9) evaluated by an independent route (Cauchy/FFT Taylor
coefficients), round trip, product-equilibrium fixed point and the Gaussian (Isserlis) closed
form at config-3 rates.
"""
from itertools import combinations, product

import numpy as np
import pytest

import oracle as O

RNG = np.random.default_rng(1234)
EPS = np.finfo(np.float64).eps


@pytest.fixture(autouse=True)
def _reseed(request):
    """Per-test seeded states: the draws do not depend on test order (xdist, -k selections)."""
    global RNG
    import zlib
    RNG = np.random.default_rng(zlib.crc32(request.node.nodeid.encode()))


def _random_state(Q, amp=0.02):
    rho = 1 + RNG.uniform(-0.05, 0.05)
    u = RNG.uniform(-0.05, 0.05, 3)
    feq = O.equilibrium_cell(Q, rho, u)
    _, w, _ = O.stencil_arrays(Q)
    return feq + amp * w * RNG.uniform(-1, 1, Q)


METHODS = [
    O.Method(Q=19, op="srt", rates=(1.8,)),
    O.Method(Q=27, op="srt", rates=(0.7,)),
    O.Method(Q=19, op="trt", rates=(1.6, 0.5)),
    O.Method(Q=27, op="trt", rates=(1.3, 1.1)),
    O.Method(Q=19, op="mrt", rates=(1.9, 1.3, 1.1, 0.8)),
    O.Method(Q=27, op="mrt", rates=(1.9, 1.3, 1.1, 0.8)),  # D3Q27 MRT (generated GPU operator)
    O.Method(Q=27, op="cumulant", rates=(1.95, 1.2, 1.1, 0.9, 1.3, 0.7)),
]


@pytest.mark.parametrize("m", METHODS, ids=lambda m: f"{m.op}{m.Q}")
def test_collision_conserves_mass_momentum(m):
    c, _, _ = O.stencil_arrays(m.Q)
    for _ in range(10):
        f = _random_state(m.Q)
        g = O.collide_cell(m, f)
        assert abs(g.sum() - f.sum()) < 1e-15
        np.testing.assert_allclose(c.T @ g, c.T @ f, atol=1e-16)
        assert np.abs(g - f).max() > 1e-6  # it does something


@pytest.mark.parametrize("m", METHODS, ids=lambda m: f"{m.op}{m.Q}")
def test_equilibrium_is_fixed_point(m):
    rho, u = 1.02, np.array([0.03, -0.02, 0.05])
    feq = (O.product_equilibrium_cell if m.op == "cumulant" else O.equilibrium_cell)(m.Q, rho, u)
    np.testing.assert_allclose(O.collide_cell(m, feq), feq, rtol=0, atol=1e-15)


def test_srt_literal_eq1():
    """Eq. (1): f* = omega f_eq + (1-omega) f with rho, u from Eq. (2)."""
    m = METHODS[0]
    c, w, _ = O.stencil_arrays(19)
    f = _random_state(19)
    rho = f.sum()
    u = c.T @ f / rho
    cu = c @ u
    feq = w * rho * (1 + 3 * cu + 4.5 * cu ** 2 - 1.5 * u @ u)
    np.testing.assert_allclose(O.collide_cell(m, f), 1.8 * feq + (1 - 1.8) * f, rtol=0, atol=1e-15)


@pytest.mark.parametrize("force", [(0, 0, 0), (1e-3, -2e-3, 5e-4)])
def test_trt_equal_rates_is_srt(force):
    for Q in (19, 27):
        f = _random_state(Q)
        a = O.collide_cell(O.Method(Q=Q, op="trt", rates=(1.37, 1.37), force=force), f)
        b = O.collide_cell(O.Method(Q=Q, op="srt", rates=(1.37,), force=force), f)
        np.testing.assert_allclose(a, b, rtol=0, atol=1e-16)


@pytest.mark.parametrize("Q", [19, 27])
def test_mrt_equal_rates_is_srt(Q):
    f = _random_state(Q)
    a = O.collide_cell(O.Method(Q=Q, op="mrt", rates=(1.37, 1.37, 1.37, 1.37)), f)
    b = O.collide_cell(O.Method(Q=Q, op="srt", rates=(1.37,)), f)
    np.testing.assert_allclose(a, b, rtol=0, atol=1e-15)


@pytest.mark.parametrize("Q", [19, 27])
def test_mrt_config2_closed_form(Q):
    """G6: with omega_shear = ws and every other rate 1, weighted MRT gives
    f* = f_eq - (ws - 1) (9/2) w_q c_q c_q : dev(Pi_neq), Pi_neq = sum_q c c (f - f_eq)
    (D3Q27 too: the projector needs only the 4th-order isotropy of the weights)."""
    c, w, _ = O.stencil_arrays(Q)
    m = O.Method(Q=Q, op="mrt", rates=(1.9, 1.0, 1.0, 1.0))
    for _ in range(5):
        f = _random_state(Q)
        rho = f.sum()
        u = c.T @ f / rho
        feq = O.equilibrium_cell(Q, rho, u)
        Pi = np.einsum("qa,qb,q->ab", c, c, f - feq)
        dev = Pi - np.trace(Pi) / 3 * np.eye(3)
        ref = feq - (1.9 - 1) * 4.5 * w * np.einsum("qa,qb,ab->q", c, c, dev)
        # rounding-order bound (G16): the two routes each sum Q products of O(|f|) terms
        np.testing.assert_allclose(O.collide_cell(m, f), ref, rtol=0, atol=Q * EPS * np.abs(f).max())


def test_mrt_unweighted_differs_at_config2_rates():
    f = _random_state(19)
    a = O.collide_cell(O.Method(Q=19, op="mrt", rates=(1.9, 1.0, 1.0, 1.0)), f)
    b = O.collide_cell(O.Method(Q=19, op="mrt", rates=(1.9, 1.0, 1.0, 1.0), mrt_weighted=False), f)
    assert np.abs(a - b).max() > 1e-7  # G5: the reading matters


def test_trt_guo_momentum_gain_and_source_parity():
    """G4: one collision adds exactly F to the momentum and leaves the mass unchanged."""
    F = np.array([1e-3, -2e-3, 5e-4])
    for Q in (19, 27):
        c, _, _ = O.stencil_arrays(Q)
        f = _random_state(Q)
        g = O.collide_cell(O.Method(Q=Q, op="trt", rates=(1.6, 0.5), force=F), f)
        assert abs(g.sum() - f.sum()) < 1e-15
        np.testing.assert_allclose(c.T @ g - c.T @ f, F, rtol=1e-12, atol=1e-17)


# ---------------------------------------------------------------------------------------
# Cumulants
# ---------------------------------------------------------------------------------------
def _taylor_coeffs_of_K(f, c, r=0.3, N=16):
    """[xi^abc] K(xi), K = ln sum_q f_q exp(c_q . xi) (Eq. 9), by the Cauchy integral on a
    polydisc of radius r (trapezoidal rule = FFT; aliasing error ~ r^N)."""
    th = 2 * np.pi * np.arange(N) / N
    z = r * np.exp(1j * th)
    X, Y, Z = np.meshgrid(z, z, z, indexing="ij")
    S = sum(fq * np.exp(cq[0] * X + cq[1] * Y + cq[2] * Z) for fq, cq in zip(f, c))
    K = np.log(S)
    coef = np.fft.fftn(K) / N ** 3
    out = np.zeros((3, 3, 3))
    for a, b, cc in product(range(3), repeat=3):
        out[a, b, cc] = (coef[a, b, cc] / r ** (a + b + cc)).real
    return out


def test_cumulants_match_generating_function_eq9():
    c, _, _ = O.stencil_arrays(27)
    fact = np.array([1.0, 1.0, 2.0])
    for _ in range(3):
        f = _random_state(27, amp=0.2)
        rho, kap = O.cumulants_cell(f)
        tay = _taylor_coeffs_of_K(f, c)
        ref = tay * fact[:, None, None] * fact[None, :, None] * fact[None, None, :]
        assert abs(rho - f.sum()) < 1e-15
        ref[0, 0, 0] = 0.0
        k2 = kap.copy()
        k2[0, 0, 0] = 0.0
        np.testing.assert_allclose(k2, ref, rtol=0, atol=1e-12)


def test_cumulant_second_order_is_central_moment():
    c, _, _ = O.stencil_arrays(27)
    f = _random_state(27, amp=0.3)
    rho, kap = O.cumulants_cell(f)
    u = c.T @ f / rho
    d = c - u
    Sig = np.einsum("qa,qb,q->ab", d, d, f) / rho
    e2 = {(0, 0): (2, 0, 0), (1, 1): (0, 2, 0), (2, 2): (0, 0, 2), (0, 1): (1, 1, 0), (0, 2): (1, 0, 1), (1, 2): (0, 1, 1)}
    for (a, b), e in e2.items():
        assert abs(kap[e] - Sig[a, b]) < 1e-15
    np.testing.assert_allclose([kap[1, 0, 0], kap[0, 1, 0], kap[0, 0, 1]], u, atol=1e-16)


def test_cumulant_round_trip():
    for _ in range(5):
        f = _random_state(27, amp=0.3)
        rho, kap = O.cumulants_cell(f)
        np.testing.assert_allclose(O.from_cumulants_cell(rho, kap), f, rtol=0, atol=1e-15)


def test_cumulant_all_rates_one_gives_product_equilibrium():
    m = O.Method(Q=27, op="cumulant", rates=(1, 1, 1, 1, 1, 1))
    c, _, _ = O.stencil_arrays(27)
    f = _random_state(27, amp=0.3)
    rho = f.sum()
    u = c.T @ f / rho
    np.testing.assert_allclose(O.collide_cell(m, f), O.product_equilibrium_cell(27, rho, u), rtol=0, atol=2e-16)


def _gaussian_raw_moment(e, mean, cov):
    """E[X^a Y^b Z^c] for a Gaussian by Isserlis' theorem (independent of the series)."""
    idx = [d for d in range(3) for _ in range(e[d])]
    n = len(idx)
    tot = 0.0
    for k in range(n + 1):
        for S in combinations(range(n), k):  # positions taking the fluctuation
            rest = [i for i in range(n) if i not in S]
            mterm = np.prod([mean[idx[i]] for i in rest]) if rest else 1.0
            tot += mterm * _pairings([idx[i] for i in S], cov)
    return tot


def _pairings(ax, cov):
    if not ax:
        return 1.0
    if len(ax) % 2:
        return 0.0
    first, rest = ax[0], ax[1:]
    return sum(cov[first, rest[j]] * _pairings(rest[:j] + rest[j + 1:], cov) for j in range(len(rest)))


def test_cumulant_config3_isserlis_closed_form():
    """G7: ws = 1.95, every other rate 1 -> f* = V^-1 [rho E_{N(u, S')} X^a Y^b Z^c] with
    S' = cs2 I + (1 - ws) dev(S), S = second-order cumulants (central second moments / rho)."""
    c, _, _ = O.stencil_arrays(27)
    m = O.Method(Q=27, op="cumulant", rates=(1.95,))
    A = np.array([[np.prod(np.asarray(cq, float) ** np.array(e)) for cq in c] for e in product(range(3), repeat=3)])
    for _ in range(3):
        f = _random_state(27, amp=0.2)
        rho = f.sum()
        u = c.T @ f / rho
        d = c - u
        Sig = np.einsum("qa,qb,q->ab", d, d, f) / rho
        Sp = np.eye(3) / 3 + (1 - 1.95) * (Sig - np.trace(Sig) / 3 * np.eye(3))
        mom = np.array([rho * _gaussian_raw_moment(e, u, Sp) for e in product(range(3), repeat=3)])
        ref = np.linalg.solve(A, mom)
        np.testing.assert_allclose(O.collide_cell(m, f), ref, rtol=0, atol=2e-15)


# ---------------------------------------------------------------------------------------
# D3Q19 cumulant ("cumulant methods not only for D3Q27 ... but also for D3Q19"): the
# cumulants of the 19 basis monomials are relaxed as in G7 and mapped back through the
# basis moments. Pins: Eq. (9) by the Cauchy/FFT route, round trip, fixed point, conservation, the
# Maxwellian (all rates 1) and Gaussian/Isserlis (C3-like rates) closed forms on the basis moments.
# ---------------------------------------------------------------------------------------
def _basis19():
    c, _, _ = O.stencil_arrays(19)
    es = [e for e in product(range(3), repeat=3) if min(e) == 0]  # the 19 non-zero-row monomials
    A = np.array([[np.prod(np.asarray(cq, float) ** np.array(e)) for cq in c] for e in es])
    return c, es, A


def test_d3q19_cumulants_match_generating_function_eq9():
    c, es, _ = _basis19()
    fact = np.array([1.0, 1.0, 2.0])
    for _ in range(3):
        f = _random_state(19, amp=0.2)
        rho, kap = O.cumulants_any(19, f)
        ref = _taylor_coeffs_of_K(f, c) * fact[:, None, None] * fact[None, :, None] * fact[None, None, :]
        assert abs(rho - f.sum()) < 1e-15
        for e in es[1:]:
            assert abs(kap[e] - ref[e]) < 1e-12, e


def test_d3q19_cumulant_round_trip_and_fixed_point():
    m = O.Method(Q=19, op="cumulant", rates=(1.8, 1.3, 1.1, 0.9))
    c, _, _ = O.stencil_arrays(19)
    for _ in range(5):
        f = _random_state(19, amp=0.3)
        rho, kap = O.cumulants_any(19, f)
        np.testing.assert_allclose(O.from_cumulants_any(19, rho, kap), f, rtol=0, atol=1e-15)
        u = c.T @ f / rho
        feq = O.maxwellian_equilibrium_cell(19, rho, u)
        np.testing.assert_allclose(O.collide_cell(m, feq), feq, rtol=0, atol=2e-16)
        out = O.collide_cell(m, f)
        assert abs(out.sum() - f.sum()) < 1e-15
        np.testing.assert_allclose(c.T @ out, c.T @ f, rtol=0, atol=1e-16)


def test_d3q19_cumulant_all_rates_one_gives_maxwellian_moments():
    """kappa' = kappa_eq -> the basis moments of f* are the untruncated Maxwellian moments
    rho prod_d mu_{e_d}(u_d) (Gaussian factorisation of Eq. 7)."""
    c, es, A = _basis19()
    m = O.Method(Q=19, op="cumulant", rates=(1, 1, 1, 1))
    for _ in range(3):
        f = _random_state(19, amp=0.3)
        rho = f.sum()
        u = c.T @ f / rho
        mu = lambda k, v: 1.0 if k == 0 else v if k == 1 else 1 / 3 + v * v
        ref = np.array([rho * mu(e[0], u[0]) * mu(e[1], u[1]) * mu(e[2], u[2]) for e in es])
        np.testing.assert_allclose(A @ O.collide_cell(m, f), ref, rtol=0, atol=5e-16)


def test_d3q19_cumulant_isserlis_closed_form():
    """C3-like rates (ws = 1.95, others 1): the basis moments of f* are rho E_{N(u, S')}[X^a Y^b Z^c]
    with S' = cs2 I + (1 - ws) dev(S), S the central second moments / rho (Isserlis, brute-force pairings)."""
    c, es, A = _basis19()
    m = O.Method(Q=19, op="cumulant", rates=(1.95,))
    for _ in range(3):
        f = _random_state(19, amp=0.2)
        rho = f.sum()
        u = c.T @ f / rho
        d = c - u
        Sig = np.einsum("qa,qb,q->ab", d, d, f) / rho
        Sp = np.eye(3) / 3 + (1 - 1.95) * (Sig - np.trace(Sig) / 3 * np.eye(3))
        mom = np.array([rho * _gaussian_raw_moment(e, u, Sp) for e in es])
        np.testing.assert_allclose(O.collide_cell(m, f), np.linalg.solve(A, mom), rtol=0, atol=2e-15)


# ---------------------------------------------------------------------------------------
# MRT with one rate per moment: the rows are the paper's weighted
# Gram-Schmidt basis in its order (pinned by the D2Q9 tableau, tests/golden/d2q9_mrt_weighted.txt).
# ---------------------------------------------------------------------------------------
ROW_RATES = (1.9, 1.7, 1.5, 1.3, 1.1, 1.05, 0.9, 1.2, 1.4, 0.8, 1.6, 1.0, 1.25, 0.7, 1.35)


def test_mrt_per_row_rates_reduce_to_group_rates():
    groups = (1.9, 1.3, 1.1, 0.8)
    per_row = (groups[0],) * 5 + (groups[1],) + (groups[2],) * 6 + (groups[3],) * 3
    a = O.Method(Q=19, op="mrt", rates=per_row)
    b = O.Method(Q=19, op="mrt", rates=groups)
    for _ in range(5):
        f = _random_state(19, amp=0.1)
        np.testing.assert_allclose(O.collide_cell(a, f), O.collide_cell(b, f), rtol=0, atol=1e-16)


def test_mrt_per_row_rates_conservation_fixed_point_and_row_relaxation():
    """Each non-conserved moment m_k = <P_k, f> relaxes by its own rate: m_k' - m_k,eq = (1 - w_k)(m_k - m_k,eq)."""
    from oracle import methods
    m = O.Method(Q=19, op="mrt", rates=ROW_RATES)
    M, _, S = m.mrt_matrices()
    c, _, _ = O.stencil_arrays(19)
    for _ in range(5):
        f = _random_state(19, amp=0.1)
        out = O.collide_cell(m, f)
        assert abs(out.sum() - f.sum()) < 1e-15
        np.testing.assert_allclose(c.T @ out, c.T @ f, atol=1e-16)
        rho = f.sum()
        feq = O.equilibrium_cell(19, rho, c.T @ f / rho)
        # rounding bound of a Q-term dot product (G16): Q eps sum_q |M_kq| |f_q| per moment
        bound = 19 * EPS * (np.abs(M) @ np.abs(f))
        np.testing.assert_allclose(M @ (out - feq), (1 - S) * (M @ (f - feq)) * (S > 0) + (M @ (out - feq)) * (S == 0),
                                   rtol=0, atol=bound.max())
        np.testing.assert_allclose(O.collide_cell(m, feq), feq, rtol=0, atol=2e-16)
    assert list(S[4:]) == list(ROW_RATES)


# ---------------------------------------------------------------------------------------
# Independent pins of the general-rate operators (round-2 verdict, "restated pins"):
#  * cumulant with omega_bulk, omega_3..omega_6 != 1: the post-collision cumulants, recomputed from f*
#    by the Cauchy/FFT route of Eq. (9) (no series code), obey each relaxation rule cumulant by
#    cumulant (G7 / G21);
#  * weighted MRT with four distinct group rates: f* = f - sum_g omega_g P_g (f - f_eq), with the
#    weighted projectors P_g built here in floating point from the group monomials (shear
#    combinations, bulk, orders 3 and 4, orthogonalised against all lower groups) — not from the
#    oracle's Gram-Schmidt basis, which the oracle builds in exact rationals (G5/G6).
# ---------------------------------------------------------------------------------------
GENERAL_CUMULANT_RATES = (1.8, 1.3, 1.2, 0.9, 1.1, 0.7)  # omega_s, omega_b, omega_3, omega_4, omega_5, omega_6


@pytest.mark.parametrize("Q", [27, 19])
def test_cumulant_general_rates_each_rule_via_generating_function(Q):
    c, _, _ = O.stencil_arrays(Q)
    rates = GENERAL_CUMULANT_RATES if Q == 27 else GENERAL_CUMULANT_RATES[:4]
    ws, wb = rates[0], rates[1]
    m = O.Method(Q=Q, op="cumulant", rates=rates)
    fact = np.array([1.0, 1.0, 2.0])
    F3 = fact[:, None, None] * fact[None, :, None] * fact[None, None, :]
    es = [e for e in product(range(3), repeat=3) if Q == 27 or min(e) == 0]
    for _ in range(3):
        f = _random_state(Q, amp=0.2)
        fs = O.collide_cell(m, f)
        k0 = _taylor_coeffs_of_K(f, c) * F3
        k1 = _taylor_coeffs_of_K(fs, c) * F3
        assert abs(fs.sum() - f.sum()) < 1e-15
        for e in ((1, 0, 0), (0, 1, 0), (0, 0, 1)):  # order 1 (velocity) unchanged
            assert abs(k1[e] - k0[e]) < 1e-12, e
        diag = [(2, 0, 0), (0, 2, 0), (0, 0, 2)]
        T0, T1 = sum(k0[e] for e in diag), sum(k1[e] for e in diag)
        assert abs(T1 - (T0 + wb * (1.0 - T0))) < 1e-12  # trace -> its equilibrium 3 c_s^2 = 1 at rate omega_b
        for e in diag:  # deviator -> (1 - omega_s) deviator
            assert abs((k1[e] - T1 / 3) - (1 - ws) * (k0[e] - T0 / 3)) < 1e-12, e
        for e in ((1, 1, 0), (1, 0, 1), (0, 1, 1)):  # off-diagonal -> (1 - omega_s)
            assert abs(k1[e] - (1 - ws) * k0[e]) < 1e-12, e
        n_checked = 0
        for e in es:
            n = sum(e)
            if n >= 3:  # order n -> (1 - omega_n) kappa (Maxwellian value 0)
                assert abs(k1[e] - (1 - rates[n - 1]) * k0[e]) < 1e-11, e
                assert abs(k0[e]) > 1e-6  # the check is not vacuous
                n_checked += 1
        assert n_checked == (17 if Q == 27 else 9)  # all orders 3..6 (D3Q27) / 3..4 (D3Q19)


def _group_polys(Q):
    """Non-conserved moment groups of the weighted MRT (G6) as monomial-exponent combinations."""
    sq = {"x2": (2, 0, 0), "y2": (0, 2, 0), "z2": (0, 0, 2)}
    shear = [[(1, sq["x2"]), (-1, sq["y2"])], [(1, (1, 1, 0))], [(1, (1, 0, 1))], [(1, sq["y2"]), (-1, sq["z2"])],
             [(1, (0, 1, 1))]]
    bulk = [[(1, sq["x2"]), (1, sq["y2"]), (1, sq["z2"])]]
    es = [e for e in product(range(3), repeat=3) if Q == 27 or min(e) == 0]
    order3 = [[(1, e)] for e in es if sum(e) == 3]
    higher = [[(1, e)] for e in es if sum(e) >= 4]
    conserved = [[(1, (0, 0, 0))], [(1, (1, 0, 0))], [(1, (0, 1, 0))], [(1, (0, 0, 1))]]
    return conserved, [shear, bulk, order3, higher]


def _projectors(Q):
    c, w, _ = O.stencil_arrays(Q)
    ev = lambda p: np.array([sum(s * np.prod(np.asarray(cq, float) ** np.array(e)) for s, e in p) for cq in c])
    conserved, groups = _group_polys(Q)
    lower = np.array([ev(p) for p in conserved]).T  # columns: functions of q
    W = np.diag(w)
    out = []
    for g in groups:
        B = np.array([ev(p) for p in g]).T
        # weighted-orthogonal complement of the lower groups' span: G = B - L (L^T W L)^-1 L^T W B
        G = B - lower @ np.linalg.solve(lower.T @ W @ lower, lower.T @ W @ B)
        out.append(W @ G @ np.linalg.solve(G.T @ W @ G, G.T))  # population-space projector of the group
        lower = np.hstack([lower, B])
    return out


@pytest.mark.parametrize("Q", [19, 27])
def test_mrt_distinct_group_rates_independent_projectors(Q):
    rates = (1.9, 1.3, 1.1, 0.8)  # shear, bulk, order 3, order >= 4
    m = O.Method(Q=Q, op="mrt", rates=rates)
    c, _, _ = O.stencil_arrays(Q)
    P = _projectors(Q)
    for i, Pi in enumerate(P):  # complementary projectors: P_i P_j = delta_ij P_i
        for j, Pj in enumerate(P):
            np.testing.assert_allclose(Pi @ Pj, Pi if i == j else 0 * Pi, atol=1e-13)
    for _ in range(5):
        f = _random_state(Q, amp=0.1)
        rho = f.sum()
        feq = O.equilibrium_cell(Q, rho, c.T @ f / rho)
        ref = f - sum(wg * (Pg @ (f - feq)) for wg, Pg in zip(rates, P))
        np.testing.assert_allclose(O.collide_cell(m, f), ref, rtol=0, atol=1e-15)
