"""Oracle pins: stencils, moment bases and the equilibrium (CPU, no GPU).

Each test checks the oracle against something other than itself: values printed in the paper
(tests/golden/, with citations), closed-form lattice isotropy, or exact identities.
"""
import os
from fractions import Fraction as Fr
from itertools import product

import numpy as np
import pytest

import oracle as O
from oracle import methods

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _golden(name):
    rows = []
    with open(os.path.join(GOLD, name)) as fh:
        for line in fh:
            line = line.strip()
            if line and not line.startswith("#"):
                rows.append([s.strip() for s in line.split("|")] if "|" in line else line.split())
    return rows


# ---------------------------------------------------------------------------------------
# Stencils: isotropy up to 4th order is a closed form for the weights.
# ---------------------------------------------------------------------------------------
@pytest.mark.parametrize("Q", [19, 27])
def test_stencil_isotropy_c_oracle(Q):
    c, w, opp = O.stencil_arrays(Q)
    assert len(set(map(tuple, c.tolist()))) == Q
    assert abs(w.sum() - 1) < 1e-15
    for a in range(3):
        assert abs((w * c[:, a]).sum()) < 1e-16
        for b in range(3):
            assert abs((w * c[:, a] * c[:, b]).sum() - (a == b) / 3) < 1e-15
            for g in range(3):
                assert abs((w * c[:, a] * c[:, b] * c[:, g]).sum()) < 1e-16
    assert abs((w * c[:, 0] ** 4).sum() - 1 / 3) < 1e-15
    assert abs((w * c[:, 0] ** 2 * c[:, 1] ** 2).sum() - 1 / 9) < 1e-15
    np.testing.assert_array_equal(c[opp], -c)


@pytest.mark.parametrize("name", ["D2Q9", "D3Q15", "D3Q19", "D3Q27"])
def test_stencil_isotropy_exact(name):
    dirs, w = methods.stencil(name), methods.weights(name)
    d = len(dirs[0])
    assert sum(w) == 1
    for a, b in product(range(d), repeat=2):
        assert sum(wi * c[a] * c[b] for c, wi in zip(dirs, w)) == (Fr(1, 3) if a == b else 0)
    assert sum(wi * c[0] ** 4 for c, wi in zip(dirs, w)) == Fr(1, 3)


def test_stencil_order_matches_between_c_and_python():
    for Q in (19, 27):
        c, w, opp = O.stencil_arrays(Q)
        dirs = methods.stencil(f"D3Q{Q}")
        assert [tuple(r) for r in c.tolist()] == dirs
        assert [float(v) for v in methods.weights(f"D3Q{Q}")] == w.tolist()
        assert methods.opposite(f"D3Q{Q}") == opp.tolist()
    # D3Q19 = D3Q27 minus the corners
    assert set(methods.stencil("D3Q27")) - set(methods.stencil("D3Q19")) == set(product((-1, 1), repeat=3))


# ---------------------------------------------------------------------------------------
# Monomial basis construction
# ---------------------------------------------------------------------------------------
def test_d3q19_zero_row_monomials_paper():
    gold = {tuple(int(v) for v in r) for r in _golden("d3q19_zero_row_monomials.txt")}
    got = set(methods.zero_row_monomials("D3Q19"))
    assert got == gold and len(got) == 8           # "8 out of the 27"
    assert (2, 1, 1) in got and (1, 1, 1) in got    # the two examples named at P:336
    assert methods.zero_row_monomials("D3Q27") == []  # D3Q27: all 27 independent


def test_d3q15_group_example_paper():
    # group [x^2 y, y z^2, x^2 y z^2] -> keep lowest order, sum: x^2 y + y z^2
    basis = methods.monomial_basis("D3Q15")
    assert {(2, 1, 0): Fr(1), (0, 1, 2): Fr(1)} in basis
    assert len(basis) == 15


def test_d2q9_trt_raw_moments_paper():
    gold = _golden("d2q9_trt_tableau.txt")
    got = [methods.poly_str(p) for p in methods.monomial_basis("D2Q9")]
    assert sorted(got) == sorted(r[0] for r in gold)
    # even/odd classification of the tableau: parity of total degree
    for r in gold:
        p = next(p for p in methods.monomial_basis("D2Q9") if methods.poly_str(p) == r[0])
        assert (methods.order(p) % 2 == 0) == (r[1] == "omega_e")


def test_d2q9_weighted_gram_schmidt_paper():
    gold = _golden("d2q9_mrt_weighted.txt")
    polys, groups = methods.mrt_method("D2Q9", weighted=True)
    got = [methods.poly_str(p) for p in polys]
    assert got == [r[0] for r in gold]
    rate_of = {"conserved": "0", "shear": "omega_0", "bulk": "omega_1", "order3": "omega_2", "order4+": "omega_3"}
    assert [rate_of[g] for g in groups] == [r[1] for r in gold]
    # the standard (unweighted) product gives a different basis (P:345 offers both)
    un = [methods.poly_str(p) for p in methods.mrt_method("D2Q9", weighted=False)[0]]
    assert un != got


@pytest.mark.parametrize("weighted", [True, False])
def test_d3q19_mrt_basis_orthogonal_and_invertible(weighted):
    name = "D3Q19"
    dirs, w = methods.stencil(name), methods.weights(name)
    polys, groups = methods.mrt_method(name, weighted=weighted)
    M = methods.moment_matrix(polys, dirs)
    Minv = methods.mat_inverse(M)
    n = len(M)
    for i in range(n):
        for j in range(n):
            assert sum(M[i][k] * Minv[k][j] for k in range(n)) == (1 if i == j else 0)
    ww = w if weighted else [Fr(1)] * n
    for i in range(n):
        for j in range(i):
            assert sum(ww[q] * M[i][q] * M[j][q] for q in range(n)) == 0
    assert groups.count("shear") == 5 and groups.count("bulk") == 1
    assert groups.count("order3") == 6 and groups.count("order4+") == 3 and groups.count("conserved") == 4


# ---------------------------------------------------------------------------------------
# Equilibrium, Eq. (3): moments are closed forms.
# ---------------------------------------------------------------------------------------
@pytest.mark.parametrize("Q", [19, 27])
def test_equilibrium_moments_closed_form(Q):
    c, w, _ = O.stencil_arrays(Q)
    rng = np.random.default_rng(1)
    for _ in range(20):
        rho = 1 + rng.uniform(-0.1, 0.1)
        u = rng.uniform(-0.1, 0.1, 3)
        f = O.equilibrium_cell(Q, rho, u)
        assert abs(f.sum() - rho) < 1e-15
        np.testing.assert_allclose(c.T @ f, rho * u, atol=1e-16)
        Pi = np.einsum("qa,qb,q->ab", c, c, f)
        np.testing.assert_allclose(Pi, rho * (np.eye(3) / 3 + np.outer(u, u)), atol=2e-16)
    # u = 0 -> w_q rho
    np.testing.assert_allclose(O.equilibrium_cell(Q, 1.25, np.zeros(3)), 1.25 * w, rtol=0, atol=1e-16)


def _maxwellian_moment_trunc2(e, rho, u):
    """Continuous Maxwellian raw moment E[xi^e] (Eqs. 7-8) = rho prod_d mu_{e_d}(u_d)
    with mu_0 = 1, mu_1 = u, mu_2 = u^2 + cs^2, truncated to 2nd order in u (Gaussian factorises)."""
    from itertools import product as P
    # each factor as polynomial in (u-order, coef): mu_0=[(0,1)], mu_1=[(1,u)], mu_2=[(0,1/3),(2,u^2)]
    facs = []
    for d, k in enumerate(e):
        facs.append({0: [(0, 1.0)], 1: [(1, u[d])], 2: [(0, 1 / 3), (2, u[d] ** 2)]}[k])
    tot = 0.0
    for terms in P(*facs):
        order = sum(t[0] for t in terms)
        if order <= 2:
            tot += np.prod([t[1] for t in terms])
    return rho * tot


def test_d3q27_equilibrium_equals_maxwellian_moments_paper():
    """for D3Q27 the moment-matched (Maxwellian) equilibrium is exactly Eq. (3);
    for D3Q19 it differs."""
    c, _, _ = O.stencil_arrays(27)
    rho, u = 1.03, np.array([0.04, -0.03, 0.02])
    f = O.equilibrium_cell(27, rho, u)
    for e in product(range(3), repeat=3):
        m = float((f * np.prod(c.astype(float) ** np.array(e), axis=1)).sum())
        assert abs(m - _maxwellian_moment_trunc2(e, rho, u)) < 1e-15, e
    c19, _, _ = O.stencil_arrays(19)
    f19 = O.equilibrium_cell(19, rho, u)
    worst = max(abs(float((f19 * np.prod(c19.astype(float) ** np.array(e), axis=1)).sum())
                    - _maxwellian_moment_trunc2(e, rho, u)) for e in product(range(3), repeat=3)
                if not all(k >= 1 for k in e))
    assert worst > 1e-5
    # SURVEY G1 scratch: the x^2 y^2 moment differs by -rho u_z^2 / 6
    m22 = float((f19 * c19[:, 0] ** 2 * c19[:, 1] ** 2).sum())
    assert abs(m22 - _maxwellian_moment_trunc2((2, 2, 0), rho, u) - (-rho * u[2] ** 2 / 6)) < 1e-15


def test_g6_group_rate_mrt_is_invariant_under_within_order_gram_schmidt_permutations():
    """DESIGN G6: with one rate per group {shear, bulk, order 3, order >= 4} the MRT operator M^-1 S M does
    not depend on the order in which Gram-Schmidt meets the moments of one order (each group's span is
    canonical; shear is weighted-orthogonal to bulk). 12 random within-order permutations of the D3Q19
    input sequence (shear moments permuted among themselves, bulk kept after them): M^-1 S M is EQUAL in
    exact rationals."""
    import random
    from fractions import Fraction as Fr
    import numpy as np
    from oracle import methods as Mt
    name = "D3Q19"
    dirs, w = Mt.stencil(name), Mt.weights(name)
    basis = Mt.monomial_basis(name)
    basis, bulk = Mt.split_shear_bulk(basis, 3)
    basis = Mt.sort_moments(basis, bulk)
    rates = {"conserved": Fr(0), "shear": Fr(19, 10), "bulk": Fr(13, 10), "order3": Fr(11, 10), "order4+": Fr(4, 5)}

    def operator(seq):
        polys = Mt.gram_schmidt(seq, dirs, w)
        groups = []
        for raw in seq:
            o = Mt.order(raw)
            groups.append("conserved" if o <= 1 else ("bulk" if raw == bulk else "shear") if o == 2 else
                          "order3" if o == 3 else "order4+")
        M = Mt.moment_matrix(polys, dirs)
        Mi = Mt.mat_inverse(M)
        n = len(M)
        SM = [[rates[groups[i]] * M[i][j] for j in range(n)] for i in range(n)]
        return [[sum((Mi[i][k] * SM[k][j] for k in range(n)), Fr(0)) for j in range(n)] for i in range(n)]

    ref = operator(basis)
    rng = random.Random(7)
    for _ in range(12):
        seq = []
        for o in range(5):
            block = [p for p in basis if Mt.order(p) == o and p != bulk]
            rng.shuffle(block)
            seq += block
            if o == 2:
                seq.append(bulk)
        assert len(seq) == len(basis) and seq != basis
        assert operator(seq) == ref
    # the check is not vacuous: an order-4 moment met before the (even, non-orthogonal) order-2 ones changes
    # the operator (before the odd order-3 ones it would not: odd and even moments are orthogonal)
    o4 = [p for p in basis if Mt.order(p) == 4]
    seq = [p for p in basis if Mt.order(p) <= 1] + o4[:1] + [p for p in basis if Mt.order(p) in (2, 3)] + o4[1:]
    assert operator(seq) != ref
