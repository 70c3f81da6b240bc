"""Exact-rational construction of the LB method tables used by the oracle.

TEST INFRASTRUCTURE — part of the CPU oracle. Only ``tests/``, ``__graft_entry__.smoke()``
and ``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may import anything under
``oracle/``. The product path (``paper_2001_11806_b200``) never does.

Everything here is computed in :class:`fractions.Fraction` and follows the paper
(``/root/reference/PAPER.md``, cited as ``P:<line>``) step by step:

* stencils DdQq with weights and c_s^2 = 1/3 (ordering = SURVEY G10);
* moment polynomials as exponent dictionaries, the discrete moment Eq. (5) and the
  moment matrix M_kq = P_k(c_q) (typo "f_q" read away);
* monomial basis construction with aliasing Eq. (6): exponents in {0,1,2}, zero
  rows dropped (D3Q19: 8 of 27), equal rows grouped (D3Q15);
* shear/bulk split of the 2nd-order moments, sort by order then
  lexicographically, (weighted) Gram-Schmidt;
* relaxation-rate assignment per moment group (shear, bulk, order 3, order >= 4).

Parity unpinned items (definitional readings): the within-order input order
of Gram-Schmidt (G6 — irrelevant when rates are assigned per group, which the tests check).
"""
from __future__ import annotations

from fractions import Fraction as Fr
from itertools import product
from typing import Dict, List, Sequence, Tuple

Poly = Dict[Tuple[int, ...], Fr]  # exponent tuple -> coefficient

CS2 = Fr(1, 3)  # speed of sound squared for first-neighbourhood stencils


# ----------------------------------------------------------------------------------------
# Stencils. Order: centre first, then by |c|_1, then lexicographic with -1<0<1.
# ----------------------------------------------------------------------------------------
def stencil(name: str) -> List[Tuple[int, ...]]:
    """Directions of D2Q9, D3Q15, D3Q19 or D3Q27 in the ABI order."""
    d = int(name[1])
    q = int(name[3:])
    dirs = list(product((-1, 0, 1), repeat=d))
    if name == "D3Q19":
        dirs = [c for c in dirs if sum(abs(v) for v in c) <= 2]  # drop the 8 corners
    elif name == "D3Q15":
        dirs = [c for c in dirs if sum(abs(v) for v in c) in (0, 1, 3)]  # drop the 12 edges
    elif name not in ("D2Q9", "D3Q27"):
        raise ValueError(name)
    dirs.sort(key=lambda c: (sum(abs(v) for v in c), c))
    assert len(dirs) == q
    return dirs


def weights(name: str) -> List[Fr]:
    """Lattice weights by shell |c|^2 (standard values; pinned by isotropy in the tests)."""
    table = {
        "D2Q9": {0: Fr(4, 9), 1: Fr(1, 9), 2: Fr(1, 36)},
        "D3Q15": {0: Fr(2, 9), 1: Fr(1, 9), 3: Fr(1, 72)},
        "D3Q19": {0: Fr(1, 3), 1: Fr(1, 18), 2: Fr(1, 36)},
        "D3Q27": {0: Fr(8, 27), 1: Fr(2, 27), 2: Fr(1, 54), 3: Fr(1, 216)},
    }[name]
    return [table[sum(v * v for v in c)] for c in stencil(name)]


def opposite(name: str) -> List[int]:
    dirs = stencil(name)
    return [dirs.index(tuple(-v for v in c)) for c in dirs]


# ----------------------------------------------------------------------------------------
# Polynomials
# ----------------------------------------------------------------------------------------
def mono(e: Sequence[int]) -> Poly:
    return {tuple(e): Fr(1)}


def padd(a: Poly, b: Poly, s: Fr = Fr(1)) -> Poly:
    out = dict(a)
    for k, v in b.items():
        out[k] = out.get(k, Fr(0)) + s * v
        if out[k] == 0:
            del out[k]
    return out


def pscale(a: Poly, s: Fr) -> Poly:
    return {k: v * s for k, v in a.items() if v * s != 0}


def peval(p: Poly, c: Sequence[int]) -> Fr:
    tot = Fr(0)
    for e, coef in p.items():
        t = coef
        for ci, ei in zip(c, e):
            t *= Fr(ci) ** ei
        tot += t
    return tot


def order(p: Poly) -> int:
    return max(sum(e) for e in p)


def moment_row(p: Poly, dirs) -> List[Fr]:
    """Row k of M: P_k(c_q) for all q (read as M_kq = P_k(c_q), G15)."""
    return [peval(p, c) for c in dirs]


def discrete_moment(p: Poly, dirs, f) -> Fr:
    """Eq. (5): Pi_P(f) = sum_q P(c_q) f_q."""
    return sum((peval(p, c) * fq for c, fq in zip(dirs, f)), Fr(0))


# ----------------------------------------------------------------------------------------
# Monomial basis
# ----------------------------------------------------------------------------------------
def monomial_basis(name: str) -> List[Poly]:
    """Independent monomial moments: exponents in {0,1,2} (aliasing Eq. 6), zero rows dropped,
    equal rows grouped (lowest order kept, summed if several)."""
    dirs = stencil(name)
    d = len(dirs[0])
    groups: Dict[Tuple[Fr, ...], List[Tuple[int, ...]]] = {}
    for e in product((0, 1, 2), repeat=d):
        row = tuple(moment_row(mono(e), dirs))
        if all(v == 0 for v in row):
            continue
        groups.setdefault(row, []).append(e)
    basis = []
    for row, es in groups.items():
        lo = min(sum(e) for e in es)
        keep = [e for e in es if sum(e) == lo]
        p: Poly = {}
        for e in keep:
            p = padd(p, mono(e))
        basis.append(p)
    assert len(basis) == len(dirs), (name, len(basis))
    return basis


def zero_row_monomials(name: str) -> List[Tuple[int, ...]]:
    dirs = stencil(name)
    d = len(dirs[0])
    return [e for e in product((0, 1, 2), repeat=d)
            if all(v == 0 for v in moment_row(mono(e), dirs))]


def _lex_key(p: Poly):
    # lexicographic on the exponent tuples, highest power of x first (x^2 y before x y^2)
    return tuple(sorted((tuple(-v for v in e) for e in p)))


def split_shear_bulk(basis: List[Poly], d: int) -> Tuple[List[Poly], Poly]:
    """Replace {x^2, y^2, (z^2), xy, ...} by shear {x^2-y^2, (y^2-z^2), xy, ...} and the bulk
    moment x^2+y^2(+z^2). Returns (new basis, bulk polynomial)."""
    sq = [tuple(2 if i == j else 0 for i in range(d)) for j in range(d)]
    out = [p for p in basis if not (len(p) == 1 and next(iter(p)) in sq)]
    assert len(out) == len(basis) - d
    bulk: Poly = {}
    for e in sq:
        bulk = padd(bulk, mono(e))
    shear = [padd(mono(sq[j]), mono(sq[j + 1]), Fr(-1)) for j in range(d - 1)]
    # keep second-order group order: shear diagonal, off-diagonal, then bulk
    res = []
    inserted = False
    for p in out:
        if order(p) == 2 and not inserted:
            res.extend(shear)
            inserted = True
        res.append(p)
    if not inserted:
        res.extend(shear)
    res.append(bulk)
    return res, bulk


def sort_moments(basis: List[Poly], bulk: Poly | None = None) -> List[Poly]:
    """Sort by moment order, then lexicographically; within order 2 the split shear
    moments precede the bulk moment as in the D2Q9 tableau."""
    def key(p):
        return (order(p), 1 if (bulk is not None and p == bulk) else 0, _lex_key(p))
    return sorted(basis, key=key)


def inner(p: Poly, q: Poly, dirs, w=None) -> Fr:
    if w is None:
        return sum((peval(p, c) * peval(q, c) for c in dirs), Fr(0))
    return sum((wi * peval(p, c) * peval(q, c) for c, wi in zip(dirs, w)), Fr(0))


def normalise(p: Poly) -> Poly:
    """Integer coefficients, gcd 1, positive leading coefficient (highest order, then lex)."""
    from math import gcd
    den = 1
    for v in p.values():
        den = den * v.denominator // gcd(den, v.denominator)
    p = pscale(p, Fr(den))
    g = 0
    for v in p.values():
        g = gcd(g, abs(v.numerator))
    p = pscale(p, Fr(1, g))
    lead = sorted(p, key=lambda e: (-sum(e), tuple(-v for v in e)))[0]
    if p[lead] < 0:
        p = pscale(p, Fr(-1))
    return p


def gram_schmidt(basis: List[Poly], dirs, w=None) -> List[Poly]:
    """Classical Gram-Schmidt in the order given, weighted by w if given."""
    out: List[Poly] = []
    for p in basis:
        v = dict(p)
        for u in out:
            v = padd(v, u, -inner(p, u, dirs, w) / inner(u, u, dirs, w))
        assert v, "linearly dependent moment"
        out.append(normalise(v))
    return out


# ----------------------------------------------------------------------------------------
# Full MRT method (O4)
# ----------------------------------------------------------------------------------------
def mrt_method(name: str, weighted: bool = True):
    """Orthogonal MRT basis of `name`: returns (polys, groups) with groups[k] in
    {'conserved', 'shear', 'bulk', 'order3', 'order4+'}."""
    dirs = stencil(name)
    d = len(dirs[0])
    w = weights(name)
    basis = monomial_basis(name)
    basis, bulk = split_shear_bulk(basis, d)
    basis = sort_moments(basis, bulk)
    polys = gram_schmidt(basis, dirs, w if weighted else None)
    groups = []
    for raw, p in zip(basis, polys):
        o = order(raw)
        if o <= 1:
            groups.append("conserved")
        elif o == 2:
            groups.append("bulk" if raw == bulk else "shear")
        elif o == 3:
            groups.append("order3")
        else:
            groups.append("order4+")
    return polys, groups


def moment_matrix(polys: List[Poly], dirs) -> List[List[Fr]]:
    return [moment_row(p, dirs) for p in polys]


def mat_inverse(a: List[List[Fr]]) -> List[List[Fr]]:
    """Exact Gauss-Jordan inverse; raises if singular (checks invertibility)."""
    n = len(a)
    m = [list(r) + [Fr(int(i == j)) for j in range(n)] for i, r in enumerate(a)]
    for col in range(n):
        piv = next((r for r in range(col, n) if m[r][col] != 0), None)
        if piv is None:
            raise ValueError("singular moment matrix")
        m[col], m[piv] = m[piv], m[col]
        pv = m[col][col]
        m[col] = [v / pv for v in m[col]]
        for r in range(n):
            if r != col and m[r][col] != 0:
                fac = m[r][col]
                m[r] = [a_ - fac * b_ for a_, b_ in zip(m[r], m[col])]
    return [r[n:] for r in m]


def mrt_rates_per_row(groups: List[str], omega_shear, omega_bulk, omega3, omega4,
                      conserved=0.0) -> List[float]:
    """Diagonal of S (Eq. 4) from the group rates; conserved rows get an arbitrary rate
    ("the relaxation rate can be chosen arbitrarily")."""
    table = {"conserved": conserved, "shear": omega_shear, "bulk": omega_bulk,
             "order3": omega3, "order4+": omega4}
    return [float(table[g]) for g in groups]


def poly_str(p: Poly, names="xyz") -> str:
    """Human-readable polynomial, used by golden fixtures (e.g. '9x^2y^2-3x^2-3y^2+1')."""
    terms = sorted(p.items(), key=lambda kv: (-sum(kv[0]), tuple(-v for v in kv[0])))
    s = ""
    for e, c in terms:
        mon = "".join(names[i] + (f"^{k}" if k > 1 else "") for i, k in enumerate(e) if k)
        coef = c
        sign = "-" if coef < 0 else "+"
        a = abs(coef)
        if mon and a == 1:
            body = mon
        else:
            body = (str(a) if a.denominator == 1 else f"{a.numerator}/{a.denominator}") + mon
        s += sign + body
    return s[1:] if s.startswith("+") else s
