"""Symbolic LB method description for the kernel generator (sympy, exact rationals).

Product-side code (it writes CUDA that is compiled into ``liblbm_b200.so``); it never imports
``oracle/``. It restates the paper's construction of a moment-based method:

* stencils D3Q19 / D3Q27 with weights, c_s^2 = 1/3, direction order = ABI
  order (centre, then |c|_1, then lexicographic with -1 < 0 < 1; DESIGN G10);
* monomial moments with exponents in {0, 1, 2} (aliasing, Eq. 6), zero rows dropped;
* 2nd-order split into shear (x^2 - y^2, y^2 - z^2, xy, xz, yz) and bulk (x^2 + y^2 + z^2) moments
  (P:347), sorted by order then lexicographically (DESIGN G6);
* weighted Gram-Schmidt (DESIGN G5) and the relaxation-rate groups shear,
  bulk, order 3, order >= 4;
* the 2nd-order compressible equilibrium Eq. (3), written for zero-centred storage
  g = f - w (DESIGN G12): g_eq = w drho + w rho (3 c.u + 9/2 (c.u)^2 - 3/2 u^2), rho = 1 + drho.
"""
from __future__ import annotations

from functools import lru_cache
from itertools import product
from typing import List, Tuple

import sympy as sp

X, Y, Z = sp.symbols("x y z")
CS2 = sp.Rational(1, 3)


@lru_cache(maxsize=None)
def stencil(Q: int) -> Tuple[Tuple[int, int, int], ...]:
    dirs = list(product((-1, 0, 1), repeat=3))
    if Q == 19:
        dirs = [c for c in dirs if sum(abs(v) for v in c) <= 2]
    elif Q != 27:
        raise ValueError(f"D3Q{Q} is not generated")
    dirs.sort(key=lambda c: (sum(abs(v) for v in c), c))
    return tuple(dirs)


@lru_cache(maxsize=None)
def weights(Q: int) -> Tuple[sp.Rational, ...]:
    shell = {19: {0: sp.Rational(1, 3), 1: sp.Rational(1, 18), 2: sp.Rational(1, 36)},
             27: {0: sp.Rational(8, 27), 1: sp.Rational(2, 27), 2: sp.Rational(1, 54), 3: sp.Rational(1, 216)}}[Q]
    return tuple(shell[sum(v * v for v in c)] for c in stencil(Q))


def opposite(Q: int) -> List[int]:
    d = stencil(Q)
    return [d.index(tuple(-v for v in c)) for c in d]


def evaluate(p: sp.Expr, c) -> sp.Rational:
    return sp.Rational(p.subs({X: c[0], Y: c[1], Z: c[2]}))


def _order(p: sp.Expr) -> int:
    return sp.Poly(p, X, Y, Z).total_degree()


@lru_cache(maxsize=None)
def moment_basis(Q: int, weighted: bool = True):
    """Orthogonal moment polynomials and their groups: list of (poly, group), group in
    {'conserved', 'shear', 'bulk', 'order3', 'order4'}."""
    dirs = stencil(Q)
    w = weights(Q)
    monos = []
    for e in product((0, 1, 2), repeat=3):
        m = X ** e[0] * Y ** e[1] * Z ** e[2]
        if any(evaluate(m, c) != 0 for c in dirs):
            monos.append((e, m))
    assert len(monos) == Q, (Q, len(monos))
    sq = {(2, 0, 0), (0, 2, 0), (0, 0, 2)}
    rest = [(e, m) for e, m in monos if e not in sq]
    bulk = X ** 2 + Y ** 2 + Z ** 2
    shear = [X ** 2 - Y ** 2, Y ** 2 - Z ** 2]

    def lex(e):
        return tuple(-v for v in e)

    # order, then bulk after shear, then lexicographic with the highest power of x first
    items = [(sum(e), 0, lex(e), m) for e, m in rest]
    items += [(2, 0, (-2, 0, 0), shear[0]), (2, 0, (0, -2, 0), shear[1]), (2, 1, (0, 0, 0), bulk)]
    items.sort(key=lambda t: (t[0], t[1], t[2]))
    raw = [t[3] for t in items]

    def inner(a, b):
        return sum((wi if weighted else 1) * evaluate(a, c) * evaluate(b, c) for c, wi in zip(dirs, w))

    out = []
    for p in raw:
        v = p
        for u in out:
            v = v - inner(p, u) / inner(u, u) * u
        out.append(sp.expand(v))
    groups = []
    for p0 in raw:
        o = _order(p0)
        groups.append("conserved" if o <= 1 else ("bulk" if p0 == bulk else "shear") if o == 2
                      else "order3" if o == 3 else "order4")
    return tuple(zip(out, groups))


def moment_matrix(Q: int, weighted: bool = True) -> sp.Matrix:
    dirs = stencil(Q)
    return sp.Matrix([[evaluate(p, c) for c in dirs] for p, _ in moment_basis(Q, weighted)])


def relaxation_rates(Q: int, op: str, rates) -> List[sp.Expr]:
    """Diagonal of S per basis row: SRT one rate; TRT omega_e on even, omega_o on odd rows
    (P:422-460); MRT one rate per group (shear, bulk, order 3, order >= 4). Conserved rows: 0."""
    basis = moment_basis(Q)
    S = []
    for p, grp in basis:
        if grp == "conserved":
            S.append(sp.Integer(0))
        elif op == "srt":
            S.append(rates[0])
        elif op == "trt":
            S.append(rates[0] if _order(p) % 2 == 0 else rates[1])
        elif op == "mrt":
            S.append({"shear": rates[0], "bulk": rates[1], "order3": rates[2], "order4": rates[3]}[grp])
        else:
            raise ValueError(op)
    return S
