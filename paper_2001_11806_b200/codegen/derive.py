"""Derivation of the collision operator and the FLOP-minimising simplification pipeline.

Follows the paper's "Compute Kernel Generation / Simplification" section (Tables I
and II):

* the operator is first written the way an automatic derivation produces it: moments
  m = M g, equilibrium moments m_eq = M g_eq(rho, u), relaxation in moment space and the
  transformation back, g' = g - M^-1 S (m - m_eq) (Eq. 4), with rho and u as subexpressions;
* "only CSE": sympy's CSE on that form;
* the custom pipeline in the paper's order: expand; quadratic velocity products
  u_i u_j -> ((u_i + u_j)^2 - u_i^2 - u_j^2) / 2 with a new subexpression e = u_i + u_j; expand;
  factor the relaxation rates; the common quadratic term (the centre expression with all
  pre-collision values 0 and rates 1); substitution of existing subexpressions; CSE;
* the "direction CSE" variant: the two expressions of a direction pair q, q-bar are
  rewritten as (even part) +- (odd part) before the global CSE;
* the cheapest variant is kept.

FLOPs are counted as additions (incl. subtractions), multiplications (a coefficient -1 is free,
it becomes a subtraction), divisions and square roots, the convention of Tables I/II.
Everything is in zero-centred variables g = f - w (DESIGN G12) so the emitted code serves fp32
and fp64 alike.
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import Dict, List, Sequence, Tuple

import sympy as sp

from . import methods

Assign = Tuple[sp.Symbol, sp.Expr]


@dataclass
class Flops:
    adds: int = 0
    muls: int = 0
    divs: int = 0
    sqrts: int = 0

    @property
    def total(self) -> int:
        return self.adds + self.muls + self.divs + self.sqrts

    def __add__(self, o: "Flops") -> "Flops":
        return Flops(self.adds + o.adds, self.muls + o.muls, self.divs + o.divs, self.sqrts + o.sqrts)

    def as_dict(self):
        return {"adds": self.adds, "muls": self.muls, "divs": self.divs, "sqrts": self.sqrts, "total": self.total}


def count_flops(e: sp.Expr) -> Flops:
    """Operations to evaluate `e` as written (no re-association)."""
    if e.is_Atom or e.is_number:  # constants (e.g. sqrt(2)) fold at compile time
        return Flops()
    f = Flops()
    if e.is_Add:
        f.adds += len(e.args) - 1
    elif e.is_Mul:
        args = list(e.args)
        if args[0] == -1:  # negation folds into the enclosing add/sub
            args = args[1:]
        num = [x for x in args if not (x.is_Pow and x.exp.is_Integer and x.exp < 0)]
        den = [x for x in args if x.is_Pow and x.exp.is_Integer and x.exp < 0]
        f.muls += max(len(num) - 1, 0)
        for x in num:
            f = f + count_flops(x)
        if den:  # n / (b1^k1 b2^k2 ...): build the denominator, one division
            f.divs += 1
            f.muls += sum(-int(x.exp) for x in den) - 1
            for x in den:
                f = f + count_flops(x.base)
        return f
    elif e.is_Pow:
        if e.exp == sp.Rational(1, 2):
            f.sqrts += 1
        elif e.exp.is_Integer and e.exp > 0:
            f.muls += int(e.exp) - 1
        elif e.exp.is_Integer and e.exp < 0:
            f.divs += 1
            f.muls += -int(e.exp) - 1
        else:
            raise ValueError(f"unsupported power {e}")
        return f + count_flops(e.base)
    for a in e.args:
        f = f + count_flops(a)
    return f


def count_assignments(subs: Sequence[Assign], main: Sequence[sp.Expr]) -> Flops:
    f = Flops()
    for _, e in subs:
        f = f + count_flops(e)
    for e in main:
        f = f + count_flops(e)
    return f


@dataclass
class Operator:
    """A collision operator as subexpressions + one expression per population."""
    Q: int
    op: str
    g: Tuple[sp.Symbol, ...]
    rates: Tuple[sp.Symbol, ...]
    subs: List[Assign]
    main: List[sp.Expr]
    macro: Tuple[sp.Symbol, ...]          # drho, ux, uy, uz
    history: List[Tuple[str, Flops]] = field(default_factory=list)
    relax: Tuple[sp.Symbol, ...] = ()     # the relaxation-rate symbols the pipeline factors out
    equilibrium: str = "compressible"

    def __post_init__(self):
        if not self.relax:
            self.relax = self.rates

    def flops(self) -> Flops:
        return count_assignments(self.subs, self.main)

    def record(self, label: str):
        self.history.append((label, self.flops()))
        return self


def n_rates(op: str) -> int:
    return {"srt": 1, "trt": 2, "mrt": 4, "smagorinsky": 2}[op]


def derive(Q: int, op: str, equilibrium: str = "compressible") -> Operator:
    """The moment-space form of SRT / TRT / weighted MRT / Smagorinsky-SRT with Eq. (3),
    compressible (rho0 = rho) or incompressible (rho0 = 1 in Eqs. 2 and 3, DESIGN G19).

    Conserved rows: their relaxation rate "can be chosen arbitrarily" because
    m - m_eq vanishes there; SRT gives them omega, TRT omega_e / omega_o by parity (then
    M^-1 S M is omega I, resp. the parity projectors), MRT 0.
    Smagorinsky (Eqs. 11-14; DESIGN G18): SRT with the local rate
    omega = 2 / (tau0 + sqrt(tau0^2 + 18 C_S^2 sqrt(2 Pi:Pi) / rho)), Pi = sum c c (g - g_eq);
    rates = [omega_0, C_S]."""
    incompressible = equilibrium == "incompressible"
    dirs = methods.stencil(Q)
    w = methods.weights(Q)
    g = sp.symbols(f"g0:{Q}")
    rates = sp.symbols(f"omega0:{n_rates(op)}")
    drho, rho, irho, jx, jy, jz, ux, uy, uz = sp.symbols("drho rho inv_rho j_x j_y j_z u_x u_y u_z")
    subs: List[Assign] = [(drho, sp.Add(*g)), (rho, drho + 1)]
    if not incompressible:
        subs.append((irho, 1 / rho))
    for sym, a in ((jx, 0), (jy, 1), (jz, 2)):
        subs.append((sym, sp.Add(*[c[a] * gq for c, gq in zip(dirs, g) if c[a] != 0])))
    for sym, j in ((ux, jx), (uy, jy), (uz, jz)):
        # one division by the density; none with rho0 = 1
        subs.append((sym, j if incompressible else j * irho))
    rho0 = 1 if incompressible else rho
    usq = ux ** 2 + uy ** 2 + uz ** 2
    geq = []
    for c, wq in zip(dirs, w):
        cu = c[0] * ux + c[1] * uy + c[2] * uz
        geq.append(wq * drho + wq * rho0 * (3 * cu + sp.Rational(9, 2) * cu ** 2 - sp.Rational(3, 2) * usq))
    relax = rates
    kind = op
    if op == "smagorinsky":
        om = sp.Symbol("omega_eff")
        tau0, P = sp.symbols("tau0 Pi_norm")
        pis = []
        for a, b in ((0, 0), (1, 1), (2, 2), (0, 1), (0, 2), (1, 2)):
            s_ab = sp.Symbol(f"Pi_{'xyz'[a]}{'xyz'[b]}")
            # non-equilibrium moment: population moment minus the (simplified) equilibrium moment
            m_ab = sp.Add(*[c[a] * c[b] * gq for c, gq in zip(dirs, g) if c[a] * c[b] != 0])
            meq_ab = sp.factor(sp.expand(sum(c[a] * c[b] * eq for c, eq in zip(dirs, geq))))
            subs.append((s_ab, m_ab - meq_ab))
            pis.append((s_ab, a == b))
        subs.append((P, sp.sqrt(2 * sp.Add(*[(1 if diag else 2) * s_ab ** 2 for s_ab, diag in pis]))))
        subs.append((tau0, 1 / rates[0]))
        subs.append((om, 2 / (tau0 + sp.sqrt(tau0 ** 2 + 18 * rates[1] ** 2 * P / rho))))
        relax = (om,)
        kind = "srt"
    M = methods.moment_matrix(Q)
    Minv = M.inv()
    S = methods.relaxation_rates(Q, kind, relax)
    basis = methods.moment_basis(Q)
    for k, (p, grp) in enumerate(basis):
        if grp == "conserved" and kind in ("srt", "trt"):
            order = sp.Poly(p, methods.X, methods.Y, methods.Z).total_degree()
            S[k] = relax[0] if (kind == "srt" or order == 0) else relax[1]
    m = [sp.Add(*[M[k, q] * g[q] for q in range(Q) if M[k, q] != 0]) for k in range(Q)]
    meq = [sp.factor(sp.expand(sum(M[k, q] * geq[q] for q in range(Q)))) for k in range(Q)]
    main = []
    for q in range(Q):
        terms = [Minv[q, k] * S[k] * (m[k] - meq[k]) for k in range(Q) if S[k] != 0 and Minv[q, k] != 0]
        main.append(g[q] - sp.Add(*terms))
    return Operator(Q, op, g, rates, subs, main, (drho, ux, uy, uz), relax=relax,
                    equilibrium=equilibrium).record("initial")


def subs_linear(e: sp.Expr, pattern: sp.Expr, sym: sp.Symbol) -> sp.Expr:
    """Replace every multiple lam * pattern contained term by term in the expanded sum `e` by
    lam * sym (lam a monomial factor, e.g. -omega/18). sympy's subs only finds exact sub-sums."""
    e = sp.expand(e)
    pat = sp.expand(pattern).as_coefficients_dict()
    pterms = list(pat.items())
    if len(pterms) < 2:
        return e
    t0, a0 = pterms[0]
    while True:
        terms = e.as_coefficients_dict()
        done = True
        for t, b in list(terms.items()):
            lam = sp.cancel(b * t / (a0 * t0))
            if not (lam.is_Mul or lam.is_Symbol or lam.is_Number) or any(
                    x.is_Pow and x.exp < 0 for x in sp.Mul.make_args(lam)):
                continue
            ok = True
            for tp, ap in pterms[1:]:
                need = sp.expand(lam * ap * tp)
                nt = need.as_coefficients_dict()
                if len(nt) != 1:
                    ok = False
                    break
                (mt, mc), = nt.items()
                if terms.get(mt, 0) != mc:
                    ok = False
                    break
            if ok:
                e = sp.expand(e - lam * pattern) + lam * sym
                done = False
                break
        if done:
            return e


# ---------------------------------------------------------------------------------------------
# transformations
# ---------------------------------------------------------------------------------------------
def _copy(o: Operator, subs=None, main=None) -> Operator:
    return Operator(o.Q, o.op, o.g, o.rates, list(o.subs if subs is None else subs),
                    list(o.main if main is None else main), o.macro, list(o.history), o.relax, o.equilibrium)


def expand(o: Operator) -> Operator:
    return _copy(o, main=[sp.expand(e) for e in o.main]).record("expand")


def quadratic_velocity_products(o: Operator) -> Operator:
    _, ux, uy, uz = o.macro
    new = list(o.subs)
    rep = {}
    for a, b, name in ((ux, uy, "e_xy"), (ux, uz, "e_xz"), (uy, uz, "e_yz")):
        e = sp.Symbol(name)
        new.append((e, a + b))
        rep[a * b] = (e ** 2 - a ** 2 - b ** 2) / 2
    main = [e.subs(rep) for e in o.main]
    return _copy(o, subs=new, main=main).record("quadratic velocity prod.")


def factor_rates(o: Operator) -> Operator:
    return _copy(o, main=[sp.collect(e, o.relax) for e in o.main]).record("factor omegas")


def common_quadratic_term(o: Operator) -> Operator:
    """Centre expression with g = 0 and all rates 1, as a subexpression."""
    zero = {s: 0 for s in o.g}
    ones = {r: 1 for r in o.relax}
    w0 = methods.weights(o.Q)[0]
    cq = sp.expand(o.main[0].subs(zero).subs(ones) / w0)
    if cq == 0:
        return _copy(o).record("common quadratic term")
    sym = sp.Symbol("c_q")
    new = list(o.subs) + [(sym, cq)]
    main = [sp.collect(subs_linear(e, cq, sym), o.relax) for e in o.main]
    return _copy(o, subs=new, main=main).record("common quadratic term")


def substitute_subexpressions(o: Operator) -> Operator:
    """Search the definitions of existing subexpressions (drho, j) inside the expressions."""
    main = list(o.main)
    for sym, d in o.subs:
        if d.is_Add and len(d.args) > 2:
            main = [subs_linear(e, d, sym) for e in main]
    main = [sp.collect(e, o.relax) for e in main]
    return _copy(o, main=main).record("substitute existing subexpr.")


def cse(o: Operator, label: str = "sympy CSE") -> Operator:
    gen = sp.numbered_symbols("x")
    exprs = [d for _, d in o.subs] + list(o.main)
    repl, red = sp.cse(exprs, symbols=gen, optimizations="basic")
    n = len(o.subs)
    subs = list(repl) + [(s, e) for (s, _), e in zip(o.subs, red[:n])]
    # keep dependency order: a subexpression may use cse symbols and vice versa
    subs = _toposort(subs)
    return _copy(o, subs=subs, main=list(red[n:])).record(label)


def direction_split(o: Operator) -> Operator:
    """Direction-aware form: for each pair (q, q-bar) define s = (e_q + e_qbar)/2 and
    a = (e_q - e_qbar)/2 as subexpressions, e_q = s + a, e_qbar = s - a."""
    opp = methods.opposite(o.Q)
    main = list(o.main)
    subs = list(o.subs)
    for q in range(1, o.Q):
        b = opp[q]
        if q > b:
            continue
        s_sym, a_sym = sp.Symbol(f"s_{q}"), sp.Symbol(f"a_{q}")
        s = sp.collect(sp.expand((main[q] + main[b]) / 2), o.relax)
        a = sp.collect(sp.expand((main[q] - main[b]) / 2), o.relax)
        subs += [(s_sym, s), (a_sym, a)]
        main[q], main[b] = s_sym + a_sym, s_sym - a_sym
    return _copy(o, subs=subs, main=main).record("direction split")


def _toposort(subs: List[Assign]) -> List[Assign]:
    defined = {s for s, _ in subs}
    done, out, pending = set(), [], list(subs)
    while pending:
        rest = []
        for s, e in pending:
            if all((d not in defined) or (d in done) for d in e.free_symbols):
                out.append((s, e))
                done.add(s)
            else:
                rest.append((s, e))
        if len(rest) == len(pending):
            raise RuntimeError("cyclic subexpressions")
        pending = rest
    return out


# ---------------------------------------------------------------------------------------------
# the three strategies and the choice
# ---------------------------------------------------------------------------------------------
def only_cse(o: Operator) -> Operator:
    return cse(o)


def custom(o: Operator, direction: bool = False) -> Operator:
    o = expand(o)
    o = quadratic_velocity_products(o)
    o = expand(o)
    o = factor_rates(o)
    o = common_quadratic_term(o)
    o = substitute_subexpressions(o)
    if direction:
        o = direction_split(o)
    return cse(o)


def strategies(Q: int, op: str, equilibrium: str = "compressible") -> Dict[str, Operator]:
    base = derive(Q, op, equilibrium)
    return {"only_cse": only_cse(base), "custom_direction_cse": custom(base, True), "custom": custom(base)}


def best(results: Dict[str, Operator]) -> Tuple[str, Operator]:
    name = min(results, key=lambda k: results[k].flops().total)
    return name, results[name]


def evaluate(o: Operator, g_values, rate_values) -> List[float]:
    """Numeric evaluation of the assignments in order (used by the tests)."""
    env = {s: sp.Float(v, 30) for s, v in zip(o.g, g_values)}
    env.update({r: sp.Float(v, 30) for r, v in zip(o.rates, rate_values)})
    for s, e in o.subs:
        env[s] = e.xreplace(env).evalf(30)
    return [float(e.xreplace(env).evalf(30)) for e in o.main]
