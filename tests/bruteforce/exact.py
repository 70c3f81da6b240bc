"""Exact-rational brute force of one LB time step on tiny lattices (pins the C oracle).

Independent re-statement of the paper's equations in :class:`fractions.Fraction`:
Eq. (2) moments, Eq. (3) 2nd-order compressible equilibrium, Eq. (1)
SRT, TRT with the parity-split Guo source (G4), Eq. (4) MRT
and the cumulant collision via Eq. (9) as a truncated power series (exact in Q
because xi^3 = 0 per axis on {-1,0,1} velocities). Streaming is pull with the
flag-field rules of O6 / G8 (UBB: f_q = f_qbar(x) + 6 w_q rho_w c_q.u_w).

Slow by design: a dict of Fractions per cell. Used only on 4^3 lattices for 1-3 steps.
"""
from __future__ import annotations

from fractions import Fraction as Fr
from itertools import product
from typing import Dict, List, Sequence

from oracle import methods

FLUID, NOSLIP, UBB = 0, 1, 2


def to_fr(x: float) -> Fr:
    return Fr(x)  # exact binary value of the double


class Exact:
    def __init__(self, Q: int, op: str, rates: Sequence, force=(0, 0, 0), ubb_u=(0, 0, 0), equilibrium="compressible"):
        self.equilibrium = equilibrium
        self.name = f"D3Q{Q}"
        self.dirs = methods.stencil(self.name)
        self.w = methods.weights(self.name)
        self.opp = methods.opposite(self.name)
        self.Q = Q
        self.op = op
        self.rates = [to_fr(r) for r in rates]
        self.F = [to_fr(v) for v in force]
        self.uw = [to_fr(v) for v in ubb_u]
        if op in ("mrt", "kbc"):
            polys, groups = methods.mrt_method(self.name, weighted=True)
            self.M = methods.moment_matrix(polys, self.dirs)
            self.Minv = methods.mat_inverse(self.M)
            r = list(self.rates) + [Fr(1)] * 4
            tab = {"conserved": Fr(0), "shear": r[0], "bulk": r[1], "order3": r[2], "order4+": r[3]}
            self.S = [tab[g] for g in groups]
            self.groups = groups
        if op == "cumulant":
            self.rates = list(self.rates) + [Fr(1)] * (6 - len(self.rates))

    # ---- Eq. (2), (3) ---------------------------------------------------------------
    def macro(self, f):
        rho = sum(f, Fr(0))
        j = [sum((c[d] * fq for c, fq in zip(self.dirs, f)), Fr(0)) for d in range(3)]
        rho0 = Fr(1) if self.equilibrium == "incompressible" else rho  # Eq. (2)
        u = [(j[d] + self.F[d] / 2) / rho0 for d in range(3)]
        return rho, u

    def feq(self, rho, u):
        out = []
        uu = sum(v * v for v in u)
        rho0 = Fr(1) if self.equilibrium == "incompressible" else rho
        for c, w in zip(self.dirs, self.w):
            cu = sum(c[d] * u[d] for d in range(3))
            out.append(w * rho + w * rho0 * (3 * cu + Fr(9, 2) * cu * cu - Fr(3, 2) * uu))
        if self.equilibrium == "moment_matched" and self.Q == 19:
            # hand-derived correction (independent of the oracle's M^-1 route): the Maxwellian x^2 y^2
            # moment truncated at 2nd order is rho (cs^4 + cs^2 (ux^2 + uy^2)), Eq. (3) gives
            # rho/9 + rho (ux^2 + uy^2)/3 - rho uz^2/6; the 4 xy-edges carry +rho uz^2/24 each (and
            # cyclically), the faces -2 (a + b) so that orders 0-3 are unchanged, the centre 4 (a + b + c).
            a = {2: rho * u[2] ** 2 / 24, 1: rho * u[1] ** 2 / 24, 0: rho * u[0] ** 2 / 24}  # keyed by the zero axis
            for q, c in enumerate(self.dirs):
                nz = [d for d in range(3) if c[d] != 0]
                if len(nz) == 2:
                    out[q] += a[3 - nz[0] - nz[1]]
                elif len(nz) == 1:
                    out[q] += -2 * sum(a[k] for k in range(3) if k != nz[0])
                else:
                    out[q] += 4 * (a[0] + a[1] + a[2])
        return out

    def guo(self, q, u, we, wo):
        c = self.dirs[q]
        cF = sum(c[d] * self.F[d] for d in range(3))
        cu = sum(c[d] * u[d] for d in range(3))
        uF = sum(u[d] * self.F[d] for d in range(3))
        return (1 - wo / 2) * self.w[q] * 3 * cF + (1 - we / 2) * self.w[q] * (9 * cu * cF - 3 * uF)

    # ---- collision --------------------------------------------------------------------
    def collide(self, f: List[Fr]) -> List[Fr]:
        if self.op == "identity":
            return list(f)
        if self.op == "cumulant":
            return self._cumulant(f)
        rho, u = self.macro(f)
        fe = self.feq(rho, u)
        if self.op == "srt":
            w = self.rates[0]
            return [w * fe[q] + (1 - w) * f[q] + self.guo(q, u, w, w) for q in range(self.Q)]
        if self.op == "trt":
            we, wo = self.rates[0], self.rates[1]
            out = []
            for q in range(self.Q):
                b = self.opp[q]
                fp, fm = (f[q] + f[b]) / 2, (f[q] - f[b]) / 2
                ep, em = (fe[q] + fe[b]) / 2, (fe[q] - fe[b]) / 2
                out.append(f[q] - we * (fp - ep) - wo * (fm - em) + self.guo(q, u, we, wo))
            return out
        if self.op == "mrt":
            Q = self.Q
            m = [sum((self.M[k][q] * f[q] for q in range(Q)), Fr(0)) for k in range(Q)]
            me = [sum((self.M[k][q] * fe[q] for q in range(Q)), Fr(0)) for k in range(Q)]
            mp = [self.S[k] * me[k] + (1 - self.S[k]) * m[k] for k in range(Q)]
            return [sum((self.Minv[q][k] * mp[k] for k in range(Q)), Fr(0)) for q in range(Q)]
        if self.op == "kbc":  # Eqs. (16), (19): s = shear rows, h = the other non-conserved rows
            Q = self.Q
            dm = [sum((self.M[k][q] * (f[q] - fe[q]) for q in range(Q)), Fr(0)) for k in range(Q)]
            ms = [dm[k] if self.groups[k] == "shear" else Fr(0) for k in range(Q)]
            mh = [dm[k] if self.groups[k] not in ("shear", "conserved") else Fr(0) for k in range(Q)]
            ds = [sum((self.Minv[q][k] * ms[k] for k in range(Q)), Fr(0)) for q in range(Q)]
            dh = [sum((self.Minv[q][k] * mh[k] for k in range(Q)), Fr(0)) for q in range(Q)]
            sh = sum((ds[q] * dh[q] / fe[q] for q in range(Q)), Fr(0))
            hh = sum((dh[q] * dh[q] / fe[q] for q in range(Q)), Fr(0))
            ws = self.rates[0]
            wh = 1 + (1 - ws) * sh / hh if hh != 0 else Fr(1)
            return [f[q] - ws * ds[q] - wh * dh[q] for q in range(Q)]
        raise ValueError(self.op)

    # truncated series in xi with exponents <= 2 per axis: dict (a,b,c) -> Fr
    @staticmethod
    def _smul(A: Dict, B: Dict) -> Dict:
        out: Dict = {}
        for ea, va in A.items():
            for eb, vb in B.items():
                e = (ea[0] + eb[0], ea[1] + eb[1], ea[2] + eb[2])
                if max(e) > 2:
                    continue
                out[e] = out.get(e, Fr(0)) + va * vb
        return out

    def _cumulant(self, f):
        fac = [1, 1, 2]
        idx = list(product(range(3), repeat=3))
        m = {e: sum((fq * c[0] ** e[0] * c[1] ** e[1] * c[2] ** e[2] for c, fq in zip(self.dirs, f)), Fr(0))
             for e in idx}
        rho = m[(0, 0, 0)]
        X = {e: m[e] / (rho * fac[e[0]] * fac[e[1]] * fac[e[2]]) for e in idx if e != (0, 0, 0)}
        K: Dict = {}
        P = dict(X)
        for n in range(1, 7):
            if n > 1:
                P = self._smul(P, X)
            for e, v in P.items():
                K[e] = K.get(e, Fr(0)) + (-1) ** (n + 1) * v / n
        kap = {e: K.get(e, Fr(0)) * fac[e[0]] * fac[e[1]] * fac[e[2]] for e in idx if e != (0, 0, 0)}
        ws, wb = self.rates[0], self.rates[1]
        T = kap[(2, 0, 0)] + kap[(0, 2, 0)] + kap[(0, 0, 2)]
        Tn = T + wb * (1 - T)
        for e in ((2, 0, 0), (0, 2, 0), (0, 0, 2)):
            kap[e] = Tn / 3 + (1 - ws) * (kap[e] - T / 3)
        for e in ((1, 1, 0), (1, 0, 1), (0, 1, 1)):
            kap[e] = (1 - ws) * kap[e]
        for e in idx:
            n = sum(e)
            if n >= 3:
                kap[e] = (1 - self.rates[n - 1]) * kap[e]
        Kp = {e: kap[e] / (fac[e[0]] * fac[e[1]] * fac[e[2]]) for e in kap}
        E = {(0, 0, 0): Fr(1)}
        P = dict(Kp)
        nf = 1
        for n in range(1, 7):
            if n > 1:
                P = self._smul(P, Kp)
                nf *= n
            for e, v in P.items():
                E[e] = E.get(e, Fr(0)) + v / nf
        mp = {e: rho * fac[e[0]] * fac[e[1]] * fac[e[2]] * E.get(e, Fr(0)) for e in idx}
        if self.Q == 19:
            return self._d3q19_from_moments(mp)
        out = []
        for c in self.dirs:
            v = Fr(0)
            for e in idx:
                coef = Fr(1)
                for d in range(3):
                    if c[d] == 0:
                        k = {0: Fr(1), 1: Fr(0), 2: Fr(-1)}[e[d]]
                    elif c[d] == 1:
                        k = {0: Fr(0), 1: Fr(1, 2), 2: Fr(1, 2)}[e[d]]
                    else:
                        k = {0: Fr(0), 1: Fr(-1, 2), 2: Fr(1, 2)}[e[d]]
                    coef *= k
                v += coef * mp[e]
            out.append(v)
        return out

    def _d3q19_from_moments(self, M):
        """Hand-derived inverse of the D3Q19 monomial moment map (edges from their 4 plane moments,
        faces from the axis moments minus the edges, centre from the mass) — independent of the
        oracle's M^-1 route."""
        out = []
        for c in self.dirs:
            nz = [d for d in range(3) if c[d] != 0]
            if not nz:
                v = (M[(0, 0, 0)] - M[(2, 0, 0)] - M[(0, 2, 0)] - M[(0, 0, 2)]
                     + M[(2, 2, 0)] + M[(2, 0, 2)] + M[(0, 2, 2)])
            elif len(nz) == 1:
                a = nz[0]
                o = [d for d in range(3) if d != a]
                e2 = tuple(2 if d == a else 0 for d in range(3))
                e1 = tuple(1 if d == a else 0 for d in range(3))
                s_ = M[e2] - sum(M[tuple(2 if d in (a, b) else 0 for d in range(3))] for b in o)
                d_ = M[e1] - sum(M[tuple(1 if d == a else 2 if d == b else 0 for d in range(3))] for b in o)
                v = (s_ + c[a] * d_) / 2
            else:
                a, b = nz
                e = lambda ka, kb: tuple(ka if d == a else kb if d == b else 0 for d in range(3))
                v = (M[e(2, 2)] + c[a] * M[e(1, 2)] + c[b] * M[e(2, 1)] + c[a] * c[b] * M[e(1, 1)]) / 4
            out.append(v)
        return out

    # ---- pull step on an n^3 periodic lattice with flags -------------------------------
    def step_pull(self, f, flags, shape):
        """f: dict (x,y,z) -> list of Q Fractions; flags: dict (x,y,z) -> int."""
        nx, ny, nz = shape
        out = {}
        for (x, y, z), fc in f.items():
            if flags[(x, y, z)] != FLUID:
                out[(x, y, z)] = list(fc)
                continue
            g = []
            for q, c in enumerate(self.dirs):
                nb = ((x - c[0]) % nx, (y - c[1]) % ny, (z - c[2]) % nz)
                fl = flags[nb]
                if fl == FLUID:
                    g.append(f[nb][q])
                else:
                    v = fc[self.opp[q]]
                    if fl == UBB:
                        v += 6 * self.w[q] * sum(c[d] * self.uw[d] for d in range(3))
                    g.append(v)
            out[(x, y, z)] = self.collide(g)
        return out
