"""CPU oracle for the fused lattice Boltzmann stream-collide path (arXiv 2001.11806).

TEST INFRASTRUCTURE. Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may import this package. The product path
(``paper_2001_11806_b200``) shares no code with it; see DESIGN.md "Oracle".

The arithmetic lives in ``lbm_oracle.c`` (plain fp64 C, OpenMP over z) and the exact-rational
method tables in ``methods.py``. This module only builds/loads the C library and marshals
numpy arrays. Arrays use the canonical layout ``f[q, z(+ghosts), y, x]`` (x fastest).
"""
from __future__ import annotations

import ctypes as C
import functools
import os
import subprocess
from dataclasses import dataclass, field
from typing import Optional, Sequence

import numpy as np

from . import methods

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(HERE, "lbm_oracle.c")
LIB = os.path.join(HERE, "liblbm_oracle.so")

SRT, TRT, MRT, CUMULANT, IDENTITY, SMAGORINSKY, KBC, KBC_EXACT = 0, 1, 2, 3, 4, 5, 6, 7
OPS = {"srt": SRT, "trt": TRT, "mrt": MRT, "cumulant": CUMULANT, "identity": IDENTITY,
       "smagorinsky": SMAGORINSKY, "kbc": KBC, "kbc_exact": KBC_EXACT}
FLUID, NOSLIP, UBB = 0, 1, 2


@functools.lru_cache(maxsize=None)
def _monomial_tables(Q: int):
    name = f"D3Q{Q}"
    basis = methods.monomial_basis(name)
    assert all(len(p) == 1 for p in basis), "D3Q19/D3Q27 monomial bases are single monomials"
    exps = [next(iter(p)) for p in basis]
    Mr = methods.moment_matrix(basis, methods.stencil(name))
    Minv = methods.mat_inverse(Mr)
    exps = np.array(exps, dtype=np.int32)
    minv = np.array([[float(v) for v in row] for row in Minv])
    exps.setflags(write=False)
    minv.setflags(write=False)
    return exps, minv


def build(force: bool = False) -> str:
    """Compile the oracle with gcc: fp64, no FMA contraction, OpenMP."""
    if force or not os.path.exists(LIB) or os.path.getmtime(LIB) < os.path.getmtime(SRC):
        cmd = ["gcc", "-O2", "-std=c11", "-fPIC", "-shared", "-fopenmp", "-ffp-contract=off",
               "-fno-fast-math", SRC, "-o", LIB + ".tmp", "-lm"]
        subprocess.check_call(cmd)
        os.replace(LIB + ".tmp", LIB)
    return LIB


class _Cfg(C.Structure):
    _fields_ = [("Q", C.c_int32), ("op", C.c_int32),
                ("nx", C.c_int64), ("ny", C.c_int64), ("nz", C.c_int64),
                ("zghost", C.c_int32), ("nthreads", C.c_int32),
                ("rates", C.c_double * 8), ("force", C.c_double * 3),
                ("ubb_u", C.c_double * 3), ("ubb_rho", C.c_double),
                ("M", C.c_void_p), ("Minv", C.c_void_p), ("S", C.c_void_p),
                ("eq_kind", C.c_int32), ("mono_exp", C.c_void_p), ("Mmono_inv", C.c_void_p),
                ("wall_u", C.c_void_p)]


EQ_KINDS = {"compressible": 0, "incompressible": 1, "moment_matched": 2}


_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = C.CDLL(build())
        P = C.c_void_p
        for name, args, res in [
            ("ora_stencil", [C.c_int, P, P, P], None),
            ("ora_step_pull", [P, P, P, P], C.c_int),
            ("ora_step_push", [P, P, P, P], C.c_int),
            ("ora_stream", [P, P, P, P], C.c_int),
            ("ora_collide_all", [P, P, P], C.c_int),
            ("ora_aa_even", [P, P, P], C.c_int),
            ("ora_aa_odd", [P, P, P], C.c_int),
            ("ora_eso_even", [P, P, P], C.c_int),
            ("ora_eso_odd", [P, P, P], C.c_int),
            ("ora_eso_layout", [P, P, P, C.c_int, C.c_int], C.c_int),
            ("ora_init_equilibrium", [P, P, P, P], C.c_int),
            ("ora_macroscopic", [P, P, C.c_double, P, P], C.c_int),
            ("ora_collide_cell", [P, P, P], None),
            ("ora_smagorinsky_omega_cell", [P, P], C.c_double),
            ("ora_equilibrium_cell", [C.c_int, C.c_double, P, P], None),
            ("ora_product_equilibrium_cell", [C.c_int, C.c_double, P, P], None),
            ("ora_equilibrium_kind_cell", [P, C.c_double, P, P], None),
            ("ora_maxwellian_equilibrium_cell", [P, C.c_double, P, P], None),
            ("ora_from_cumulants_cfg_cell", [P, C.c_double, P, P], None),
            ("ora_cumulants_cell", [C.c_int, P, P], C.c_double),
            ("ora_from_cumulants_cell", [C.c_int, C.c_double, P, P], None),
            ("ora_pull_cell", [P, P, P, C.c_int64, C.c_int64, C.c_int64, P], None),
            ("ora_pack_face", [P, P, C.c_int64, C.c_int, P], C.c_int64),
            ("ora_unpack_face", [P, P, C.c_int64, C.c_int, P], C.c_int64),
        ]:
            fn = getattr(_lib, name)
            fn.argtypes = args
            fn.restype = res
    return _lib


def _p(a: Optional[np.ndarray]):
    if a is None:
        return None
    assert a.flags["C_CONTIGUOUS"], "oracle arrays must be C-contiguous"
    return a.ctypes.data


def stencil_arrays(Q: int):
    c = np.zeros((Q, 3), np.int32)
    w = np.zeros(Q, np.float64)
    opp = np.zeros(Q, np.int32)
    lib().ora_stencil(Q, _p(c), _p(w), _p(opp))
    return c, w, opp


@dataclass
class Method:
    """What the oracle computes: stencil, operator and its parameters (SURVEY §8(b) rates)."""
    Q: int = 19
    op: str = "srt"
    rates: Sequence[float] = (1.8,)
    force: Sequence[float] = (0.0, 0.0, 0.0)
    ubb_u: Sequence[float] = (0.0, 0.0, 0.0)
    ubb_rho: float = 1.0
    mrt_weighted: bool = True
    nthreads: int = 0
    equilibrium: str = "compressible"  # | "incompressible" (rho0 = 1) | "moment_matched"
    _mats: tuple = field(default=None, repr=False)
    _mono: tuple = field(default=None, repr=False)

    def monomial_tables(self):
        """Exponents of the monomial moment basis and the exact inverse of its moment
        matrix (moment-matched equilibrium; D3Q19 cumulant)."""
        return _monomial_tables(self.Q)

    def mrt_matrices(self):
        """M (rows = weighted-orthogonal moment polynomials), M^-1 (exact) and S (Eq. 4)."""
        if self._mats is None:
            name = f"D3Q{self.Q}"
            polys, groups = methods.mrt_method(name, weighted=self.mrt_weighted)
            dirs = methods.stencil(name)
            Mr = methods.moment_matrix(polys, dirs)
            Minv = methods.mat_inverse(Mr)
            if self.op in ("kbc", "kbc_exact"):  # row parts: 0 conserved, 1 shear (s), 2 higher order (h)
                S = [0.0 if g == "conserved" else 1.0 if g == "shear" else 2.0 for g in groups]
            elif len(self.rates) == 15:  # one rate per non-conserved row, in the basis order
                assert groups[:4] == ["conserved"] * 4
                S = [0.0] * 4 + [float(v) for v in self.rates]
            else:
                r = list(self.rates) + [1.0] * 4
                S = methods.mrt_rates_per_row(groups, r[0], r[1], r[2], r[3])
            self._mats = (np.array([[float(v) for v in row] for row in Mr]),
                          np.array([[float(v) for v in row] for row in Minv]),
                          np.array(S, dtype=np.float64))
        return self._mats


class Domain:
    """Local lattice of nx*ny*nz cells; zghost=1 adds ghost planes z=-1 and z=nz (slab mode)."""

    def __init__(self, method: Method, nx: int, ny: int, nz: int, zghost: int = 0,
                 flags: Optional[np.ndarray] = None, wall_u: Optional[np.ndarray] = None):
        """wall_u: optional per-cell wall velocity (3, nz+2*zghost, ny, nx) used by UBB cells instead
        of method.ubb_u (per-link boundary data)."""
        self.m = method
        self.nx, self.ny, self.nz, self.zghost = nx, ny, nz, zghost
        self.Q = method.Q
        self.shape = (self.Q, nz + 2 * zghost, ny, nx)
        if flags is not None:
            flags = np.ascontiguousarray(flags, dtype=np.uint8)
            assert flags.shape == self.shape[1:], (flags.shape, self.shape)
        self.flags = flags
        cfg = _Cfg()
        cfg.Q = self.Q
        cfg.op = OPS[method.op]
        cfg.nx, cfg.ny, cfg.nz = nx, ny, nz
        cfg.zghost = zghost
        cfg.nthreads = method.nthreads
        r = list(method.rates) + [0.0] * (8 - len(method.rates))
        if method.op == "cumulant":  # unspecified higher-order rates default to 1 (G7)
            r = list(method.rates) + [1.0] * (6 - len(method.rates))
            r = r + [0.0] * (8 - len(r))
        cfg.rates = (C.c_double * 8)(*r[:8])
        cfg.force = (C.c_double * 3)(*method.force)
        cfg.ubb_u = (C.c_double * 3)(*method.ubb_u)
        cfg.ubb_rho = method.ubb_rho
        self._keep = []
        if method.op in ("mrt", "kbc", "kbc_exact"):
            M, Minv, S = method.mrt_matrices()
            self._keep = [np.ascontiguousarray(M), np.ascontiguousarray(Minv), np.ascontiguousarray(S)]
            cfg.M, cfg.Minv, cfg.S = (_p(a) for a in self._keep)
        if wall_u is not None:
            wall_u = np.ascontiguousarray(wall_u, np.float64)
            assert wall_u.shape == (3,) + self.shape[1:], wall_u.shape
            self._wall_u = wall_u
            cfg.wall_u = _p(wall_u)
        cfg.eq_kind = EQ_KINDS[method.equilibrium]
        if method.equilibrium == "moment_matched" or method.op == "cumulant":
            exps, minv = method.monomial_tables()
            self._keep += [np.ascontiguousarray(exps), np.ascontiguousarray(minv)]
            cfg.mono_exp, cfg.Mmono_inv = _p(self._keep[-2]), _p(self._keep[-1])
        self.cfg = cfg

    # -- allocation ------------------------------------------------------------------
    def zeros(self) -> np.ndarray:
        return np.zeros(self.shape, np.float64)

    def _pc(self):
        return C.byref(self.cfg)

    def _fl(self):
        return _p(self.flags) if self.flags is not None else None

    # -- steps --------------------------------------------------------------------------
    def init_equilibrium(self, rho: np.ndarray, u: np.ndarray) -> np.ndarray:
        """f = f_eq(rho, u) (product equilibrium for the cumulant). rho: (nz,ny,nx); u: (3,nz,ny,nx)."""
        rho = np.ascontiguousarray(rho, np.float64)
        u = np.ascontiguousarray(u, np.float64)
        assert rho.shape == (self.nz, self.ny, self.nx) and u.shape == (3,) + rho.shape
        f = self.zeros()
        lib().ora_init_equilibrium(self._pc(), _p(rho), _p(u), _p(f))
        return f

    def step_pull(self, src: np.ndarray, dst: np.ndarray) -> None:
        lib().ora_step_pull(self._pc(), _p(src), _p(dst), self._fl())

    def step_push(self, f: np.ndarray, tmp: Optional[np.ndarray] = None) -> None:
        tmp = self.zeros() if tmp is None else tmp
        lib().ora_step_push(self._pc(), _p(f), _p(tmp), self._fl())

    def stream(self, src: np.ndarray, dst: np.ndarray) -> None:
        lib().ora_stream(self._pc(), _p(src), _p(dst), self._fl())

    def collide_all(self, a: np.ndarray) -> None:
        lib().ora_collide_all(self._pc(), _p(a), self._fl())

    def aa_even(self, a: np.ndarray) -> None:
        assert lib().ora_aa_even(self._pc(), _p(a), self._fl()) == 0

    def aa_odd(self, a: np.ndarray) -> None:
        assert lib().ora_aa_odd(self._pc(), _p(a), self._fl()) == 0

    def eso_step(self, a: np.ndarray, odd: int) -> None:
        """One EsoTwist step on the raw array (ghost planes included in slab mode)."""
        assert (lib().ora_eso_odd if odd else lib().ora_eso_even)(self._pc(), _p(a), self._fl()) == 0

    def run_pull(self, f0: np.ndarray, n: int) -> np.ndarray:
        """P(n) = (C o S)^n P(0) with two arrays (G11). Wall cells keep their initial values."""
        a, b = f0.copy(), f0.copy()
        for _ in range(n):
            self.step_pull(a, b)
            a, b = b, a
        return a

    def run_push(self, f0: np.ndarray, n: int) -> np.ndarray:
        """F(n) = (S o C)^n f0."""
        f, tmp = f0.copy(), self.zeros()
        for _ in range(n):
            self.step_push(f, tmp)
        return f

    def run_aa(self, f0: np.ndarray, n: int) -> np.ndarray:
        """AA pattern: even, odd, even, ... on one array; returns the raw array (slot layout of
        the last parity)."""
        a = f0.copy()
        for t in range(n):
            (self.aa_even if t % 2 == 0 else self.aa_odd)(a)
        return a

    def eso_from_canonical(self, f: np.ndarray, parity: int = 0) -> np.ndarray:
        """EsoTwist storage holding the canonical (pre-collision) state f."""
        assert not self.zghost
        f = np.ascontiguousarray(f, np.float64)
        a = self.zeros()
        assert lib().ora_eso_layout(self._pc(), _p(f), _p(a), parity, 1) == 0
        return a

    def eso_to_canonical(self, a: np.ndarray, parity: int) -> np.ndarray:
        f = self.zeros()
        assert lib().ora_eso_layout(self._pc(), _p(f), _p(np.ascontiguousarray(a)), parity, 0) == 0
        return f

    def run_eso(self, f0: np.ndarray, n: int) -> np.ndarray:
        """EsoTwist even/odd steps on one array starting from the canonical state f0; returns the raw
        array after n steps (slot layout of parity n % 2)."""
        a = self.eso_from_canonical(f0, 0)
        for t in range(n):
            assert (lib().ora_eso_even if t % 2 == 0 else lib().ora_eso_odd)(self._pc(), _p(a), self._fl()) == 0
        return a

    # -- readout ---------------------------------------------------------------------
    def macroscopic(self, f: np.ndarray, post_collision: bool = False):
        rho = np.zeros((self.nz, self.ny, self.nx))
        u = np.zeros((3, self.nz, self.ny, self.nx))
        lib().ora_macroscopic(self._pc(), _p(f), -1.0 if post_collision else 1.0, _p(rho), _p(u))
        return rho, u

    def pull_cell(self, src: np.ndarray, x: int, y: int, z: int) -> np.ndarray:
        out = np.zeros(self.Q)
        lib().ora_pull_cell(self._pc(), _p(src), self._fl(), x, y, z, _p(out))
        return out

    def pack_face(self, f: np.ndarray, z: int, direction: int) -> np.ndarray:
        nq = 5 if self.Q == 19 else 9
        out = np.zeros(nq * self.ny * self.nx)
        n = lib().ora_pack_face(self._pc(), _p(f), z, direction, _p(out))
        assert n == out.size
        return out

    def unpack_face(self, f: np.ndarray, z: int, direction: int, buf: np.ndarray) -> None:
        buf = np.ascontiguousarray(buf, np.float64)
        lib().ora_unpack_face(self._pc(), _p(f), z, direction, _p(buf))


def collide_cell(method: Method, f: np.ndarray) -> np.ndarray:
    d = Domain(method, 1, 1, 1)
    f = np.ascontiguousarray(f, np.float64)
    out = np.zeros(method.Q)
    lib().ora_collide_cell(d._pc(), _p(f), _p(out))
    return out


def equilibrium_cell(Q: int, rho: float, u) -> np.ndarray:
    u = np.ascontiguousarray(u, np.float64)
    out = np.zeros(Q)
    lib().ora_equilibrium_cell(Q, rho, _p(u), _p(out))
    return out


def equilibrium_kind_cell(method: Method, rho: float, u) -> np.ndarray:
    """Equilibrium of `method.equilibrium`'s kind at (rho, u)."""
    d = Domain(method, 1, 1, 1)
    u = np.ascontiguousarray(u, np.float64)
    out = np.zeros(method.Q)
    lib().ora_equilibrium_kind_cell(d._pc(), rho, _p(u), _p(out))
    return out


def maxwellian_equilibrium_cell(Q: int, rho: float, u) -> np.ndarray:
    """Populations with the untruncated Maxwellian basis moments (the cumulant fixed point; D3Q27:
    the product equilibrium)."""
    d = Domain(Method(Q=Q, op="cumulant", rates=(1.0,)), 1, 1, 1)
    u = np.ascontiguousarray(u, np.float64)
    out = np.zeros(Q)
    lib().ora_maxwellian_equilibrium_cell(d._pc(), rho, _p(u), _p(out))
    return out


def from_cumulants_any(Q: int, rho: float, kappa: np.ndarray) -> np.ndarray:
    """Inverse cumulant transform on D3Q19 or D3Q27 (basis-moment route)."""
    d = Domain(Method(Q=Q, op="cumulant", rates=(1.0,)), 1, 1, 1)
    k = np.ascontiguousarray(kappa, np.float64).reshape(27)
    out = np.zeros(Q)
    lib().ora_from_cumulants_cfg_cell(d._pc(), rho, _p(k), _p(out))
    return out


def cumulants_any(Q: int, f: np.ndarray):
    f = np.ascontiguousarray(f, np.float64)
    k = np.zeros(27)
    rho = lib().ora_cumulants_cell(Q, _p(f), _p(k))
    return rho, k.reshape(3, 3, 3)


def product_equilibrium_cell(Q: int, rho: float, u) -> np.ndarray:
    u = np.ascontiguousarray(u, np.float64)
    out = np.zeros(Q)
    lib().ora_product_equilibrium_cell(Q, rho, _p(u), _p(out))
    return out


def cumulants_cell(f: np.ndarray):
    """(rho, kappa[3,3,3]) of a D3Q27 population vector (Eq. 9, O5)."""
    f = np.ascontiguousarray(f, np.float64)
    k = np.zeros(27)
    rho = lib().ora_cumulants_cell(27, _p(f), _p(k))
    return rho, k.reshape(3, 3, 3)


def from_cumulants_cell(rho: float, kappa: np.ndarray) -> np.ndarray:
    k = np.ascontiguousarray(kappa, np.float64).reshape(27)
    out = np.zeros(27)
    lib().ora_from_cumulants_cell(27, rho, _p(k), _p(out))
    return out


def smagorinsky_omega_cell(method: Method, f: np.ndarray) -> float:
    d = Domain(method, 1, 1, 1)
    f = np.ascontiguousarray(f, np.float64)
    return lib().ora_smagorinsky_omega_cell(d._pc(), _p(f))
