"""Shared helpers of the GPU parity tests: the BASELINE configs, building a CUDA-path simulation
and the matching oracle domain from the same seeded inputs, and error metrics."""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import Optional, Tuple

import numpy as np

import lbminputs as LI
import oracle as O

TOL = {"f64": 1e-12, "f32": 2e-5}  # north_star: max relative population error vs the oracle


@dataclass
class Case:
    name: str
    shape: Tuple[int, int, int]
    Q: int = 19
    op: str = "srt"
    rates: tuple = (1.8,)
    dtype: str = "f64"
    pattern: str = "pull"
    force: tuple = (0.0, 0.0, 0.0)
    geometry: str = "periodic"  # periodic | channel | cavity | obstacles
    ubb: tuple = (0.0, 0.0, 0.0)
    init: str = "random"        # random | rest | shear
    rho_amp: float = 1e-3
    u_amp: float = 0.01
    steps: int = 10
    seed: int = 0
    equilibrium: str = "compressible"  # | incompressible | moment_matched (SRT/TRT/MRT)
    extra: dict = field(default_factory=dict)

    def flags(self) -> Optional[np.ndarray]:
        nx, ny, nz = self.shape
        if self.geometry == "channel":
            return LI.channel_flags(nx, ny, nz)
        if self.geometry == "cavity":
            assert nx == ny == nz
            return LI.cavity_flags(nx)
        if self.geometry == "obstacles":
            return LI.random_obstacles(self.seed, nx, ny, nz)
        return None

    def periodic(self):
        return {"channel": (1, 0, 1), "cavity": (0, 0, 0)}.get(self.geometry, (1, 1, 1))

    def fields(self, z0=0, nz=None):
        nx, ny, nzg = self.shape
        if self.init == "rest":
            n = nzg if nz is None else nz
            return np.ones((n, ny, nx)), np.zeros((3, n, ny, nx))
        prof = LI.PROFILE_SHEAR_WAVE if self.init == "shear" else LI.PROFILE_NONE
        return LI.random_fields(self.seed, nx, ny, nzg, self.rho_amp, self.u_amp, prof, 0.01, z0=z0, nz=nz)

    def profile(self):
        return (LI.PROFILE_SHEAR_WAVE, 0.01) if self.init == "shear" else (LI.PROFILE_NONE, 0.0)

    def method(self, nthreads=0) -> O.Method:
        # the generated operators (codegen/) compute the same operator as their hand-written kin
        return O.Method(Q=self.Q, op=self.op.removeprefix("gen_"), rates=self.rates, force=self.force, ubb_u=self.ubb, nthreads=nthreads,
                        equilibrium=self.equilibrium)


def make_sim(case: Case, **kw):
    from paper_2001_11806_b200 import lbm as L
    args = dict(shape=case.shape, stencil=case.Q, collision=case.op, rates=case.rates, dtype=case.dtype,
                pattern=case.pattern, force=case.force, flags=case.flags(), ubb_velocity=case.ubb,
                periodic=case.periodic(), equilibrium=case.equilibrium)
    args.update(case.extra)
    args.update(kw)
    return L.Simulation(**args)


def init_sim(sim, case: Case, use_random_kernel: bool = True):
    """Random-init cases use the GPU's own generator (lbm_init_random); others upload arrays."""
    if case.init in ("random", "shear") and use_random_kernel:
        prof, amp = case.profile()
        sim.init_random(case.seed, case.rho_amp, case.u_amp, prof, amp)
    else:
        rho, u = case.fields()
        sim.init_equilibrium(rho, u)


def oracle_run(case: Case, steps: Optional[int] = None) -> np.ndarray:
    """Canonical populations of the oracle after `steps` with the case's pattern semantics."""
    nx, ny, nz = case.shape
    d = O.Domain(case.method(), nx, ny, nz, flags=case.flags())
    rho, u = case.fields()
    f0 = d.init_equilibrium(rho, u)
    n = case.steps if steps is None else steps
    if case.pattern in ("aa", "esotwist", "push"):  # all hold the push state F(n) (G11)
        return d.run_push(f0, n)
    return d.run_pull(f0, n)


def fluid_mask(case: Case, Q: int) -> np.ndarray:
    fl = case.flags()
    nx, ny, nz = case.shape
    m = np.ones((nz, ny, nx), bool) if fl is None else fl == 0
    return np.broadcast_to(m, (Q, nz, ny, nx))


def max_rel_err(got: np.ndarray, ref: np.ndarray, mask: Optional[np.ndarray] = None) -> float:
    if mask is not None:
        got, ref = got[mask], ref[mask]
    return float(np.max(np.abs(got - ref) / np.abs(ref)))


# ------------------------------------------------------------------------------------------
# BASELINE.json configs (full size) and the reduced-size proxies used for full-step parity.
# ------------------------------------------------------------------------------------------
FULL = {
    "c0": Case("c0", (32, 32, 32), 19, "srt", (1.8,), "f64", steps=100),
    "c1_f64": Case("c1_f64", (256, 256, 256), 19, "trt", (1.6, 0.5), "f64", force=(1e-6, 0, 0),
                   geometry="channel", init="rest", steps=2000),
    "c1_f32": Case("c1_f32", (256, 256, 256), 19, "trt", (1.6, 0.5), "f32", force=(1e-6, 0, 0),
                   geometry="channel", init="rest", steps=2000),
    "c2": Case("c2", (512, 512, 512), 19, "mrt", (1.9, 1.0, 1.0, 1.0), "f32", pattern="aa",
               init="shear", rho_amp=0.0, u_amp=1e-4, steps=500),
    "c3": Case("c3", (384, 384, 384), 27, "cumulant", (1.95,), "f64", geometry="cavity",
               ubb=(0.05, 0, 0), init="rest", steps=1000),
    "c4": Case("c4", (512, 512, 512), 19, "trt", (1.6, 0.5), "f64", steps=200),
    "c4_strong": Case("c4_strong", (1024, 1024, 1024), 19, "trt", (1.6, 0.5), "f32", steps=200),
}
