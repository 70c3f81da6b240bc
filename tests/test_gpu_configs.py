"""GPU parity of the BASELINE configs at their OWN step counts (north_star: "GPU results must match the
oracle ... after the config's step count"; C1 "checked against the Poiseuille profile").

Where a config's flow is translation-invariant the full-size GPU run is compared element by element with
an oracle run on the invariant cross-section (C1: the channel flow from rest under a uniform force is
x/z-invariant, so every fluid cell of the 256^3 lattice is compared with one 1x256x1 oracle column; C2
without its noise is x/y-invariant: every cell of the 512^3 lattice against one 1x1x512 column). Where it
is not (C2 with noise, C3, C4), a reduced lattice runs the config's full step count against the full oracle
run, and the full-size GPU run is checked on properties that hold at any size (viscosity of the decaying
wave, mirror symmetry, conservation).

Bars: max relative population error <= 1e-12 (fp64) / 2e-5 (fp32) (north_star); the Poiseuille start-up
series at t = n - 1/2 to 2.5e-4 of the maximum; the shear-wave viscosity to 1e-3
(SURVEY §8(c) "Viscosity" gate). Comparisons of the large fields run in torch on the device.
"""
import functools

import numpy as np
import pytest

import lbminputs as LI
import oracle as O
from tests import closed_forms as CF
from tests.gpu_common import FULL, TOL, Case, fluid_mask, init_sim, make_sim, max_rel_err, oracle_run

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _lib():
    from paper_2001_11806_b200 import build
    build.build()
    import torch
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"


def _torch():
    import torch
    return torch


def _device_populations(sim):
    torch = _torch()
    out = torch.empty((sim.Q, sim.nz_local, sim.ny, sim.nx), dtype=torch.float64, device="cuda")
    sim.populations(out=out)
    return out


def _device_macroscopic(sim):
    torch = _torch()
    rho = torch.empty((sim.nz_local, sim.ny, sim.nx), dtype=torch.float64, device="cuda")
    u = torch.empty((3, sim.nz_local, sim.ny, sim.nx), dtype=torch.float64, device="cuda")
    sim.macroscopic(rho, u)
    return rho, u


def _max_rel(got, ref) -> float:
    """max |got - ref| / |ref| over broadcast torch tensors (ref broadcasts along invariant axes)."""
    return float(((got - ref).abs() / ref.abs()).max())


# -----------------------------------------------------------------------------------------
# C1: D3Q19 TRT + Guo, 256^3 channel, 2000 steps, fp64 and fp32 — every fluid cell vs the oracle column
# -----------------------------------------------------------------------------------------
@functools.lru_cache(maxsize=None)
def _c1_column(steps: int):
    """Oracle pull state P(steps) on the 1 x 256 x 1 cross-section of config 1 (x/z-invariant flow)."""
    base = FULL["c1_f64"]
    ny = base.shape[1]
    d = O.Domain(base.method(), 1, ny, 1, flags=LI.channel_flags(1, ny, 1))
    f0 = d.init_equilibrium(np.ones((1, ny, 1)), np.zeros((3, 1, ny, 1)))
    return d.run_pull(f0, steps)


@pytest.mark.parametrize("boundary_mode", ["flags", "links"])
@pytest.mark.parametrize("dtype", ["f64", "f32"])
def test_c1_full_size_2000_steps_vs_oracle_column_and_poiseuille(dtype, boundary_mode):
    torch = _torch()
    case = FULL[f"c1_{dtype}"]
    nx, ny, nz = case.shape
    sim = make_sim(case, boundary_mode=boundary_mode)
    sim.init_random(0, 0.0, 0.0)  # rho = 1, u = 0 exactly (U(-0, 0) = 0): the config's rest start
    sim.step(case.steps)
    got = _device_populations(sim)[:, :, 1:ny - 1, :]  # fluid rows y = 1..254
    ref = torch.from_numpy(_c1_column(case.steps)).cuda()[:, :, 1:ny - 1, :]  # (19, 1, 254, 1)
    err = _max_rel(got, ref)
    assert err <= TOL[dtype], err
    # the flow is x/z-invariant and every cell of a row runs the same arithmetic on the same values
    spread = float((got.amax(dim=(1, 3)) - got.amin(dim=(1, 3))).abs().max())
    assert spread == 0.0, spread
    del got
    # Poiseuille start-up series at t = n - 1/2 (pull state P(n) from P(0) = f_eq; G11)
    _, u = _device_macroscopic(sim)
    ux = u[0].mean(dim=(0, 2)).cpu().numpy()[1:ny - 1]
    H = ny - 2
    nu = CF.lattice_viscosity(case.rates[0])
    series = CF.poiseuille_startup(np.arange(1, H + 1), H, case.force[0], nu, case.steps - 0.5)
    assert np.abs(ux - series).max() / series.max() < 2.5e-4
    wrong = CF.poiseuille_startup(np.arange(1, H + 1), H, case.force[0], nu, case.steps + 0.5)
    assert np.abs(ux - wrong).max() / wrong.max() > 2.5e-4  # a half-step bookkeeping error would be caught
    sim.close()


# -----------------------------------------------------------------------------------------
# C2: D3Q19 weighted MRT fp32 AA, 512^3 shear wave, 500 steps
# -----------------------------------------------------------------------------------------
def test_c2_full_size_500_steps_noise_free_vs_oracle_column():
    """The config without its 1e-4 noise is x/y-invariant: every cell of the 512^3 AA lattice after 500 steps
    (even: canonical slots) against one 1 x 1 x 512 oracle column run in the push semantics (G11)."""
    torch = _torch()
    base = FULL["c2"]
    nx, ny, nz = base.shape
    sim = make_sim(base)
    sim.init_random(0, 0.0, 0.0, LI.PROFILE_SHEAR_WAVE, 0.01)
    sim.step(base.steps)
    d = O.Domain(base.method(), 1, 1, nz)
    rho, u = LI.random_fields(0, 1, 1, nz, 0.0, 0.0, LI.PROFILE_SHEAR_WAVE, 0.01)
    ref = torch.from_numpy(d.run_push(d.init_equilibrium(rho, u), base.steps)).cuda()  # (19, 512, 1, 1)
    got = _device_populations(sim)
    err = _max_rel(got, ref)
    assert err <= TOL[base.dtype], err
    sim.close()


@pytest.mark.parametrize("dtype,gate", [("f64", 1e-3), ("f32", 5e-2)])
def test_c2_full_size_viscosity_fit(dtype, gate):
    """The config's 512^3 wave with its noise: the x/y-averaged u_x projected on sin(2 pi z/512) decays with
    the lattice viscosity of omega_shear = 1.9 (nu = (1/1.9 - 1/2)/3), fitted between steps 100 and 500
    (after the initial non-equilibrium layer).

    fp64 (the config's geometry, noise and steps in double precision): gate 1e-3 (measured 1.2e-5, the same
    as the oracle column). fp32 (the config itself): the relative decay per step, nu k^2 = 1.3e-6, is only
    ~22 fp32 ulps (eps = 6e-8), so the deterministic per-step rounding of the stored populations biases the
    fitted rate by a few percent whatever the kernel does (a plain numpy fp32 column with the same
    zero-centred formulation gives -1.6 %; G26); gate 5e-2. The fp32 state itself matches the oracle
    to 2e-5 (test_c2_full_size_500_steps_noise_free_vs_oracle_column)."""
    base = FULL["c2"]
    case = Case(base.name, base.shape, base.Q, base.op, base.rates, dtype, base.pattern, init=base.init,
                rho_amp=base.rho_amp, u_amp=base.u_amp, steps=base.steps)
    sim = make_sim(case)
    init_sim(sim, case)
    amps = {}
    for t0, t1 in ((0, 100), (100, 500)):
        sim.step(t1 - t0)
        _, u = _device_macroscopic(sim)
        amps[t1] = CF.shear_wave_amplitude(u[0].mean(dim=(1, 2)).cpu().numpy())
        del u
    nu_fit = CF.fitted_viscosity(amps[100], amps[500], 100, 500, base.shape[2])
    nu = CF.lattice_viscosity(base.rates[0])
    assert abs(nu_fit / nu - 1) <= gate, (nu_fit, nu)
    sim.close()


def test_c2_noisy_proxy_500_steps_vs_oracle():
    """Config 2 with its noise, full wavelength (nz = 512) and full step count on a 32 x 32 x 512 lattice."""
    case = Case("c2_proxy_512", (32, 32, 512), 19, "mrt", (1.9, 1.0, 1.0, 1.0), "f32", pattern="aa", init="shear",
                rho_amp=0.0, u_amp=1e-4, steps=500)
    sim = make_sim(case)
    init_sim(sim, case)
    sim.step(case.steps)
    err = max_rel_err(sim.populations(), oracle_run(case))
    assert err <= TOL["f32"], err


# -----------------------------------------------------------------------------------------
# C3: D3Q27 cumulant fp64 lid-driven cavity, 1000 steps
# -----------------------------------------------------------------------------------------
C3_PROXY = Case("c3_proxy_48", (48, 48, 48), 27, "cumulant", (1.95,), "f64", geometry="cavity", ubb=(0.05, 0, 0),
                init="rest", steps=1000)


@functools.lru_cache(maxsize=None)
def _c3_oracle():
    return oracle_run(C3_PROXY)


@pytest.mark.parametrize("boundary_mode", ["flags", "links"])
def test_c3_cavity_48_1000_steps_vs_oracle(boundary_mode):
    sim = make_sim(C3_PROXY, boundary_mode=boundary_mode)
    init_sim(sim, C3_PROXY)
    sim.step(C3_PROXY.steps)
    err = max_rel_err(sim.populations(), _c3_oracle(), fluid_mask(C3_PROXY, 27))
    assert err <= TOL["f64"], err


def test_c3_full_size_1000_steps_mirror_symmetry_and_mass():
    """384^3 cavity, 1000 steps: the lid moves along x, so the solution is mirror-symmetric under
    y -> 383 - y (rho, u_x, u_z even, u_y odd); the fluid mass is conserved (bounce-back and a tangential
    UBB lid add no mass: the UBB terms 6 w_q c_q.u_w of the +-c_x links cancel)."""
    torch = _torch()
    base = FULL["c3"]
    n = base.shape[0]
    sim = make_sim(base, boundary_mode="links")
    sim.init_random(0, 0.0, 0.0)
    fl = torch.from_numpy(base.flags() == 0).cuda()
    rho0, _ = _device_macroscopic(sim)
    mass0 = float(rho0[fl].sum())
    del rho0
    sim.step(base.steps)
    rho, u = _device_macroscopic(sim)
    inner = (slice(1, n - 1), slice(1, n - 1), slice(1, n - 1))  # (z, y, x) fluid box
    r = rho[inner]
    assert float((r - r.flip(1)).abs().max()) <= 1e-13
    for d, sign in ((0, 1.0), (1, -1.0), (2, 1.0)):
        ud = u[d][inner]
        assert float((ud - sign * ud.flip(1)).abs().max()) <= 1e-13, d
    assert float(u[0][inner].abs().max()) > 1e-3  # the lid did drive a flow
    mass = float(rho[fl].sum())
    assert abs(mass / mass0 - 1) <= 1e-12, mass / mass0 - 1
    sim.close()


# -----------------------------------------------------------------------------------------
# C4: D3Q19 TRT fp64 pull, 512^3 per GPU, 200 steps
# -----------------------------------------------------------------------------------------
def test_c4_64_cubed_200_steps_vs_oracle():
    case = Case("c4_proxy_64", (64, 64, 64), 19, "trt", (1.6, 0.5), "f64", steps=200)
    sim = make_sim(case)
    init_sim(sim, case)
    sim.step(case.steps)
    err = max_rel_err(sim.populations(), oracle_run(case))
    assert err <= TOL["f64"], err


def test_c4_full_size_200_steps_conservation():
    """512^3 periodic, F = 0, 200 steps: total mass and momentum are invariants of every step
    (collision conserves rho and j per cell, streaming permutes populations)."""
    torch = _torch()
    base = FULL["c4"]
    sim = make_sim(base)
    init_sim(sim, base)

    def totals():
        rho, u = _device_macroscopic(sim)
        out = [float(rho.sum())] + [float((rho * u[d]).sum()) for d in range(3)]
        del rho, u
        return np.array(out)

    t0 = totals()
    sim.step(base.steps)
    t1 = totals()
    assert abs(t1[0] / t0[0] - 1) <= 1e-13, t1[0] / t0[0] - 1
    assert np.abs(t1[1:] - t0[1:]).max() <= 1e-14 * t0[0], (t1[1:] - t0[1:])
    sim.close()
