"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle on the same seeded inputs.

Bars (north_star): max relative population error <= 1e-12 (fp64) / <= 2e-5 (fp32) after the
case's step count; data movement (streaming, flag-driven boundaries, AA slots, halo planes,
slab decomposition) bit-exact.
"""
import numpy as np
import pytest

import lbminputs as LI
import oracle as O
from tests.gpu_common import FULL, TOL, Case, fluid_mask, init_sim, make_sim, max_rel_err, oracle_run

pytestmark = pytest.mark.gpu

ROW_RATES = (1.9, 1.7, 1.5, 1.3, 1.1, 1.05, 0.9, 1.2, 1.4, 0.8, 1.6, 1.0, 1.25, 0.7, 1.35)  # per-moment MRT


@pytest.fixture(scope="module", autouse=True)
def _lib():
    from paper_2001_11806_b200 import build
    build.build()
    import torch
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"


def _markers(Q, shape, seed=1):
    """Distinct dyadic marker values, exact in fp32 and fp64."""
    rng = np.random.default_rng(seed)
    nx, ny, nz = shape
    return rng.integers(1, 2 ** 20, size=(Q, nz, ny, nx)).astype(np.float64) / 2 ** 12


# -----------------------------------------------------------------------------------------
# Data movement, bit-exact
# -----------------------------------------------------------------------------------------
@pytest.mark.parametrize("Q", [19, 27])
@pytest.mark.parametrize("dtype", ["f64", "f32"])
@pytest.mark.parametrize("geometry", ["periodic", "obstacles"])
def test_pull_streaming_and_bounce_back_bit_exact(Q, dtype, geometry):
    case = Case("mark", (13, 11, 7), Q, "identity", (), dtype, geometry=geometry)
    sim = make_sim(case)
    m = _markers(Q, case.shape)
    sim.set_populations(m, raw=True)
    d = O.Domain(O.Method(Q=Q, op="identity", rates=()), *case.shape, flags=case.flags())
    ref = d.run_pull(m, 3)
    sim.step(3)
    got = sim.populations(raw=True)
    mask = fluid_mask(case, Q)
    np.testing.assert_array_equal(got[mask], ref[mask])


@pytest.mark.parametrize("Q", [19, 27])
@pytest.mark.parametrize("geometry", ["periodic", "obstacles"])
def test_aa_slots_bit_exact(Q, geometry):
    case = Case("mark", (9, 7, 6), Q, "identity", (), "f64", pattern="aa", geometry=geometry)
    sim = make_sim(case)
    m = _markers(Q, case.shape, 2)
    sim.set_populations(m, raw=True)
    d = O.Domain(O.Method(Q=Q, op="identity", rates=()), *case.shape, flags=case.flags())
    mask = fluid_mask(case, Q)
    for n in (1, 2, 3):
        sim.step(1)
        np.testing.assert_array_equal(sim.populations(raw=True)[mask], d.run_aa(m, n)[mask])     # slot layout
        np.testing.assert_array_equal(sim.populations(raw=False)[mask],                          # canonical gather
                                      _centre_free(d.run_push(m, n), Q, True)[mask])


@pytest.mark.parametrize("Q", [19, 27])
@pytest.mark.parametrize("geometry", ["periodic", "obstacles"])
def test_esotwist_slots_bit_exact(Q, geometry):
    """EsoTwist storage (identity collision, dyadic markers): raw array == oracle's EsoTwist array after
    every step, and the canonical gather == the push pattern; both parities."""
    case = Case("emark", (9, 7, 6), Q, "identity", (), "f64", pattern="esotwist", geometry=geometry)
    sim = make_sim(case)
    m = _markers(Q, case.shape, 3)
    d = O.Domain(O.Method(Q=Q, op="identity", rates=()), *case.shape, flags=case.flags())
    sim.set_populations(d.eso_from_canonical(m, 0), raw=True)  # storage layout written directly
    _, w, _ = O.stencil_arrays(Q)
    mask = fluid_mask(case, Q)
    for n in (1, 2, 3):
        sim.step(1)
        raw_ref = d.run_eso(m, n)  # identity: the stored values are the markers (no w offset)
        np.testing.assert_array_equal(sim.populations(raw=True)[mask], raw_ref[mask])
        np.testing.assert_array_equal(sim.populations(raw=False)[mask], (d.run_push(m, n) + w[:, None, None, None])[mask])


def _centre_free(f_raw_stream, Q, add_w):
    # identity collision: canonical value = raw marker + w_q (the library adds w back)
    _, w, _ = O.stencil_arrays(Q)
    return f_raw_stream + (w[:, None, None, None] if add_w else 0.0)


@pytest.mark.parametrize("Q", [19, 27])
def test_pack_face_layout_bit_exact(Q):
    case = Case("pack", (10, 7, 6), Q, "trt", (1.6, 0.5), "f64")
    sim = make_sim(case)
    init_sim(sim, case)
    sim.step(2)
    raw = sim.populations(raw=True)
    d = O.Domain(O.Method(Q=Q, op="identity", rates=()), *case.shape)
    for z in (0, 3, 5):
        for direction in (1, -1):
            np.testing.assert_array_equal(sim.pack_face(z, direction), d.pack_face(raw, z, direction))


# -----------------------------------------------------------------------------------------
# Initialisation and readout
# -----------------------------------------------------------------------------------------
@pytest.mark.parametrize("Q,op,rates", [(19, "srt", (1.8,)), (27, "cumulant", (1.95,)), (19, "cumulant", (1.95,))])
def test_init_random_matches_seeded_inputs(Q, op, rates):
    case = Case("init", (16, 12, 10), Q, op, rates, "f64", init="shear")
    sim = make_sim(case)
    init_sim(sim, case, use_random_kernel=True)
    d = O.Domain(case.method(), *case.shape)
    rho, u = case.fields()
    ref = d.init_equilibrium(rho, u)
    assert max_rel_err(sim.populations(), ref) < 1e-14


@pytest.mark.parametrize("equilibrium", ["compressible", "incompressible"])
def test_macroscopic_readout_equilibrium_kinds(equilibrium):
    """u = (j -+ F/2) / rho0 with rho0 = rho (compressible) or 1 (incompressible)."""
    case = Case("mro", (12, 16, 8), 19, "trt", (1.6, 0.5), "f64", force=(1e-5, 0, 0), geometry="channel",
                steps=9, equilibrium=equilibrium)
    sim = make_sim(case)
    init_sim(sim, case)
    sim.step(case.steps)
    d = O.Domain(case.method(), *case.shape, flags=case.flags())
    rho_o, u_o = d.macroscopic(oracle_run(case), post_collision=True)
    rho, u = sim.macroscopic()
    fl = case.flags() == 0
    np.testing.assert_allclose(rho[fl], rho_o[fl], rtol=1e-13)
    np.testing.assert_allclose(u[:, fl], u_o[:, fl], rtol=0, atol=1e-15)


def test_macroscopic_readout():
    case = FULL["c1_f64"]
    case = Case("c1s", (12, 16, 8), **{k: getattr(case, k) for k in ("Q", "op", "rates", "dtype", "force", "geometry")},
                init="random", steps=30)
    sim = make_sim(case)
    init_sim(sim, case)
    sim.step(case.steps)
    d = O.Domain(case.method(), *case.shape, flags=case.flags())
    ref = oracle_run(case)
    rho_o, u_o = d.macroscopic(ref, post_collision=True)
    rho, u = sim.macroscopic()
    fl = case.flags() == 0
    np.testing.assert_allclose(rho[fl], rho_o[fl], rtol=1e-13)
    np.testing.assert_allclose(u[:, fl], u_o[:, fl], rtol=0, atol=1e-15)


# -----------------------------------------------------------------------------------------
# Numerical parity per operator / config (reduced sizes, many steps, ragged extents)
# -----------------------------------------------------------------------------------------
PARITY = [
    Case("c0_full", (32, 32, 32), 19, "srt", (1.8,), "f64", steps=100),
    Case("c1_proxy_f64", (16, 32, 8), 19, "trt", (1.6, 0.5), "f64", force=(1e-6, 0, 0), geometry="channel",
         init="rest", steps=300),
    Case("c1_proxy_f32", (16, 32, 8), 19, "trt", (1.6, 0.5), "f32", force=(1e-6, 0, 0), geometry="channel",
         init="rest", steps=300),
    Case("c1_proxy_f32_random", (16, 32, 8), 19, "trt", (1.6, 0.5), "f32", force=(1e-6, 0, 0), geometry="channel",
         steps=100),
    Case("c2_proxy", (32, 32, 32), 19, "mrt", (1.9, 1.0, 1.0, 1.0), "f32", pattern="aa", init="shear", rho_amp=0.0,
         u_amp=1e-4, steps=100),
    Case("c2_proxy_f64", (24, 20, 32), 19, "mrt", (1.9, 1.0, 1.0, 1.0), "f64", pattern="aa", init="shear",
         rho_amp=0.0, u_amp=1e-4, steps=40),
    # two-cells-per-thread AA kernels of C2 (k_aa_*_x2): a ragged row end (nx = 100: cell B exists for x < 100
    # only) and a row of exactly 64 (cell B of lane 31 is x = nx - 1, whose +x neighbour wraps to 0)
    Case("c2_x2_ragged", (100, 12, 10), 19, "mrt", (1.9, 1.0, 1.0, 1.0), "f32", pattern="aa", u_amp=0.03, steps=13),
    Case("c2_x2_row64", (64, 6, 8), 19, "mrt", (1.9, 1.0, 1.0, 1.0), "f32", pattern="aa", u_amp=0.03, steps=12),
    Case("c3_proxy", (20, 20, 20), 27, "cumulant", (1.95,), "f64", geometry="cavity", ubb=(0.05, 0, 0),
         init="rest", steps=100),
    Case("c3_proxy_random", (16, 16, 16), 27, "cumulant", (1.95,), "f64", geometry="cavity", ubb=(0.05, 0, 0),
         steps=30),
    Case("c4_proxy", (24, 24, 24), 19, "trt", (1.6, 0.5), "f64", steps=50),
    Case("ragged_q27_trt_f32", (37, 23, 19), 27, "trt", (1.3, 0.9), "f32", force=(2e-5, -1e-5, 3e-5),
         geometry="obstacles", ubb=(0.02, -0.01, 0.03), steps=20),
    Case("ragged_q19_srt_f64_obst", (37, 23, 19), 19, "srt", (1.1,), "f64", geometry="obstacles",
         ubb=(0.02, -0.01, 0.03), steps=20),
    Case("mrt_general_rates_walls", (20, 18, 12), 19, "mrt", (1.9, 1.3, 1.1, 0.8), "f64", geometry="channel", steps=25),
    Case("mrt_general_f32_pull", (20, 18, 12), 19, "mrt", (1.7, 1.2, 0.9, 1.4), "f32", steps=25),
    Case("cumulant_general_rates", (14, 12, 10), 27, "cumulant", (1.8, 1.3, 1.2, 0.9, 1.1, 0.7), "f64", steps=20),
    Case("cumulant_f32", (14, 12, 10), 27, "cumulant", (1.95,), "f32", steps=20),
    Case("aa_trt_force_odd", (18, 14, 10), 19, "trt", (1.6, 0.5), "f64", pattern="aa", force=(1e-5, 2e-5, 0), steps=21),
    Case("aa_q27_trt_f32", (18, 14, 10), 27, "trt", (1.5, 1.2), "f32", pattern="aa", steps=12),
    Case("aa_cumulant_f64", (12, 12, 12), 27, "cumulant", (1.95,), "f64", pattern="aa", steps=10),
    Case("aa_trt_obstacles_odd", (17, 13, 11), 19, "trt", (1.6, 0.5), "f64", pattern="aa", force=(1e-5, 0, 0),
         geometry="obstacles", ubb=(0.02, -0.01, 0.03), steps=15),
    Case("aa_trt_obstacles_f32", (17, 13, 11), 27, "trt", (1.4, 1.1), "f32", pattern="aa", geometry="obstacles",
         ubb=(0.02, -0.01, 0.03), steps=16),
    Case("aa_cumulant_cavity", (14, 14, 14), 27, "cumulant", (1.95,), "f64", pattern="aa", geometry="cavity",
         ubb=(0.05, 0, 0), steps=20),
    Case("aa_mrt_f32_channel", (16, 20, 12), 19, "mrt", (1.9, 1.0, 1.0, 1.0), "f32", pattern="aa",
         geometry="channel", steps=24),
    Case("tiny_1x1x4", (1, 1, 4), 19, "srt", (1.5,), "f64", steps=7),
    Case("smagorinsky_q19_f64_channel", (16, 20, 10), 19, "smagorinsky", (1.95, 0.17), "f64", geometry="channel",
         u_amp=0.05, steps=30),
    Case("smagorinsky_q27_f32_obst", (17, 13, 11), 27, "smagorinsky", (1.9, 0.12), "f32", geometry="obstacles",
         ubb=(0.02, -0.01, 0.03), u_amp=0.05, steps=20),
    Case("smagorinsky_aa_q19_f64", (18, 14, 10), 19, "smagorinsky", (1.95, 0.2), "f64", pattern="aa", u_amp=0.05,
         steps=13),
    Case("kbc_q19_f64_cavity", (14, 14, 14), 19, "kbc", (1.99,), "f64", geometry="cavity", ubb=(0.05, 0, 0),
         steps=30),
    Case("kbc_q19_f32", (16, 12, 10), 19, "kbc", (1.9,), "f32", u_amp=0.05, steps=20),
    Case("kbc_aa_q19_f64_obst", (17, 13, 11), 19, "kbc", (1.95,), "f64", pattern="aa", geometry="obstacles",
         ubb=(0.02, -0.01, 0.03), u_amp=0.05, steps=15),
    # equilibrium variants: incompressible Eq. (3), moment-matched
    Case("inc_trt_force_channel_f64", (16, 20, 8), 19, "trt", (1.6, 0.5), "f64", force=(1e-5, 0, 0), geometry="channel",
         steps=40, equilibrium="incompressible"),
    Case("inc_trt_q27_f32_aa", (18, 14, 10), 27, "trt", (1.5, 1.2), "f32", pattern="aa", steps=12,
         equilibrium="incompressible"),
    Case("inc_mrt_f64_obst", (17, 13, 11), 19, "mrt", (1.9, 1.3, 1.1, 0.8), "f64", geometry="obstacles",
         ubb=(0.02, -0.01, 0.03), steps=20, equilibrium="incompressible"),
    Case("inc_srt_f32_aa_mrt_rates", (32, 16, 8), 19, "mrt", (1.9, 1.0, 1.0, 1.0), "f32", pattern="aa", init="shear",
         rho_amp=0.0, u_amp=1e-4, steps=16, equilibrium="incompressible"),
    Case("mm_trt_q19_f64_walls", (17, 13, 11), 19, "trt", (1.6, 0.5), "f64", force=(1e-5, 2e-5, 0), geometry="obstacles",
         ubb=(0.02, -0.01, 0.03), u_amp=0.05, steps=20, equilibrium="moment_matched"),
    Case("mm_srt_q19_f32_aa", (18, 14, 10), 19, "srt", (1.7,), "f32", pattern="aa", u_amp=0.05, steps=13,
         equilibrium="moment_matched"),
    Case("mm_mrt_q19_f64_aa_channel", (16, 20, 12), 19, "mrt", (1.9, 1.3, 1.1, 0.8), "f64", pattern="aa",
         geometry="channel", u_amp=0.05, steps=14, equilibrium="moment_matched"),
    Case("mm_trt_q27_is_eq3", (14, 12, 10), 27, "trt", (1.3, 0.9), "f64", u_amp=0.05, steps=10,
         equilibrium="moment_matched"),
    # KBC on D3Q27
    Case("kbc_q27_f64_cavity", (14, 14, 14), 27, "kbc", (1.99,), "f64", geometry="cavity", ubb=(0.05, 0, 0), steps=25),
    Case("kbc_q27_f32_aa_obst", (17, 13, 11), 27, "kbc", (1.9,), "f32", pattern="aa", geometry="obstacles",
         ubb=(0.02, -0.01, 0.03), u_amp=0.05, steps=14),
    # D3Q19 cumulant
    Case("cum19_f64_periodic", (16, 14, 12), 19, "cumulant", (1.95,), "f64", u_amp=0.05, steps=20),
    Case("cum19_general_rates_cavity", (14, 14, 14), 19, "cumulant", (1.8, 1.3, 1.2, 0.9), "f64", geometry="cavity",
         ubb=(0.05, 0, 0), steps=25),
    Case("cum19_f32_channel", (16, 20, 12), 19, "cumulant", (1.9,), "f32", geometry="channel", u_amp=0.03, steps=20),
    Case("cum19_aa_f64_obst", (17, 13, 11), 19, "cumulant", (1.95, 1.1, 1.0, 1.2), "f64", pattern="aa",
         geometry="obstacles", ubb=(0.02, -0.01, 0.03), u_amp=0.05, steps=15),
    # MRT with one rate per moment
    Case("mrt_rows_f64_walls", (17, 13, 11), 19, "mrt", ROW_RATES, "f64", geometry="obstacles", ubb=(0.02, -0.01, 0.03),
         u_amp=0.05, steps=15),
    Case("mrt_rows_f32_aa", (32, 16, 8), 19, "mrt", ROW_RATES, "f32", pattern="aa", u_amp=0.03, steps=12),
    Case("mrt_rows_f64_eso_channel", (16, 20, 12), 19, "mrt", ROW_RATES, "f64", pattern="esotwist", geometry="channel",
         steps=11),
    # collide-stream-push, two arrays
    Case("push_trt_force_obst_f64", (17, 13, 11), 19, "trt", (1.6, 0.5), "f64", pattern="push", force=(1e-5, 2e-5, 0),
         geometry="obstacles", ubb=(0.02, -0.01, 0.03), steps=15),
    Case("push_cumulant_cavity", (14, 14, 14), 27, "cumulant", (1.95,), "f64", pattern="push", geometry="cavity",
         ubb=(0.05, 0, 0), steps=12),
    Case("push_mrt_f32_channel32", (32, 20, 12), 19, "mrt", (1.9, 1.3, 1.1, 0.8), "f32", pattern="push",
         geometry="channel", steps=13),
    Case("push_kbc27_periodic", (16, 12, 10), 27, "kbc", (1.95,), "f64", pattern="push", u_amp=0.05, steps=9),
    # EsoTwist
    Case("eso_trt_force_f64_odd", (18, 14, 10), 19, "trt", (1.6, 0.5), "f64", pattern="esotwist", force=(1e-5, 2e-5, 0),
         steps=21),
    Case("eso_srt_q27_f32_even", (18, 14, 10), 27, "srt", (1.7,), "f32", pattern="esotwist", steps=12),
    Case("eso_trt_obstacles_odd", (17, 13, 11), 19, "trt", (1.6, 0.5), "f64", pattern="esotwist", force=(1e-5, 0, 0),
         geometry="obstacles", ubb=(0.02, -0.01, 0.03), steps=15),
    Case("eso_cumulant_cavity", (14, 14, 14), 27, "cumulant", (1.95,), "f64", pattern="esotwist", geometry="cavity",
         ubb=(0.05, 0, 0), steps=20),
    Case("eso_mrt_f32_channel", (16, 20, 12), 19, "mrt", (1.9, 1.3, 1.1, 0.8), "f32", pattern="esotwist",
         geometry="channel", steps=13),
    Case("eso_kbc_obst_f64", (17, 13, 11), 19, "kbc", (1.95,), "f64", pattern="esotwist", geometry="obstacles",
         ubb=(0.02, -0.01, 0.03), u_amp=0.05, steps=14),
    # generated operators (codegen/)
    Case("gen_srt_q19_f64_cavity", (14, 14, 14), 19, "gen_srt", (1.9,), "f64", geometry="cavity", ubb=(0.05, 0, 0),
         steps=20),
    Case("gen_trt_q19_f32_channel", (16, 20, 12), 19, "gen_trt", (1.6, 0.5), "f32", geometry="channel", u_amp=0.05,
         steps=20),
    Case("gen_trt_q19_f64_obst_aa", (17, 13, 11), 19, "gen_trt", (1.7, 1.1), "f64", pattern="aa", geometry="obstacles",
         ubb=(0.02, -0.01, 0.03), u_amp=0.05, steps=13),
    Case("gen_mrt_q19_f64_aa", (18, 14, 10), 19, "gen_mrt", (1.9, 1.3, 1.1, 0.8), "f64", pattern="aa", u_amp=0.05,
         steps=12),
    Case("gen_mrt_q19_f32_pull_walls", (32, 20, 12), 19, "gen_mrt", (1.9, 1.0, 1.0, 1.0), "f32", geometry="channel",
         u_amp=0.03, steps=11),
    Case("gen_srt_q27_f32_aa", (18, 14, 10), 27, "gen_srt", (1.7,), "f32", pattern="aa", u_amp=0.05, steps=12),
    Case("gen_mrt_q27_f64_cavity", (14, 14, 14), 27, "gen_mrt", (1.9, 1.3, 1.1, 0.8), "f64", geometry="cavity",
         ubb=(0.05, 0, 0), steps=15),
    Case("gen_mrt_q27_f32_aa_obst", (17, 13, 11), 27, "gen_mrt", (1.8, 1.0, 1.0, 1.0), "f32", pattern="aa",
         geometry="obstacles", ubb=(0.02, -0.01, 0.03), u_amp=0.05, steps=12),
    Case("gen_trt_q27_f64_push_obst", (17, 13, 11), 27, "gen_trt", (1.6, 0.5), "f64", pattern="push",
         geometry="obstacles", ubb=(0.02, -0.01, 0.03), u_amp=0.05, steps=11),
    Case("gen_trt_q19_f64_eso", (18, 14, 10), 19, "gen_trt", (1.6, 0.5), "f64", pattern="esotwist", u_amp=0.05,
         steps=9),
    Case("gen_smag_q19_f64_channel", (16, 20, 10), 19, "gen_smagorinsky", (1.95, 0.17), "f64", geometry="channel",
         u_amp=0.05, steps=20),
    Case("gen_smag_q27_f32_aa_obst", (17, 13, 11), 27, "gen_smagorinsky", (1.9, 0.12), "f32", pattern="aa",
         geometry="obstacles", ubb=(0.02, -0.01, 0.03), u_amp=0.05, steps=12),
    Case("gen_inc_srt_q19_f64_walls", (17, 13, 11), 19, "gen_srt", (1.8,), "f64", geometry="obstacles",
         ubb=(0.02, -0.01, 0.03), u_amp=0.05, steps=15, equilibrium="incompressible"),
    Case("gen_inc_trt_q27_f32_aa", (18, 14, 10), 27, "gen_trt", (1.5, 1.2), "f32", pattern="aa", steps=12,
         u_amp=0.05, equilibrium="incompressible"),
    Case("gen_inc_trt_q19_f64_push", (16, 12, 10), 19, "gen_trt", (1.6, 0.5), "f64", pattern="push", steps=9,
         u_amp=0.05, equilibrium="incompressible"),
    # KBC with the exact entropy maximum by Newton's method
    Case("kbcx_q19_f64_cavity", (14, 14, 14), 19, "kbc_exact", (1.99,), "f64", geometry="cavity", ubb=(0.08, 0, 0),
         u_amp=0.1, steps=20),
    Case("kbcx_q27_f64_aa_obst", (17, 13, 11), 27, "kbc_exact", (1.95,), "f64", pattern="aa", geometry="obstacles",
         ubb=(0.02, -0.01, 0.03), u_amp=0.1, steps=12),
    Case("kbcx_q19_f32", (16, 12, 10), 19, "kbc_exact", (1.9,), "f32", u_amp=0.08, steps=15),
    Case("kbcx_q27_f32_push_channel", (16, 20, 12), 27, "kbc_exact", (1.97,), "f32", pattern="push", geometry="channel",
         u_amp=0.08, steps=11),
    Case("kbcx_q19_f64_eso_odd", (18, 14, 10), 19, "kbc_exact", (1.95,), "f64", pattern="esotwist", u_amp=0.1, steps=9),
]


@pytest.fixture(params=["plain", "staged"])
def kernel_path(request):
    """Run the test with the bulk kernels forced to one path (include/lbm.h lbm_set_kernel_path)."""
    from paper_2001_11806_b200 import lbm as L
    L.set_kernel_path(request.param)
    yield request.param
    L.set_kernel_path("auto")


@pytest.mark.parametrize("case", PARITY, ids=lambda c: c.name)
def test_parity_vs_oracle(case, kernel_path):
    sim = make_sim(case)
    init_sim(sim, case)
    sim.step(case.steps)
    got = sim.populations()
    ref = oracle_run(case)
    err = max_rel_err(got, ref, fluid_mask(case, case.Q))
    assert err <= TOL[case.dtype], err


STAGED_CASES = [
    Case("st_trt_f64_ragged_rows", (32, 13, 9), 19, "trt", (1.6, 0.5), "f64", force=(1e-5, 0, 0), steps=9),
    Case("st_mrt_f32_aa_walls16", (32, 20, 12), 19, "mrt", (1.9, 1.3, 1.1, 0.8), "f32", pattern="aa",
         geometry="channel", steps=11),
    Case("st_cumulant_pull_cavity16", (16, 16, 16), 27, "cumulant", (1.95,), "f64", geometry="cavity",
         ubb=(0.05, 0, 0), steps=9),
    Case("st_kbc_aa_obst", (48, 10, 8), 19, "kbc", (1.95,), "f64", pattern="aa", geometry="obstacles",
         ubb=(0.02, -0.01, 0.03), u_amp=0.05, steps=9),
    Case("st_smag_q27_f32", (64, 6, 5), 27, "smagorinsky", (1.9, 0.12), "f32", u_amp=0.05, steps=8),
    Case("st_kbc27_pull_f64", (32, 9, 7), 27, "kbc", (1.95,), "f64", u_amp=0.05, steps=7),
    Case("st_kbcx27_pull_f64", (32, 9, 7), 27, "kbc_exact", (1.95,), "f64", u_amp=0.1, steps=7),
    Case("st_kbcx19_aa_f32_walls16", (32, 12, 10), 19, "kbc_exact", (1.95,), "f32", pattern="aa", geometry="channel",
         u_amp=0.08, steps=9),
    Case("st_eso_mrt_f32_walls16", (32, 14, 10), 19, "mrt", (1.9, 1.3, 1.1, 0.8), "f32", pattern="esotwist",
         geometry="channel", steps=9),
    Case("st_eso_cum27_f64_odd", (16, 9, 7), 27, "cumulant", (1.95,), "f64", pattern="esotwist", u_amp=0.03, steps=7),
    Case("st_mrt_rows_aa_f64", (32, 9, 7), 19, "mrt", ROW_RATES, "f64", pattern="aa", u_amp=0.03, steps=8),
    Case("st_cum19_aa_f32_walls16", (32, 12, 10), 19, "cumulant", (1.95,), "f32", pattern="aa", geometry="channel",
         u_amp=0.03, steps=9),
]


@pytest.mark.parametrize("case", STAGED_CASES, ids=lambda c: c.name)
def test_staged_and_plain_paths_agree(case):
    """Shapes the TMA-staged kernels accept (nx * sizeof(real) % 16 == 0; staged flag rows at nx % 16 == 0;
    several rows per tile and a ragged last tile): both paths against the oracle, and against each other."""
    from paper_2001_11806_b200 import lbm as L
    out = {}
    try:
        for path in ("plain", "staged"):
            L.set_kernel_path(path)
            sim = make_sim(case)
            init_sim(sim, case)
            sim.step(case.steps)
            out[path] = sim.populations(raw=True)
            err = max_rel_err(sim.populations(), oracle_run(case), fluid_mask(case, case.Q))
            assert err <= TOL[case.dtype], (path, err)
            sim.close()
    finally:
        L.set_kernel_path("auto")
    mask = fluid_mask(case, case.Q)
    d = np.abs(out["plain"][mask] - out["staged"][mask])
    assert float(d.max()) <= (1e-14 if case.dtype == "f64" else 1e-6)


GRAPH_CASES = [
    PARITY[0],
    Case("g_links_pull", (16, 16, 16), 27, "cumulant", (1.95,), "f64", geometry="cavity", ubb=(0.05, 0, 0), steps=13,
         extra={"boundary_mode": "links"}),
    Case("g_split_aa_staged", (32, 20, 12), 19, "trt", (1.6, 0.5), "f64", pattern="aa", geometry="channel", steps=13),
    Case("g_faces_pull", (20, 18, 12), 19, "trt", (1.6, 0.5), "f64", force=(1e-5, 0, 0), geometry="channel", steps=13),
    Case("g_eso_obst", (17, 13, 11), 19, "trt", (1.6, 0.5), "f64", pattern="esotwist", geometry="obstacles", steps=13),
    Case("g_push_links_f32", (32, 16, 12), 19, "mrt", (1.9, 1.0, 1.0, 1.0), "f32", pattern="push", geometry="channel",
         steps=13, extra={"boundary_mode": "links"}),
]


@pytest.mark.parametrize("case", GRAPH_CASES, ids=lambda c: c.name)
def test_cuda_graph_path_bit_identical(case):
    """use_graph = 1: the two-step cycle captured once and replayed (odd step counts end with a plain step)
    is bit-identical to plain launches, for every boundary implementation and pattern."""
    a = make_sim(case)
    b = make_sim(case, use_graph=True)
    for s in (a, b):
        init_sim(s, case)
        s.step(case.steps)
        s.step(4)
    mask = fluid_mask(case, case.Q)
    np.testing.assert_array_equal(a.populations(raw=True)[mask], b.populations(raw=True)[mask])


PERSISTENT = [
    Case("p_c0", (32, 32, 32), 19, "srt", (1.8,), "f64", steps=37),
    Case("p_walls_force", (17, 13, 11), 19, "trt", (1.6, 0.5), "f64", force=(1e-5, 0, 0), geometry="obstacles",
         ubb=(0.02, -0.01, 0.03), steps=15),
    Case("p_aa_cumulant_cavity", (12, 12, 12), 27, "cumulant", (1.95,), "f64", pattern="aa", geometry="cavity",
         ubb=(0.05, 0, 0), steps=13),
    Case("p_aa_mrt_f32", (20, 16, 12), 19, "mrt", (1.9, 1.0, 1.0, 1.0), "f32", pattern="aa", init="shear",
         rho_amp=0.0, u_amp=1e-4, steps=12),
]


@pytest.mark.parametrize("case", PERSISTENT, ids=lambda c: c.name)
def test_persistent_multistep_kernel(case):
    """use_graph = 2: one cooperative launch per lbm_step call (grid barrier between steps); split
    into uneven calls and NaN-check chunks to exercise the phase bookkeeping."""
    sim = make_sim(case, use_graph=2, check_nan_every=4)
    init_sim(sim, case)
    l0 = sim.launches
    sim.step(case.steps // 2)
    sim.step(case.steps - case.steps // 2)
    assert sim.launches - l0 <= 2 + case.steps // 4 + 2  # one launch per chunk, not per step
    err = max_rel_err(sim.populations(), oracle_run(case), fluid_mask(case, case.Q))
    assert err <= TOL[case.dtype], err


@pytest.mark.parametrize("pattern", ["pull", "aa", "esotwist", "push"])
def test_zero_steps_is_identity_and_counters(pattern):
    """lbm_step(0) launches nothing and leaves the state bit-identical (degenerate call)."""
    case = Case("zero", (16, 8, 6), 19, "trt", (1.6, 0.5), "f64", pattern=pattern, steps=0)
    sim = make_sim(case)
    init_sim(sim, case)
    before, l0 = sim.populations(raw=True), sim.launches
    sim.step(0)
    assert sim.launches == l0
    np.testing.assert_array_equal(sim.populations(raw=True), before)


def test_nan_detection():
    from paper_2001_11806_b200 import lbm as L
    case = Case("nan", (8, 8, 8), 19, "srt", (1.8,), "f64")
    sim = make_sim(case, check_nan_every=1)
    init_sim(sim, case)
    f = sim.populations()
    f[3, 2, 2, 2] = np.nan
    sim.set_populations(f)
    with pytest.raises(L.LBMError) as e:
        sim.step(2)
    assert e.value.status == L.LBM_ENAN


# -----------------------------------------------------------------------------------------
# Slab decomposition (loopback slabs on one GPU run the same kernels as NCCL ranks)
# -----------------------------------------------------------------------------------------
@pytest.mark.parametrize("P", [2, 4])
@pytest.mark.parametrize("halo_mode", [0, 1])
def test_slab_decomposition_bit_identical(P, halo_mode):
    case = Case("dec", (20, 16, 16), 19, "trt", (1.6, 0.5), "f64", force=(1e-5, 0, 0), geometry="channel", steps=30)
    one = make_sim(case)
    many = make_sim(case, n_local_slabs=P, halo_mode=halo_mode)
    for s in (one, many):
        init_sim(s, case)
        s.step(case.steps)
    np.testing.assert_array_equal(one.populations(raw=True), many.populations(raw=True))
    # and host-array init goes through the ghost exchange
    many2 = make_sim(case, n_local_slabs=P, halo_mode=halo_mode)
    init_sim(many2, case, use_random_kernel=False)
    many2.step(case.steps)
    np.testing.assert_array_equal(one.populations(raw=True), many2.populations(raw=True))


@pytest.mark.parametrize("Q,op,rates,dtype", [(27, "cumulant", (1.95,), "f64"), (19, "srt", (1.8,), "f32"),
                                              (27, "kbc_exact", (1.95,), "f64")])
def test_slab_decomposition_other_ops(Q, op, rates, dtype):
    case = Case("dec2", (12, 10, 12), Q, op, rates, dtype, steps=9)
    one = make_sim(case)
    many = make_sim(case, n_local_slabs=3)
    for s in (one, many):
        init_sim(s, case)
        s.step(case.steps)
    np.testing.assert_array_equal(one.populations(raw=True), many.populations(raw=True))


@pytest.mark.parametrize("P", [2, 4])
@pytest.mark.parametrize("halo_mode", [0, 1])
@pytest.mark.parametrize("Q,op,rates,geometry,force", [(19, "trt", (1.6, 0.5), "channel", (1e-5, 0, 0)),
                                                       (19, "srt", (1.7,), "obstacles", (0, 0, 0)),
                                                       (27, "cumulant", (1.95,), "periodic", (0, 0, 0)),
                                                       (19, "mrt", (1.9, 1.0, 1.0, 1.0), "periodic", (0, 0, 0))])
def test_aa_slab_decomposition_bit_identical(P, halo_mode, Q, op, rates, geometry, force):
    """AA with slabs: ghost fill after even steps, return of ghost-plane writes after odd steps
    (masked by the producing cell's flag with walls). Odd and even step counts."""
    case = Case("aadec", (14, 12, 16), Q, op, rates, "f64", pattern="aa", force=force, geometry=geometry,
                ubb=(0.02, -0.01, 0.03))
    if op == "mrt":  # C2's fp32 shear-only MRT: the two-cells-per-thread kernels (nx = 72: ragged second cell)
        case = Case("aadec_x2", (72, 6, 16), Q, op, rates, "f32", pattern="aa", u_amp=0.03)
    for steps in (7, 10):
        one = make_sim(case)
        many = make_sim(case, n_local_slabs=P, halo_mode=halo_mode)
        for s in (one, many):
            init_sim(s, case)
            s.step(steps)
        mask = fluid_mask(case, Q)
        np.testing.assert_array_equal(one.populations(raw=True)[mask], many.populations(raw=True)[mask])
        np.testing.assert_array_equal(one.populations()[mask], many.populations()[mask])


@pytest.mark.parametrize("halo_mode", [0, 1, 2])
@pytest.mark.parametrize("Q,op,rates,geometry,pattern", [(19, "trt", (1.6, 0.5), "channel", "pull"),
                                                         (27, "cumulant", (1.95,), "periodic", "pull"),
                                                         (19, "trt", (1.6, 0.5), "obstacles", "aa"),
                                                         (27, "cumulant", (1.95,), "cavity", "aa"),
                                                         (19, "mrt", (1.9, 1.3, 1.1, 0.8), "channel", "aa")])
def test_nccl_self_exchange_bit_identical(halo_mode, Q, op, rates, geometry, pattern):
    """The NCCL exchange path (ghost planes, schedule, comm stream overlapped with the interior
    launch, event ordering) on one GPU through a 1-rank communicator: bit-identical to local z wrap."""
    case = Case("self", (16, 16, 16) if geometry == "cavity" else (16, 12, 10), Q, op, rates, "f64", geometry=geometry,
                steps=13, pattern=pattern, ubb=(0.02, -0.01, 0.03))
    one = make_sim(case)
    nc = make_sim(case, nccl_self=True, halo_mode=halo_mode)
    for s in (one, nc):
        init_sim(s, case)
        s.step(case.steps)
    np.testing.assert_array_equal(one.populations(raw=True), nc.populations(raw=True))
    nc2 = make_sim(case, nccl_self=True, halo_mode=halo_mode)
    init_sim(nc2, case, use_random_kernel=False)  # host arrays + exchange of the initial ghosts
    nc2.step(case.steps)
    np.testing.assert_array_equal(one.populations(raw=True), nc2.populations(raw=True))


# -----------------------------------------------------------------------------------------
# Full BASELINE sizes (the launch configuration bench.py times): sampled cells vs the oracle
# evaluated on the (2k+1)^3 neighbourhood each sample depends on after k steps.
# -----------------------------------------------------------------------------------------
def _sample_cells(case, n=48, seed=5):
    rng = np.random.default_rng(seed)
    nx, ny, nz = case.shape
    pts = [(rng.integers(nx), rng.integers(ny), rng.integers(nz)) for _ in range(n)]
    # boundary-adjacent and domain-edge cells
    pts += [(0, 1, 0), (nx - 1, ny - 2, nz - 1), (nx // 2, 1, nz // 2), (1, ny - 2, nz - 2), (nx - 1, 0, 0)]
    fl = case.flags()
    return [p for p in pts if fl is None or fl[p[2], p[1], p[0]] == 0]


def _oracle_at(case, pts, k):
    nx, ny, nz = case.shape
    B = 2 * k + 1
    out = []
    gfl = case.flags()
    prof, amp = case.profile()
    for (x, y, z) in pts:
        xs = np.arange(x - k, x + k + 1)
        ys = np.arange(y - k, y + k + 1)
        zs = np.arange(z - k, z + k + 1)
        Z, Y, X = np.meshgrid(zs, ys, xs, indexing="ij")
        fl = None if gfl is None else np.ascontiguousarray(gfl[Z % nz, Y % ny, X % nx])
        d = O.Domain(case.method(nthreads=1), B, B, B, flags=fl)
        if case.init == "rest":
            rho, u = np.ones((B, B, B)), np.zeros((3, B, B, B))
        else:
            rho, u = LI.fields_at(case.seed, nx, ny, nz, X, Y, Z, case.rho_amp, case.u_amp, prof, amp)
        f0 = d.init_equilibrium(rho, u)
        f = d.run_push(f0, k) if case.pattern == "aa" else d.run_pull(f0, k)
        out.append(f[:, k, k, k])
    return np.array(out).T


@pytest.mark.parametrize("name,boundary_mode,op", [("c0", "flags", None), ("c1_f64", "flags", None), ("c1_f32", "flags", None),
                                                   ("c2", "flags", None), ("c3", "flags", None), ("c4", "flags", None),
                                                   ("c1_f64", "links", None), ("c1_f32", "links", None), ("c3", "links", None),
                                                   # generated operators and compiled-in boundaries at full size
                                                   ("c4", "flags", "gen_trt"), ("c2", "flags", "gen_mrt"),
                                                   ("c1_f64", "inline", None), ("c3", "inline", None)])
def test_full_size_sampled_parity(name, boundary_mode, op):
    base = FULL[name]
    if op is not None:
        base = Case(base.name, base.shape, base.Q, op, base.rates, base.dtype, base.pattern, base.force, base.geometry,
                    base.ubb, init=base.init, rho_amp=base.rho_amp, u_amp=base.u_amp)
    # random near-equilibrium start (instead of rest) so every sampled cell does non-trivial work
    case = Case(base.name, base.shape, base.Q, base.op, base.rates, base.dtype, base.pattern, base.force,
                base.geometry, base.ubb, init="shear" if base.init == "shear" else "random",
                rho_amp=base.rho_amp if base.init == "shear" else 1e-3, u_amp=base.u_amp if base.init == "shear" else 0.01)
    k = 2 if case.pattern == "aa" else 3
    sim = make_sim(case, boundary_mode=boundary_mode)
    init_sim(sim, case)
    sim.step(k)
    pts = _sample_cells(case)
    nx, ny, _ = case.shape
    idx = np.array([x + nx * (y + ny * z) for (x, y, z) in pts], np.int64)
    got = sim.populations_at(idx)
    ref = _oracle_at(case, pts, k)
    err = float(np.max(np.abs(got - ref) / np.abs(ref)))
    assert err <= TOL[case.dtype], err
    sim.close()


# -----------------------------------------------------------------------------------------
# Low-level kernel ABI on caller-owned (torch) device memory
# -----------------------------------------------------------------------------------------
@pytest.mark.parametrize("pattern", ["pull", "aa"])
@pytest.mark.parametrize("nx,flag_offset", [(19, 0), (32, 0), (32, 1)])
def test_low_level_kernel_abi(pattern, nx, flag_offset):
    """Caller-owned torch memory. nx = 32 (rows of 16-byte multiples) reaches the TMA-staged AA even kernel,
    whose flag rows move by bulk copy only from a 16-byte aligned flag base: flag_offset = 1 passes a
    misaligned torch view of the flag bytes, which must fall back to global flag reads, not fault."""
    import ctypes as C
    import torch
    from paper_2001_11806_b200 import lbm as L
    case = Case("ll", (nx, 14, 9), 19, "trt", (1.6, 0.5), "f64", pattern=pattern, force=(1e-5, 0, 0),
                geometry="obstacles", ubb=(0.02, 0.0, -0.01), steps=6)
    nx, ny, nz = case.shape
    d = O.Domain(case.method(), nx, ny, nz, flags=case.flags())
    rho, u = case.fields()
    f0 = d.init_equilibrium(rho, u)
    _, w, _ = O.stencil_arrays(19)
    g0 = torch.from_numpy(f0 - w[:, None, None, None]).cuda()
    g1 = g0.clone()
    fl_buf = torch.empty(nx * ny * nz + 16, dtype=torch.uint8, device="cuda")
    fl = fl_buf[flag_offset:flag_offset + nx * ny * nz]
    stream = torch.cuda.Stream()
    hf = np.ascontiguousarray(case.flags())
    assert L.lbm_prepare_flags(hf.ctypes.data, nx, ny, nz, 0, fl.data_ptr(), stream.cuda_stream) == 0
    k = L.lbm_kernel_args()
    k.stencil, k.collision, k.dtype = 19, L.TRT, L.F64
    k.flags = fl.data_ptr()
    k.shape[0], k.shape[1], k.shape[2] = nx, ny, nz
    k.ghost, k.z_begin, k.z_end = 0, 0, nz
    k.rates[0], k.rates[1] = case.rates
    for i in range(3):
        k.force[i] = case.force[i]
        k.ubb_velocity[i] = case.ubb[i]
    k.stream = stream.cuda_stream
    a, b = g0, g1
    for t in range(case.steps):
        if pattern == "pull":
            k.src, k.dst = a.data_ptr(), b.data_ptr()
            assert L.lbm_kernel_pull(C.byref(k)) == 0
            a, b = b, a
        else:
            k.dst = a.data_ptr()
            assert L.lbm_kernel_aa(C.byref(k), t % 2) == 0
    stream.synchronize()
    got = a.cpu().numpy() + w[:, None, None, None]
    ref = d.run_pull(f0, case.steps) if pattern == "pull" else d.run_push(f0, case.steps)
    assert max_rel_err(got, ref, fluid_mask(case, 19)) <= 1e-12


# -----------------------------------------------------------------------------------------
# Index-list boundaries: flag-free update kernels + link kernel
# -----------------------------------------------------------------------------------------
LINK_CASES = [
    Case("lk_trt_f64_cavity_pull", (14, 14, 14), 19, "trt", (1.6, 0.5), "f64", force=(1e-5, 0, 0), geometry="cavity",
         ubb=(0.05, 0, 0), steps=21),
    Case("lk_trt_f32_obst_aa", (17, 13, 11), 19, "trt", (1.6, 0.5), "f32", pattern="aa", geometry="obstacles",
         ubb=(0.02, -0.01, 0.03), steps=15),
    Case("lk_cum27_cavity_aa", (12, 12, 12), 27, "cumulant", (1.95,), "f64", pattern="aa", geometry="cavity",
         ubb=(0.05, 0, 0), steps=12),
    Case("lk_mrt_f32_channel32_pull", (32, 20, 12), 19, "mrt", (1.9, 1.3, 1.1, 0.8), "f32", geometry="channel", steps=14),
    Case("lk_kbc_obst_pull", (16, 12, 10), 19, "kbc", (1.95,), "f64", geometry="obstacles", ubb=(0.02, -0.01, 0.03),
         u_amp=0.05, steps=12),
    # EsoTwist with index lists (P:875-891 + P:904-914): the fix moves the departing slot of the link location
    Case("lk_eso_trt_f64_obst_odd", (17, 13, 11), 19, "trt", (1.6, 0.5), "f64", pattern="esotwist", force=(1e-5, 0, 0),
         geometry="obstacles", ubb=(0.02, -0.01, 0.03), steps=15),
    Case("lk_eso_cum27_cavity_even", (12, 12, 12), 27, "cumulant", (1.95,), "f64", pattern="esotwist",
         geometry="cavity", ubb=(0.05, 0, 0), steps=12),
    Case("lk_eso_mrt_f32_channel32", (32, 20, 12), 19, "mrt", (1.9, 1.3, 1.1, 0.8), "f32", pattern="esotwist",
         geometry="channel", steps=13),
]


def _links_brute_force(fl, Q):
    c, _, _ = O.stencil_arrays(Q)
    nz, ny, nx = fl.shape
    out = set()
    for z, y, x in zip(*np.nonzero(fl)):
        for q in range(1, Q):
            xx, yy, zz = (x + c[q, 0]) % nx, (y + c[q, 1]) % ny, (z + c[q, 2]) % nz
            if fl[zz, yy, xx] == 0:
                out.add((int(x + nx * (y + ny * z)), q, int(fl[z, y, x])))
    return out


@pytest.mark.parametrize("case", LINK_CASES, ids=lambda c: c.name)
def test_index_list_boundaries_vs_oracle(case, kernel_path):
    sim = make_sim(case, boundary_mode="links")
    cells, dirs, types = sim.boundary_links()
    assert set(zip(cells.tolist(), dirs.tolist(), types.tolist())) == _links_brute_force(case.flags(), case.Q)
    assert len(cells) == len(set(zip(cells.tolist(), dirs.tolist())))
    init_sim(sim, case)
    sim.step(case.steps)
    mask = fluid_mask(case, case.Q)
    err = max_rel_err(sim.populations(), oracle_run(case), mask)
    assert err <= TOL[case.dtype], err
    # same update as the compiled-in flag handling
    ref = make_sim(case)
    init_sim(ref, case)
    ref.step(case.steps)
    assert max_rel_err(sim.populations(), ref.populations(), mask) <= (1e-13 if case.dtype == "f64" else 1e-6)


@pytest.mark.parametrize("pattern,steps", [("pull", 17), ("aa", 16), ("aa", 17)])
def test_index_list_per_link_wall_velocities(pattern, steps):
    """Custom per-link boundary data: every UBB link gets the wall velocity of its wall cell
    from a seeded field; the oracle uses the same field per wall cell."""
    case = Case("lkv", (14, 14, 14), 19, "trt", (1.6, 0.5), "f64", pattern=pattern, geometry="cavity",
                ubb=(0.05, 0, 0), steps=steps)
    nx, ny, nz = case.shape
    fl = case.flags().copy()
    fl[fl == LI.NOSLIP] = LI.UBB  # every wall moves, with its own velocity
    rng = np.random.default_rng(9)
    field = rng.uniform(-0.03, 0.03, (3, nz, ny, nx))
    sim = make_sim(case, boundary_mode="links", flags=fl)
    cells, dirs, types = sim.boundary_links()
    assert (types == LI.UBB).all()
    sim.set_link_velocities(field.reshape(3, -1)[:, cells].T)
    init_sim(sim, case)
    sim.step(steps)
    d = O.Domain(case.method(), nx, ny, nz, flags=fl, wall_u=field)
    rho, u = case.fields()
    f0 = d.init_equilibrium(rho, u)
    ref = d.run_push(f0, steps) if pattern == "aa" else d.run_pull(f0, steps)
    mask = np.broadcast_to(fl == 0, ref.shape)
    assert max_rel_err(sim.populations(), ref, mask) <= 1e-12
    rho_g, u_g = sim.macroscopic()
    rho_o, u_o = d.macroscopic(ref, post_collision=pattern == "pull")
    np.testing.assert_allclose(u_g[:, fl == 0], u_o[:, fl == 0], rtol=0, atol=1e-15)


IN_KERNEL_LINK_CASES = [c for c in LINK_CASES if c.pattern in ("pull", "aa")] + [
    # face-aligned walls (FM_FACEL: walls and links from coordinates): C1-like channel, C3-like cavity
    Case("lk_trt_f32_channel_force_pull", (24, 18, 10), 19, "trt", (1.6, 0.5), "f32", geometry="channel",
         force=(1e-5, 0, 0), steps=11),
    Case("lk_trt_f64_channel_force_aa", (24, 18, 10), 19, "trt", (1.6, 0.5), "f64", pattern="aa", geometry="channel",
         force=(1e-5, 0, 0), steps=11),
    Case("lk_cum27_cavity_pull", (12, 12, 12), 27, "cumulant", (1.95,), "f64", geometry="cavity",
         ubb=(0.05, 0, 0), steps=12),
    Case("lk_cum27_f32_cavity_aa", (12, 12, 12), 27, "cumulant", (1.95,), "f32", pattern="aa", geometry="cavity",
         ubb=(0.05, 0, 0), steps=12),
    Case("lk_trt_f64_box_aa", (40, 12, 10), 19, "trt", (1.6, 0.5), "f64", pattern="aa", geometry="obstacles",
         ubb=(0.03, 0.01, -0.02), steps=9, extra={"flags": np.maximum(LI.channel_flags(40, 12, 10), LI.random_obstacles(3, 40, 12, 10))}),
]


@pytest.mark.parametrize("use_graph", [False, True])
@pytest.mark.parametrize("case", IN_KERNEL_LINK_CASES, ids=lambda c: c.name)
def test_in_kernel_links_identical_to_link_kernel(case, use_graph, kernel_path, monkeypatch):
    """Index lists folded into the pull / AA update kernels (FM_LINKS: each near-wall fluid cell stores the
    wall slots of its links after its collision) against the separate link kernel: the link stores
    are the link kernel's values (bit for bit on the plain fp64 path); the two kernel instantiations may
    contract the collision arithmetic differently (G16), so the comparison allows 1e-14 (fp64) / 2e-6 (fp32)
    relative — at odd and even step counts, across several lbm_step calls, with the CUDA-graph cycle, and
    after set_populations (the full list primes the wall slots again)."""
    monkeypatch.setenv("LBM_LINKS_FUSED", "1")
    fused = make_sim(case, boundary_mode="links", use_graph=use_graph)
    assert fused.boundary_impl == "links_fused"
    monkeypatch.setenv("LBM_LINKS_FUSED", "0")
    sep = make_sim(case, boundary_mode="links")
    assert sep.boundary_impl == "links"
    fl = case.extra.get("flags", case.flags())
    mask = np.broadcast_to(fl == 0, (case.Q,) + fl.shape)
    for s in (fused, sep):
        init_sim(s, case)
    tol = 1e-14 if case.dtype == "f64" else 2e-6

    def same(a, b):
        if case.dtype == "f64" and kernel_path == "plain":
            np.testing.assert_array_equal(a, b)
        else:
            assert max_rel_err(a, b) <= tol

    for n in (1, 2, case.steps):
        for s in (fused, sep):
            s.step(n)
        same(fused.populations()[mask], sep.populations()[mask])
    for s in (fused, sep):
        s.set_populations(s.populations())
        s.step(3)
    same(fused.populations()[mask], sep.populations()[mask])
    if case.extra.get("flags") is None:
        assert max_rel_err(fused.populations(), oracle_run(case, case.steps + 6), mask) <= TOL[case.dtype]


@pytest.mark.parametrize("P,halo_mode,nccl_self", [(2, 0, False), (4, 1, False), (1, 0, True), (1, 1, True), (1, 2, True)])
@pytest.mark.parametrize("pattern", ["pull", "aa", "push", "esotwist"])
@pytest.mark.parametrize("in_kernel", ["0", "1"])
def test_index_list_boundaries_slabs_bit_identical(P, halo_mode, nccl_self, pattern, in_kernel, monkeypatch):
    """Index-list boundaries with slab decomposition: the link kernel also fills the wall slots of ghost
    planes after the exchange (fused halo: after the next LSA gate, plus a closing gate per lbm_step call);
    loopback slabs, NCCL self-exchange and the fused NVLink halo are bit-identical to the single slab, for
    every pattern, and the concatenated link lists are the global list. With the in-kernel links (pull, AA,
    not the fused halo) the links whose wall cell lies in a ghost plane stay with the link kernel."""
    monkeypatch.setenv("LBM_LINKS_FUSED", in_kernel)
    case = Case("lkdec", (16, 12, 16), 19, "trt", (1.6, 0.5), "f64", force=(1e-5, 0, 0), geometry="obstacles",
                ubb=(0.02, -0.01, 0.03), steps=13, pattern=pattern)
    one = make_sim(case, boundary_mode="links")
    many = make_sim(case, boundary_mode="links", n_local_slabs=P, halo_mode=halo_mode, nccl_self=nccl_self)
    a, b = one.boundary_links(), many.boundary_links()
    assert sorted(zip(*[v.tolist() for v in a])) == sorted(zip(*[v.tolist() for v in b]))
    for s in (one, many):
        init_sim(s, case)
        s.step(case.steps)
    mask = fluid_mask(case, case.Q)
    np.testing.assert_array_equal(one.populations()[mask], many.populations()[mask])


@pytest.mark.parametrize("P,halo_mode,nccl_self", [(2, 0, False), (4, 1, False), (1, 0, True), (1, 1, True)])
@pytest.mark.parametrize("pattern,geometry,Q,op,rates", [("pull", "channel", 19, "trt", (1.6, 0.5)),
                                                         ("aa", "channel", 19, "trt", (1.6, 0.5)),
                                                         ("aa", "cavity", 27, "cumulant", (1.95,)),
                                                         ("pull", "cavity", 27, "cumulant", (1.95,))])
def test_in_kernel_links_walled_slabs_bit_identical(P, halo_mode, nccl_self, pattern, geometry, Q, op, rates, monkeypatch):
    """In-kernel links (FM_LINKS) on the channel and the cavity across slabs: the links whose wall cell lies in
    a ghost plane stay with the residual link kernel (after the exchange); bit-identical to the single slab."""
    monkeypatch.setenv("LBM_LINKS_FUSED", "1")
    shape = (16, 16, 16)
    case = Case("fl", shape, Q, op, rates, "f64", pattern=pattern, geometry=geometry, ubb=(0.03, 0, 0),
                force=(1e-5, 0, 0) if op == "trt" else (0, 0, 0), steps=9)
    one = make_sim(case, boundary_mode="links")
    many = make_sim(case, boundary_mode="links", n_local_slabs=P, halo_mode=halo_mode, nccl_self=nccl_self)
    assert one.boundary_impl == many.boundary_impl == "links_fused"
    for s in (one, many):
        init_sim(s, case)
        s.step(case.steps)
    mask = fluid_mask(case, Q)
    np.testing.assert_array_equal(one.populations()[mask], many.populations()[mask])
    assert max_rel_err(one.populations(), oracle_run(case), mask) <= TOL["f64"]


@pytest.mark.parametrize("P,halo_mode,nccl_self", [(2, 0, False), (4, 1, False), (1, 0, True), (1, 1, True), (1, 2, True)])
@pytest.mark.parametrize("Q,op,rates,geometry", [(19, "trt", (1.6, 0.5), "obstacles"), (27, "cumulant", (1.95,), "periodic"),
                                                 (19, "mrt", (1.9, 1.3, 1.1, 0.8), "channel")])
def test_esotwist_slab_decomposition_bit_identical(P, halo_mode, nccl_self, Q, op, rates, geometry):
    """EsoTwist across slabs: after every step the slots the next step reads from the lower ghost plane come
    from the down neighbour's top plane, and the slots the bottom plane wrote into the lower ghost go to it
    (masked by the producing cell with walls); odd and even step counts, loopback slabs and NCCL."""
    case = Case("esodec", (14, 12, 16), Q, op, rates, "f64", pattern="esotwist", force=(0, 0, 0), geometry=geometry,
                ubb=(0.02, -0.01, 0.03))
    for steps in (7, 10):
        one = make_sim(case)
        many = make_sim(case, n_local_slabs=P, halo_mode=halo_mode, nccl_self=nccl_self)
        for s in (one, many):
            init_sim(s, case)
            s.step(steps)
        mask = fluid_mask(case, Q)
        np.testing.assert_array_equal(one.populations()[mask], many.populations()[mask])
    many2 = make_sim(case, n_local_slabs=P, halo_mode=halo_mode, nccl_self=nccl_self)
    init_sim(many2, case, use_random_kernel=False)
    many2.step(5)
    np.testing.assert_allclose(many2.populations()[mask], oracle_run(case, 5)[mask], rtol=1e-12, atol=0)


@pytest.mark.parametrize("P,halo_mode,nccl_self", [(2, 0, False), (4, 1, False), (1, 0, True), (1, 1, True), (1, 2, True)])
@pytest.mark.parametrize("Q,op,rates,geometry", [(19, "trt", (1.6, 0.5), "obstacles"), (27, "cumulant", (1.95,), "cavity")])
def test_push_slab_decomposition_bit_identical(P, halo_mode, nccl_self, Q, op, rates, geometry):
    """Collide-stream-push across slabs: the pushes that land in ghost planes go home after every step
    (masked by the producing cell with walls), or go straight to the neighbour's plane (fused)."""
    case = Case("pushdec", (16, 16, 16), Q, op, rates, "f64", pattern="push", geometry=geometry, ubb=(0.02, -0.01, 0.03),
                steps=11)
    one = make_sim(case)
    many = make_sim(case, n_local_slabs=P, halo_mode=halo_mode, nccl_self=nccl_self)
    for s in (one, many):
        init_sim(s, case)
        s.step(case.steps)
    mask = fluid_mask(case, Q)
    np.testing.assert_array_equal(one.populations(raw=True)[mask], many.populations(raw=True)[mask])


@pytest.mark.parametrize("kind", ["push", "collide"])
def test_low_level_push_and_collide_kernels(kind):
    """lbm_kernel_push (walls inline) and lbm_kernel_collide on caller-owned torch memory vs the oracle."""
    import ctypes as C
    import torch
    from paper_2001_11806_b200 import lbm as L
    case = Case("llp", (19, 14, 9), 19, "trt", (1.6, 0.5), "f64", force=(1e-5, 0, 0), geometry="obstacles",
                ubb=(0.02, 0.0, -0.01), steps=5)
    nx, ny, nz = case.shape
    d = O.Domain(case.method(), nx, ny, nz, flags=case.flags())
    rho, u = case.fields()
    f0 = d.init_equilibrium(rho, u)
    _, w, _ = O.stencil_arrays(19)
    a = torch.from_numpy(f0 - w[:, None, None, None]).cuda()
    b = a.clone()
    fl = torch.empty(nx * ny * nz, dtype=torch.uint8, device="cuda")
    stream = torch.cuda.Stream()
    hf = np.ascontiguousarray(case.flags())
    assert L.lbm_prepare_flags(hf.ctypes.data, nx, ny, nz, 0, fl.data_ptr(), stream.cuda_stream) == 0
    k = L.lbm_kernel_args()
    k.stencil, k.collision, k.dtype = 19, L.TRT, L.F64
    k.flags = fl.data_ptr()
    k.shape[0], k.shape[1], k.shape[2] = nx, ny, nz
    k.ghost, k.z_begin, k.z_end = 0, 0, nz
    k.rates[0], k.rates[1] = case.rates
    for i in range(3):
        k.force[i] = case.force[i]
        k.ubb_velocity[i] = case.ubb[i]
    k.stream = stream.cuda_stream
    if kind == "push":
        for _ in range(case.steps):
            k.src, k.dst = a.data_ptr(), b.data_ptr()
            assert L.lbm_kernel_push(C.byref(k)) == 0
            a, b = b, a
        ref = d.run_push(f0, case.steps)
    else:
        k.dst = a.data_ptr()
        assert L.lbm_kernel_collide(C.byref(k)) == 0
        ref = f0.copy()
        d.collide_all(ref)
    stream.synchronize()
    got = a.cpu().numpy() + w[:, None, None, None]
    assert max_rel_err(got, ref, fluid_mask(case, 19)) <= 1e-12


def test_copy_q_probe():
    """The copy-q roofline probe runs and reports a plausible HBM bandwidth (it is a measurement, not a
    parity check: > 1 TB/s on a B200)."""
    from paper_2001_11806_b200 import lbm as L
    gbs = L.probe_copy(19, "f64", True, (256, 128, 64), reps=3)
    assert 1000.0 < gbs < 20000.0, gbs


@pytest.mark.gpu
@pytest.mark.parametrize("gen,hand,Q,rates,dtype,pattern", [
    ("gen_trt", "trt", 19, (1.6, 0.5), "f64", "pull"), ("gen_srt", "srt", 27, (1.8,), "f32", "aa"),
    ("gen_mrt", "mrt", 19, (1.9, 1.0, 1.0, 1.0), "f32", "aa"), ("gen_mrt", "mrt", 19, (1.9, 1.3, 1.1, 0.8), "f64", "pull"),
    ("gen_smagorinsky", "smagorinsky", 27, (1.9, 0.17), "f64", "aa")])
def test_generated_equals_hand_written(gen, hand, Q, rates, dtype, pattern):
    """The generated operator (codegen/) and the hand-written kernel are the same operator: same
    states after several steps up to FP reassociation."""
    out = []
    for op in (gen, hand):
        case = Case(f"gh_{op}", (32, 12, 10), Q, op, rates, dtype, pattern=pattern, geometry="obstacles",
                    ubb=(0.02, -0.01, 0.03), u_amp=0.05, steps=10)
        sim = make_sim(case)
        init_sim(sim, case)
        sim.step(case.steps)
        out.append(sim.populations())
    tol = 1e-13 if dtype == "f64" else 1e-5
    np.testing.assert_allclose(out[0], out[1], rtol=0, atol=tol)


# -----------------------------------------------------------------------------------------
# Compiled-in boundaries (LBM_BOUNDARY_INLINE): every cell tests its neighbours' flags
# -----------------------------------------------------------------------------------------
INLINE_CASES = [
    Case("in_trt_f64_cavity_pull", (14, 14, 14), 19, "trt", (1.6, 0.5), "f64", force=(1e-5, 0, 0), geometry="cavity",
         ubb=(0.05, 0, 0), steps=21),
    Case("in_trt_f32_obst_aa", (17, 13, 11), 19, "trt", (1.6, 0.5), "f32", pattern="aa", geometry="obstacles",
         ubb=(0.02, -0.01, 0.03), steps=15),
    Case("in_cum27_cavity_push", (12, 12, 12), 27, "cumulant", (1.95,), "f64", pattern="push", geometry="cavity",
         ubb=(0.05, 0, 0), steps=9),
    Case("in_mrt_f64_channel_eso", (16, 20, 12), 19, "mrt", (1.9, 1.3, 1.1, 0.8), "f64", pattern="esotwist",
         geometry="channel", steps=11),
]


@pytest.mark.parametrize("case", INLINE_CASES, ids=lambda c: c.name)
def test_inline_boundaries_vs_oracle_and_flags(case):
    sim = make_sim(case, boundary_mode="inline")
    init_sim(sim, case)
    sim.step(case.steps)
    got = sim.populations()
    mask = fluid_mask(case, case.Q)
    assert max_rel_err(got, oracle_run(case), mask) <= TOL[case.dtype]
    ref = make_sim(case)  # split mode (bulk + edge-list kernel): the same per-cell arithmetic
    init_sim(ref, case)
    ref.step(case.steps)
    np.testing.assert_allclose(got[mask], ref.populations()[mask], rtol=0,
                               atol=1e-14 if case.dtype == "f64" else 1e-6)


@pytest.mark.parametrize("P", [2, 3])
def test_inline_boundaries_slabs_bit_identical(P):
    case = Case("in_slabs", (16, 12, 12), 19, "trt", (1.6, 0.5), "f64", pattern="aa", geometry="obstacles",
                ubb=(0.02, -0.01, 0.03), steps=8)
    one = make_sim(case, boundary_mode="inline")
    many = make_sim(case, boundary_mode="inline", n_local_slabs=P if 12 % P == 0 else 2)
    for s in (one, many):
        init_sim(s, case)
        s.step(case.steps)
    np.testing.assert_array_equal(one.populations(raw=True), many.populations(raw=True))


# -----------------------------------------------------------------------------------------
# Borrowed (caller-owned torch) device buffers (SURVEY §8(b) ownership)
# -----------------------------------------------------------------------------------------
@pytest.mark.parametrize("pattern,geometry,extra", [("pull", "channel", {}), ("aa", "obstacles", {}),
                                                    ("esotwist", "channel", {}), ("push", "periodic", {}),
                                                    ("pull", "channel", {"nccl_self": True, "halo_mode": 1}),
                                                    ("aa", "periodic", {"nccl_self": True, "halo_mode": 0})])
def test_borrowed_torch_buffers(pattern, geometry, extra):
    """lbm_create on torch tensors (pdf_dev / flags_dev / halo_dev): same results as library-owned memory
    (bit-exact) and as the oracle; the state lives in the caller's tensors."""
    import torch
    case = Case("borrow", (32, 16, 12), 19, "trt", (1.6, 0.5), "f64", pattern=pattern, force=(1e-5, 0, 0),
                geometry=geometry, ubb=(0.02, -0.01, 0.03), steps=8)
    own = make_sim(case, **extra)
    lent = make_sim(case, borrow=True, **extra)
    assert "pdf0" in lent.buffers and ("flags" in lent.buffers) == (case.flags() is not None)
    assert ("halo" in lent.buffers) == bool(extra)
    before = lent.buffers["pdf0"].clone()
    for s in (own, lent):
        init_sim(s, case)
        s.step(case.steps)
    mask = fluid_mask(case, 19)
    np.testing.assert_array_equal(lent.populations(raw=True)[mask], own.populations(raw=True)[mask])
    assert max_rel_err(lent.populations(), oracle_run(case), mask) <= TOL["f64"]
    assert not torch.equal(before, lent.buffers["pdf0"])  # the library wrote into the caller's tensor
    if pattern == "pull" and not extra:  # even step count: the state is in pdf_dev[0], canonical layout
        st = lent.buffers["pdf0"].view(torch.float64).reshape(19, 12, 16, 32).cpu().numpy()
        np.testing.assert_array_equal(st[mask], lent.populations(raw=True)[mask])
    lent.close()
    own.close()


@pytest.mark.parametrize("pattern,geometry,dtype", [("pull", "cavity", "f64"), ("aa", "periodic", "f64"),
                                                    ("esotwist", "cavity", "f64"), ("pull", "periodic", "f32")])
def test_cumulant_unit_rate_kernels_match_general(pattern, geometry, dtype, monkeypatch):
    """D3Q27 cumulant with omega_bulk = omega_3..6 = 1 (C3's rates) runs the specialised kernels
    (collide_cumulant27_unit: second moments only, Gaussian closure); they match the general kernels
    (LBM_CUMULANT_GENERAL=1) to rounding and the oracle to the north_star bar."""
    case = Case("cumu", (16, 16, 16), 27, "cumulant", (1.95,), dtype, pattern=pattern, geometry=geometry,
                ubb=(0.05, 0, 0), u_amp=0.05, steps=11)
    unit = make_sim(case)
    monkeypatch.setenv("LBM_CUMULANT_GENERAL", "1")
    general = make_sim(case)
    monkeypatch.delenv("LBM_CUMULANT_GENERAL")
    for s in (unit, general):
        init_sim(s, case)
        s.step(case.steps)
    mask = fluid_mask(case, 27)
    assert max_rel_err(unit.populations(), general.populations(), mask) <= (1e-13 if dtype == "f64" else 2e-6)
    assert max_rel_err(unit.populations(), oracle_run(case), mask) <= TOL[dtype]


# -----------------------------------------------------------------------------------------
# Face-aligned walls (FM_FACES): walls recognised from coordinates (channel / cavity flag fields)
# -----------------------------------------------------------------------------------------
FACE_CASES = [  # (default: D3Q19 fp64 pull; the others with LBM_FACES=1)
    Case("fc_trt_f64_channel_pull", (20, 18, 12), 19, "trt", (1.6, 0.5), "f64", force=(1e-5, 0, 0), geometry="channel",
         steps=21),
    Case("fc_srt_f64_cavity_pull", (14, 14, 14), 19, "srt", (1.8,), "f64", geometry="cavity", ubb=(0.05, 0, 0),
         u_amp=0.03, steps=17),
    Case("fc_trt_f32_channel_pull", (32, 18, 12), 19, "trt", (1.6, 0.5), "f32", force=(1e-5, 0, 0), geometry="channel",
         steps=21),
    Case("fc_trt_q27_cavity_aa_odd", (13, 13, 13), 27, "trt", (1.5, 1.2), "f64", pattern="aa", geometry="cavity",
         ubb=(0.03, -0.02, 0), steps=11),
    Case("fc_srt_f32_channel_aa", (32, 16, 10), 19, "srt", (1.7,), "f32", pattern="aa", geometry="channel", steps=12),
    Case("fc_gtrt_f64_cavity_pull", (14, 14, 14), 19, "gen_trt", (1.7, 1.1), "f64", geometry="cavity", ubb=(0.05, 0, 0),
         u_amp=0.03, steps=12),
]


@pytest.mark.parametrize("case", FACE_CASES, ids=lambda c: c.name)
def test_face_aligned_walls_vs_oracle_and_flag_kernels(case, monkeypatch):
    """The channel and cavity flag fields run the face-aligned kernels (boundary_impl == "faces"; chosen by
    default for D3Q19 fp64 pull, forced with LBM_FACES=1 otherwise): parity with the oracle, and the same
    update as the split flag kernels (LBM_FACES=0) to rounding."""
    default = case.Q == 19 and case.dtype == "f64" and case.pattern == "pull"
    if not default:
        monkeypatch.setenv("LBM_FACES", "1")
    sim = make_sim(case)
    assert sim.boundary_impl == "faces"
    monkeypatch.setenv("LBM_FACES", "0")
    ref = make_sim(case)
    monkeypatch.delenv("LBM_FACES")
    assert ref.boundary_impl == "split"
    for s in (sim, ref):
        init_sim(s, case)
        s.step(case.steps)
    mask = fluid_mask(case, case.Q)
    assert max_rel_err(sim.populations(), oracle_run(case), mask) <= TOL[case.dtype]
    assert max_rel_err(sim.populations(), ref.populations(), mask) <= (1e-13 if case.dtype == "f64" else 1e-6)


@pytest.mark.parametrize("extra", [{"n_local_slabs": 2}, {"n_local_slabs": 4, "halo_mode": 1}, {"nccl_self": True},
                                   {"nccl_self": True, "halo_mode": 2}])
@pytest.mark.parametrize("pattern", ["pull", "aa"])
def test_face_aligned_walls_slabs_bit_identical(extra, pattern, monkeypatch):
    """FM_FACES with a z-slab decomposition: the z walls are global faces (rank 0 bottom, rank P-1 top)."""
    monkeypatch.setenv("LBM_FACES", "1")
    case = Case("fcdec", (16, 16, 16), 19, "trt", (1.6, 0.5), "f64", pattern=pattern, geometry="cavity",
                ubb=(0.05, 0, 0), u_amp=0.03, steps=9)
    one = make_sim(case)
    many = make_sim(case, **extra)
    assert one.boundary_impl == many.boundary_impl == "faces"
    for s in (one, many):
        init_sim(s, case)
        s.step(case.steps)
    mask = fluid_mask(case, case.Q)
    np.testing.assert_array_equal(one.populations(raw=True)[mask], many.populations(raw=True)[mask])


def test_non_face_geometries_keep_flag_kernels():
    case = Case("nofc", (16, 12, 10), 19, "trt", (1.6, 0.5), "f64", geometry="obstacles", steps=1)
    assert make_sim(case).boundary_impl == "split"
    assert make_sim(Case("mrtfc", (16, 16, 16), 19, "mrt", (1.9, 1.0, 1.0, 1.0), "f64", geometry="cavity")).boundary_impl == "split"
    assert make_sim(Case("cumfc", (16, 16, 16), 27, "cumulant", (1.95,), "f64", geometry="cavity")).boundary_impl == "split"
    assert make_sim(Case("esofc", (16, 16, 16), 19, "trt", (1.6, 0.5), "f64", pattern="esotwist",
                         geometry="cavity")).boundary_impl == "split"


@pytest.mark.parametrize("pattern,geometry,dtype,Q", [("aa", "periodic", "f32", 19), ("pull", "channel", "f64", 19),
                                                      ("esotwist", "obstacles", "f64", 19), ("push", "cavity", "f32", 19)])
def test_mrt_shear_only_kernels_match_general(pattern, geometry, dtype, Q, monkeypatch):
    """Weighted MRT with omega_bulk = omega_3 = omega_4 = 1 (C2's rates) runs the shear-only kernels
    (collide_mrt_shear, the G6 closed form); they match the general group-projection kernels
    (LBM_MRT_GENERAL=1) to rounding and the oracle to the north_star bar."""
    case = Case("mrts", (16, 16, 16) if geometry == "cavity" else (32, 14, 12), Q, "mrt", (1.9, 1.0, 1.0, 1.0), dtype,
                pattern=pattern, geometry=geometry, ubb=(0.02, -0.01, 0.03), u_amp=0.03, steps=11)
    fast = make_sim(case)
    monkeypatch.setenv("LBM_MRT_GENERAL", "1")
    general = make_sim(case)
    monkeypatch.delenv("LBM_MRT_GENERAL")
    for s in (fast, general):
        init_sim(s, case)
        s.step(case.steps)
    mask = fluid_mask(case, Q)
    assert max_rel_err(fast.populations(), general.populations(), mask) <= (1e-13 if dtype == "f64" else 2e-6)
    assert max_rel_err(fast.populations(), oracle_run(case), mask) <= TOL[dtype]

