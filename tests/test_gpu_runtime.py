"""GPU tests of the runtime's auxiliary subsystems: bit-exact checkpoint / resume through the
C ABI (lbm_save_state / lbm_load_state) for every storage pattern, decomposition and halo transport, and the
phase timeline of decomposed steps (lbm_step_phases_ms; the NVTX ranges mark the same phases)."""
import numpy as np
import pytest

from tests.gpu_common import Case, fluid_mask, init_sim, make_sim

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _lib():
    from paper_2001_11806_b200 import build
    build.build()
    import torch
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"


RESUME = [
    ("pull", "channel", "flags", {}), ("pull", "cavity", "links", {}), ("aa", "obstacles", "flags", {}),
    ("aa", "channel", "links", {}), ("esotwist", "channel", "flags", {}), ("push", "obstacles", "flags", {}),
    ("pull", "channel", "flags", {"n_local_slabs": 2}), ("aa", "obstacles", "flags", {"n_local_slabs": 2, "halo_mode": 1}),
    ("esotwist", "channel", "flags", {"n_local_slabs": 4}), ("push", "periodic", "flags", {"n_local_slabs": 2}),
    ("pull", "channel", "flags", {"nccl_self": True, "halo_mode": 0}),
    ("pull", "periodic", "flags", {"nccl_self": True, "halo_mode": 2}),
    ("aa", "channel", "flags", {"nccl_self": True, "halo_mode": 2}),
    ("esotwist", "obstacles", "flags", {"nccl_self": True, "halo_mode": 1}),
]


@pytest.mark.parametrize("k", [5, 6])
@pytest.mark.parametrize("pattern,geometry,boundary_mode,extra", RESUME,
                         ids=[f"{p}-{g}-{b}-{'-'.join(f'{a}{v}' for a, v in e.items()) or 'single'}" for p, g, b, e in RESUME])
def test_resume_bit_exact(pattern, geometry, boundary_mode, extra, k):
    """n steps == k steps, save, load into a FRESH handle, n - k steps (odd and even k: both AA / EsoTwist
    parities), bit for bit on the stored state and the canonical populations."""
    shape = (16, 16, 16) if geometry == "cavity" else (16, 12, 16)
    case = Case("resume", shape, 19, "trt", (1.6, 0.5), "f64", pattern=pattern, force=(1e-5, 0, 0) if geometry != "cavity" else (0, 0, 0),
                geometry=geometry, ubb=(0.02, -0.01, 0.03), steps=13)
    kw = dict(boundary_mode=boundary_mode, **extra)
    ref = make_sim(case, **kw)
    init_sim(ref, case)
    ref.step(case.steps)
    a = make_sim(case, **kw)
    init_sim(a, case)
    a.step(k)
    state, steps = a.save_state()
    assert steps == k
    a.close()
    b = make_sim(case, **kw)
    b.load_state(state, steps)
    assert b.steps_done == k
    b.step(case.steps - k)
    mask = fluid_mask(case, 19)
    np.testing.assert_array_equal(b.populations(raw=True)[mask], ref.populations(raw=True)[mask])
    np.testing.assert_array_equal(b.populations()[mask], ref.populations()[mask])
    s2, n2 = b.save_state()
    s1, n1 = ref.save_state()
    assert n1 == n2 == case.steps


def test_resume_into_same_handle_rewinds():
    """Loading an earlier checkpoint into the running handle rewinds it (the CUDA-graph cycle is re-captured
    for the restored parity)."""
    case = Case("rewind", (32, 8, 8), 19, "srt", (1.8,), "f64", pattern="aa", steps=9)
    sim = make_sim(case, use_graph=True)
    init_sim(sim, case)
    sim.step(3)
    st, n = sim.save_state()
    sim.step(6)
    first = sim.populations(raw=True)
    sim.load_state(st, n)
    sim.step(6)
    np.testing.assert_array_equal(sim.populations(raw=True), first)


@pytest.mark.parametrize("extra", [{"n_local_slabs": 2}, {"nccl_self": True, "halo_mode": 0},
                                   {"nccl_self": True, "halo_mode": 1}, {"nccl_self": True, "halo_mode": 2}])
def test_step_phase_timeline(extra):
    """lbm_step_phases_ms: the boundary planes run first, the interior starts after them on the compute
    stream, the exchange starts after the boundary planes (NCCL: on the comm stream, concurrently with the
    interior); every interval is non-empty and well ordered."""
    case = Case("phases", (128, 128, 32), 19, "trt", (1.6, 0.5), "f64", steps=3)
    sim = make_sim(case, **extra)
    init_sim(sim, case)
    sim.step(2)
    sim.enable_kernel_timing()
    sim.step(1)
    ph = sim.step_phases_ms()
    (b0, b1), (x0, x1), (i0, i1) = ph["boundary"], ph["exchange"], ph["interior"]
    assert b0 == 0.0 and b1 > b0 and i1 > i0 and x1 >= x0
    assert i0 >= b1 - 1e-3
    if extra.get("halo_mode") != 2:  # the fused halo's gate runs before the boundary planes
        assert x0 >= b1 - 1e-3
    sim.close()


@pytest.mark.parametrize("pattern", ["pull", "aa"])
def test_async_host_io_jobs_match_synchronous(pattern):
    """LBM_HOST_ASYNC: three back-to-back jobs (init from pinned host arrays, steps, macroscopic readout to
    pinned host arrays) enqueued without host waits — uploads and downloads on their own streams, staging
    double-buffered — give bit-identical outputs to the synchronous calls, once lbm_sync returned."""
    import torch
    from paper_2001_11806_b200 import lbm as L
    import lbminputs as LI
    case = Case("aio", (32, 20, 16), 19, "trt", (1.6, 0.5), "f64", pattern=pattern, force=(1e-5, 0, 0),
                geometry="channel", steps=7)
    sim = make_sim(case)
    nx, ny, nz = case.shape
    cells = nx * ny * nz
    ins, outs, refs = [], [], []
    for seed in range(3):
        rho, u = LI.random_fields(seed, nx, ny, nz, 1e-3, 0.01)
        r_h = torch.from_numpy(rho.reshape(-1).copy()).pin_memory()
        u_h = torch.from_numpy(u.reshape(-1).copy()).pin_memory()
        ins.append((r_h, u_h))
        outs.append((torch.empty(cells, dtype=torch.float64).pin_memory(), torch.empty(3 * cells, dtype=torch.float64).pin_memory()))
        ref = make_sim(case)
        ref.init_equilibrium(rho, u)
        ref.step(case.steps + seed)
        refs.append(ref.macroscopic())
        ref.close()
    for seed in range(3):
        (r_h, u_h), (r_o, u_o) = ins[seed], outs[seed]
        assert L.lbm_init_equilibrium(sim.h, r_h.data_ptr(), u_h.data_ptr(), L.HOST_ASYNC) == 0
        assert L.lbm_step(sim.h, case.steps + seed) == 0
        assert L.lbm_get_macroscopic(sim.h, r_o.data_ptr(), u_o.data_ptr(), L.HOST_ASYNC) == 0
    sim.sync()
    for seed in range(3):
        r_o, u_o = outs[seed]
        np.testing.assert_array_equal(r_o.numpy().reshape(nz, ny, nx), refs[seed][0])
        np.testing.assert_array_equal(u_o.numpy().reshape(3, nz, ny, nx), refs[seed][1])


FLAT = [("pull", "periodic", "flags"), ("pull", "channel", "flags"), ("pull", "channel", "links"), ("aa", "periodic", "flags"),
        ("aa", "channel", "flags"), ("aa", "channel", "links"), ("aa", "obstacles", "flags"), ("esotwist", "channel", "flags"),
        ("push", "periodic", "flags")]


@pytest.mark.parametrize("dtype", ["f64", "f32"])
@pytest.mark.parametrize("nx", [44, 300])
@pytest.mark.parametrize("pattern,geometry,boundary_mode", FLAT, ids=["-".join(f) for f in FLAT])
def test_flat_rows_bit_identical_to_box_blocks(pattern, geometry, boundary_mode, nx, dtype):
    """Flat-row launch indexing (full x-rows with nx % block_x != 0: the cells of the rows are indexed linearly,
    DESIGN §6.3; the Fig. 7 / 8 domain has nx = 300) updates exactly the cells of the (bx, by)
    block launch: the stored state after an odd and an even number of steps is bit-identical to a handle with
    block_x forced (which keeps the box blocks), on the plain kernel path (test_gpu_parity runs its odd-extent
    cases, nx = 19 etc., through the flat rows by default, against the oracle). fp32 AA without flags in the
    kernel (periodic, or index lists applied by the link kernel): the box launch runs the two-cell even-step
    kernel, whose second cell is another compiled instance of the same collision (differently contracted), so
    there the canonical populations agree within that rounding (2e-6, the bound of the in-kernel links test)."""
    from tests.gpu_common import max_rel_err
    from paper_2001_11806_b200 import lbm as L
    case = Case("flat", (nx, 11, 6), 19, "trt", (1.6, 0.5), dtype, pattern=pattern, geometry=geometry,
                force=(1e-5, 0, 0) if geometry == "channel" else (0, 0, 0), steps=5)
    L.set_kernel_path("plain")
    try:
        got = []
        for kw in ({}, {"block_x": 64 if nx == 300 else 32}):
            sim = make_sim(case, boundary_mode=boundary_mode, **kw)
            init_sim(sim, case)
            out = []
            for n in (3, 2):
                sim.step(n)
                out.append((sim.populations(raw=True).copy(), sim.populations().copy()))
            got.append(out)
            sim.close()
    finally:
        L.set_kernel_path("auto")
    mask = fluid_mask(case, 19)
    two_cell_even = dtype == "f32" and pattern == "aa" and (geometry == "periodic" or boundary_mode == "links")
    for (raw_a, can_a), (raw_b, can_b) in zip(*got):
        if two_cell_even:
            assert max_rel_err(can_a, can_b, mask) <= 2e-6
        else:
            np.testing.assert_array_equal(raw_a[mask], raw_b[mask])
            np.testing.assert_array_equal(can_a[mask], can_b[mask])
