"""Oracle pins: streaming, boundaries, patterns and closed-form flows (CPU, no GPU).

* hand-checkable first step on 4^3 (SURVEY §8(c) "Streaming / BC / patterns");
* pattern identities (G11): AA(2N) = push(2N), pull from C(f0) = C(push(n));
* conservation per step (periodic: mass + momentum; walled box: mass);
* UBB(u_w = 0) == NoSlip bit-exactly; Couette exact linear profile (UBB sign, half-way wall);
* Poiseuille: exact steady parabola (TRT, Lambda = 3/16) and the start-up series at t = n - 1/2;
* shear-wave decay: nu = (1/omega - 1/2)/3 (P:507-513 relation; north_star);
* slab decomposition with pack/unpack halo exchange bit-identical to the undecomposed run.
"""
import numpy as np
import pytest

import lbminputs as LI
import oracle as O


def _rand_f0(d, seed=3, rho_amp=1e-3, u_amp=0.01):
    rho, u = LI.random_fields(seed, d.nx, d.ny, d.nz, rho_amp, u_amp)
    return d.init_equilibrium(rho, u)


# ---------------------------------------------------------------------------------------
def test_hand_checked_first_step_push_4cubed():
    """All cells f = w_q except x0 with f = w_q (1 + delta): u = 0 there, so C leaves it
    unchanged for any omega; after one push step cell x0 + c_q holds w_q (1 + delta) in slot q."""
    m = O.Method(Q=19, op="srt", rates=(1.7,))
    d = O.Domain(m, 4, 4, 4, 0)
    c, w, _ = O.stencil_arrays(19)
    delta = 0.25
    f = np.empty(d.shape)
    f[:] = w[:, None, None, None]
    x0 = (1, 2, 3)  # (x, y, z)
    f[:, x0[2], x0[1], x0[0]] *= 1 + delta
    d.step_push(f)
    for q in range(19):
        for z in range(4):
            for y in range(4):
                for x in range(4):
                    tgt = ((x0[0] + c[q, 0]) % 4, (x0[1] + c[q, 1]) % 4, (x0[2] + c[q, 2]) % 4)
                    exp = w[q] * (1 + delta) if (x, y, z) == tgt else w[q]
                    assert abs(f[q, z, y, x] - exp) < 1e-15, (q, x, y, z)
    rho, u = d.macroscopic(f)
    for q in range(1, 19):
        tgt = ((x0[0] + c[q, 0]) % 4, (x0[1] + c[q, 1]) % 4, (x0[2] + c[q, 2]) % 4)
        r = 1 + w[q] * delta
        assert abs(rho[tgt[2], tgt[1], tgt[0]] - r) < 1e-15
        np.testing.assert_allclose(u[:, tgt[2], tgt[1], tgt[0]], w[q] * delta * c[q] / r, atol=1e-16)
    assert abs(rho[x0[2], x0[1], x0[0]] - (1 + w[0] * delta)) < 1e-15


@pytest.mark.parametrize("op,Q,rates", [("srt", 19, (1.8,)), ("trt", 19, (1.6, 0.5)),
                                         ("mrt", 19, (1.9, 1.0, 1.0, 1.0)), ("cumulant", 27, (1.95,))])
def test_pattern_identities(op, Q, rates):
    """G11: AA after 2N steps equals push after 2N (same arithmetic: bit-exact); pull started
    from P(0) = C(f0) equals C(F(n))."""
    m = O.Method(Q=Q, op=op, rates=rates, nthreads=1)
    d = O.Domain(m, 5, 4, 3)
    rng = np.random.default_rng(5)
    f0 = _rand_f0(d) * (1 + 0.01 * rng.uniform(-1, 1, d.shape))  # non-equilibrium start
    n = 4
    Fn = d.run_push(f0, n)
    np.testing.assert_array_equal(d.run_aa(f0, n), Fn)
    P0 = f0.copy()
    d.collide_all(P0)
    Pn = d.run_pull(P0, n)
    CF = Fn.copy()
    d.collide_all(CF)
    np.testing.assert_array_equal(Pn, CF)


@pytest.mark.parametrize("op,Q,rates", [("trt", 19, (1.6, 0.5)), ("cumulant", 27, (1.95,)), ("identity", 27, ())])
def test_aa_with_walls_equals_push(op, Q, rates):
    """AA with NoSlip/UBB walls (odd-step slot rules) reproduces the push pattern F(2N) bit-exactly,
    and after an odd number of steps the reversed-slot layout plus the wall rule gives F(2N+1)."""
    n = 7
    fl = LI.random_obstacles(4, n, n, n, frac=0.2, ubb_frac=0.5)
    m = O.Method(Q=Q, op=op, rates=rates, ubb_u=(0.03, -0.02, 0.01), nthreads=1)
    d = O.Domain(m, n, n, n, flags=fl)
    f0 = _rand_f0(d, u_amp=0.03) * (1 + 0.01 * np.random.default_rng(9).uniform(-1, 1, d.shape))
    fluid = np.broadcast_to(fl == 0, d.shape)
    for N in (2, 4):
        np.testing.assert_array_equal(d.run_aa(f0, N)[fluid], d.run_push(f0, N)[fluid])
    a = d.run_aa(f0, 3)
    F3 = d.run_push(f0, 3)
    c, w, opp = O.stencil_arrays(Q)
    for q in range(Q):
        gathered = np.roll(a[opp[q]], shift=(c[q, 2], c[q, 1], c[q, 0]), axis=(0, 1, 2))
        nbw = np.roll(fl, shift=(c[q, 2], c[q, 1], c[q, 0]), axis=(0, 1, 2))  # flag of x - c_q
        cu = c[q] @ np.array(m.ubb_u)
        bounced = a[q] + np.where(nbw == LI.UBB, 6.0 * w[q] * 1.0 * cu, 0.0)
        can = np.where(nbw == 0, gathered, bounced)
        np.testing.assert_array_equal(can[fl == 0], F3[q][fl == 0])


@pytest.mark.parametrize("op,Q,rates", [("identity", 19, ()), ("srt", 19, (1.8,)), ("trt", 27, (1.6, 0.5)),
                                         ("mrt", 19, (1.9, 1.3, 1.1, 0.8)), ("cumulant", 27, (1.95, 1.1))])
@pytest.mark.parametrize("walls", [False, True])
def test_esotwist_equals_push(op, Q, rates, walls):
    """EsoTwist reproduces the push pattern F(n) bit-exactly for even and odd n, with and
    without NoSlip/UBB walls; the canonical state is gathered here with np.roll (independent of the
    oracle's layout routine): F_q(x) = a(x - c_q^+)(q) after even n, a(x - c_q^+)(qbar) after odd n."""
    n = 7
    fl = LI.random_obstacles(5, n, n, n, frac=0.2, ubb_frac=0.5) if walls else None
    m = O.Method(Q=Q, op=op, rates=rates, ubb_u=(0.03, -0.02, 0.01), nthreads=1)
    d = O.Domain(m, n, n, n, flags=fl)
    f0 = _rand_f0(d, u_amp=0.03) * (1 + 0.01 * np.random.default_rng(9).uniform(-1, 1, d.shape))
    fluid = np.ones((n, n, n), bool) if fl is None else fl == 0
    c, _, opp = O.stencil_arrays(Q)
    cp = np.maximum(c, 0)
    for N in (1, 2, 5, 6):
        a = d.run_eso(f0, N)
        F = d.run_push(f0, N)
        for q in range(Q):
            slot = opp[q] if N % 2 else q
            can = np.roll(a[slot], shift=(cp[q, 2], cp[q, 1], cp[q, 0]), axis=(0, 1, 2))
            np.testing.assert_array_equal(can[fluid], F[q][fluid])
        np.testing.assert_array_equal(d.eso_to_canonical(a, N % 2)[:, fluid], F[:, fluid])


def test_aa_odd_parity_layout():
    """After an odd number of AA steps the array holds C(F(n-1)) with reversed slots:
    F(n)_q(y) = a[y - c_q](qbar)."""
    m = O.Method(Q=19, op="trt", rates=(1.6, 0.5), nthreads=1)
    d = O.Domain(m, 4, 5, 3)
    f0 = _rand_f0(d)
    a = d.run_aa(f0, 3)
    F3 = d.run_push(f0, 3)
    c, _, opp = O.stencil_arrays(19)
    for q in range(19):
        shifted = np.roll(a[opp[q]], shift=(c[q, 2], c[q, 1], c[q, 0]), axis=(0, 1, 2))
        np.testing.assert_array_equal(shifted, F3[q])


@pytest.mark.parametrize("op,Q,rates", [("srt", 19, (1.8,)), ("trt", 27, (1.6, 0.5)),
                                         ("mrt", 19, (1.9, 1.3, 1.1, 0.8)), ("cumulant", 27, (1.95, 1.1))])
def test_conservation_periodic(op, Q, rates):
    m = O.Method(Q=Q, op=op, rates=rates, nthreads=1)
    d = O.Domain(m, 6, 5, 4)
    c, _, _ = O.stencil_arrays(Q)
    f = _rand_f0(d, u_amp=0.03)
    f *= 1 + 0.01 * np.random.default_rng(2).uniform(-1, 1, f.shape)
    mass0 = np.sum(f)
    mom0 = np.einsum("qa,qzyx->a", c, f)
    g = f.copy()
    for _ in range(3):
        d.step_pull(f, g)
        f, g = g, f
        assert abs(np.sum(f) / mass0 - 1) < 1e-13
        np.testing.assert_allclose(np.einsum("qa,qzyx->a", c, f), mom0, atol=1e-13 * mass0)


def test_mass_conservation_walled_box():
    n = 8
    m = O.Method(Q=19, op="trt", rates=(1.6, 0.5), nthreads=1)
    fl = LI.cavity_flags(n)
    fl[fl == LI.UBB] = LI.NOSLIP
    d = O.Domain(m, n, n, n, flags=fl)
    f = _rand_f0(d, u_amp=0.05)
    fluid = fl == 0
    mass0 = f[:, fluid].sum()
    g = f.copy()
    for _ in range(20):
        d.step_pull(f, g)
        f, g = g, f
    assert abs(f[:, fluid].sum() / mass0 - 1) < 1e-13


def test_ubb_zero_velocity_equals_noslip():
    n = 6
    fl = LI.cavity_flags(n)
    f0 = None
    outs = []
    for ubb_as_noslip in (False, True):
        flags = fl.copy()
        if ubb_as_noslip:
            flags[flags == LI.UBB] = LI.NOSLIP
        m = O.Method(Q=27, op="trt", rates=(1.6, 0.5), ubb_u=(0.0, 0.0, 0.0), nthreads=1)
        d = O.Domain(m, n, n, n, flags=flags)
        if f0 is None:
            f0 = _rand_f0(d, u_amp=0.05)
        outs.append(d.run_pull(f0, 3))
    np.testing.assert_array_equal(outs[0], outs[1])


@pytest.mark.parametrize("omega,tol,steps", [(1.0, 1e-12, 6000), (1.8, 1e-11, 60000)])
def test_couette_ubb_exact_linear_profile(omega, tol, steps):
    """NoSlip at y = 0, UBB u_w = (0.05, 0, 0) at y = H+1: the steady profile is exactly linear,
    u_x = u_w (y - 1/2) / H (half-way walls), which fixes the sign and placement of the UBB term."""
    H = 16
    uw = 0.05
    fl = LI.couette_flags(1, H, 1)
    m = O.Method(Q=19, op="srt", rates=(omega,), ubb_u=(uw, 0, 0), nthreads=1)
    d = O.Domain(m, 1, H + 2, 1, flags=fl)
    f0 = d.init_equilibrium(np.ones((1, H + 2, 1)), np.zeros((3, 1, H + 2, 1)))
    f = d.run_pull(f0, steps)
    rho, u = d.macroscopic(f, post_collision=True)
    y = np.arange(1, H + 1)
    np.testing.assert_allclose(u[0, 0, 1:H + 1, 0], uw * (y - 0.5) / H, rtol=0, atol=tol)


def test_poiseuille_steady_exact_parabola_trt_magic():
    """TRT with Lambda = (1/we - 1/2)(1/wo - 1/2) = 3/16 (we = 1.6, wo = 0.5, G14) and Guo
    forcing gives the exact parabola u = F/(2 nu) (y - 1/2)(H + 1/2 - y)."""
    H, F = 10, 1e-6
    we, wo = 1.6, 0.5
    nu = (1 / we - 0.5) / 3
    m = O.Method(Q=19, op="trt", rates=(we, wo), force=(F, 0, 0), nthreads=1)
    d = O.Domain(m, 1, H + 2, 1, flags=LI.channel_flags(1, H + 2, 1))
    f0 = d.init_equilibrium(np.ones((1, H + 2, 1)), np.zeros((3, 1, H + 2, 1)))
    f = d.run_pull(f0, 20000)
    _, u = d.macroscopic(f, post_collision=True)
    y = np.arange(1, H + 1)
    exact = F / (2 * nu) * (y - 0.5) * (H + 0.5 - y)
    assert np.abs(u[0, 0, 1:H + 1, 0] - exact).max() / exact.max() < 1e-10


def test_poiseuille_transient_series_config1_shape():
    """Config 1 channel (H = 254) after n = 2000 pull steps from P(0) = f_eq(1, 0), compared with
    the start-up series at t = n - 1/2 (G11): error / max <= 2.5e-4."""
    Ny, F, n = 256, 1e-6, 2000
    H = Ny - 2
    we, wo = 1.6, 0.5
    nu = (1 / we - 0.5) / 3
    m = O.Method(Q=19, op="trt", rates=(we, wo), force=(F, 0, 0), nthreads=1)
    d = O.Domain(m, 1, Ny, 1, flags=LI.channel_flags(1, Ny, 1))
    f0 = d.init_equilibrium(np.ones((1, Ny, 1)), np.zeros((3, 1, Ny, 1)))
    f = d.run_pull(f0, n)
    _, u = d.macroscopic(f, post_collision=True)
    y = np.arange(1, H + 1)
    eta = (y - 0.5) / H
    t = n - 0.5
    us = F * H ** 2 / (2 * nu) * eta * (1 - eta)
    series = us.copy()
    for k in range(1, 2000, 2):
        series -= 4 * F * H ** 2 / (nu * k ** 3 * np.pi ** 3) * np.sin(k * np.pi * eta) * np.exp(-k * k * np.pi ** 2 * nu * t / H ** 2)
    err = np.abs(u[0, 0, 1:H + 1, 0] - series).max() / series.max()
    assert err < 2.5e-4
    # a half-step bookkeeping error (t = n + 1/2) is caught
    t2 = n + 0.5
    s2 = us.copy()
    for k in range(1, 2000, 2):
        s2 -= 4 * F * H ** 2 / (nu * k ** 3 * np.pi ** 3) * np.sin(k * np.pi * eta) * np.exp(-k * k * np.pi ** 2 * nu * t2 / H ** 2)
    assert np.abs(u[0, 0, 1:H + 1, 0] - s2).max() / s2.max() > 2.5e-4


def test_momentum_gain_per_step_periodic():
    F = np.array([1e-5, 0, -2e-5])
    m = O.Method(Q=19, op="trt", rates=(1.6, 0.5), force=F, nthreads=1)
    d = O.Domain(m, 4, 4, 4)
    c, _, _ = O.stencil_arrays(19)
    f = _rand_f0(d)
    g = f.copy()
    p0 = np.einsum("qa,qzyx->a", c, f)
    for k in range(1, 4):
        d.step_pull(f, g)
        f, g = g, f
        np.testing.assert_allclose(np.einsum("qa,qzyx->a", c, f) - p0, k * 64 * F, rtol=1e-9, atol=1e-14)


@pytest.mark.parametrize("op,rates", [("srt", (1.8,)), ("mrt", (1.9, 1.0, 1.0, 1.0))])
def test_shear_wave_viscosity(op, rates):
    """u_x = A sin(2 pi z / L) decays as exp(-nu k^2 t) with nu = (1/omega - 1/2)/3, omega the
    shear rate. Fitted between two late times on a quasi-1D L = 256 lattice; gate 1e-3 (SURVEY §8(c)
    "Viscosity": <= 1e-3 at L >= 256; measured ~5e-5)."""
    L, A = 256, 1e-3
    m = O.Method(Q=19, op=op, rates=rates, nthreads=1)
    d = O.Domain(m, 1, 1, L)
    z = np.arange(L)
    u = np.zeros((3, L, 1, 1))
    u[0, :, 0, 0] = A * np.sin(2 * np.pi * z / L)
    f = d.init_equilibrium(np.ones((L, 1, 1)), u)
    g = f.copy()
    amps = {}
    for t in range(1, 1201):
        d.step_pull(f, g)
        f, g = g, f
        if t in (200, 1200):
            _, uu = d.macroscopic(f, post_collision=True)
            amps[t] = 2 * np.mean(uu[0, :, 0, 0] * np.sin(2 * np.pi * z / L))
    k = 2 * np.pi / L
    nu_fit = np.log(amps[200] / amps[1200]) / (k * k * 1000)
    nu = (1 / rates[0] - 0.5) / 3
    assert abs(nu_fit / nu - 1) < 1e-3


def test_slab_decomposition_bit_identical():
    """O7 / §8(e): P z-slabs with one ghost plane per side, crossing populations packed in
    canonical order and unpacked into the neighbour's ghost plane, reproduce the undecomposed
    pull run bit-for-bit (channel with walls, TRT + force)."""
    nx, ny, nz, P, steps = 5, 6, 8, 4, 3
    fl = LI.channel_flags(nx, ny, nz)
    m = O.Method(Q=19, op="trt", rates=(1.6, 0.5), force=(1e-4, 0, 0), nthreads=1)
    full = O.Domain(m, nx, ny, nz, flags=fl)
    f0 = _rand_f0(full)
    ref = full.run_pull(f0, steps)
    nzl = nz // P
    slabs = []
    for r in range(P):
        z0 = r * nzl
        zg = [(z0 + k) % nz for k in range(-1, nzl + 1)]
        d = O.Domain(m, nx, ny, nzl, zghost=1, flags=fl[zg])
        a = np.ascontiguousarray(f0[:, zg])
        slabs.append([d, a, a.copy()])
    for _ in range(steps):
        for d, a, b in slabs:
            d.step_pull(a, b)
        for r, (d, a, b) in enumerate(slabs):  # exchange on the freshly written arrays (b)
            up = slabs[(r + 1) % P]
            dn = slabs[(r - 1) % P]
            up[0].unpack_face(up[2], -1, +1, d.pack_face(b, nzl - 1, +1))
            dn[0].unpack_face(dn[2], nzl, -1, d.pack_face(b, 0, -1))
        for s in slabs:
            s[1], s[2] = s[2], s[1]
    got = np.concatenate([a[:, 1:-1] for _, a, _ in slabs], axis=1)
    fluid = np.broadcast_to(fl == 0, ref.shape)
    np.testing.assert_array_equal(got[fluid], ref[fluid])


@pytest.mark.parametrize("omega,tol,steps", [(1.0, 2e-12, 6000), (1.8, 1e-11, 60000)])
def test_couette_two_moving_walls_wall_velocity_field(omega, tol, steps):
    """Per-link wall data: both walls UBB, bottom u1 = (0.02, 0, 0), top u2 = (-0.03, 0, 0),
    given as a per-cell wall-velocity field. The steady profile is exactly linear between the half-way
    walls, u_x = u1 + (u2 - u1) (y - 1/2) / H; a uniform field equals the global ubb_u bit-exactly."""
    H, u1, u2 = 16, 0.02, -0.03
    fl = np.zeros((1, H + 2, 1), np.uint8)
    fl[:, 0, :] = LI.UBB
    fl[:, H + 1, :] = LI.UBB
    wall = np.zeros((3, 1, H + 2, 1))
    wall[0, :, 0, :] = u1
    wall[0, :, H + 1, :] = u2
    m = O.Method(Q=19, op="srt", rates=(omega,), nthreads=1)
    d = O.Domain(m, 1, H + 2, 1, flags=fl, wall_u=wall)
    f0 = d.init_equilibrium(np.ones((1, H + 2, 1)), np.zeros((3, 1, H + 2, 1)))
    f = d.run_pull(f0, steps)
    _, u = d.macroscopic(f, post_collision=True)
    y = np.arange(1, H + 1)
    np.testing.assert_allclose(u[0, 0, 1:H + 1, 0], u1 + (u2 - u1) * (y - 0.5) / H, rtol=0, atol=tol)
    # uniform field == global velocity
    uw = (0.05, -0.01, 0.02)
    fl2 = LI.couette_flags(3, H, 2)
    wall2 = np.broadcast_to(np.array(uw)[:, None, None, None], (3,) + fl2.shape).copy()
    a = O.Domain(O.Method(Q=19, op="trt", rates=(1.6, 0.5), ubb_u=uw, nthreads=1), 3, H + 2, 2, flags=fl2)
    b = O.Domain(O.Method(Q=19, op="trt", rates=(1.6, 0.5), nthreads=1), 3, H + 2, 2, flags=fl2, wall_u=wall2)
    g0 = a.init_equilibrium(np.ones((2, H + 2, 3)), np.zeros((3, 2, H + 2, 3)))
    np.testing.assert_array_equal(a.run_pull(g0, 7), b.run_pull(g0, 7))
    np.testing.assert_array_equal(a.run_aa(g0, 7), b.run_aa(g0, 7))
