// collide.cuh — register-resident collision operators for the fused kernels.
//
// All operators act on ZERO-CENTRED populations g_q = f_q - w_q (G12) held in registers, so
// the O(1) lattice weights never enter the arithmetic: drho = sum g, j = sum c g,
// g_eq,q = w_q drho + w_q rho (3 c.u + 9/2 (c.u)^2 - 3/2 u.u)   (Eq. 3 minus w_q).
// Because w_q = w_qbar the centring commutes with bounce-back and AA slot swaps.
//
// SRT  Eq. (1), P:263-267 — run as TRT with omega_e = omega_o = omega (exact special case).
// TRT  P:422-460 — symmetric/antisymmetric pair split, Guo source split by parity (G4).
// MRT  Eq. (4), P:294-300 — weighted-orthogonal D3Q19 moments; relaxed per group
//      (shear / bulk / order 3 / order 4). This file uses its own
//      orthogonal basis of each group's span (hand-derived): the
//      result depends only on the spans when rates are assigned per group (G6).
// CUM  P:391-415 — D3Q27 cumulants via the per-axis central-moment ("chimera") transform and
//      the explicit mean-zero moment<->cumulant relations (Faa di Bruno), G7 rates.
#pragma once
#include "stencil.cuh"

namespace lbm {

// Operator template parameter: low 4 bits = collision (enum Op below), bits 4-5 = equilibrium
// variant (EQ_*): Eq. (3) compressible (rho0 = rho), incompressible (rho0 = 1), or the
// moment-matched D3Q19 equilibrium (identical to Eq. (3) for D3Q27).
enum EqKind { EQ_COMPRESSIBLE = 0, EQ_INCOMPRESSIBLE = 1, EQ_MOMENT_MATCHED = 2 };
__host__ __device__ constexpr int op_base(int op) { return op & 15; }
__host__ __device__ constexpr int op_eq(int op) { return op >> 4; }
__host__ __device__ constexpr int op_with_eq(int op, int eq) { return op | (eq << 4); }

// Moment-matched correction of the symmetric equilibrium part of direction q (D3Q19; zero for
// D3Q27): the 2nd-order-truncated Maxwellian x^2 y^2 moment exceeds Eq. (3)'s by rho u_z^2 / 6
// (and cyclically); the correction that fixes the three order-4 moments and leaves orders 0-3
// unchanged puts rho u_k^2 / 24 on each edge in the plane normal to axis k, -rho (u^2 - u_k^2) / 12
// on the two faces along axis k and rho u^2 / 6 on the centre (derivation; pinned by the
// oracle's M^-1 route in tests/test_bruteforce.py).
template <int Q, typename T>
__device__ __forceinline__ T mm_delta(int q, T rho, T ux, T uy, T uz) {
    if (Q != 19) return T(0);
    const int cx = kC27[q][0], cy = kC27[q][1], cz = kC27[q][2];
    const int n = cx * cx + cy * cy + cz * cz;
    const T r24 = rho * T(1.0 / 24.0);
    if (n == 2) return r24 * (cx == 0 ? ux * ux : cy == 0 ? uy * uy : uz * uz);
    if (n == 1) return T(-2) * r24 * (cx != 0 ? uy * uy + uz * uz : cy != 0 ? ux * ux + uz * uz : ux * ux + uy * uy);
    return T(4) * r24 * (ux * ux + uy * uy + uz * uz);
}

// Reciprocal for weights (the KBC entropic scalar product): fp64 = hardware approximation
// (rcp.approx.ftz.f64, ~20 bits) refined by two Newton steps (~1 ulp, no division slow path);
// fp32 = IEEE division.
__device__ __forceinline__ double fast_rcp(double x) {
    double r;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
    r = r * (2.0 - x * r);
    r = r * (2.0 - x * r);
    return r;
}
__device__ __forceinline__ float fast_rcp(float x) { return 1.0f / x; }

template <typename T>
struct Rates {
    T r[16];
    T F[3];
};

// ---------------------------------------------------------------------------------------
// Macroscopic values from centred populations. Pre-collision (pull-gathered) state.
// ---------------------------------------------------------------------------------------
template <int Q, typename T>
__device__ __forceinline__ void moments0(const T (&g)[Q], T &drho, T &jx, T &jy, T &jz) {
    using S = Stencil<Q>;
    drho = T(0);
    jx = T(0);
    jy = T(0);
    jz = T(0);
#pragma unroll
    for (int q = 0; q < Q; ++q) {
        drho += g[q];
        if (S::cx(q) > 0) jx += g[q];
        if (S::cx(q) < 0) jx -= g[q];
        if (S::cy(q) > 0) jy += g[q];
        if (S::cy(q) < 0) jy -= g[q];
        if (S::cz(q) > 0) jz += g[q];
        if (S::cz(q) < 0) jz -= g[q];
    }
}

// The same moments as balanced-tree sums (depth log2 Q instead of a Q-long chain of dependent adds): for the
// latency-bound fp64 operators (KBC, cumulant) the dependent-add chains of the sequential sums sit on the
// critical path of every cell. Different rounding order than moments0 (both are Eq. (2) exactly up to
// rounding; G16).
__host__ __device__ constexpr int dir_set_n(int Q, int axis, int sign) {
    int n = 0;
    for (int q = 0; q < Q; ++q)
        if (axis < 0 || kC27[q][axis] == sign) ++n;
    return n;
}
__host__ __device__ constexpr int dir_set_idx(int Q, int axis, int sign, int k) {
    for (int q = 0; q < Q; ++q)
        if (axis < 0 || kC27[q][axis] == sign) {
            if (k == 0) return q;
            --k;
        }
    return 0;
}
template <int Q, int AX, int SG, int LO, int HI, typename T>
__device__ __forceinline__ T tree_sum_dirs(const T (&g)[Q]) {
    if constexpr (HI - LO == 1) {
        return g[dir_set_idx(Q, AX, SG, LO)];
    } else {
        constexpr int M = (LO + HI) / 2;
        return tree_sum_dirs<Q, AX, SG, LO, M, T>(g) + tree_sum_dirs<Q, AX, SG, M, HI, T>(g);
    }
}
template <int Q, typename T>
__device__ __forceinline__ void moments0_tree(const T (&g)[Q], T &drho, T &jx, T &jy, T &jz) {
    drho = tree_sum_dirs<Q, -1, 0, 0, Q, T>(g);
    jx = tree_sum_dirs<Q, 0, 1, 0, dir_set_n(Q, 0, 1), T>(g) - tree_sum_dirs<Q, 0, -1, 0, dir_set_n(Q, 0, -1), T>(g);
    jy = tree_sum_dirs<Q, 1, 1, 0, dir_set_n(Q, 1, 1), T>(g) - tree_sum_dirs<Q, 1, -1, 0, dir_set_n(Q, 1, -1), T>(g);
    jz = tree_sum_dirs<Q, 2, 1, 0, dir_set_n(Q, 2, 1), T>(g) - tree_sum_dirs<Q, 2, -1, 0, dir_set_n(Q, 2, -1), T>(g);
}

// ---------------------------------------------------------------------------------------
// TRT (+ Guo). SRT passes we == wo.
// ---------------------------------------------------------------------------------------
template <int Q, typename T, bool FORCE, int EQ = EQ_COMPRESSIBLE>
__device__ __forceinline__ void collide_trt(T (&g)[Q], const Rates<T> &p) {
    using S = Stencil<Q>;
    const T we = p.r[0], wo = p.r[1];
    T drho, jx, jy, jz;
    moments0<Q, T>(g, drho, jx, jy, jz);
    const T rho = T(1) + drho;
    const T rho0 = EQ == EQ_INCOMPRESSIBLE ? T(1) : rho;  // reference density of Eq. (2)/(3)
    const T inv = EQ == EQ_INCOMPRESSIBLE ? T(1) : T(1) / rho;
    T ux, uy, uz;
    if (FORCE) {
        ux = (jx + T(0.5) * p.F[0]) * inv;
        uy = (jy + T(0.5) * p.F[1]) * inv;
        uz = (jz + T(0.5) * p.F[2]) * inv;
    } else {
        ux = jx * inv;
        uy = jy * inv;
        uz = jz * inv;
    }
    const T uu15 = T(1.5) * (ux * ux + uy * uy + uz * uz);
    const T se = T(1) - T(0.5) * we, so = T(1) - T(0.5) * wo;
    T uF3 = T(0);
    if (FORCE) uF3 = T(3) * (ux * p.F[0] + uy * p.F[1] + uz * p.F[2]);
    {  // centre
        const T w0 = T(S::w(0));
        T eq = w0 * drho - w0 * rho0 * uu15;
        if (EQ == EQ_MOMENT_MATCHED) eq += mm_delta<Q, T>(0, rho, ux, uy, uz);
        g[0] = g[0] - we * (g[0] - eq);
        if (FORCE) g[0] -= se * w0 * uF3;
    }
#pragma unroll
    for (int q = 1; q < Q; ++q) {
        constexpr int dummy = 0;
        (void)dummy;
        if (q < S::opp(q)) {
            const int b = S::opp(q);
            const T w = T(S::w(q));
            const T cu = T(S::cx(q)) * ux + T(S::cy(q)) * uy + T(S::cz(q)) * uz;
            const T wr = w * rho0;
            T eqs = w * drho + wr * (T(4.5) * cu * cu - uu15);
            if (EQ == EQ_MOMENT_MATCHED) eqs += mm_delta<Q, T>(q, rho, ux, uy, uz);
            const T eqa = wr * T(3) * cu;
            const T fp = T(0.5) * (g[q] + g[b]);
            const T fm = T(0.5) * (g[q] - g[b]);
            const T ds = we * (fp - eqs);
            const T da = wo * (fm - eqa);
            T gq = g[q] - ds - da;
            T gb = g[b] - ds + da;
            if (FORCE) {
                const T cF = T(S::cx(q)) * p.F[0] + T(S::cy(q)) * p.F[1] + T(S::cz(q)) * p.F[2];
                const T sa = so * w * T(3) * cF;
                const T ss = se * w * (T(9) * cu * cF - uF3);
                gq += ss + sa;
                gb += ss - sa;
            }
            g[q] = gq;
            g[b] = gb;
        }
    }
}

// ---------------------------------------------------------------------------------------
// Weighted-orthogonal MRT, D3Q19. Basis per rate group (integer-valued polynomials, their
// weighted norms N_k = sum_q w_q P_k(c_q)^2):
//   shear : xy, xz, yz (1/9 each), 2x^2-y^2-z^2 (4/3), y^2-z^2 (4/9)
//   bulk  : c^2 - 1 (2/3)
//   order3: 3(y^2+z^2)x - 2x (2/3), (y^2-z^2)x (2/9), and the y, z analogues
//   order4: 6(x^2y^2+x^2z^2+y^2z^2) - 3c^2 + 1 (2), (2x^2-1)(y^2-z^2) (4/9),
//           2(x^2y^2+x^2z^2-2y^2z^2) - (2x^2-y^2-z^2) (4/3)
// Together with 1, x, y, z they are a complete weighted-orthogonal basis of R^19, so
// f* = f - sum_k omega_k w P_k <P_k, f - f_eq> / N_k is Eq. (4) with per-group rates.
// ---------------------------------------------------------------------------------------
__host__ __device__ constexpr int mrt_poly(int k, int x, int y, int z) {
    const int xx = x * x, yy = y * y, zz = z * z, cc = xx + yy + zz;
    switch (k) {
        case 0: return x * y;
        case 1: return x * z;
        case 2: return y * z;
        case 3: return 2 * xx - yy - zz;
        case 4: return yy - zz;
        case 5: return cc - 1;
        case 6: return 3 * (yy + zz) * x - 2 * x;
        case 7: return (yy - zz) * x;
        case 8: return 3 * (xx + zz) * y - 2 * y;
        case 9: return (xx - zz) * y;
        case 10: return 3 * (xx + yy) * z - 2 * z;
        case 11: return (xx - yy) * z;
        case 12: return 6 * (xx * yy + xx * zz + yy * zz) - 3 * cc + 1;
        case 13: return (2 * xx - 1) * (yy - zz);
        default: return 2 * (xx * yy + xx * zz - 2 * yy * zz) - (2 * xx - yy - zz);
    }
}
__host__ __device__ constexpr double mrt_inv_norm(int k) {
    return k <= 2 ? 9.0 : k == 3 ? 0.75 : k == 4 ? 2.25 : k == 5 ? 1.5
         : (k >= 6 && k <= 11) ? ((k % 2 == 0) ? 1.5 : 4.5)
         : k == 12 ? 0.5 : k == 13 ? 2.25 : 0.75;
}
__host__ __device__ constexpr int mrt_group(int k) { return k <= 4 ? 0 : k == 5 ? 1 : k <= 11 ? 2 : 3; }
// index of polynomial k inside its group (0..5)
__host__ __device__ constexpr int mrt_slot(int k) { return k <= 4 ? k : k == 5 ? 0 : k <= 11 ? k - 6 : k - 12; }

// Eq. (4) with per-group rates, written as f* = f_eq + sum_g (1 - omega_g) P_g (f - f_eq): the
// projectors of the four non-conserved groups plus the conserved one sum to the identity and
// d = f - f_eq has no conserved part, so f - sum_g omega_g P_g d = f_eq + sum_g (1 - omega_g) P_g d.
// A group relaxed with omega_g = 1 contributes nothing and is skipped by a uniform branch — the
// run-time counterpart of the paper's pre-evaluation of constant relaxation rates.
template <typename T, int EQ = EQ_COMPRESSIBLE>
__device__ __forceinline__ void collide_mrt19(T (&g)[19], const Rates<T> &p) {
    using S = Stencil<19>;
    T drho, jx, jy, jz;
    moments0<19, T>(g, drho, jx, jy, jz);
    const T rho = T(1) + drho;
    const T rho0 = EQ == EQ_INCOMPRESSIBLE ? T(1) : rho;
    const T inv = EQ == EQ_INCOMPRESSIBLE ? T(1) : T(1) / rho;
    const T ux = jx * inv, uy = jy * inv, uz = jz * inv;
    const T uu15 = T(1.5) * (ux * ux + uy * uy + uz * uz);
    // Non-equilibrium part d = g - g_eq, split over the direction pairs (q, qbar): even moment
    // polynomials (shear, bulk, order 4) see only dp = d_q + d_qbar, odd ones (order 3) only
    // dm = d_q - d_qbar — half the work of the plain 15 x 19 transform. g is overwritten with g_eq.
    const T w0 = T(S::w(0));
    T eq0 = w0 * drho - w0 * rho0 * uu15;
    if (EQ == EQ_MOMENT_MATCHED) eq0 += mm_delta<19, T>(0, rho, ux, uy, uz);
    const T d0 = g[0] - eq0;
    g[0] -= d0;
    T dp[19], dm[19];
#pragma unroll
    for (int q = 1; q < 19; ++q) {
        if (q < S::opp(q)) {
            const int b = S::opp(q);
            const T w = T(S::w(q));
            const T cu = T(S::cx(q)) * ux + T(S::cy(q)) * uy + T(S::cz(q)) * uz;
            const T wr = w * rho0;
            T eqs = w * drho + wr * (T(4.5) * cu * cu - uu15);
            if (EQ == EQ_MOMENT_MATCHED) eqs += mm_delta<19, T>(q, rho, ux, uy, uz);
            const T eqa = wr * T(3) * cu;
            dp[q] = (g[q] + g[b]) - T(2) * eqs;
            dm[q] = (g[q] - g[b]) - T(2) * eqa;
            g[q] = eqs + eqa;
            g[b] = eqs - eqa;
        }
    }
#pragma unroll
    for (int grp = 0; grp < 4; ++grp) {
        const T keep = T(1) - p.r[grp];
        if (keep == T(0)) continue;  // uniform: omega_g = 1 relaxes the group to equilibrium
        const bool odd = grp == 2;
        T a[6];
#pragma unroll
        for (int k = 0; k < 15; ++k) {
            if (mrt_group(k) != grp) continue;
            T m = T(0);
            if (!odd) {
                const int c0 = mrt_poly(k, 0, 0, 0);
                if (c0 != 0) m = T(c0) * d0;
            }
#pragma unroll
            for (int q = 1; q < 19; ++q) {
                if (q < S::opp(q)) {
                    const int c = mrt_poly(k, S::cx(q), S::cy(q), S::cz(q));
                    const T v = odd ? dm[q] : dp[q];
                    if (c == 1) m += v;
                    else if (c == -1) m -= v;
                    else if (c != 0) m += T(c) * v;
                }
            }
            a[mrt_slot(k)] = keep * T(mrt_inv_norm(k)) * m;
        }
        if (!odd) {
            T s = T(0);
#pragma unroll
            for (int k = 0; k < 15; ++k) {
                if (mrt_group(k) != grp) continue;
                const int c = mrt_poly(k, 0, 0, 0);
                if (c != 0) s += T(c) * a[mrt_slot(k)];
            }
            g[0] += w0 * s;
        }
#pragma unroll
        for (int q = 1; q < 19; ++q) {
            if (q < S::opp(q)) {
                const int b = S::opp(q);
                T acc = T(0);
#pragma unroll
                for (int k = 0; k < 15; ++k) {
                    if (mrt_group(k) != grp) continue;
                    const int c = mrt_poly(k, S::cx(q), S::cy(q), S::cz(q));
                    if (c == 1) acc += a[mrt_slot(k)];
                    else if (c == -1) acc -= a[mrt_slot(k)];
                    else if (c != 0) acc += T(c) * a[mrt_slot(k)];
                }
                const T w = T(S::w(q));
                g[q] += w * acc;
                g[b] += odd ? -w * acc : w * acc;
            }
        }
    }
}

// ---------------------------------------------------------------------------------------
// MRT with one relaxation rate per moment ("a relaxation rate separately for each of the
// previously selected moments"), D3Q19. Here the rows themselves matter (G6), so the basis is the
// paper's: the weighted Gram-Schmidt of the monomial sequence sorted by order, then
// lexicographically with the highest power of x first, the second-order moments split into shear
// and bulk parts with shear first:
//   1 | x y z | x^2-y^2, xy, xz, y^2-z^2, yz, x^2+y^2+z^2 | x^2y x^2z xy^2 xz^2 y^2z yz^2 | x^2y^2 x^2z^2 y^2z^2
// (the 8 monomials with every exponent >= 1 have zero rows on D3Q19 and are dropped).
// The orthogonalisation runs at compile time on the value vectors P(c_q); rows are used only through
// the projector w P <P, .> / <P, P>_w, so their normalisation is irrelevant. rates r[0..14] belong to
// the 15 non-conserved rows in this order.
// ---------------------------------------------------------------------------------------
__host__ __device__ constexpr int mrt_input19(int r, int x, int y, int z) {
    const int xx = x * x, yy = y * y, zz = z * z;
    switch (r) {
        case 0: return 1;
        case 1: return x;
        case 2: return y;
        case 3: return z;
        case 4: return xx - yy;
        case 5: return x * y;
        case 6: return x * z;
        case 7: return yy - zz;
        case 8: return y * z;
        case 9: return xx + yy + zz;
        case 10: return xx * y;
        case 11: return xx * z;
        case 12: return x * yy;
        case 13: return x * zz;
        case 14: return yy * z;
        case 15: return y * zz;
        case 16: return xx * yy;
        case 17: return xx * zz;
        default: return yy * zz;
    }
}

struct MrtRows19 {
    double v[19][19];     // v[k][q] = P_k(c_q), rows 0..3 conserved
    double inv_norm[19];  // 1 / sum_q w_q P_k(c_q)^2
};

__host__ __device__ constexpr MrtRows19 make_mrt_rows19() {
    MrtRows19 b{};
    for (int k = 0; k < 19; ++k) {
        for (int q = 0; q < 19; ++q) b.v[k][q] = mrt_input19(k, kC27[q][0], kC27[q][1], kC27[q][2]);
        for (int j = 0; j < k; ++j) {  // classical Gram-Schmidt, weighted inner product
            double num = 0.0, den = 0.0;
            for (int q = 0; q < 19; ++q) {
                const double w = Stencil<19>::w(q);
                num += w * mrt_input19(k, kC27[q][0], kC27[q][1], kC27[q][2]) * b.v[j][q];
                den += w * b.v[j][q] * b.v[j][q];
            }
            for (int q = 0; q < 19; ++q) b.v[k][q] -= num / den * b.v[j][q];
        }
        double nn = 0.0;
        for (int q = 0; q < 19; ++q) nn += Stencil<19>::w(q) * b.v[k][q] * b.v[k][q];
        b.inv_norm[k] = 1.0 / nn;
    }
    return b;
}
// The rows live in __constant__ memory of k_mrt_rows.cu (filled once from make_mrt_rows19() on the host);
// the unrolled loops read them as constant-bank operands. Defined only in that translation unit.
template <typename T>
__device__ void collide_mrt19_rows(T (&g)[19], const Rates<T> &p);

// ---------------------------------------------------------------------------------------
// Smagorinsky SRT (Eqs. 11-14), rates = [omega_0, C_S]. The local omega solves
// Eq. (14) with |S| of Eq. (12): omega = 2 / (tau_0 + sqrt(tau_0^2 + 18 C_S^2 P / rho)),
// P = sqrt(2 Pi^neq : Pi^neq), tau_0 = 1/omega_0; then Eq. (1) with that omega.
// ---------------------------------------------------------------------------------------
template <int Q, typename T>
__device__ __forceinline__ void collide_smagorinsky(T (&g)[Q], const Rates<T> &p) {
    using S = Stencil<Q>;
    T drho, jx, jy, jz;
    moments0<Q, T>(g, drho, jx, jy, jz);
    const T rho = T(1) + drho;
    const T inv = T(1) / rho;
    const T ux = jx * inv, uy = jy * inv, uz = jz * inv;
    const T uu15 = T(1.5) * (ux * ux + uy * uy + uz * uz);
    T d[Q];  // non-equilibrium part g - g_eq
    {
        const T w0 = T(S::w(0));
        d[0] = g[0] - (w0 * drho - w0 * rho * uu15);
    }
#pragma unroll
    for (int q = 1; q < Q; ++q) {
        if (q < S::opp(q)) {
            const int b = S::opp(q);
            const T w = T(S::w(q));
            const T cu = T(S::cx(q)) * ux + T(S::cy(q)) * uy + T(S::cz(q)) * uz;
            const T wr = w * rho;
            const T eqs = w * drho + wr * (T(4.5) * cu * cu - uu15);
            const T eqa = wr * T(3) * cu;
            d[q] = g[q] - (eqs + eqa);
            d[b] = g[b] - (eqs - eqa);
        }
    }
    // Pi^neq_ab = sum_q c_a c_b d_q (only the non-zero products of the stencil)
    T pxx = T(0), pyy = T(0), pzz = T(0), pxy = T(0), pxz = T(0), pyz = T(0);
#pragma unroll
    for (int q = 1; q < Q; ++q) {
        if (S::cx(q) != 0) pxx += d[q];
        if (S::cy(q) != 0) pyy += d[q];
        if (S::cz(q) != 0) pzz += d[q];
        if (S::cx(q) * S::cy(q) > 0) pxy += d[q];
        if (S::cx(q) * S::cy(q) < 0) pxy -= d[q];
        if (S::cx(q) * S::cz(q) > 0) pxz += d[q];
        if (S::cx(q) * S::cz(q) < 0) pxz -= d[q];
        if (S::cy(q) * S::cz(q) > 0) pyz += d[q];
        if (S::cy(q) * S::cz(q) < 0) pyz -= d[q];
    }
    const T pp = pxx * pxx + pyy * pyy + pzz * pzz + T(2) * (pxy * pxy + pxz * pxz + pyz * pyz);
    const T P = sqrt(T(2) * pp);
    const T tau0 = T(1) / p.r[0];
    const T cs = p.r[1];
    const T omega = T(2) / (tau0 + sqrt(tau0 * tau0 + T(18) * cs * cs * P * inv));
#pragma unroll
    for (int q = 0; q < Q; ++q) g[q] -= omega * d[q];
}

// ---------------------------------------------------------------------------------------
// KBC entropic operator, D3Q19 and D3Q27 (Eqs. 15-19), rates = [omega_s]. Delta_s = shear-group
// projection, Delta_h = bulk + order 3 + order 4 projections of g - g_eq (the weighted basis of
// collide_mrt19); omega_h = 1 + (1 - omega_s) <Ds,Dh>_E / <Dh,Dh>_E, <a,b>_E = sum a b / f_eq.
// ---------------------------------------------------------------------------------------
// Only the shear part is projected: d = g - g_eq has no conserved moments, so the higher-order part
// is Delta_h = d - Delta_s exactly (f = f_eq + Delta_s + Delta_h, Eq. 15), and
// f' = f - w_s Ds - w_h Dh = f_eq + (1 - w_h) d + (w_h - w_s) Ds. The shear polynomials are even
// and vanish at c = 0, so Ds is the same for q and qbar and zero at the centre.
//
// EXACT: omega_h maximises the entropy S of Eq. (17) itself ("solved numerically in every cell using
// Newton's method"): Newton on G(w) = sum_q Dh_q ln(f'_q(w) / f_eq,q) = 0
// (the "+1" term of the optimality condition sums to zero, sum Dh = 0) with
// G'(w) = -sum_q Dh_q^2 / f'_q(w), started from the linearised omega_h above; with
// x_q = ((1 - w_s) Ds_q + (1 - w) Dh_q) / f_eq,q, f'_q / f_eq,q = 1 + x_q and ln = log1p(x_q).
// A step that would make some f'_q <= 0 is halved (as the oracle does). Newton converges
// quadratically, so after a full step of size s the remaining error is ~K s^2 (K = G''/2G' = O(1)):
// the loop stops after a full step with |s| <= 1e-8 (fp64) / 1e-4 (fp32), i.e. at an error the oracle's
// 1e-14 criterion would only confirm with one more evaluation (G-reading G25), or after 30 / 8 steps.
// 1/f_eq of a pair is recomputed per step (registers, not a stored array).
// ln(1 + x): near 0 (|x| < 1/16, the usual case f' ~ f_eq) by the atanh series
// 2 (s + s^3/3 + ... + s^13/13), s = x / (2 + x), |s| < 1/31 so the tail is below 1e-18 relative;
// elsewhere the library log1p. fp32 uses log1pf throughout.
__device__ __forceinline__ double ln1p_kbc(double x) {
    if (fabs(x) < 0.0625) {
        const double s = x * fast_rcp(2.0 + x), s2 = s * s;
        double p = 1.0 / 13.0;
        p = fma(p, s2, 1.0 / 11.0);
        p = fma(p, s2, 1.0 / 9.0);
        p = fma(p, s2, 1.0 / 7.0);
        p = fma(p, s2, 1.0 / 5.0);
        p = fma(p, s2, 1.0 / 3.0);
        return 2.0 * fma(s * s2, p, s);
    }
    return log1p(x);
}
__device__ __forceinline__ float ln1p_kbc(float x) { return log1pf(x); }

template <int Q, typename T>
__device__ __forceinline__ void kbc_pair_feq(int q, T drho, T rho, T ux, T uy, T uz, T uu15, T &es, T &ea, T &iq, T &ib) {
    using S = Stencil<Q>;
    const T w = T(S::w(q));
    const T cu = T(S::cx(q)) * ux + T(S::cy(q)) * uy + T(S::cz(q)) * uz;
    const T wr = w * rho;
    es = w * drho + wr * (T(4.5) * cu * cu - uu15);
    ea = wr * T(3) * cu;
    // 1/f_eq of the pair from one reciprocal: 1/(A +- B) = (A -+ B) / (A^2 - B^2)
    const T A = w + es;
    const T rr = fast_rcp(A * A - ea * ea);
    iq = (A - ea) * rr;
    ib = (A + ea) * rr;
}

template <int Q, typename T, bool EXACT = false>
__device__ __forceinline__ void collide_kbc(T (&g)[Q], const Rates<T> &p) {
    using S = Stencil<Q>;
    T drho, jx, jy, jz;
    moments0<Q, T>(g, drho, jx, jy, jz);
    const T rho = T(1) + drho;
    const T inv = T(1) / rho;
    const T ux = jx * inv, uy = jy * inv, uz = jz * inv;
    const T uu15 = T(1.5) * (ux * ux + uy * uy + uz * uz);
    const T w0 = T(S::w(0));
    const T eq0 = w0 * drho - w0 * rho * uu15;
    // g <- d = g - g_eq; shear coefficients a_k = <P_k, d> / N_k from the pair sums
    g[0] -= eq0;
    T a[5] = {T(0), T(0), T(0), T(0), T(0)};
#pragma unroll
    for (int q = 1; q < Q; ++q) {
        if (q < S::opp(q)) {
            const int b = S::opp(q);
            const T w = T(S::w(q));
            const T cu = T(S::cx(q)) * ux + T(S::cy(q)) * uy + T(S::cz(q)) * uz;
            const T wr = w * rho;
            const T es = w * drho + wr * (T(4.5) * cu * cu - uu15);
            const T ea = wr * T(3) * cu;
            g[q] -= es + ea;
            g[b] -= es - ea;
            const T dp = g[q] + g[b];
#pragma unroll
            for (int k = 0; k < 5; ++k) {
                const int c = mrt_poly(k, S::cx(q), S::cy(q), S::cz(q));
                if (c == 1) a[k] += dp;
                else if (c == -1) a[k] -= dp;
                else if (c != 0) a[k] += T(c) * dp;
            }
        }
    }
#pragma unroll
    for (int k = 0; k < 5; ++k) a[k] *= T(mrt_inv_norm(k));
    // entropic products <Ds,Dh>_E, <Dh,Dh>_E with <x,y>_E = sum x y / f_eq, f_eq = w + g_eq (Eq. 19)
    T sh = T(0), hh = g[0] * g[0] / (w0 + eq0);
    T ds[Q];
#pragma unroll
    for (int q = 1; q < Q; ++q) {
        if (q < S::opp(q)) {
            const int b = S::opp(q);
            const T w = T(S::w(q));
            T acc = T(0);
#pragma unroll
            for (int k = 0; k < 5; ++k) {
                const int c = mrt_poly(k, S::cx(q), S::cy(q), S::cz(q));
                if (c == 1) acc += a[k];
                else if (c == -1) acc -= a[k];
                else if (c != 0) acc += T(c) * a[k];
            }
            const T s = w * acc;
            ds[q] = s;
            const T cu = T(S::cx(q)) * ux + T(S::cy(q)) * uy + T(S::cz(q)) * uz;
            const T wr = w * rho;
            const T es = w * drho + wr * (T(4.5) * cu * cu - uu15);
            const T ea = wr * T(3) * cu;
            // 1/f_eq of the pair from one reciprocal: 1/(A +- B) = (A -+ B) / (A^2 - B^2)
            const T A = w + es;
            const T rr = fast_rcp(A * A - ea * ea);
            const T iq = (A - ea) * rr;
            const T ib = (A + ea) * rr;
            const T hq = g[q] - s, hb = g[b] - s;
            sh += s * (hq * iq + hb * ib);
            hh += hq * hq * iq + hb * hb * ib;
        }
    }
    const T ws = p.r[0];
    T wh = hh > T(0) ? T(1) + (T(1) - ws) * sh / hh : T(1);
    if constexpr (EXACT) {
        if (hh > T(0)) {
            constexpr bool f64 = sizeof(T) == 8;
            constexpr int kMaxIt = f64 ? 30 : 8;
            const T tol = f64 ? T(1e-8) : T(1e-4);
            const T i0 = T(1) / (w0 + eq0);
            const T kw = T(1) - ws;
            // x_q(w) and positivity at a trial w; G and G' at w
            auto positive = [&](T w) {
                bool ok = T(1) + (T(1) - w) * g[0] * i0 > T(0);
#pragma unroll
                for (int q = 1; q < Q; ++q) {
                    if (q < S::opp(q)) {
                        const int b = S::opp(q);
                        T es, ea, iq, ib;
                        kbc_pair_feq<Q, T>(q, drho, rho, ux, uy, uz, uu15, es, ea, iq, ib);
                        ok = ok && (T(1) + (kw * ds[q] + (T(1) - w) * (g[q] - ds[q])) * iq > T(0)) &&
                             (T(1) + (kw * ds[q] + (T(1) - w) * (g[b] - ds[q])) * ib > T(0));
                    }
                }
                return ok;
            };
            for (int it = 0; it < kMaxIt; ++it) {
                const T km = T(1) - wh;
                T x0 = km * g[0] * i0;
                T G = g[0] * ln1p_kbc(x0);
                // G' only sets the convergence rate, not the root: approximate reciprocals suffice
                T Gp = -g[0] * g[0] * i0 * fast_rcp(T(1) + x0);
                // min_q f'/f_eq and max_q |Dh/f_eq| bound f' at the next iterate: f'(w - s)/f_eq =
                // 1 + x + s Dh/f_eq stays positive when min(1 + x) > |s| max|Dh/f_eq|
                T lo = T(1) + x0, hi = fabs(g[0] * i0);
#pragma unroll
                for (int q = 1; q < Q; ++q) {
                    if (q < S::opp(q)) {
                        const int b = S::opp(q);
                        T es, ea, iq, ib;
                        kbc_pair_feq<Q, T>(q, drho, rho, ux, uy, uz, uu15, es, ea, iq, ib);
                        const T hq = g[q] - ds[q], hb = g[b] - ds[q];
                        const T xq = (kw * ds[q] + km * hq) * iq, xb = (kw * ds[q] + km * hb) * ib;
                        G += hq * ln1p_kbc(xq) + hb * ln1p_kbc(xb);
                        Gp -= hq * hq * iq * fast_rcp(T(1) + xq) + hb * hb * ib * fast_rcp(T(1) + xb);
                        lo = fmin(lo, fmin(T(1) + xq, T(1) + xb));
                        hi = fmax(hi, fmax(fabs(hq * iq), fabs(hb * ib)));
                    }
                }
                T step = G / Gp;
                if (!(fabs(step) <= T(1e30))) {  // NaN state (a non-positive f' already): keep it NaN
                    wh = step;
                    break;
                }
                T wn = wh - step;
                bool full = true;
                for (int tries = 0; tries < 60 && !(lo > fabs(step) * hi) && !positive(wn); ++tries) {
                    step *= T(0.5);
                    wn = wh - step;
                    full = false;
                }
                wh = wn;
                if (full && fabs(step) <= tol) break;
            }
        }
    }
    // f' = f_eq + (1 - w_h) d + (w_h - w_s) Ds
    const T kd = T(1) - wh, ks = wh - ws;
    g[0] = eq0 + kd * g[0];
#pragma unroll
    for (int q = 1; q < Q; ++q) {
        if (q < S::opp(q)) {
            const int b = S::opp(q);
            const T w = T(S::w(q));
            const T cu = T(S::cx(q)) * ux + T(S::cy(q)) * uy + T(S::cz(q)) * uz;
            const T wr = w * rho;
            const T es = w * drho + wr * (T(4.5) * cu * cu - uu15);
            const T ea = wr * T(3) * cu;
            const T sk = ks * ds[q];
            g[q] = (es + ea) + kd * g[q] + sk;
            g[b] = (es - ea) + kd * g[b] + sk;
        }
    }
}

// Weighted MRT with only the shear group relaxed (omega_bulk = omega_3 = omega_4 = 1: config C2, G6): every
// other group relaxes to equilibrium, and the weighted shear projector of a non-equilibrium part d is
// (9/2) w_q (c_q c_q - c^2/3 I) : Pi~ with Pi~ the traceless part of sum_q c c d (the closed form of G6,
// pinned by the oracle test test_mrt_config2_closed_form; D3Q19 and D3Q27). So
//   f* = f_eq + (1 - omega_s) (9/2) w_q c_q c_q : Pi~^neq,  Pi^neq = sum_q c c f - rho (c_s^2 I + u u)
// (Eq. 3), computed from the pair sums: ~60 % of the group-projection operations of collide_mrt19. The
// run-time counterpart of lbmpy's pre-evaluation of constant relaxation rates.
template <int Q, typename T>
__device__ __forceinline__ void collide_mrt_shear(T (&g)[Q], const Rates<T> &p) {
    using S = Stencil<Q>;
    T drho, jx, jy, jz;
    moments0<Q, T>(g, drho, jx, jy, jz);
    const T rho = T(1) + drho;
    const T inv = T(1) / rho;
    const T ux = jx * inv, uy = jy * inv, uz = jz * inv;
    const T uu15 = T(1.5) * (ux * ux + uy * uy + uz * uz);
    // second moments of g from the pair sums g_q + g_qbar (f = g + w adds c_s^2 I)
    T pxx = T(0), pyy = T(0), pzz = T(0), pxy = T(0), pxz = T(0), pyz = T(0);
#pragma unroll
    for (int q = 1; q < Q; ++q) {
        if (q < S::opp(q)) {
            const int cx = S::cx(q), cy = S::cy(q), cz = S::cz(q);
            const T sp = g[q] + g[S::opp(q)];
            if (cx != 0) pxx += sp;
            if (cy != 0) pyy += sp;
            if (cz != 0) pzz += sp;
            if (cx * cy > 0) pxy += sp;
            if (cx * cy < 0) pxy -= sp;
            if (cx * cz > 0) pxz += sp;
            if (cx * cz < 0) pxz -= sp;
            if (cy * cz > 0) pyz += sp;
            if (cy * cz < 0) pyz -= sp;
        }
    }
    // non-equilibrium part: Pi(f) - rho (c_s^2 I + u u) = Pi(g) - drho / 3 - rho u u
    const T third = T(1) / T(3);
    const T rx = rho * ux, ry = rho * uy, rz = rho * uz;
    const T nxx = pxx - third * drho - rx * ux, nyy = pyy - third * drho - ry * uy, nzz = pzz - third * drho - rz * uz;
    const T nxy = pxy - rx * uy, nxz = pxz - rx * uz, nyz = pyz - ry * uz;
    const T tr3 = third * (nxx + nyy + nzz);
    const T k = T(4.5) * (T(1) - p.r[0]);
    const T dxx = k * (nxx - tr3), dyy = k * (nyy - tr3), dzz = k * (nzz - tr3);
    const T dxy = T(2) * k * nxy, dxz = T(2) * k * nxz, dyz = T(2) * k * nyz;
    const T w0 = T(S::w(0));
    g[0] = w0 * drho - w0 * rho * uu15;  // c = 0: the traceless part does not reach the centre
#pragma unroll
    for (int q = 1; q < Q; ++q) {
        if (q < S::opp(q)) {
            const int b = S::opp(q);
            const int cx = S::cx(q), cy = S::cy(q), cz = S::cz(q);
            const T w = T(S::w(q));
            const T cu = T(cx) * ux + T(cy) * uy + T(cz) * uz;
            const T wr = w * rho;
            const T es = w * drho + wr * (T(4.5) * cu * cu - uu15);
            const T ea = wr * T(3) * cu;
            T qq = T(0);  // c c : (k Pi~), compile-time coefficients
            if (cx != 0) qq += dxx;
            if (cy != 0) qq += dyy;
            if (cz != 0) qq += dzz;
            if (cx * cy > 0) qq += dxy;
            if (cx * cy < 0) qq -= dxy;
            if (cx * cz > 0) qq += dxz;
            if (cx * cz < 0) qq -= dxz;
            if (cy * cz > 0) qq += dyz;
            if (cy * cz < 0) qq -= dyz;
            const T sh = w * qq;
            g[q] = (es + ea) + sh;
            g[b] = (es - ea) + sh;
        }
    }
}

// ---------------------------------------------------------------------------------------
// Cumulant, D3Q27.
// Tensor index of a direction: t = (cx+1)*9 + (cy+1)*3 + (cz+1); after the forward transform
// slot (a,b,c) holds the central moment K_abc = sum_q (cx-ux)^a (cy-uy)^b (cz-uz)^c f_q.
// ---------------------------------------------------------------------------------------
__host__ __device__ constexpr int tidx(int q) { return (kC27[q][0] + 1) * 9 + (kC27[q][1] + 1) * 3 + (kC27[q][2] + 1); }

// forward per-line transform: (f-, f0, f+) -> (K0, K1, K2) about velocity u
template <typename T>
__device__ __forceinline__ void chim_fwd(T &m, T &z, T &p, T u) {
    const T k0 = m + z + p;
    const T d = p - m;
    const T s = p + m;
    const T k1 = d - u * k0;
    const T k2 = s - T(2) * u * d + u * u * k0;
    m = k0;
    z = k1;
    p = k2;
}
// inverse: (K0, K1, K2) -> (f-, f0, f+)
template <typename T>
__device__ __forceinline__ void chim_bwd(T &m, T &z, T &p, T u) {
    const T k0 = m, k1 = z, k2 = p;
    const T uu = u * u;
    const T f0 = (T(1) - uu) * k0 - T(2) * u * k1 - k2;
    const T fp = T(0.5) * ((uu + u) * k0 + (T(2) * u + T(1)) * k1 + k2);
    const T fm = T(0.5) * ((uu - u) * k0 + (T(2) * u - T(1)) * k1 + k2);
    m = fm;
    z = f0;
    p = fp;
}

template <typename T>
__device__ __forceinline__ void collide_cumulant27(T (&g)[27], const Rates<T> &p) {
    using S = Stencil<27>;
    T K[27];
#pragma unroll
    for (int q = 0; q < 27; ++q) K[tidx(q)] = g[q] + T(S::w(q));
    T rho = T(0), jx = T(0), jy = T(0), jz = T(0);
#pragma unroll
    for (int q = 0; q < 27; ++q) {
        rho += K[tidx(q)];
    }
    T drho, ax, ay, az;
    moments0<27, T>(g, drho, ax, ay, az);
    jx = ax;
    jy = ay;
    jz = az;
    rho = T(1) + drho;
    const T inv = T(1) / rho;
    const T ux = jx * inv, uy = jy * inv, uz = jz * inv;
#define KI(a, b, c) K[(a) * 9 + (b) * 3 + (c)]
    // forward: x, then y, then z
#pragma unroll
    for (int b = 0; b < 3; ++b)
#pragma unroll
        for (int c = 0; c < 3; ++c) chim_fwd(KI(0, b, c), KI(1, b, c), KI(2, b, c), ux);
#pragma unroll
    for (int a = 0; a < 3; ++a)
#pragma unroll
        for (int c = 0; c < 3; ++c) chim_fwd(KI(a, 0, c), KI(a, 1, c), KI(a, 2, c), uy);
#pragma unroll
    for (int a = 0; a < 3; ++a)
#pragma unroll
        for (int b = 0; b < 3; ++b) chim_fwd(KI(a, b, 0), KI(a, b, 1), KI(a, b, 2), uz);

    // normalised central moments c_abc = K_abc / rho (orders 2..6; order 1 vanish)
    const T c200 = KI(2, 0, 0) * inv, c020 = KI(0, 2, 0) * inv, c002 = KI(0, 0, 2) * inv;
    const T c110 = KI(1, 1, 0) * inv, c101 = KI(1, 0, 1) * inv, c011 = KI(0, 1, 1) * inv;
    const T c111 = KI(1, 1, 1) * inv;
    const T c210 = KI(2, 1, 0) * inv, c201 = KI(2, 0, 1) * inv, c120 = KI(1, 2, 0) * inv;
    const T c021 = KI(0, 2, 1) * inv, c102 = KI(1, 0, 2) * inv, c012 = KI(0, 1, 2) * inv;
    const T c211 = KI(2, 1, 1) * inv, c121 = KI(1, 2, 1) * inv, c112 = KI(1, 1, 2) * inv;
    const T c220 = KI(2, 2, 0) * inv, c202 = KI(2, 0, 2) * inv, c022 = KI(0, 2, 2) * inv;
    const T c221 = KI(2, 2, 1) * inv, c212 = KI(2, 1, 2) * inv, c122 = KI(1, 2, 2) * inv;
    const T c222 = KI(2, 2, 2) * inv;

    // cumulants (mean zero: sum over set partitions without singleton blocks)
    const T k211 = c211 - c200 * c011 - T(2) * c110 * c101;
    const T k121 = c121 - c020 * c101 - T(2) * c110 * c011;
    const T k112 = c112 - c002 * c110 - T(2) * c101 * c011;
    const T k220 = c220 - c200 * c020 - T(2) * c110 * c110;
    const T k202 = c202 - c200 * c002 - T(2) * c101 * c101;
    const T k022 = c022 - c020 * c002 - T(2) * c011 * c011;
    const T k221 = c221 - c200 * c021 - c020 * c201 - T(2) * c011 * c210 - T(2) * c101 * c120 - T(4) * c110 * c111;
    const T k212 = c212 - c200 * c012 - c002 * c210 - T(2) * c011 * c201 - T(2) * c110 * c102 - T(4) * c101 * c111;
    const T k122 = c122 - c020 * c102 - c002 * c120 - T(2) * c101 * c021 - T(2) * c110 * c012 - T(4) * c011 * c111;
    const T k222 = c222 - c200 * c022 - c020 * c202 - c002 * c220
                 - T(4) * (c110 * c112 + c101 * c121 + c011 * c211)
                 - T(2) * (c210 * c012 + c201 * c021 + c120 * c102) - T(4) * c111 * c111
                 + T(2) * c200 * c020 * c002
                 + T(4) * (c200 * c011 * c011 + c020 * c101 * c101 + c002 * c110 * c110)
                 + T(16) * c110 * c101 * c011;

    // relaxation (G7): trace to 3 cs^2 = 1 with omega_bulk, deviator/off-diagonal with omega_shear,
    // order n >= 3 to zero with omega_n
    const T ws = p.r[0], wb = p.r[1];
    const T r3 = T(1) - p.r[2], r4 = T(1) - p.r[3], r5 = T(1) - p.r[4], r6 = T(1) - p.r[5];
    const T tr = c200 + c020 + c002;
    const T trn = tr + wb * (T(1) - tr);
    const T rs = T(1) - ws;
    const T third = T(1) / T(3);
    const T n200 = third * trn + rs * (c200 - third * tr);
    const T n020 = third * trn + rs * (c020 - third * tr);
    const T n002 = third * trn + rs * (c002 - third * tr);
    const T n110 = rs * c110, n101 = rs * c101, n011 = rs * c011;
    const T n111 = r3 * c111;
    const T n210 = r3 * c210, n201 = r3 * c201, n120 = r3 * c120, n021 = r3 * c021, n102 = r3 * c102, n012 = r3 * c012;
    const T q211 = r4 * k211, q121 = r4 * k121, q112 = r4 * k112;
    const T q220 = r4 * k220, q202 = r4 * k202, q022 = r4 * k022;
    const T q221 = r5 * k221, q212 = r5 * k212, q122 = r5 * k122;
    const T q222 = r6 * k222;

    // back to central moments: c = sum over partitions without singletons of prod kappa_B
    const T m211 = q211 + n200 * n011 + T(2) * n110 * n101;
    const T m121 = q121 + n020 * n101 + T(2) * n110 * n011;
    const T m112 = q112 + n002 * n110 + T(2) * n101 * n011;
    const T m220 = q220 + n200 * n020 + T(2) * n110 * n110;
    const T m202 = q202 + n200 * n002 + T(2) * n101 * n101;
    const T m022 = q022 + n020 * n002 + T(2) * n011 * n011;
    const T m221 = q221 + n200 * n021 + n020 * n201 + T(2) * n011 * n210 + T(2) * n101 * n120 + T(4) * n110 * n111;
    const T m212 = q212 + n200 * n012 + n002 * n210 + T(2) * n011 * n201 + T(2) * n110 * n102 + T(4) * n101 * n111;
    const T m122 = q122 + n020 * n102 + n002 * n120 + T(2) * n101 * n021 + T(2) * n110 * n012 + T(4) * n011 * n111;
    const T m222 = q222 + n200 * q022 + n020 * q202 + n002 * q220
                 + T(4) * (n110 * q112 + n101 * q121 + n011 * q211)
                 + T(2) * (n210 * n012 + n201 * n021 + n120 * n102) + T(4) * n111 * n111
                 + n200 * n020 * n002
                 + T(2) * (n200 * n011 * n011 + n020 * n101 * n101 + n002 * n110 * n110)
                 + T(8) * n110 * n101 * n011;

    KI(0, 0, 0) = rho;
    KI(1, 0, 0) = T(0);
    KI(0, 1, 0) = T(0);
    KI(0, 0, 1) = T(0);
    KI(2, 0, 0) = rho * n200; KI(0, 2, 0) = rho * n020; KI(0, 0, 2) = rho * n002;
    KI(1, 1, 0) = rho * n110; KI(1, 0, 1) = rho * n101; KI(0, 1, 1) = rho * n011;
    KI(1, 1, 1) = rho * n111;
    KI(2, 1, 0) = rho * n210; KI(2, 0, 1) = rho * n201; KI(1, 2, 0) = rho * n120;
    KI(0, 2, 1) = rho * n021; KI(1, 0, 2) = rho * n102; KI(0, 1, 2) = rho * n012;
    KI(2, 1, 1) = rho * m211; KI(1, 2, 1) = rho * m121; KI(1, 1, 2) = rho * m112;
    KI(2, 2, 0) = rho * m220; KI(2, 0, 2) = rho * m202; KI(0, 2, 2) = rho * m022;
    KI(2, 2, 1) = rho * m221; KI(2, 1, 2) = rho * m212; KI(1, 2, 2) = rho * m122;
    KI(2, 2, 2) = rho * m222;

    // backward: z, y, x
#pragma unroll
    for (int a = 0; a < 3; ++a)
#pragma unroll
        for (int b = 0; b < 3; ++b) chim_bwd(KI(a, b, 0), KI(a, b, 1), KI(a, b, 2), uz);
#pragma unroll
    for (int a = 0; a < 3; ++a)
#pragma unroll
        for (int c = 0; c < 3; ++c) chim_bwd(KI(a, 0, c), KI(a, 1, c), KI(a, 2, c), uy);
#pragma unroll
    for (int b = 0; b < 3; ++b)
#pragma unroll
        for (int c = 0; c < 3; ++c) chim_bwd(KI(0, b, c), KI(1, b, c), KI(2, b, c), ux);
#undef KI
#pragma unroll
    for (int q = 0; q < 27; ++q) g[q] = K[tidx(q)] - T(S::w(q));
}

// Cumulant D3Q27 with omega_bulk = omega_3 = ... = omega_6 = 1 (the rates of config C3, G7): the
// run-time counterpart of lbmpy's pre-evaluation of constant relaxation rates for the
// cumulant. Every cumulant of order >= 3 is relaxed to its Maxwellian value 0 and the trace to 3 cs^2, so
// only the second-order central moments of the pre-collision state are needed (from the raw second
// moments, not the full forward transform), and the post-collision central moments are the Gaussian
// (Isserlis) ones of the relaxed covariance: order 4 m211 = n200 n011 + 2 n110 n101, m220 = n200 n020 +
// 2 n110^2 (and permutations), order 6 m222, odd orders 0 (the closed form the oracle pin G7 checks).
// The first backward pass (z) uses the parity structure of those moments: lines (a, b) with a + b even
// hold (K_ab0, 0, K_ab2), odd ones (0, K_ab1, 0). About 600 instead of 1135 FP64 operations per cell.
template <typename T>
__device__ __forceinline__ void chim_bwd_even(T &m, T &z, T &p, T u) {  // (k0, 0, k2)
    const T k0 = m, k2 = p;
    const T uu = u * u;
    z = (T(1) - uu) * k0 - k2;
    p = T(0.5) * ((uu + u) * k0 + k2);
    m = T(0.5) * ((uu - u) * k0 + k2);
}
template <typename T>
__device__ __forceinline__ void chim_bwd_odd(T &m, T &z, T &p, T u) {  // (0, k1, 0)
    const T k1 = z;
    z = T(-2) * u * k1;
    p = T(0.5) * (T(2) * u + T(1)) * k1;
    m = T(0.5) * (T(2) * u - T(1)) * k1;
}

template <typename T>
__device__ __forceinline__ void collide_cumulant27_unit(T (&g)[27], const Rates<T> &p) {
    using S = Stencil<27>;
    T drho, jx, jy, jz;
    moments0_tree<27, T>(g, drho, jx, jy, jz);
    const T rho = T(1) + drho;
    const T inv = T(1) / rho;
    const T ux = jx * inv, uy = jy * inv, uz = jz * inv;
    // raw second moments of g; f = g + w adds delta_ab / 3 (sum_q w_q c_a c_b = c_s^2 delta_ab)
    T pxx = T(0), pyy = T(0), pzz = T(0), pxy = T(0), pxz = T(0), pyz = T(0);
#pragma unroll
    for (int q = 1; q < 27; ++q) {
        const int cx = S::cx(q), cy = S::cy(q), cz = S::cz(q);
        if (cx != 0) pxx += g[q];
        if (cy != 0) pyy += g[q];
        if (cz != 0) pzz += g[q];
        if (cx * cy > 0) pxy += g[q];
        if (cx * cy < 0) pxy -= g[q];
        if (cx * cz > 0) pxz += g[q];
        if (cx * cz < 0) pxz -= g[q];
        if (cy * cz > 0) pyz += g[q];
        if (cy * cz < 0) pyz -= g[q];
    }
    const T third = T(1) / T(3);
    // normalised central second moments (= second-order cumulants) c_ab = P_ab / rho - u_a u_b
    const T c200 = (pxx + third) * inv - ux * ux, c020 = (pyy + third) * inv - uy * uy, c002 = (pzz + third) * inv - uz * uz;
    const T c110 = pxy * inv - ux * uy, c101 = pxz * inv - ux * uz, c011 = pyz * inv - uy * uz;
    // relaxation: deviator and off-diagonals with omega_shear, trace to 1 (omega_bulk = 1)
    const T rs = T(1) - p.r[0];
    const T tr3 = third * (c200 + c020 + c002);
    const T n200 = third + rs * (c200 - tr3), n020 = third + rs * (c020 - tr3), n002 = third + rs * (c002 - tr3);
    const T n110 = rs * c110, n101 = rs * c101, n011 = rs * c011;
    // post-collision central moments (all cumulants of order >= 3 are zero)
    const T m211 = n200 * n011 + T(2) * n110 * n101;
    const T m121 = n020 * n101 + T(2) * n110 * n011;
    const T m112 = n002 * n110 + T(2) * n101 * n011;
    const T m220 = n200 * n020 + T(2) * n110 * n110;
    const T m202 = n200 * n002 + T(2) * n101 * n101;
    const T m022 = n020 * n002 + T(2) * n011 * n011;
    const T m222 = n200 * n020 * n002 + T(2) * (n200 * n011 * n011 + n020 * n101 * n101 + n002 * n110 * n110) +
                   T(8) * n110 * n101 * n011;
    T K[27];
#define KI(a, b, c) K[(a) * 9 + (b) * 3 + (c)]
    KI(0, 0, 0) = rho;            KI(0, 0, 1) = T(0);           KI(0, 0, 2) = rho * n002;
    KI(0, 1, 0) = T(0);           KI(0, 1, 1) = rho * n011;     KI(0, 1, 2) = T(0);
    KI(0, 2, 0) = rho * n020;     KI(0, 2, 1) = T(0);           KI(0, 2, 2) = rho * m022;
    KI(1, 0, 0) = T(0);           KI(1, 0, 1) = rho * n101;     KI(1, 0, 2) = T(0);
    KI(1, 1, 0) = rho * n110;     KI(1, 1, 1) = T(0);           KI(1, 1, 2) = rho * m112;
    KI(1, 2, 0) = T(0);           KI(1, 2, 1) = rho * m121;     KI(1, 2, 2) = T(0);
    KI(2, 0, 0) = rho * n200;     KI(2, 0, 1) = T(0);           KI(2, 0, 2) = rho * m202;
    KI(2, 1, 0) = T(0);           KI(2, 1, 1) = rho * m211;     KI(2, 1, 2) = T(0);
    KI(2, 2, 0) = rho * m220;     KI(2, 2, 1) = T(0);           KI(2, 2, 2) = rho * m222;
    // backward: z (parity-structured lines), y, x
#pragma unroll
    for (int a = 0; a < 3; ++a)
#pragma unroll
        for (int b = 0; b < 3; ++b) {
            if ((a + b) % 2 == 0) chim_bwd_even(KI(a, b, 0), KI(a, b, 1), KI(a, b, 2), uz);
            else chim_bwd_odd(KI(a, b, 0), KI(a, b, 1), KI(a, b, 2), uz);
        }
#pragma unroll
    for (int a = 0; a < 3; ++a)
#pragma unroll
        for (int c = 0; c < 3; ++c) chim_bwd(KI(a, 0, c), KI(a, 1, c), KI(a, 2, c), uy);
#pragma unroll
    for (int b = 0; b < 3; ++b)
#pragma unroll
        for (int c = 0; c < 3; ++c) chim_bwd(KI(0, b, c), KI(1, b, c), KI(2, b, c), ux);
#undef KI
#pragma unroll
    for (int q = 0; q < 27; ++q) g[q] = K[tidx(q)] - T(S::w(q));
}

// ---------------------------------------------------------------------------------------
// Cumulant, D3Q19 (cumulant methods "also for D3Q19"): the 19 populations are embedded in
// the 3x3x3 tensor with zero corners, transformed to central moments by the same per-axis chimera
// transform, the cumulants of the 19 basis monomials (at least one exponent 0; the set is
// closed under taking sub-indices, so none of them needs a dropped monomial) are relaxed as in G7
// (orders 2, 3, 4), shifted back to raw moments per axis and mapped to populations with the
// closed-form inverse of the D3Q19 monomial moment matrix (d3q19_from_raw).
// ---------------------------------------------------------------------------------------
// raw moment tensor M[a*9 + b*3 + c] (basis entries only are read) -> the 19 populations
template <typename T>
__device__ __forceinline__ void d3q19_from_raw(const T (&M)[27], T (&f)[19]) {
#define MI(a, b, c) M[(a) * 9 + (b) * 3 + (c)]
    // faces: f(+-e_x) = ((M200 - M220 - M202) +- (M100 - M120 - M102)) / 2, and cyclically
    const T sx = MI(2, 0, 0) - MI(2, 2, 0) - MI(2, 0, 2), dx = MI(1, 0, 0) - MI(1, 2, 0) - MI(1, 0, 2);
    const T sy = MI(0, 2, 0) - MI(2, 2, 0) - MI(0, 2, 2), dy = MI(0, 1, 0) - MI(2, 1, 0) - MI(0, 1, 2);
    const T sz = MI(0, 0, 2) - MI(2, 0, 2) - MI(0, 2, 2), dz = MI(0, 0, 1) - MI(2, 0, 1) - MI(0, 2, 1);
#pragma unroll
    for (int q = 0; q < 19; ++q) {
        const int cx = kC27[q][0], cy = kC27[q][1], cz = kC27[q][2];
        const int n = cx * cx + cy * cy + cz * cz;
        T v;
        if (n == 0) {
            v = MI(0, 0, 0) - MI(2, 0, 0) - MI(0, 2, 0) - MI(0, 0, 2) + MI(2, 2, 0) + MI(2, 0, 2) + MI(0, 2, 2);
        } else if (n == 1) {
            const T sgn = T(cx + cy + cz);
            v = cx ? T(0.5) * (sx + sgn * dx) : cy ? T(0.5) * (sy + sgn * dy) : T(0.5) * (sz + sgn * dz);
        } else if (cz == 0) {  // xy edge: (M220 + sx M120 + sy M210 + sx sy M110) / 4
            v = T(0.25) * (MI(2, 2, 0) + T(cx) * MI(1, 2, 0) + T(cy) * MI(2, 1, 0) + T(cx * cy) * MI(1, 1, 0));
        } else if (cy == 0) {  // xz edge
            v = T(0.25) * (MI(2, 0, 2) + T(cx) * MI(1, 0, 2) + T(cz) * MI(2, 0, 1) + T(cx * cz) * MI(1, 0, 1));
        } else {  // yz edge
            v = T(0.25) * (MI(0, 2, 2) + T(cy) * MI(0, 1, 2) + T(cz) * MI(0, 2, 1) + T(cy * cz) * MI(0, 1, 1));
        }
        f[q] = v;
    }
#undef MI
}

// central -> raw moments along one line (K0, K1, K2) about velocity u
template <typename T>
__device__ __forceinline__ void shift_raw(T &m, T &z, T &p, T u) {
    const T k0 = m, k1 = z, k2 = p;
    z = k1 + u * k0;
    p = k2 + T(2) * u * k1 + u * u * k0;
}

template <typename T>
__device__ __forceinline__ void collide_cumulant19(T (&g)[19], const Rates<T> &p) {
    using S = Stencil<19>;
    T K[27];
#pragma unroll
    for (int t = 0; t < 27; ++t) K[t] = T(0);
#pragma unroll
    for (int q = 0; q < 19; ++q) K[tidx(q)] = g[q] + T(S::w(q));
    T drho, jx, jy, jz;
    moments0<19, T>(g, drho, jx, jy, jz);
    const T rho = T(1) + drho;
    const T inv = T(1) / rho;
    const T ux = jx * inv, uy = jy * inv, uz = jz * inv;
#define KI(a, b, c) K[(a) * 9 + (b) * 3 + (c)]
#pragma unroll
    for (int b = 0; b < 3; ++b)
#pragma unroll
        for (int c = 0; c < 3; ++c) chim_fwd(KI(0, b, c), KI(1, b, c), KI(2, b, c), ux);
#pragma unroll
    for (int a = 0; a < 3; ++a)
#pragma unroll
        for (int c = 0; c < 3; ++c) chim_fwd(KI(a, 0, c), KI(a, 1, c), KI(a, 2, c), uy);
#pragma unroll
    for (int a = 0; a < 3; ++a)
#pragma unroll
        for (int b = 0; b < 3; ++b) chim_fwd(KI(a, b, 0), KI(a, b, 1), KI(a, b, 2), uz);
    const T c200 = KI(2, 0, 0) * inv, c020 = KI(0, 2, 0) * inv, c002 = KI(0, 0, 2) * inv;
    const T c110 = KI(1, 1, 0) * inv, c101 = KI(1, 0, 1) * inv, c011 = KI(0, 1, 1) * inv;
    // order 4 of the basis: kappa_220 = c220 - c200 c020 - 2 c110^2 (and cyclically)
    const T k220 = KI(2, 2, 0) * inv - c200 * c020 - T(2) * c110 * c110;
    const T k202 = KI(2, 0, 2) * inv - c200 * c002 - T(2) * c101 * c101;
    const T k022 = KI(0, 2, 2) * inv - c020 * c002 - T(2) * c011 * c011;
    const T ws = p.r[0], wb = p.r[1], r3 = T(1) - p.r[2], r4 = T(1) - p.r[3];
    const T tr = c200 + c020 + c002;
    const T trn = tr + wb * (T(1) - tr);
    const T rs = T(1) - ws;
    const T third = T(1) / T(3);
    const T n200 = third * trn + rs * (c200 - third * tr);
    const T n020 = third * trn + rs * (c020 - third * tr);
    const T n002 = third * trn + rs * (c002 - third * tr);
    const T n110 = rs * c110, n101 = rs * c101, n011 = rs * c011;
    // relaxed central moments (times rho) of the basis; the dropped entries are never read
    KI(0, 0, 0) = rho;
    KI(1, 0, 0) = T(0);
    KI(0, 1, 0) = T(0);
    KI(0, 0, 1) = T(0);
    KI(2, 0, 0) = rho * n200; KI(0, 2, 0) = rho * n020; KI(0, 0, 2) = rho * n002;
    KI(1, 1, 0) = rho * n110; KI(1, 0, 1) = rho * n101; KI(0, 1, 1) = rho * n011;
    KI(2, 1, 0) *= r3; KI(2, 0, 1) *= r3; KI(1, 2, 0) *= r3;
    KI(0, 2, 1) *= r3; KI(1, 0, 2) *= r3; KI(0, 1, 2) *= r3;
    KI(2, 2, 0) = rho * (r4 * k220 + n200 * n020 + T(2) * n110 * n110);
    KI(2, 0, 2) = rho * (r4 * k202 + n200 * n002 + T(2) * n101 * n101);
    KI(0, 2, 2) = rho * (r4 * k022 + n020 * n002 + T(2) * n011 * n011);
    KI(1, 1, 1) = T(0); KI(2, 1, 1) = T(0); KI(1, 2, 1) = T(0); KI(1, 1, 2) = T(0);
    KI(2, 2, 1) = T(0); KI(2, 1, 2) = T(0); KI(1, 2, 2) = T(0); KI(2, 2, 2) = T(0);
    // central -> raw moments per axis
#pragma unroll
    for (int a = 0; a < 3; ++a)
#pragma unroll
        for (int b = 0; b < 3; ++b) shift_raw(KI(a, b, 0), KI(a, b, 1), KI(a, b, 2), uz);
#pragma unroll
    for (int a = 0; a < 3; ++a)
#pragma unroll
        for (int c = 0; c < 3; ++c) shift_raw(KI(a, 0, c), KI(a, 1, c), KI(a, 2, c), uy);
#pragma unroll
    for (int b = 0; b < 3; ++b)
#pragma unroll
        for (int c = 0; c < 3; ++c) shift_raw(KI(0, b, c), KI(1, b, c), KI(2, b, c), ux);
#undef KI
    T f[19];
    d3q19_from_raw<T>(K, f);
#pragma unroll
    for (int q = 0; q < 19; ++q) g[q] = f[q] - T(S::w(q));
}

#include "generated/gen_collide.cuh"

// ---------------------------------------------------------------------------------------
// Dispatch
// ---------------------------------------------------------------------------------------
enum Op { OP_SRT = 0, OP_TRT = 1, OP_MRT = 2, OP_CUMULANT = 3, OP_IDENTITY = 4, OP_SMAGORINSKY = 5, OP_KBC = 6,
          OP_KBC_EXACT = 7, /* KBC, omega_h by Newton maximisation of Eq. (17) (= LBM_KBC_EXACT) */
          OP_GEN_SRT = 8, OP_GEN_TRT = 9, OP_GEN_MRT = 10, OP_GEN_SMAGORINSKY = 11, /* generated (codegen/, = LBM_GEN_*) */
          OP_CUMULANT_UNIT = 12, /* D3Q27 cumulant with omega_bulk = omega_3..6 = 1 (internal id, selected at create) */
          OP_MRT_SHEAR = 13, /* weighted MRT with omega_bulk = omega_3 = omega_4 = 1 (internal id, selected at create) */
          OP_MRT_ROWS = 15 /* MRT with one rate per moment (internal id; ABI: LBM_MRT + n_row_rates = 15) */ };

// Operator class for occupancy / kernel-path tuning: the generated operators behave like their
// hand-written counterparts (TRT-like, MRT-like).
constexpr int op_class(int op) {
    return (op == OP_GEN_SRT || op == OP_GEN_TRT) ? OP_TRT : op == OP_GEN_MRT ? OP_MRT : op == OP_GEN_SMAGORINSKY ? OP_SMAGORINSKY
         : op == OP_CUMULANT_UNIT ? OP_CUMULANT : op == OP_MRT_SHEAR ? OP_MRT : op;
}

template <int Q, int OPX, typename T, bool FORCE>
__device__ __forceinline__ void collide(T (&g)[Q], const Rates<T> &p) {
    constexpr int OP = op_base(OPX), EQ = op_eq(OPX);
    static_assert(EQ == EQ_COMPRESSIBLE || OP == OP_SRT || OP == OP_TRT || OP == OP_MRT ||
                      ((OP == OP_GEN_SRT || OP == OP_GEN_TRT) && EQ == EQ_INCOMPRESSIBLE),
                  "equilibrium variants exist for SRT/TRT/MRT (generated: incompressible SRT/TRT)");
    if constexpr (OP == OP_SRT || OP == OP_TRT) {
        collide_trt<Q, T, FORCE, EQ>(g, p);
    } else if constexpr (OP == OP_MRT) {
        static_assert(Q == 19, "MRT is implemented for D3Q19");
        collide_mrt19<T, EQ>(g, p);
    } else if constexpr (OP == OP_CUMULANT) {
        if constexpr (Q == 27) collide_cumulant27<T>(g, p);
        else collide_cumulant19<T>(g, p);
    } else if constexpr (OP == OP_MRT_SHEAR) {
        collide_mrt_shear<Q, T>(g, p);
    } else if constexpr (OP == OP_CUMULANT_UNIT) {
        static_assert(Q == 27, "the unit-rate cumulant specialisation is D3Q27");
        collide_cumulant27_unit<T>(g, p);
    } else if constexpr (OP == OP_SMAGORINSKY) {
        collide_smagorinsky<Q, T>(g, p);
    } else if constexpr (OP == OP_KBC) {
        collide_kbc<Q, T>(g, p);
    } else if constexpr (OP == OP_KBC_EXACT) {
        collide_kbc<Q, T, true>(g, p);
    } else if constexpr (OP == OP_MRT_ROWS) {
        static_assert(Q == 19, "per-moment MRT is implemented for D3Q19");
        collide_mrt19_rows<T>(g, p);
    } else if constexpr (OP == OP_GEN_SRT && EQ == EQ_INCOMPRESSIBLE) {
        if constexpr (Q == 19) gen_srt19_inc<T>(g, p);
        else gen_srt27_inc<T>(g, p);
    } else if constexpr (OP == OP_GEN_TRT && EQ == EQ_INCOMPRESSIBLE) {
        if constexpr (Q == 19) gen_trt19_inc<T>(g, p);
        else gen_trt27_inc<T>(g, p);
    } else if constexpr (OP == OP_GEN_SRT) {
        if constexpr (Q == 19) gen_srt19<T>(g, p);
        else gen_srt27<T>(g, p);
    } else if constexpr (OP == OP_GEN_TRT) {
        if constexpr (Q == 19) gen_trt19<T>(g, p);
        else gen_trt27<T>(g, p);
    } else if constexpr (OP == OP_GEN_SMAGORINSKY) {
        if constexpr (Q == 19) gen_smagorinsky19<T>(g, p);
        else gen_smagorinsky27<T>(g, p);
    } else if constexpr (OP == OP_GEN_MRT) {
        if constexpr (Q == 19) gen_mrt19<T>(g, p);
        else gen_mrt27<T>(g, p);
    }
}

}  // namespace lbm
