/*
 * lbm_oracle.c — plain, slow, obviously correct fp64 CPU oracle of the fused lattice
 * Boltzmann stream–collide time step (Bauer, Köstler, Rüde, arXiv 2001.11806 "lbmpy").
 *
 * TEST INFRASTRUCTURE ONLY. Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library. The product path
 * (paper_2001_11806_b200/) shares no code with it and never calls it.
 *
 * Citations: P:<n> = /root/reference/PAPER.md line n; G<k>/O<k> = SURVEY.md §8(c) readings
 * (restated in DESIGN.md).
 *
 *   Eq. (1)  SRT/BGK
 *   Eq. (2)  density / velocity
 *   Eq. (3)  discrete equilibrium (2nd order, compressible rho0 = rho)
 *   Eq. (4)  MRT step f' = M^-1 [S m_eq + (I-S) M f]
 *   TRT as MRT with even/odd rates
 *   Eq. (9)  cumulant generating function    P:398-402 (multi-step moments->cumulants P:409-415)
 *   UBB (link-wise, fluid->boundary c)       P:517-537, reading G8
 *   Two-array pull / push, AA pattern
 *
 * Layout: SoA, element (q, z, y, x) at q*Sq + (z+g)*ny*nx + y*nx + x, x fastest, with
 * g = 1 ghost plane per z side when cfg->zghost (slab mode) and g = 0 otherwise; x and y
 * always wrap (non-periodic axes carry wall cells on their faces, G9); z wraps when g = 0.
 *
 * Floating point: plain C, fp64, no FMA contraction (-ffp-contract=off), OpenMP static
 * schedule over z (the paper's scheme).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define ORA_SRT 0
#define ORA_TRT 1
#define ORA_MRT 2
#define ORA_CUMULANT 3
#define ORA_IDENTITY 4
#define ORA_SMAGORINSKY 5
#define ORA_KBC 6
#define ORA_KBC_EXACT 7 /* KBC with the entropy maximised exactly by Newton's method */

#define FLAG_FLUID 0
#define FLAG_NOSLIP 1
#define FLAG_UBB 2

typedef struct {
    int32_t Q;          /* 19 or 27 */
    int32_t op;         /* ORA_* */
    int64_t nx, ny, nz; /* local extent without ghost planes */
    int32_t zghost;     /* 1: storage has planes z = -1 and z = nz (slab mode) */
    int32_t nthreads;   /* OpenMP threads (<= 0: runtime default) */
    double rates[8];    /* SRT [w]; TRT [we, wo]; MRT unused (S below); CUMULANT [ws, wb, w3, w4, w5, w6] */
    double force[3];    /* Guo body force (SRT/TRT) */
    double ubb_u[3];    /* UBB wall velocity */
    double ubb_rho;     /* UBB reference density rho_w (G8: 1) */
    const double *M;    /* MRT: Q x Q moment matrix, row-major (M_kq = P_k(c_q)) */
    const double *Minv; /* MRT: its inverse */
    const double *S;    /* MRT: Q relaxation rates (diagonal of S); KBC: per-row part, 0 conserved,
                           1 = shear (s), 2 = higher order (h) */
    int32_t eq_kind;    /* ORA_EQ_*: which equilibrium SRT/TRT/MRT relax to */
    const int32_t *mono_exp;  /* ORA_EQ_MOMENT_MATCHED: Q x 3 exponents of the monomial basis */
    const double *Mmono_inv;  /* ... and the inverse of its moment matrix M_kq = c_q^e_k (row-major) */
    const double *wall_u;     /* NULL, or the wall velocity of every storage cell, [3][storage cells]:
                                 a UBB cell uses its own entry instead of ubb_u ("custom boundary data
                                 ... e.g. the wall velocity", per boundary link) */
} ora_cfg;

#define ORA_EQ_COMPRESSIBLE 0    /* Eq. (3) with rho0 = rho */
#define ORA_EQ_INCOMPRESSIBLE 1  /* Eq. (3) with rho0 = 1 (He & Luo) */
#define ORA_EQ_MOMENT_MATCHED 2  /* moments of the continuous Maxwellian Eq. (7)-(8), truncated at 2nd
                                    order in u, mapped to populations with M^-1 */

/* ------------------------------------------------------------------------------------ */
/* Stencils (ordering G10: centre, then |c|_1, then lexicographic -1<0<1).     */
/* ------------------------------------------------------------------------------------ */
typedef struct {
    int Q;
    int c[27][3];
    double w[27];
    int opp[27];
} ora_stencil_t;

static int lex_less(const int *a, const int *b) {
    int la = abs(a[0]) + abs(a[1]) + abs(a[2]);
    int lb = abs(b[0]) + abs(b[1]) + abs(b[2]);
    if (la != lb) return la < lb;
    for (int i = 0; i < 3; ++i)
        if (a[i] != b[i]) return a[i] < b[i];
    return 0;
}

static void build_stencil(int Q, ora_stencil_t *s) {
    int n = 0;
    for (int x = -1; x <= 1; ++x)
        for (int y = -1; y <= 1; ++y)
            for (int z = -1; z <= 1; ++z) {
                int l1 = abs(x) + abs(y) + abs(z);
                if (Q == 19 && l1 == 3) continue; /* D3Q19 = D3Q27 minus the 8 corners */
                s->c[n][0] = x; s->c[n][1] = y; s->c[n][2] = z;
                ++n;
            }
    /* insertion sort into the ABI order */
    for (int i = 1; i < n; ++i) {
        int t[3] = {s->c[i][0], s->c[i][1], s->c[i][2]};
        int j = i - 1;
        while (j >= 0 && lex_less(t, s->c[j])) {
            memcpy(s->c[j + 1], s->c[j], sizeof(t));
            --j;
        }
        memcpy(s->c[j + 1], t, sizeof(t));
    }
    s->Q = n;
    for (int i = 0; i < n; ++i) {
        int c2 = s->c[i][0] * s->c[i][0] + s->c[i][1] * s->c[i][1] + s->c[i][2] * s->c[i][2];
        if (Q == 19) s->w[i] = (c2 == 0) ? 1.0 / 3.0 : (c2 == 1) ? 1.0 / 18.0 : 1.0 / 36.0;
        else s->w[i] = (c2 == 0) ? 8.0 / 27.0 : (c2 == 1) ? 2.0 / 27.0 : (c2 == 2) ? 1.0 / 54.0 : 1.0 / 216.0;
        for (int j = 0; j < n; ++j)
            if (s->c[j][0] == -s->c[i][0] && s->c[j][1] == -s->c[i][1] && s->c[j][2] == -s->c[i][2])
                s->opp[i] = j;
    }
}

void ora_stencil(int Q, int *c_out, double *w_out, int *opp_out) {
    ora_stencil_t s;
    build_stencil(Q, &s);
    for (int i = 0; i < s.Q; ++i) {
        for (int d = 0; d < 3; ++d) c_out[3 * i + d] = s.c[i][d];
        w_out[i] = s.w[i];
        opp_out[i] = s.opp[i];
    }
}

/* ------------------------------------------------------------------------------------ */
/* Macroscopic values Eq. (2) and equilibrium Eq. (3).                                     */
/* ------------------------------------------------------------------------------------ */

/* Eq. (2): rho = sum_q f_q; u = (sum_q c_q f_q + fsign * F/2) / rho0 with rho0 = rho (compressible)
 * or rho0 = 1 (incompressible). fsign = +1 for a pre-collision state (Guo), -1 for a
 * post-collision state (G11). */
static void macroscopic_eq(const ora_stencil_t *s, const double *f, const double *F, double fsign, int incompressible,
                           double *rho, double u[3]) {
    double r = 0.0, j[3] = {0.0, 0.0, 0.0};
    for (int q = 0; q < s->Q; ++q) {
        r += f[q];
        for (int d = 0; d < 3; ++d) j[d] += s->c[q][d] * f[q];
    }
    double rho0 = incompressible ? 1.0 : r;
    for (int d = 0; d < 3; ++d) u[d] = (j[d] + fsign * 0.5 * F[d]) / rho0;
    *rho = r;
}
static void macroscopic(const ora_stencil_t *s, const double *f, const double *F, double fsign,
                        double *rho, double u[3]) {
    macroscopic_eq(s, f, F, fsign, 0, rho, u);
}

/* Eq. (3), second order, compressible: f_eq = w rho [1 + c.u/cs2 + (c.u)^2/(2 cs4) - u.u/(2 cs2)]
 * with cs2 = 1/3 (G1). */
static void equilibrium(const ora_stencil_t *s, double rho, const double u[3], double *feq) {
    const double cs2 = 1.0 / 3.0;
    double uu = u[0] * u[0] + u[1] * u[1] + u[2] * u[2];
    for (int q = 0; q < s->Q; ++q) {
        double cu = s->c[q][0] * u[0] + s->c[q][1] * u[1] + s->c[q][2] * u[2];
        double second = 0.0; /* (1/(2 cs^4)) u_a u_b (c_a c_b - cs2 delta_ab) */
        for (int a = 0; a < 3; ++a)
            for (int b = 0; b < 3; ++b)
                second += u[a] * u[b] * (s->c[q][a] * s->c[q][b] - (a == b ? cs2 : 0.0));
        second /= 2.0 * cs2 * cs2;
        feq[q] = s->w[q] * rho + s->w[q] * rho * (cu / cs2 + second);
    }
    (void)uu;
}

/* Eq. (3), second order, with reference density rho0: f_eq = w rho + w rho0 [c.u/cs2 +
 * u_a u_b (c_a c_b - cs2 delta_ab) / (2 cs4)]. rho0 = rho gives equilibrium() above. */
static void equilibrium_rho0(const ora_stencil_t *s, double rho, double rho0, const double u[3], double *feq) {
    const double cs2 = 1.0 / 3.0;
    for (int q = 0; q < s->Q; ++q) {
        double cu = s->c[q][0] * u[0] + s->c[q][1] * u[1] + s->c[q][2] * u[2];
        double second = 0.0;
        for (int a = 0; a < 3; ++a)
            for (int b = 0; b < 3; ++b)
                second += u[a] * u[b] * (s->c[q][a] * s->c[q][b] - (a == b ? cs2 : 0.0));
        second /= 2.0 * cs2 * cs2;
        feq[q] = s->w[q] * rho + s->w[q] * rho0 * (cu / cs2 + second);
    }
}

/* Moment-matched equilibrium: the raw moment of basis monomial x^a y^b z^c of the
 * continuous Maxwellian Eq. (7) is rho prod_d mu_{e_d}(u_d) with mu_0 = 1, mu_1 = u, mu_2 = cs2 + u^2
 * (the Gaussian factorises over the axes); the product is expanded in powers of u and truncated after
 * 2nd order ("Optionally the moments can be truncated to a given order in u"); the
 * populations are M^-1 m_eq. */
static void equilibrium_moment_matched(const ora_cfg *cfg, const ora_stencil_t *s, double rho, const double u[3],
                                       double *feq) {
    const double cs2 = 1.0 / 3.0;
    double m[27];
    for (int k = 0; k < s->Q; ++k) {
        /* factor d as coefficients of u_d^0, u_d^1, u_d^2 */
        double fac[3][3];
        for (int d = 0; d < 3; ++d) {
            int e = cfg->mono_exp[3 * k + d];
            fac[d][0] = (e == 0) ? 1.0 : (e == 2) ? cs2 : 0.0;
            fac[d][1] = (e == 1) ? u[d] : 0.0;
            fac[d][2] = (e == 2) ? u[d] * u[d] : 0.0;
        }
        double v = 0.0;
        for (int i = 0; i < 3; ++i)
            for (int j = 0; j < 3; ++j)
                for (int l = 0; l < 3; ++l)
                    if (i + j + l <= 2) v += fac[0][i] * fac[1][j] * fac[2][l];
        m[k] = rho * v;
    }
    for (int q = 0; q < s->Q; ++q) {
        double v = 0.0;
        for (int k = 0; k < s->Q; ++k) v += cfg->Mmono_inv[q * s->Q + k] * m[k];
        feq[q] = v;
    }
}

/* The equilibrium of the configured kind (cfg->eq_kind). */
static void equilibrium_cfg(const ora_cfg *cfg, const ora_stencil_t *s, double rho, const double u[3], double *feq) {
    switch (cfg->eq_kind) {
        case ORA_EQ_INCOMPRESSIBLE: equilibrium_rho0(s, rho, 1.0, u, feq); break;
        case ORA_EQ_MOMENT_MATCHED: equilibrium_moment_matched(cfg, s, rho, u, feq); break;
        default: equilibrium(s, rho, u, feq); break;
    }
}
static int incompressible(const ora_cfg *cfg) { return cfg->eq_kind == ORA_EQ_INCOMPRESSIBLE; }

/* Product equilibrium (G2): the fixed point of the cumulant collision for D3Q27,
 * prod_axes p(c_i; u_i), p(+-1) = (1/3 + u^2 +- u)/2, p(0) = 2/3 - u^2. */
static void product_equilibrium(const ora_stencil_t *s, double rho, const double u[3], double *feq) {
    for (int q = 0; q < s->Q; ++q) {
        double v = rho;
        for (int d = 0; d < 3; ++d) {
            int c = s->c[q][d];
            double p = (c == 0) ? (2.0 / 3.0 - u[d] * u[d]) : 0.5 * (1.0 / 3.0 + u[d] * u[d] + c * u[d]);
            v *= p;
        }
        feq[q] = v;
    }
}

/* ------------------------------------------------------------------------------------ */
/* Collision operators                                                                     */
/* ------------------------------------------------------------------------------------ */

/* Guo source (G4), split by moment parity:
 * S_q = (1 - wo/2) w_q 3 (c_q.F) + (1 - we/2) w_q [9 (c_q.u)(c_q.F) - 3 u.F]. */
static double guo_source(const ora_stencil_t *s, int q, const double u[3], const double F[3],
                         double we, double wo) {
    double cF = s->c[q][0] * F[0] + s->c[q][1] * F[1] + s->c[q][2] * F[2];
    double cu = s->c[q][0] * u[0] + s->c[q][1] * u[1] + s->c[q][2] * u[2];
    double uF = u[0] * F[0] + u[1] * F[1] + u[2] * F[2];
    return (1.0 - wo / 2.0) * s->w[q] * 3.0 * cF + (1.0 - we / 2.0) * s->w[q] * (9.0 * cu * cF - 3.0 * uF);
}

static int has_force(const ora_cfg *cfg) {
    return cfg->force[0] != 0.0 || cfg->force[1] != 0.0 || cfg->force[2] != 0.0;
}

/* SRT, Eq. (1): f* = omega f_eq + (1 - omega) f (+ Guo source with we = wo = omega). */
static void collide_srt(const ora_cfg *cfg, const ora_stencil_t *s, const double *f, double *out) {
    double rho, u[3], feq[27];
    double w = cfg->rates[0];
    macroscopic_eq(s, f, cfg->force, +1.0, incompressible(cfg), &rho, u);
    equilibrium_cfg(cfg, s, rho, u, feq);
    for (int q = 0; q < s->Q; ++q) {
        out[q] = w * feq[q] + (1.0 - w) * f[q];
        if (has_force(cfg)) out[q] += guo_source(s, q, u, cfg->force, w, w);
    }
}

/* TRT: f+- = (f_q +- f_qbar)/2, f* = f - we (f+ - feq+) - wo (f- - feq-) + S_q. */
static void collide_trt(const ora_cfg *cfg, const ora_stencil_t *s, const double *f, double *out) {
    double rho, u[3], feq[27];
    double we = cfg->rates[0], wo = cfg->rates[1];
    macroscopic_eq(s, f, cfg->force, +1.0, incompressible(cfg), &rho, u);
    equilibrium_cfg(cfg, s, rho, u, feq);
    for (int q = 0; q < s->Q; ++q) {
        int qb = s->opp[q];
        double fp = 0.5 * (f[q] + f[qb]), fm = 0.5 * (f[q] - f[qb]);
        double ep = 0.5 * (feq[q] + feq[qb]), em = 0.5 * (feq[q] - feq[qb]);
        out[q] = f[q] - we * (fp - ep) - wo * (fm - em);
        if (has_force(cfg)) out[q] += guo_source(s, q, u, cfg->force, we, wo);
    }
}

/* MRT, Eq. (4): f* = M^-1 [ S m_eq + (I - S) M f ], m_eq = M f_eq (Eq. 3; G1). */
static void collide_mrt(const ora_cfg *cfg, const ora_stencil_t *s, const double *f, double *out) {
    int Q = s->Q;
    double rho, u[3], feq[27], m[27], meq[27], mp[27];
    macroscopic_eq(s, f, cfg->force, +1.0, incompressible(cfg), &rho, u);
    equilibrium_cfg(cfg, s, rho, u, feq);
    for (int k = 0; k < Q; ++k) {
        m[k] = 0.0;
        meq[k] = 0.0;
        for (int q = 0; q < Q; ++q) {
            m[k] += cfg->M[k * Q + q] * f[q];
            meq[k] += cfg->M[k * Q + q] * feq[q];
        }
        mp[k] = cfg->S[k] * meq[k] + (1.0 - cfg->S[k]) * m[k];
    }
    for (int q = 0; q < Q; ++q) {
        out[q] = 0.0;
        for (int k = 0; k < Q; ++k) out[q] += cfg->Minv[q * Q + k] * mp[k];
    }
}

/* ---- Cumulant (O5): truncated power series in Q[xi]/(xi_x^3, xi_y^3, xi_z^3). ---------- */
/* A series is 27 coefficients indexed a*9 + b*3 + c for xi_x^a xi_y^b xi_z^c, a,b,c <= 2. */
static void ser_mul(const double *A, const double *B, double *C) {
    double t[27];
    for (int i = 0; i < 27; ++i) t[i] = 0.0;
    for (int a1 = 0; a1 < 3; ++a1)
        for (int b1 = 0; b1 < 3; ++b1)
            for (int c1 = 0; c1 < 3; ++c1) {
                double x = A[a1 * 9 + b1 * 3 + c1];
                if (x == 0.0) continue;
                for (int a2 = 0; a1 + a2 < 3; ++a2)
                    for (int b2 = 0; b1 + b2 < 3; ++b2)
                        for (int c2 = 0; c1 + c2 < 3; ++c2)
                            t[(a1 + a2) * 9 + (b1 + b2) * 3 + (c1 + c2)] += x * B[a2 * 9 + b2 * 3 + c2];
            }
    for (int i = 0; i < 27; ++i) C[i] = t[i];
}

static const double fact3[3] = {1.0, 1.0, 2.0};

/* c^e for a lattice velocity component c in {-1, 0, 1} and e in {0, 1, 2} (0^0 = 1): exact, the
 * value pow(c, e) returns, by repeated multiplication. */
static double ipow(int c, int e) {
    double v = 1.0;
    for (int k = 0; k < e; ++k) v *= (double)c;
    return v;
}

/* ln(1 + X) = sum_{n=1}^{6} (-1)^{n+1} X^n / n, exact in the truncated ring (X^7 = 0). */
static void ser_log1p(const double *X, double *K) {
    double P[27];
    memcpy(P, X, sizeof(P));
    for (int i = 0; i < 27; ++i) K[i] = X[i];
    for (int n = 2; n <= 6; ++n) {
        ser_mul(P, X, P);
        double sgn = (n % 2 == 0) ? -1.0 : 1.0;
        for (int i = 0; i < 27; ++i) K[i] += sgn * P[i] / n;
    }
}

/* exp(K) = sum_{n=0}^{6} K^n / n! for K without constant term (K^7 = 0). */
static void ser_exp(const double *K, double *E) {
    double P[27];
    memcpy(P, K, sizeof(P));
    for (int i = 0; i < 27; ++i) E[i] = K[i];
    E[0] += 1.0;
    double nf = 1.0;
    for (int n = 2; n <= 6; ++n) {
        ser_mul(P, K, P);
        nf *= n;
        for (int i = 0; i < 27; ++i) E[i] += P[i] / nf;
    }
}

/* Cumulants kappa_abc of f (O5 steps 1-4). kappa[a*9+b*3+c]; returns rho. */
static double cumulants(const ora_stencil_t *s, const double *f, double *kappa) {
    double m[27], Mser[27];
    for (int a = 0; a < 3; ++a)
        for (int b = 0; b < 3; ++b)
            for (int c = 0; c < 3; ++c) {
                double v = 0.0; /* raw moment m_abc = sum_q f_q cx^a cy^b cz^c (Eq. 5) */
                for (int q = 0; q < s->Q; ++q)
                    v += f[q] * ipow(s->c[q][0], a) * ipow(s->c[q][1], b) * ipow(s->c[q][2], c);
                m[a * 9 + b * 3 + c] = v;
            }
    double rho = m[0];
    for (int a = 0; a < 3; ++a)
        for (int b = 0; b < 3; ++b)
            for (int c = 0; c < 3; ++c)
                Mser[a * 9 + b * 3 + c] = m[a * 9 + b * 3 + c] / (rho * fact3[a] * fact3[b] * fact3[c]);
    Mser[0] -= 1.0; /* X = M - 1 */
    double K[27];
    ser_log1p(Mser, K);
    for (int a = 0; a < 3; ++a)
        for (int b = 0; b < 3; ++b)
            for (int c = 0; c < 3; ++c)
                kappa[a * 9 + b * 3 + c] = fact3[a] * fact3[b] * fact3[c] * K[a * 9 + b * 3 + c];
    return rho;
}

/* Inverse of cumulants(): f from (rho, kappa) (O5 steps 6-7). */
static void from_cumulants(const ora_stencil_t *s, double rho, const double *kappa, double *f) {
    double K[27], E[27], m[27];
    for (int a = 0; a < 3; ++a)
        for (int b = 0; b < 3; ++b)
            for (int c = 0; c < 3; ++c)
                K[a * 9 + b * 3 + c] = kappa[a * 9 + b * 3 + c] / (fact3[a] * fact3[b] * fact3[c]);
    K[0] = 0.0;
    ser_exp(K, E);
    for (int a = 0; a < 3; ++a)
        for (int b = 0; b < 3; ++b)
            for (int c = 0; c < 3; ++c)
                m[a * 9 + b * 3 + c] = rho * fact3[a] * fact3[b] * fact3[c] * E[a * 9 + b * 3 + c];
    /* (V x V x V)^-1 m: per axis f(-1) = (m2 - m1)/2, f(0) = m0 - m2, f(1) = (m2 + m1)/2. */
    for (int q = 0; q < s->Q; ++q) {
        double v = 0.0;
        for (int a = 0; a < 3; ++a)
            for (int b = 0; b < 3; ++b)
                for (int c = 0; c < 3; ++c) {
                    int e[3] = {a, b, c};
                    double coef = 1.0;
                    for (int d = 0; d < 3; ++d) {
                        int cd = s->c[q][d];
                        double k; /* weight of moment order e[d] in f(cd) */
                        if (cd == 0) k = (e[d] == 0) ? 1.0 : (e[d] == 2) ? -1.0 : 0.0;
                        else if (cd == 1) k = (e[d] == 0) ? 0.0 : 0.5;
                        else k = (e[d] == 0) ? 0.0 : (e[d] == 1) ? -0.5 : 0.5;
                        coef *= k;
                    }
                    v += coef * m[a * 9 + b * 3 + c];
                }
        f[q] = v;
    }
}

/* The populations whose raw moments of the monomial basis are m[a*9 + b*3 + c]:
 * D3Q27 per axis (V x V x V)^-1 as in from_cumulants(); other stencils (D3Q19) f = M^-1 m over the
 * basis exponents (cfg->mono_exp, cfg->Mmono_inv). Moments of the dropped monomials are ignored: for
 * D3Q19 they vanish identically. */
static void populations_from_moments(const ora_cfg *cfg, const ora_stencil_t *s, const double *m, double *f) {
    if (s->Q == 27) {
        for (int q = 0; q < 27; ++q) {
            double v = 0.0;
            for (int a = 0; a < 3; ++a)
                for (int b = 0; b < 3; ++b)
                    for (int c = 0; c < 3; ++c) {
                        int e[3] = {a, b, c};
                        double coef = 1.0;
                        for (int d = 0; d < 3; ++d) {
                            int cd = s->c[q][d];
                            double k;
                            if (cd == 0) k = (e[d] == 0) ? 1.0 : (e[d] == 2) ? -1.0 : 0.0;
                            else if (cd == 1) k = (e[d] == 0) ? 0.0 : 0.5;
                            else k = (e[d] == 0) ? 0.0 : (e[d] == 1) ? -0.5 : 0.5;
                            coef *= k;
                        }
                        v += coef * m[a * 9 + b * 3 + c];
                    }
            f[q] = v;
        }
        return;
    }
    for (int q = 0; q < s->Q; ++q) {
        double v = 0.0;
        for (int k = 0; k < s->Q; ++k) {
            const int32_t *e = cfg->mono_exp + 3 * k;
            v += cfg->Mmono_inv[q * s->Q + k] * m[e[0] * 9 + e[1] * 3 + e[2]];
        }
        f[q] = v;
    }
}

/* Inverse of cumulants() on any stencil: moments from exp(K) (O5 step 6), populations from the
 * moments of the basis monomials. */
static void from_cumulants_cfg(const ora_cfg *cfg, const ora_stencil_t *s, double rho, const double *kappa, double *f) {
    double K[27], E[27], m[27];
    for (int a = 0; a < 3; ++a)
        for (int b = 0; b < 3; ++b)
            for (int c = 0; c < 3; ++c)
                K[a * 9 + b * 3 + c] = kappa[a * 9 + b * 3 + c] / (fact3[a] * fact3[b] * fact3[c]);
    K[0] = 0.0;
    ser_exp(K, E);
    for (int a = 0; a < 3; ++a)
        for (int b = 0; b < 3; ++b)
            for (int c = 0; c < 3; ++c)
                m[a * 9 + b * 3 + c] = rho * fact3[a] * fact3[b] * fact3[c] * E[a * 9 + b * 3 + c];
    populations_from_moments(cfg, s, m, f);
}

/* Maxwellian-moment equilibrium (G2 generalised): the populations whose basis moments are the raw
 * moments of the continuous Maxwellian Eq. (7)-(8), rho prod_d mu_{e_d}(u_d) (NOT truncated). For
 * D3Q27 this is the product equilibrium; it is the fixed point of the cumulant collision on any
 * stencil (kappa_eq = (ln rho, u, cs2 delta, 0, ...)). */
static void maxwellian_equilibrium(const ora_cfg *cfg, const ora_stencil_t *s, double rho, const double u[3], double *feq) {
    if (s->Q == 27) {
        product_equilibrium(s, rho, u, feq);
        return;
    }
    double m[27];
    for (int a = 0; a < 3; ++a)
        for (int b = 0; b < 3; ++b)
            for (int c = 0; c < 3; ++c) {
                int e[3] = {a, b, c};
                double v = rho;
                for (int d = 0; d < 3; ++d) v *= (e[d] == 0) ? 1.0 : (e[d] == 1) ? u[d] : (1.0 / 3.0 + u[d] * u[d]);
                m[a * 9 + b * 3 + c] = v;
            }
    populations_from_moments(cfg, s, m, feq);
}

/* Cumulant collision (O5 step 5, G7 rates): order 1 unchanged; 2nd-order trace
 * T -> T + wb (3 cs2 - T); deviator and off-diagonals -> (1 - ws); order n >= 3 -> (1 - w_n). */
static void collide_cumulant(const ora_cfg *cfg, const ora_stencil_t *s, const double *f, double *out) {
    double kap[27];
    double rho = cumulants(s, f, kap);
    const double ws = cfg->rates[0], wb = cfg->rates[1];
    const double cs2 = 1.0 / 3.0;
    int i200 = 18, i020 = 6, i002 = 2;
    double T = kap[i200] + kap[i020] + kap[i002];
    double Tn = T + wb * (3.0 * cs2 - T);
    double d200 = kap[i200] - T / 3.0, d020 = kap[i020] - T / 3.0, d002 = kap[i002] - T / 3.0;
    kap[i200] = Tn / 3.0 + (1.0 - ws) * d200;
    kap[i020] = Tn / 3.0 + (1.0 - ws) * d020;
    kap[i002] = Tn / 3.0 + (1.0 - ws) * d002;
    kap[9 + 3] *= (1.0 - ws);  /* kappa_110 */
    kap[9 + 1] *= (1.0 - ws);  /* kappa_101 */
    kap[3 + 1] *= (1.0 - ws);  /* kappa_011 */
    for (int a = 0; a < 3; ++a)
        for (int b = 0; b < 3; ++b)
            for (int c = 0; c < 3; ++c) {
                int n = a + b + c;
                if (n >= 3) kap[a * 9 + b * 3 + c] *= (1.0 - cfg->rates[n - 1]); /* w3..w6 = rates[2..5] */
            }
    from_cumulants_cfg(cfg, s, rho, kap, out);
}

/* Smagorinsky SRT (Eqs. 11-14): nu_t = (C_S Delta)^2 |S|, Delta = 1,
 * |S| = sqrt(2 S_ij S_ij), S_ij = -(3 omega / (2 rho)) Pi^neq_ij, Pi^neq = sum_q c c (f - f_eq),
 * omega = 2 / (6 C_S^2 |S| + 6 nu_0 + 1). Solving the two equations for omega (the step the paper
 * leaves to sympy): with tau_0 = 1/omega_0 = 3 nu_0 + 1/2 and P = sqrt(2 Pi:Pi),
 * (9 C^2 P / rho) omega^2 + 2 tau_0 omega - 2 = 0, whose positive root is
 * omega = 2 / (tau_0 + sqrt(tau_0^2 + 18 C^2 P / rho)). rates = [omega_0, C_S]. */
static double smagorinsky_omega(const ora_stencil_t *s, const double *f, double rho, const double *feq,
                                double omega0, double cs) {
    double Pi[3][3];
    for (int a = 0; a < 3; ++a)
        for (int b = 0; b < 3; ++b) {
            double v = 0.0;
            for (int q = 0; q < s->Q; ++q) v += s->c[q][a] * s->c[q][b] * (f[q] - feq[q]);
            Pi[a][b] = v;
        }
    double pp = 0.0;
    for (int a = 0; a < 3; ++a)
        for (int b = 0; b < 3; ++b) pp += Pi[a][b] * Pi[a][b];
    double P = sqrt(2.0 * pp);
    double tau0 = 1.0 / omega0;
    return 2.0 / (tau0 + sqrt(tau0 * tau0 + 18.0 * cs * cs * P / rho));
}

static void collide_smagorinsky(const ora_cfg *cfg, const ora_stencil_t *s, const double *f, double *out) {
    double rho, u[3], feq[27];
    macroscopic(s, f, cfg->force, +1.0, &rho, u);
    equilibrium(s, rho, u, feq);
    double w = smagorinsky_omega(s, f, rho, feq, cfg->rates[0], cfg->rates[1]);
    for (int q = 0; q < s->Q; ++q) out[q] = w * feq[q] + (1.0 - w) * f[q]; /* Eq. (1) with the local omega */
}

/* KBC entropic operator: with an MRT basis split into shear moments (s) and the other
 * non-conserved moments (h), f = f_eq + Delta_s + Delta_h and (Eq. 16) f' = f - w_s Delta_s - w_h Delta_h;
 * w_h from the linearised entropy condition (Eq. 19): w_h = 1 + (1 - w_s) <Ds,Dh>_E / <Dh,Dh>_E with
 * <a,b>_E = sum_q a_q b_q / f_eq,q. Delta_s = M^-1 [s rows of M(f - f_eq)], Delta_h likewise.
 * rates = [w_s]. */
static void collide_kbc(const ora_cfg *cfg, const ora_stencil_t *s, const double *f, double *out) {
    int Q = s->Q;
    double rho, u[3], feq[27], dm[27], ms[27], mh[27], ds[27], dh[27];
    macroscopic(s, f, cfg->force, +1.0, &rho, u);
    equilibrium(s, rho, u, feq);
    for (int k = 0; k < Q; ++k) {
        dm[k] = 0.0;
        for (int q = 0; q < Q; ++q) dm[k] += cfg->M[k * Q + q] * (f[q] - feq[q]);
        ms[k] = (cfg->S[k] == 1.0) ? dm[k] : 0.0;
        mh[k] = (cfg->S[k] == 2.0) ? dm[k] : 0.0;
    }
    for (int q = 0; q < Q; ++q) {
        ds[q] = 0.0;
        dh[q] = 0.0;
        for (int k = 0; k < Q; ++k) {
            ds[q] += cfg->Minv[q * Q + k] * ms[k];
            dh[q] += cfg->Minv[q * Q + k] * mh[k];
        }
    }
    double sh = 0.0, hh = 0.0;
    for (int q = 0; q < Q; ++q) {
        sh += ds[q] * dh[q] / feq[q];
        hh += dh[q] * dh[q] / feq[q];
    }
    double ws = cfg->rates[0];
    double wh = (hh > 0.0) ? 1.0 + (1.0 - ws) * sh / hh : 1.0;
    for (int q = 0; q < Q; ++q) out[q] = f[q] - ws * ds[q] - wh * dh[q];
}

/* KBC with exact entropy maximisation ("This condition could be solved numerically in
 * every cell using Newton's method"; the "more costly but also more general numerical
 * maximization procedure for the post-collision state entropy, which is based on Newton's method").
 * f'(w_h) = f - w_s Ds - w_h Dh (Eq. 16); maximise S(w_h) = -sum f' ln(f'/f_eq) (Eq. 17): solve
 * g(w) = sum_q Dh_q [ln(f'_q(w)/f_eq,q) + 1] = 0 with g'(w) = -sum_q Dh_q^2 / f'_q(w), starting from the
 * linearised w_h of Eq. (19). Iterates until |dw| <= 1e-14 (at most 50 steps); if a step would make a
 * population non-positive it is halved. Same parts Ds, Dh as collide_kbc (G17). */
static void collide_kbc_exact(const ora_cfg *cfg, const ora_stencil_t *s, const double *f, double *out) {
    int Q = s->Q;
    double rho, u[3], feq[27], dm[27], ms[27], mh[27], ds[27], dh[27];
    macroscopic(s, f, cfg->force, +1.0, &rho, u);
    equilibrium(s, rho, u, feq);
    for (int k = 0; k < Q; ++k) {
        dm[k] = 0.0;
        for (int q = 0; q < Q; ++q) dm[k] += cfg->M[k * Q + q] * (f[q] - feq[q]);
        ms[k] = (cfg->S[k] == 1.0) ? dm[k] : 0.0;
        mh[k] = (cfg->S[k] == 2.0) ? dm[k] : 0.0;
    }
    for (int q = 0; q < Q; ++q) {
        ds[q] = 0.0;
        dh[q] = 0.0;
        for (int k = 0; k < Q; ++k) {
            ds[q] += cfg->Minv[q * Q + k] * ms[k];
            dh[q] += cfg->Minv[q * Q + k] * mh[k];
        }
    }
    double sh = 0.0, hh = 0.0;
    for (int q = 0; q < Q; ++q) {
        sh += ds[q] * dh[q] / feq[q];
        hh += dh[q] * dh[q] / feq[q];
    }
    double ws = cfg->rates[0];
    double w = (hh > 0.0) ? 1.0 + (1.0 - ws) * sh / hh : 1.0;
    if (hh > 0.0) {
        for (int it = 0; it < 50; ++it) {
            double g = 0.0, gp = 0.0;
            for (int q = 0; q < Q; ++q) {
                double fp = f[q] - ws * ds[q] - w * dh[q];
                g += dh[q] * (log(fp / feq[q]) + 1.0);
                gp -= dh[q] * dh[q] / fp;
            }
            double step = g / gp;
            double wn = w - step;
            for (int tries = 0; tries < 60; ++tries) { /* keep every population positive */
                int ok = 1;
                for (int q = 0; q < Q; ++q)
                    if (f[q] - ws * ds[q] - wn * dh[q] <= 0.0) ok = 0;
                if (ok) break;
                step *= 0.5;
                wn = w - step;
            }
            w = wn;
            if (fabs(step) <= 1e-14) break;
        }
    }
    for (int q = 0; q < Q; ++q) out[q] = f[q] - ws * ds[q] - w * dh[q];
}

static void collide(const ora_cfg *cfg, const ora_stencil_t *s, const double *f, double *out) {
    switch (cfg->op) {
        case ORA_SMAGORINSKY: collide_smagorinsky(cfg, s, f, out); break;
        case ORA_KBC: collide_kbc(cfg, s, f, out); break;
        case ORA_KBC_EXACT: collide_kbc_exact(cfg, s, f, out); break;
        case ORA_SRT: collide_srt(cfg, s, f, out); break;
        case ORA_TRT: collide_trt(cfg, s, f, out); break;
        case ORA_MRT: collide_mrt(cfg, s, f, out); break;
        case ORA_CUMULANT: collide_cumulant(cfg, s, f, out); break;
        default: for (int q = 0; q < s->Q; ++q) out[q] = f[q]; break; /* IDENTITY */
    }
}

/* ------------------------------------------------------------------------------------ */
/* Addressing                                                                              */
/* ------------------------------------------------------------------------------------ */
static inline int64_t plane_cells(const ora_cfg *cfg) {
    return (cfg->nz + 2 * cfg->zghost) * cfg->ny * cfg->nx;
}
static inline int64_t wrap(int64_t i, int64_t n) { return ((i % n) + n) % n; }
/* storage cell index of local (x, y, z); x, y wrap; z wraps unless ghost planes exist */
static inline int64_t cell(const ora_cfg *cfg, int64_t x, int64_t y, int64_t z) {
    x = wrap(x, cfg->nx);
    y = wrap(y, cfg->ny);
    if (!cfg->zghost) z = wrap(z, cfg->nz);
    return ((z + cfg->zghost) * cfg->ny + y) * cfg->nx + x;
}

/* UBB term 6 w_q rho_w c_q.u_w of direction q for the wall cell `wall` (G8); u_w = ubb_u, or the
 * wall cell's own velocity when a wall velocity field is given. */
static double ubb_term_at(const ora_cfg *cfg, const ora_stencil_t *s, int q, int64_t wall) {
    double uw[3] = {cfg->ubb_u[0], cfg->ubb_u[1], cfg->ubb_u[2]};
    if (cfg->wall_u) {
        int64_t n = plane_cells(cfg);
        for (int d = 0; d < 3; ++d) uw[d] = cfg->wall_u[d * n + wall];
    }
    double cu = s->c[q][0] * uw[0] + s->c[q][1] * uw[1] + s->c[q][2] * uw[2];
    return 6.0 * s->w[q] * cfg->ubb_rho * cu;
}

/* Pull-streaming value of direction q at fluid cell (x,y,z) from array `a` (O6):
 * neighbour n = x - c_q; fluid -> a_q(n); NOSLIP -> a_qbar(x); UBB -> a_qbar(x) + 6 w rho_w c.u_w */
static double pull_value(const ora_cfg *cfg, const ora_stencil_t *s, const double *a, const uint8_t *flags,
                         int64_t x, int64_t y, int64_t z, int q) {
    int64_t Sq = plane_cells(cfg);
    int64_t self = cell(cfg, x, y, z);
    int64_t nb = cell(cfg, x - s->c[q][0], y - s->c[q][1], z - s->c[q][2]);
    uint8_t fl = flags ? flags[nb] : FLAG_FLUID;
    if (fl == FLAG_FLUID) return a[q * Sq + nb];
    double v = a[s->opp[q] * Sq + self];
    if (fl == FLAG_UBB) v += ubb_term_at(cfg, s, q, nb);
    return v;
}

static void set_threads(const ora_cfg *cfg) {
#ifdef _OPENMP
    extern void omp_set_num_threads(int);
    if (cfg->nthreads > 0) omp_set_num_threads(cfg->nthreads);
#else
    (void)cfg;
#endif
}

/* ------------------------------------------------------------------------------------ */
/* Time steps                                                                              */
/* ------------------------------------------------------------------------------------ */

/* Fused stream-pull-collide, two arrays: dst = C(S(src)) on fluid cells. Wall
 * cells of dst are not written. Returns 0. */
int ora_step_pull(const ora_cfg *cfg, const double *src, double *dst, const uint8_t *flags) {
    ora_stencil_t s;
    build_stencil(cfg->Q, &s);
    int64_t Sq = plane_cells(cfg);
    set_threads(cfg);
#pragma omp parallel for schedule(static)
    for (int64_t z = 0; z < cfg->nz; ++z)
        for (int64_t y = 0; y < cfg->ny; ++y)
            for (int64_t x = 0; x < cfg->nx; ++x) {
                int64_t self = cell(cfg, x, y, z);
                if (flags && flags[self] != FLAG_FLUID) continue;
                double f[27], out[27];
                for (int q = 0; q < s.Q; ++q) f[q] = pull_value(cfg, &s, src, flags, x, y, z, q);
                collide(cfg, &s, f, out);
                for (int q = 0; q < s.Q; ++q) dst[q * Sq + self] = out[q];
            }
    return 0;
}

/* Collision only, in place (fluid cells): a = C(a). */
int ora_collide_all(const ora_cfg *cfg, double *a, const uint8_t *flags) {
    ora_stencil_t s;
    build_stencil(cfg->Q, &s);
    int64_t Sq = plane_cells(cfg);
    set_threads(cfg);
#pragma omp parallel for schedule(static)
    for (int64_t z = 0; z < cfg->nz; ++z)
        for (int64_t y = 0; y < cfg->ny; ++y)
            for (int64_t x = 0; x < cfg->nx; ++x) {
                int64_t self = cell(cfg, x, y, z);
                if (flags && flags[self] != FLAG_FLUID) continue;
                double f[27], out[27];
                for (int q = 0; q < s.Q; ++q) f[q] = a[q * Sq + self];
                collide(cfg, &s, f, out);
                for (int q = 0; q < s.Q; ++q) a[q * Sq + self] = out[q];
            }
    return 0;
}

/* Streaming only (S with boundary conditions), two arrays: dst = S(src) on fluid cells. */
int ora_stream(const ora_cfg *cfg, const double *src, double *dst, const uint8_t *flags) {
    ora_stencil_t s;
    build_stencil(cfg->Q, &s);
    int64_t Sq = plane_cells(cfg);
    set_threads(cfg);
#pragma omp parallel for schedule(static)
    for (int64_t z = 0; z < cfg->nz; ++z)
        for (int64_t y = 0; y < cfg->ny; ++y)
            for (int64_t x = 0; x < cfg->nx; ++x) {
                int64_t self = cell(cfg, x, y, z);
                if (flags && flags[self] != FLAG_FLUID) continue;
                for (int q = 0; q < s.Q; ++q) dst[q * Sq + self] = pull_value(cfg, &s, src, flags, x, y, z, q);
            }
    return 0;
}

/* Fused collide-stream-push, two arrays: f <- S(C(f)), tmp is scratch of f's size. */
int ora_step_push(const ora_cfg *cfg, double *f, double *tmp, const uint8_t *flags) {
    int64_t n = (int64_t)cfg->Q * plane_cells(cfg);
    memcpy(tmp, f, (size_t)n * sizeof(double));
    ora_collide_all(cfg, tmp, flags);
    return ora_stream(cfg, tmp, f, flags);
}

/* AA pattern (Fig. 3), single array, optional flag field; with ghost planes (slab mode) the
 * caller exchanges them between steps (the ghost planes are read and written like any storage).
 * Even step: in-place collision with reversed storage: read a[x](q), write a[x](qbar). Wall cells
 * are skipped; boundary conditions act in the odd step (the boundary handling follows
 * the pattern's even/odd access scheme). */
int ora_aa_even(const ora_cfg *cfg, double *a, const uint8_t *flags) {
    ora_stencil_t s;
    build_stencil(cfg->Q, &s);
    int64_t Sq = plane_cells(cfg);
    set_threads(cfg);
#pragma omp parallel for schedule(static)
    for (int64_t z = 0; z < cfg->nz; ++z)
        for (int64_t y = 0; y < cfg->ny; ++y)
            for (int64_t x = 0; x < cfg->nx; ++x) {
                int64_t self = cell(cfg, x, y, z);
                if (flags && flags[self] != FLAG_FLUID) continue;
                double f[27], out[27];
                for (int q = 0; q < s.Q; ++q) f[q] = a[q * Sq + self];
                collide(cfg, &s, f, out);
                for (int q = 0; q < s.Q; ++q) a[s.opp[q] * Sq + self] = out[q];
            }
    return 0;
}

/* Odd step: stream-pull, collide, stream-push: read a[x - c_q](qbar), write a[x + c_q](q).
 * With walls (same rules as the pull streaming O6, expressed in the AA slots):
 *   read : x - c_q a wall -> the bounced population C_qbar(x), stored by the even step in a[x](q),
 *          plus the UBB term of q;
 *   write: x + c_q a wall -> the population returns to x as qbar next step: a[x](qbar) = out_q plus
 *          the UBB term of qbar.
 * Each fluid cell reads and writes the same set of slots, so cells are independent. */
int ora_aa_odd(const ora_cfg *cfg, double *a, const uint8_t *flags) {
    ora_stencil_t s;
    build_stencil(cfg->Q, &s);
    int64_t Sq = plane_cells(cfg);
    set_threads(cfg);
#pragma omp parallel for schedule(static)
    for (int64_t z = 0; z < cfg->nz; ++z)
        for (int64_t y = 0; y < cfg->ny; ++y)
            for (int64_t x = 0; x < cfg->nx; ++x) {
                int64_t self = cell(cfg, x, y, z);
                if (flags && flags[self] != FLAG_FLUID) continue;
                double f[27], out[27];
                for (int q = 0; q < s.Q; ++q) {
                    int64_t nb = cell(cfg, x - s.c[q][0], y - s.c[q][1], z - s.c[q][2]);
                    uint8_t fl = flags ? flags[nb] : FLAG_FLUID;
                    if (fl == FLAG_FLUID) {
                        f[q] = a[s.opp[q] * Sq + nb];
                    } else {
                        double v = a[q * Sq + self];
                        if (fl == FLAG_UBB) v += ubb_term_at(cfg, &s, q, nb);
                        f[q] = v;
                    }
                }
                collide(cfg, &s, f, out);
                for (int q = 0; q < s.Q; ++q) {
                    int64_t tg = cell(cfg, x + s.c[q][0], y + s.c[q][1], z + s.c[q][2]);
                    uint8_t fl = flags ? flags[tg] : FLAG_FLUID;
                    if (fl == FLAG_FLUID) {
                        a[q * Sq + tg] = out[q];
                    } else {
                        double v = out[q];
                        if (fl == FLAG_UBB) v += ubb_term_at(cfg, &s, s.opp[q], tg);
                        a[s.opp[q] * Sq + self] = v;
                    }
                }
            }
    return 0;
}

/* EsoTwist (Fig. 4), single array, no ghost planes, optional flag field. Every
 * population is stored "on its link": the population travelling from cell y to y + c_q lives at
 * location y + min(c_q, 0) (componentwise); seen from the arriving cell x that is x - max(c_q, 0).
 * Both time steps touch the same locations of each cell (x and its neighbours in negative
 * directions); they differ only in the slot ("twist" = the pointer swap q <-> qbar the paper replaces
 * by an even and an odd kernel):
 *   even: read arriving q at (x - c_q^+, q),    write departing q at (x + c_q^-, qbar)
 *   odd : read arriving q at (x - c_q^+, qbar), write departing q at (x + c_q^-, q)
 * (c^+ = max(c, 0), c^- = min(c, 0)); the departing slot of y is the next step's arriving slot of
 * y + c_q. Walls (pull rule O6 / G8): a departing population q whose target x + c_q is a wall comes
 * back as qbar next step; it is written, plus the UBB term of qbar, into the slot the next step reads
 * arriving qbar from: the other slot of the same location. Reads need no wall rule.
 * The canonical pre-collision state after n steps (= push F(n), G11) is a(x - c_q^+)(q) for even n,
 * a(x - c_q^+)(qbar) for odd n. */
static int64_t eso_loc(const ora_cfg *cfg, const ora_stencil_t *s, int64_t x, int64_t y, int64_t z, int q, int plus) {
    int64_t d[3];
    for (int k = 0; k < 3; ++k) {
        int c = s->c[q][k];
        d[k] = plus ? -(c > 0 ? c : 0) : (c < 0 ? c : 0); /* x - c^+  or  x + c^- */
    }
    return cell(cfg, x + d[0], y + d[1], z + d[2]);
}

static int ora_eso_step(const ora_cfg *cfg, double *a, const uint8_t *flags, int odd) {
    ora_stencil_t s;
    build_stencil(cfg->Q, &s);
    int64_t Sq = plane_cells(cfg);
    set_threads(cfg);
#pragma omp parallel for schedule(static)
    for (int64_t z = 0; z < cfg->nz; ++z)
        for (int64_t y = 0; y < cfg->ny; ++y)
            for (int64_t x = 0; x < cfg->nx; ++x) {
                int64_t self = cell(cfg, x, y, z);
                if (flags && flags[self] != FLAG_FLUID) continue;
                double f[27], out[27];
                for (int q = 0; q < s.Q; ++q) {
                    int slot = odd ? s.opp[q] : q;
                    f[q] = a[slot * Sq + eso_loc(cfg, &s, x, y, z, q, 1)];
                }
                collide(cfg, &s, f, out);
                for (int q = 0; q < s.Q; ++q) {
                    int64_t loc = eso_loc(cfg, &s, x, y, z, q, 0);
                    int64_t tg = cell(cfg, x + s.c[q][0], y + s.c[q][1], z + s.c[q][2]);
                    uint8_t fl = flags ? flags[tg] : FLAG_FLUID;
                    if (fl == FLAG_FLUID) {
                        int slot = odd ? q : s.opp[q];
                        a[slot * Sq + loc] = out[q];
                    } else { /* bounced: comes back as qbar, read next step from the other slot */
                        int slot = odd ? s.opp[q] : q;
                        double v = out[q];
                        if (fl == FLAG_UBB) v += ubb_term_at(cfg, &s, s.opp[q], tg);
                        a[slot * Sq + loc] = v;
                    }
                }
            }
    return 0;
}
int ora_eso_even(const ora_cfg *cfg, double *a, const uint8_t *flags) { return ora_eso_step(cfg, a, flags, 0); }
int ora_eso_odd(const ora_cfg *cfg, double *a, const uint8_t *flags) { return ora_eso_step(cfg, a, flags, 1); }

/* Canonical state <-> EsoTwist storage after `parity` (0: even number of steps done, 1: odd).
 * to_eso = 1: a(x - c_q^+)(slot) = f_q(x); to_eso = 0: f_q(x) = a(x - c_q^+)(slot). */
int ora_eso_layout(const ora_cfg *cfg, double *canon, double *a, int parity, int to_eso) {
    if (cfg->zghost) return -1;
    ora_stencil_t s;
    build_stencil(cfg->Q, &s);
    int64_t Sq = plane_cells(cfg);
    for (int64_t z = 0; z < cfg->nz; ++z)
        for (int64_t y = 0; y < cfg->ny; ++y)
            for (int64_t x = 0; x < cfg->nx; ++x) {
                int64_t self = cell(cfg, x, y, z);
                for (int q = 0; q < s.Q; ++q) {
                    int slot = parity ? s.opp[q] : q;
                    int64_t loc = eso_loc(cfg, &s, x, y, z, q, 1);
                    if (to_eso) a[slot * Sq + loc] = canon[q * Sq + self];
                    else canon[q * Sq + self] = a[slot * Sq + loc];
                }
            }
    return 0;
}

/* ------------------------------------------------------------------------------------ */
/* Initialisation and readout                                                              */
/* ------------------------------------------------------------------------------------ */

/* f = f_eq(rho(x), u(x)) on every storage cell of the local extent (Eq. 3), or the product
 * equilibrium for the cumulant (G2). rho: cells; u: [3][cells] (local extent, no ghosts). */
int ora_init_equilibrium(const ora_cfg *cfg, const double *rho, const double *u, double *f) {
    ora_stencil_t s;
    build_stencil(cfg->Q, &s);
    int64_t Sq = plane_cells(cfg);
    int64_t n = cfg->nx * cfg->ny * cfg->nz;
    for (int64_t z = 0; z < cfg->nz; ++z)
        for (int64_t y = 0; y < cfg->ny; ++y)
            for (int64_t x = 0; x < cfg->nx; ++x) {
                int64_t i = (z * cfg->ny + y) * cfg->nx + x;
                double uu[3] = {u[i], u[n + i], u[2 * n + i]}, feq[27];
                if (cfg->op == ORA_CUMULANT) maxwellian_equilibrium(cfg, &s, rho[i], uu, feq);
                else equilibrium_cfg(cfg, &s, rho[i], uu, feq);
                int64_t self = cell(cfg, x, y, z);
                for (int q = 0; q < s.Q; ++q) f[q * Sq + self] = feq[q];
            }
    return 0;
}

/* rho, u per local cell. fsign = +1 pre-collision state, -1 post-collision (pull) state. */
int ora_macroscopic(const ora_cfg *cfg, const double *f, double fsign, double *rho, double *u) {
    ora_stencil_t s;
    build_stencil(cfg->Q, &s);
    int64_t Sq = plane_cells(cfg);
    int64_t n = cfg->nx * cfg->ny * cfg->nz;
    for (int64_t z = 0; z < cfg->nz; ++z)
        for (int64_t y = 0; y < cfg->ny; ++y)
            for (int64_t x = 0; x < cfg->nx; ++x) {
                int64_t i = (z * cfg->ny + y) * cfg->nx + x, self = cell(cfg, x, y, z);
                double fc[27], r, uu[3];
                for (int q = 0; q < s.Q; ++q) fc[q] = f[q * Sq + self];
                macroscopic_eq(&s, fc, cfg->force, fsign, incompressible(cfg), &r, uu);
                rho[i] = r;
                u[i] = uu[0]; u[n + i] = uu[1]; u[2 * n + i] = uu[2];
            }
    return 0;
}

/* Single-cell helpers for tests and sampled full-size parity. */
/* The local Smagorinsky omega of a pre-collision cell state (for the Eq. (14) pins). */
double ora_smagorinsky_omega_cell(const ora_cfg *cfg, const double *f) {
    ora_stencil_t s;
    build_stencil(cfg->Q, &s);
    double rho, u[3], feq[27];
    macroscopic(&s, f, cfg->force, +1.0, &rho, u);
    equilibrium(&s, rho, u, feq);
    return smagorinsky_omega(&s, f, rho, feq, cfg->rates[0], cfg->rates[1]);
}

void ora_collide_cell(const ora_cfg *cfg, const double *f, double *out) {
    ora_stencil_t s;
    build_stencil(cfg->Q, &s);
    collide(cfg, &s, f, out);
}
void ora_equilibrium_cell(int Q, double rho, const double *u, double *feq) {
    ora_stencil_t s;
    build_stencil(Q, &s);
    equilibrium(&s, rho, u, feq);
}
/* The equilibrium of cfg's kind (Eq. 3 compressible / incompressible, or moment-matched). */
void ora_equilibrium_kind_cell(const ora_cfg *cfg, double rho, const double *u, double *feq) {
    ora_stencil_t s;
    build_stencil(cfg->Q, &s);
    equilibrium_cfg(cfg, &s, rho, u, feq);
}
void ora_maxwellian_equilibrium_cell(const ora_cfg *cfg, double rho, const double *u, double *feq) {
    ora_stencil_t s;
    build_stencil(cfg->Q, &s);
    maxwellian_equilibrium(cfg, &s, rho, u, feq);
}
void ora_from_cumulants_cfg_cell(const ora_cfg *cfg, double rho, const double *kappa, double *f) {
    ora_stencil_t s;
    build_stencil(cfg->Q, &s);
    from_cumulants_cfg(cfg, &s, rho, kappa, f);
}
void ora_product_equilibrium_cell(int Q, double rho, const double *u, double *feq) {
    ora_stencil_t s;
    build_stencil(Q, &s);
    product_equilibrium(&s, rho, u, feq);
}
double ora_cumulants_cell(int Q, const double *f, double *kappa) {
    ora_stencil_t s;
    build_stencil(Q, &s);
    return cumulants(&s, f, kappa);
}
void ora_from_cumulants_cell(int Q, double rho, const double *kappa, double *f) {
    ora_stencil_t s;
    build_stencil(Q, &s);
    from_cumulants(&s, rho, kappa, f);
}
/* One pull update of the single fluid cell (x,y,z): out[q] = C(S(src))_q at that cell. */
void ora_pull_cell(const ora_cfg *cfg, const double *src, const uint8_t *flags, int64_t x, int64_t y,
                   int64_t z, double *out) {
    ora_stencil_t s;
    build_stencil(cfg->Q, &s);
    double f[27];
    for (int q = 0; q < s.Q; ++q) f[q] = pull_value(cfg, &s, src, flags, x, y, z, q);
    collide(cfg, &s, f, out);
}

/* ------------------------------------------------------------------------------------ */
/* Halo reference (O7): crossing populations of plane z in canonical order                 */
/* (q ascending over {q : c_qz = dir}, then y, then x).                                    */
/* ------------------------------------------------------------------------------------ */
int64_t ora_pack_face(const ora_cfg *cfg, const double *f, int64_t z, int dir, double *out) {
    ora_stencil_t s;
    build_stencil(cfg->Q, &s);
    int64_t Sq = plane_cells(cfg), n = 0;
    for (int q = 0; q < s.Q; ++q) {
        if (s.c[q][2] != dir) continue;
        for (int64_t y = 0; y < cfg->ny; ++y)
            for (int64_t x = 0; x < cfg->nx; ++x)
                out[n++] = f[q * Sq + ((z + cfg->zghost) * cfg->ny + y) * cfg->nx + x];
    }
    return n;
}
/* Inverse: write a packed face into plane z (e.g. a ghost plane, z = -1 or z = nz). */
int64_t ora_unpack_face(const ora_cfg *cfg, double *f, int64_t z, int dir, const double *in) {
    ora_stencil_t s;
    build_stencil(cfg->Q, &s);
    int64_t Sq = plane_cells(cfg), n = 0;
    for (int q = 0; q < s.Q; ++q) {
        if (s.c[q][2] != dir) continue;
        for (int64_t y = 0; y < cfg->ny; ++y)
            for (int64_t x = 0; x < cfg->nx; ++x)
                f[q * Sq + ((z + cfg->zghost) * cfg->ny + y) * cfg->nx + x] = in[n++];
    }
    return n;
}
