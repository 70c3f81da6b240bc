// k_mrt_rows.cu — MRT with one relaxation rate per moment (D3Q19, paper's weighted Gram-Schmidt rows;
// fp64 and fp32; no force; pull, AA and EsoTwist). The orthogonalised rows (collide.cuh,
// make_mrt_rows19) are computed once on the host and kept in __constant__ memory.
#include <mutex>

#include "k_pull_inst.cuh"

namespace lbm {

__constant__ double c_mrt_v[19][19];
__constant__ double c_mrt_inv_norm[19];

template <typename T>
__device__ __forceinline__ void collide_mrt19_rows(T (&g)[19], const Rates<T> &p) {
    using S = Stencil<19>;
    T drho, jx, jy, jz;
    moments0<19, T>(g, drho, jx, jy, jz);
    const T rho = T(1) + drho;
    const T inv = T(1) / rho;
    const T ux = jx * inv, uy = jy * inv, uz = jz * inv;
    const T uu15 = T(1.5) * (ux * ux + uy * uy + uz * uz);
    // g <- g_eq, with d = g - g_eq kept as pair sums/differences (even rows see dp, odd rows dm)
    const T w0 = T(S::w(0));
    const T eq0 = w0 * drho - w0 * rho * uu15;
    const T d0 = g[0] - eq0;
    g[0] = eq0;
    T dp[19], dm[19];
#pragma unroll
    for (int q = 1; q < 19; ++q) {
        if (q < S::opp(q)) {
            const int b = S::opp(q);
            const T w = T(S::w(q));
            const T cu = T(S::cx(q)) * ux + T(S::cy(q)) * uy + T(S::cz(q)) * uz;
            const T wr = w * rho;
            const T eqs = w * drho + wr * (T(4.5) * cu * cu - uu15);
            const T eqa = wr * T(3) * cu;
            dp[q] = (g[q] + g[b]) - T(2) * eqs;
            dm[q] = (g[q] - g[b]) - T(2) * eqa;
            g[q] = eqs + eqa;
            g[b] = eqs - eqa;
        }
    }
    // f* = f_eq + sum_k (1 - omega_k) w P_k <P_k, d> / N_k over the 15 non-conserved rows
#pragma unroll
    for (int k = 4; k < 19; ++k) {
        const T keep = T(1) - p.r[k - 4];
        if (keep == T(0)) continue;  // uniform: this moment relaxes to equilibrium
        const bool odd = k >= 10 && k <= 15;
        T m = odd ? T(0) : T(c_mrt_v[k][0]) * d0;
#pragma unroll
        for (int q = 1; q < 19; ++q)
            if (q < S::opp(q)) m += T(c_mrt_v[k][q]) * (odd ? dm[q] : dp[q]);
        const T a = keep * T(c_mrt_inv_norm[k]) * m;
        if (!odd) g[0] += w0 * T(c_mrt_v[k][0]) * a;
#pragma unroll
        for (int q = 1; q < 19; ++q) {
            if (q < S::opp(q)) {
                const T t = T(S::w(q)) * T(c_mrt_v[k][q]) * a;
                g[q] += t;
                g[S::opp(q)] += odd ? -t : t;
            }
        }
    }
}

Kernels select_mrt_rows(int Q, int dtype, int fm, bool force) { return select_op<OP_MRT_ROWS, false, true, false>(Q, dtype, fm, force); }

// upload the rows to the current device (once per device; called by lbm_create after cudaSetDevice)
int mrt_rows_upload() {
    static std::mutex mu;
    static bool done[64] = {};
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return -1;
    std::lock_guard<std::mutex> lock(mu);
    if (done[dev]) return 0;
    const MrtRows19 b = make_mrt_rows19();
    if (cudaMemcpyToSymbol(c_mrt_v, b.v, sizeof(b.v)) != cudaSuccess ||
        cudaMemcpyToSymbol(c_mrt_inv_norm, b.inv_norm, sizeof(b.inv_norm)) != cudaSuccess)
        return -1;
    done[dev] = true;
    return 0;
}
}  // namespace lbm
