// k_misc.cu — auxiliary kernels: initialisation, readout, halo pack/unpack, flag row mask and
// NaN check, dispatched on (stencil, dtype).
#include <atomic>
#include <cstdlib>
#include <cstring>

#include "dispatch.h"

namespace lbm {

#define LBM_DISPATCH(Q, dtype, ...)                                   \
    do {                                                              \
        if ((Q) == 19 && (dtype) == 0) { using T = double; constexpr int QQ = 19; __VA_ARGS__; } \
        else if ((Q) == 19) { using T = float; constexpr int QQ = 19; __VA_ARGS__; }             \
        else if ((dtype) == 0) { using T = double; constexpr int QQ = 27; __VA_ARGS__; }         \
        else { using T = float; constexpr int QQ = 27; __VA_ARGS__; }                            \
    } while (0)

void launch_init(int Q, int dtype, const InitArgs &a, void *f0, void *f1, dim3 grid, dim3 block, cudaStream_t s) {
    LBM_DISPATCH(Q, dtype, (k_init<QQ, T><<<grid, block, 0, s>>>(a, static_cast<T *>(f0), static_cast<T *>(f1))));
}

void launch_get_pops(int Q, int dtype, const ReadArgs &a, const void *f, double *out, dim3 grid, dim3 block, cudaStream_t s) {
    LBM_DISPATCH(Q, dtype, (k_get_pops<QQ, T><<<grid, block, 0, s>>>(a, static_cast<const T *>(f), out)));
}

void launch_get_at(int Q, int dtype, const ReadArgs &a, const void *f, const int64_t *cells, int64_t n, int64_t first,
                   int64_t last, double *out, cudaStream_t s) {
    const unsigned blocks = (unsigned)((n + 127) / 128);
    LBM_DISPATCH(Q, dtype, (k_get_at<QQ, T><<<blocks, 128, 0, s>>>(a, static_cast<const T *>(f), cells, n, first, last, out)));
}

void launch_set_pops(int Q, int dtype, const ReadArgs &a, void *f, const double *in, dim3 grid, dim3 block, cudaStream_t s) {
    LBM_DISPATCH(Q, dtype, (k_set_pops<QQ, T><<<grid, block, 0, s>>>(a, static_cast<T *>(f), in)));
}

void launch_copyq(int Q, int dtype, bool shifted, const Geo &g, const void *src, void *dst, cudaStream_t s) {
    const dim3 block(256, 1, 1), grid((unsigned)((g.nx + 255) / 256), (unsigned)g.ny, (unsigned)g.nz);
    if (shifted) {
        LBM_DISPATCH(Q, dtype, (k_copyq<QQ, T, true><<<grid, block, 0, s>>>(g, static_cast<const T *>(src), static_cast<T *>(dst))));
    } else {
        LBM_DISPATCH(Q, dtype, (k_copyq<QQ, T, false><<<grid, block, 0, s>>>(g, static_cast<const T *>(src), static_cast<T *>(dst))));
    }
}

void launch_updateq(int Q, int dtype, bool shifted, const Geo &g, void *f, cudaStream_t s) {
    const dim3 block(256, 1, 1), grid((unsigned)((g.nx + 255) / 256), (unsigned)g.ny, (unsigned)g.nz);
    if (shifted) {
        LBM_DISPATCH(Q, dtype, (k_updateq<QQ, T, true><<<grid, block, 0, s>>>(g, static_cast<T *>(f))));
    } else {
        LBM_DISPATCH(Q, dtype, (k_updateq<QQ, T, false><<<grid, block, 0, s>>>(g, static_cast<T *>(f))));
    }
}

void launch_fma_probe(int dtype, int blocks, int iters, void *sink, cudaStream_t s) {
    if (dtype == 0) k_fma_probe<double><<<blocks, 256, 0, s>>>(0.999999, 1e-7, iters, static_cast<double *>(sink));
    else k_fma_probe<float><<<blocks, 256, 0, s>>>(0.9999f, 1e-5f, iters, static_cast<float *>(sink));
}

void launch_links(int Q, int dtype, const LinkArgs &a, void *f, cudaStream_t s) {
    if (a.n == 0) return;
    const unsigned blocks = (a.n + 255) / 256;
    LBM_DISPATCH(Q, dtype, (k_links<QQ, T><<<blocks, 256, 0, s>>>(a, static_cast<T *>(f))));
}

void launch_macro(int Q, int dtype, const ReadArgs &a, const void *f, double *rho, double *u, dim3 grid, dim3 block, cudaStream_t s) {
    LBM_DISPATCH(Q, dtype, (k_macro<QQ, T><<<grid, block, 0, s>>>(a, static_cast<const T *>(f), rho, u)));
}

static unsigned blocks_for(int64_t n) {
    int64_t b = (n + 255) / 256;
    return (unsigned)(b < 148 * 16 ? (b < 1 ? 1 : b) : 148 * 16);
}

void launch_pack(int Q, int dtype, const Geo &geo, const void *f, int zs, int dir, void *out, bool out_f64, cudaStream_t s) {
    const int64_t n = (int64_t)geo.nx * geo.ny * (Q == 19 ? 5 : 9);
    if (out_f64) {
        LBM_DISPATCH(Q, dtype, (k_pack<QQ, T, double><<<blocks_for(n), 256, 0, s>>>(geo, static_cast<const T *>(f), zs, dir, static_cast<double *>(out))));
    } else {
        LBM_DISPATCH(Q, dtype, (k_pack<QQ, T, T><<<blocks_for(n), 256, 0, s>>>(geo, static_cast<const T *>(f), zs, dir, static_cast<T *>(out))));
    }
}

void launch_unpack(int Q, int dtype, const Geo &geo, void *f, int zs, int dir, const void *in, cudaStream_t s) {
    const int64_t n = (int64_t)geo.nx * geo.ny * (Q == 19 ? 5 : 9);
    LBM_DISPATCH(Q, dtype, (k_unpack<QQ, T><<<blocks_for(n), 256, 0, s>>>(geo, static_cast<T *>(f), zs, dir, static_cast<const T *>(in))));
}

void launch_unpack_masked_eso(int Q, int dtype, const Geo &geo, void *f, int zs, int dir, const void *in, const uint8_t *flags,
                              int parity_done, cudaStream_t s) {
    const int64_t n = (int64_t)geo.nx * geo.ny * (Q == 19 ? 5 : 9);
    LBM_DISPATCH(Q, dtype, (k_unpack_masked_eso<QQ, T><<<blocks_for(n), 256, 0, s>>>(geo, static_cast<T *>(f), zs, dir,
                                                                                    static_cast<const T *>(in), flags,
                                                                                    parity_done)));
}

void launch_unpack_masked(int Q, int dtype, const Geo &geo, void *f, int zs, int dir, const void *in, const uint8_t *flags,
                          cudaStream_t s) {
    const int64_t n = (int64_t)geo.nx * geo.ny * (Q == 19 ? 5 : 9);
    LBM_DISPATCH(Q, dtype, (k_unpack_masked<QQ, T><<<blocks_for(n), 256, 0, s>>>(geo, static_cast<T *>(f), zs, dir,
                                                                                static_cast<const T *>(in), flags)));
}

__global__ void k_mark_near_wall(const Geo geo, int nplanes, const uint8_t *__restrict__ in, uint8_t *__restrict__ out) {
    const int64_t plane = (int64_t)geo.nx * geo.ny;
    const int64_t n = plane * nplanes;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const int zs = (int)(i / plane);
        const int y = (int)((i / geo.nx) % geo.ny);
        const int x = (int)(i % geo.nx);
        uint8_t v = in[i] & 3;
        if (v == 0) {
            bool near = false;
            for (int dz = -1; dz <= 1; ++dz) {
                int z2 = zs + dz;
                if (geo.g) {
                    if (z2 < 0 || z2 >= nplanes) continue;
                } else {
                    z2 = (z2 + nplanes) % nplanes;
                }
                for (int dy = -1; dy <= 1; ++dy) {
                    const int y2 = (y + dy + geo.ny) % geo.ny;
                    for (int dx = -1; dx <= 1; ++dx) {
                        const int x2 = (x + dx + geo.nx) % geo.nx;
                        near |= (in[(int64_t)z2 * plane + (int64_t)y2 * geo.nx + x2] & 3) != 0;
                    }
                }
            }
            if (near) v |= 0x80;
        }
        out[i] = v;
    }
}

void launch_mark_near_wall(const Geo &geo, int nplanes, const uint8_t *in, uint8_t *out, cudaStream_t s) {
    const int64_t n = (int64_t)geo.nx * geo.ny * nplanes;
    k_mark_near_wall<<<blocks_for(n), 256, 0, s>>>(geo, nplanes, in, out);
}

void launch_nan_check(int dtype, const void *f, int64_t n, int *flag, cudaStream_t s) {
    if (dtype == 0)
        k_nan_check<double><<<blocks_for(n), 256, 0, s>>>(static_cast<const double *>(f), n, flag);
    else
        k_nan_check<float><<<blocks_for(n), 256, 0, s>>>(static_cast<const float *>(f), n, flag);
}

}  // namespace lbm

namespace lbm {
// Kernel path of the bulk update kernels (staged.cuh): LBM_PATH_AUTO (measured per-family policy),
// LBM_PATH_PLAIN (register-gather kernels everywhere) or LBM_PATH_STAGED (TMA-staged wherever the
// layout allows). Initial value from LBM_KERNEL_PATH=auto|plain|staged; lbm_set_kernel_path changes
// it process-wide. LBM_STAGES sets the pipeline depth (tiles in flight per CTA, 2..6).
static std::atomic<int> g_kernel_path{-1};
int staged_path() {
    int v = g_kernel_path.load(std::memory_order_relaxed);
    if (v < 0) {
        const char *e = getenv("LBM_KERNEL_PATH");
        v = !e ? 0 : (!strcmp(e, "plain") ? 1 : (!strcmp(e, "staged") ? 2 : 0));
        g_kernel_path.store(v, std::memory_order_relaxed);
    }
    return v;
}
void set_staged_path(int v) { g_kernel_path.store(v, std::memory_order_relaxed); }
int staged_nstages() {
    static const int n = [] {
        const char *e = getenv("LBM_STAGES");
        const int v = e ? atoi(e) : 2;
        return v < 2 ? 2 : (v > 6 ? 6 : v);
    }();
    return n;
}
}  // namespace lbm
