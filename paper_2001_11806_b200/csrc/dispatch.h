// dispatch.h — type-erased launchers for the kernel template instantiations (k_*.cu).
#pragma once
#include <cuda_runtime.h>

#include "kernels.cuh"

namespace lbm {

using PullLaunch = void (*)(const StepArgs &, const void *src, void *dst, dim3 grid, dim3 block, cudaStream_t);
using AALaunch = void (*)(const StepArgs &, void *f, int odd, dim3 grid, dim3 block, cudaStream_t);
// near-wall cell list launch (split wall mode): pull edge kernel, or the AA odd edge kernel (src unused)
using EdgeLaunch = void (*)(const StepArgs &, const void *src, void *dst, const uint32_t *cells, uint32_t n, cudaStream_t);

// The kernels of one (operator, stencil, dtype, wall mode, force) combination; null members = not
// instantiated. fm: FM_NONE, FM_INLINE or FM_BULK (kernels.cuh); the edge launchers go with FM_BULK.
// persistent multi-step launch (cooperative); returns 0, or -1 if the launch failed
using PersistLaunch = int (*)(const StepArgs &, void *A, void *B, int phase, int nsteps, cudaStream_t);

struct Kernels {
    PullLaunch pull = nullptr;
    AALaunch aa = nullptr;
    EdgeLaunch pull_edges = nullptr;
    EdgeLaunch aa_edges = nullptr;
    PersistLaunch persist_pull = nullptr;  // walls inline (FM_INLINE) when a flag field exists
    PersistLaunch persist_aa = nullptr;
    AALaunch eso = nullptr;          // EsoTwist even/odd (odd flag)
    EdgeLaunch eso_edges = nullptr;  // near-wall cells; src != nullptr marks the odd step
    PullLaunch push = nullptr;       // collide-stream-push, two arrays
    EdgeLaunch push_edges = nullptr;
    AALaunch collide = nullptr;      // collision only, in place (odd argument unused)
};

Kernels select_trt(int Q, int dtype, int fm, bool force);
Kernels select_mrt(int Q, int dtype, int fm, bool force);
Kernels select_mrt_rows(int Q, int dtype, int fm, bool force);
int mrt_rows_upload();  // per-moment MRT rows -> __constant__ memory of the current device
Kernels select_cumulant(int Q, int dtype, int fm, bool force);
Kernels select_cumulant_unit(int Q, int dtype, int fm, bool force);  // D3Q27, omega_bulk = omega_3..6 = 1
Kernels select_mrt_shear(int Q, int dtype, int fm, bool force);      // D3Q19, omega_bulk = omega_3 = omega_4 = 1
Kernels select_identity(int Q, int dtype, int fm, bool force);
Kernels select_smagorinsky(int Q, int dtype, int fm, bool force);
Kernels select_kbc(int Q, int dtype, int fm, bool force);
Kernels select_kbc_exact(int Q, int dtype, int fm, bool force);
Kernels select_generated(int op, int Q, int dtype, int fm, bool force, int eq);
// equilibrium variants (EQ_INCOMPRESSIBLE / EQ_MOMENT_MATCHED of collide.cuh); all in k_select.cu
Kernels select_trt_eq(int Q, int dtype, int fm, bool force, int eq);
Kernels select_mrt_eq(int Q, int dtype, int fm, bool force, int eq);
// Operator dispatch used by the handle API and the low-level kernel ABI (runtime.cu); SRT runs the
// TRT kernel with equal rates.
Kernels select_kernels(int collision, int Q, int dtype, int fm, bool force, int eq = 0);

// Auxiliary kernels (k_misc.cu), dispatched on (Q, dtype).
void launch_init(int Q, int dtype, const InitArgs &a, void *f0, void *f1, dim3 grid, dim3 block, cudaStream_t s);
void launch_get_pops(int Q, int dtype, const ReadArgs &a, const void *f, double *out, dim3 grid, dim3 block, cudaStream_t s);
void launch_get_at(int Q, int dtype, const ReadArgs &a, const void *f, const int64_t *cells, int64_t n, int64_t first,
                   int64_t last, double *out, cudaStream_t s);
void launch_set_pops(int Q, int dtype, const ReadArgs &a, void *f, const double *in, dim3 grid, dim3 block, cudaStream_t s);
void launch_macro(int Q, int dtype, const ReadArgs &a, const void *f, double *rho, double *u, dim3 grid, dim3 block, cudaStream_t s);
void launch_pack(int Q, int dtype, const Geo &geo, const void *f, int zs, int dir, void *out, bool out_f64, cudaStream_t s);
void launch_unpack(int Q, int dtype, const Geo &geo, void *f, int zs, int dir, const void *in, cudaStream_t s);
void launch_unpack_masked(int Q, int dtype, const Geo &geo, void *f, int zs, int dir, const void *in, const uint8_t *flags,
                          cudaStream_t s);
void launch_unpack_masked_eso(int Q, int dtype, const Geo &geo, void *f, int zs, int dir, const void *in, const uint8_t *flags,
                              int parity_done, cudaStream_t s);
void launch_copyq(int Q, int dtype, bool shifted, const Geo &g, const void *src, void *dst, cudaStream_t s);
void launch_updateq(int Q, int dtype, bool shifted, const Geo &g, void *f, cudaStream_t s);
void launch_fma_probe(int dtype, int blocks, int iters, void *sink, cudaStream_t s);
void launch_links(int Q, int dtype, const LinkArgs &a, void *f, cudaStream_t s);
void launch_mark_near_wall(const Geo &geo, int nplanes, const uint8_t *in, uint8_t *out, cudaStream_t s);
int staged_path();           // bulk kernel path: 0 auto, 1 plain, 2 staged (k_misc.cu)
void set_staged_path(int v);
void launch_nan_check(int dtype, const void *f, int64_t n, int *flag, cudaStream_t s);

}  // namespace lbm
