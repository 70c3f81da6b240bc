// dispatch.h — type-erased launchers for the kernel template instantiations (k_*.cu).
#pragma once
#include <cuda_runtime.h>

#include "kernels.cuh"

namespace lbm {

using PullLaunch = void (*)(const StepArgs &, const void *src, void *dst, dim3 grid, dim3 block, cudaStream_t);
using AALaunch = void (*)(const StepArgs &, void *f, int odd, dim3 grid, dim3 block, cudaStream_t);

// Per-operator selection (nullptr = combination not instantiated). dtype: 0 = f64, 1 = f32.
PullLaunch select_pull_trt(int Q, int dtype, bool flags, bool force);
PullLaunch select_pull_mrt(int Q, int dtype, bool flags, bool force);
PullLaunch select_pull_cumulant(int Q, int dtype, bool flags, bool force);
PullLaunch select_pull_identity(int Q, int dtype, bool flags, bool force);
PullLaunch select_pull_smagorinsky(int Q, int dtype, bool flags, bool force);
PullLaunch select_pull_kbc(int Q, int dtype, bool flags, bool force);
AALaunch select_aa_smagorinsky(int Q, int dtype, bool flags, bool force);
AALaunch select_aa_kbc(int Q, int dtype, bool flags, bool force);

// Operator dispatch used by the handle API and the low-level kernel ABI (runtime.cu); SRT runs the
// TRT kernel with equal rates. nullptr = combination not instantiated.
PullLaunch select_pull(int collision, int Q, int dtype, bool flags, bool force);
AALaunch select_aa(int collision, int Q, int dtype, bool flags, bool force);
AALaunch select_aa_trt(int Q, int dtype, bool flags, bool force);
AALaunch select_aa_mrt(int Q, int dtype, bool flags, bool force);
AALaunch select_aa_cumulant(int Q, int dtype, bool flags, bool force);
AALaunch select_aa_identity(int Q, int dtype, bool flags, bool force);

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
void launch_mark_near_wall(const Geo &geo, int nplanes, const uint8_t *in, uint8_t *out, cudaStream_t s);
void launch_nan_check(int dtype, const void *f, int64_t n, int *flag, cudaStream_t s);

}  // namespace lbm
