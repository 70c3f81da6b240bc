// k_pull_inst.cuh — helpers to instantiate pull/AA launchers for one collision operator.
#pragma once
#include "dispatch.h"

namespace lbm {

template <int Q, int OP, typename T, bool FLAGS, bool FORCE>
void pull_launcher(const StepArgs &a, const void *src, void *dst, dim3 grid, dim3 block, cudaStream_t s) {
    k_pull<Q, OP, T, FLAGS, FORCE><<<grid, block, 0, s>>>(a, static_cast<const T *>(src), static_cast<T *>(dst));
}

template <int Q, int OP, typename T, bool FORCE>
void aa_launcher(const StepArgs &a, void *f, int odd, dim3 grid, dim3 block, cudaStream_t s) {
    if (odd)
        k_aa_odd<Q, OP, T, FORCE><<<grid, block, 0, s>>>(a, static_cast<T *>(f));
    else
        k_aa_even<Q, OP, T, FORCE><<<grid, block, 0, s>>>(a, static_cast<T *>(f));
}

template <int Q, int OP, typename T>
PullLaunch pick_pull(bool flags, bool force) {
    if (flags) return force ? &pull_launcher<Q, OP, T, true, true> : &pull_launcher<Q, OP, T, true, false>;
    return force ? &pull_launcher<Q, OP, T, false, true> : &pull_launcher<Q, OP, T, false, false>;
}

template <int Q, int OP, typename T>
PullLaunch pick_pull_noforce(bool flags, bool force) {
    if (force) return nullptr;
    return flags ? &pull_launcher<Q, OP, T, true, false> : &pull_launcher<Q, OP, T, false, false>;
}

}  // namespace lbm
