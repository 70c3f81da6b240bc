// k_pull_inst.cuh — helpers to instantiate pull/AA launchers for one collision operator.
#pragma once
#include "dispatch.h"

namespace lbm {

template <int Q, int OP, typename T, bool FLAGS, bool FORCE>
void pull_launcher(const StepArgs &a, const void *src, void *dst, dim3 grid, dim3 block, cudaStream_t s) {
    k_pull<Q, OP, T, FLAGS, FORCE><<<grid, block, 0, s>>>(a, static_cast<const T *>(src), static_cast<T *>(dst));
}

template <int Q, int OP, typename T, bool FLAGS, bool FORCE>
void aa_launcher(const StepArgs &a, void *f, int odd, dim3 grid, dim3 block, cudaStream_t s) {
    if (odd)
        k_aa_odd<Q, OP, T, FLAGS, FORCE><<<grid, block, 0, s>>>(a, static_cast<T *>(f));
    else
        k_aa_even<Q, OP, T, FLAGS, FORCE><<<grid, block, 0, s>>>(a, static_cast<T *>(f));
}

// FORCE variants are instantiated only for operators with a forcing term (SRT/TRT).
template <int Q, int OP, typename T, bool WITH_FORCE>
PullLaunch pick_pull(bool flags, bool force) {
    if constexpr (WITH_FORCE) {
        if (force) return flags ? &pull_launcher<Q, OP, T, true, true> : &pull_launcher<Q, OP, T, false, true>;
    } else {
        if (force) return nullptr;
    }
    return flags ? &pull_launcher<Q, OP, T, true, false> : &pull_launcher<Q, OP, T, false, false>;
}

template <int Q, int OP, typename T, bool WITH_FORCE>
AALaunch pick_aa(bool flags, bool force) {
    if constexpr (WITH_FORCE) {
        if (force) return flags ? &aa_launcher<Q, OP, T, true, true> : &aa_launcher<Q, OP, T, false, true>;
    } else {
        if (force) return nullptr;
    }
    return flags ? &aa_launcher<Q, OP, T, true, false> : &aa_launcher<Q, OP, T, false, false>;
}

// (Q, dtype) dispatch of one operator; Qs lists the stencils it is instantiated for
template <int OP, bool WITH_FORCE, bool Q19, bool Q27>
PullLaunch select_pull_op(int Q, int dtype, bool flags, bool force) {
    if constexpr (Q19)
        if (Q == 19) return dtype == 0 ? pick_pull<19, OP, double, WITH_FORCE>(flags, force) : pick_pull<19, OP, float, WITH_FORCE>(flags, force);
    if constexpr (Q27)
        if (Q == 27) return dtype == 0 ? pick_pull<27, OP, double, WITH_FORCE>(flags, force) : pick_pull<27, OP, float, WITH_FORCE>(flags, force);
    return nullptr;
}

template <int OP, bool WITH_FORCE, bool Q19, bool Q27>
AALaunch select_aa_op(int Q, int dtype, bool flags, bool force) {
    if constexpr (Q19)
        if (Q == 19) return dtype == 0 ? pick_aa<19, OP, double, WITH_FORCE>(flags, force) : pick_aa<19, OP, float, WITH_FORCE>(flags, force);
    if constexpr (Q27)
        if (Q == 27) return dtype == 0 ? pick_aa<27, OP, double, WITH_FORCE>(flags, force) : pick_aa<27, OP, float, WITH_FORCE>(flags, force);
    return nullptr;
}

}  // namespace lbm
