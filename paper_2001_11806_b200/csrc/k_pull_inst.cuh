// k_pull_inst.cuh — helpers to instantiate pull/AA launchers for one collision operator.
#pragma once
#include <cstdlib>

#include "dispatch.h"
#include "staged.cuh"

namespace lbm {

template <int Q, int OP, typename T, int FM, bool FORCE>
void pull_launcher(const StepArgs &a, const void *src, void *dst, dim3 grid, dim3 block, cudaStream_t s) {
    // peer stores (fused halo, boundary-plane launches only) are a separate instantiation so the
    // interior kernel carries no extra live registers
    if (a.peer_up == nullptr && staged_launch<Q, OP, T, FM, FORCE, SM_PULL>(a, src, dst, (int)grid.z, s)) return;
    if constexpr (FM != FM_INLINE && FM != FM_LINKS)  // inline walls (low-level ABI) / FM_LINKS: no peer stores
        if (a.peer_up != nullptr) {
            k_pull<Q, OP, T, FM, FORCE, true><<<grid, block, 0, s>>>(a, static_cast<const T *>(src), static_cast<T *>(dst));
            return;
        }
    k_pull<Q, OP, T, FM, FORCE, false><<<grid, block, 0, s>>>(a, static_cast<const T *>(src), static_cast<T *>(dst));
}

template <int Q, int OP, typename T, bool FORCE>
void pull_edge_launcher(const StepArgs &a, const void *src, void *dst, const uint32_t *cells, uint32_t n, cudaStream_t s) {
    if (n == 0) return;
    const unsigned blocks = (n + 127) / 128;
    if (a.peer_up != nullptr)
        k_pull_edges<Q, OP, T, FORCE, true><<<blocks, 128, 0, s>>>(a, static_cast<const T *>(src), static_cast<T *>(dst), cells, n);
    else
        k_pull_edges<Q, OP, T, FORCE, false><<<blocks, 128, 0, s>>>(a, static_cast<const T *>(src), static_cast<T *>(dst), cells, n);
}

template <int Q, int OP, typename T, int FM, bool FORCE>
void aa_launcher(const StepArgs &a, void *f, int odd, dim3 grid, dim3 block, cudaStream_t s) {
    if constexpr (FM != FM_INLINE && FM != FM_LINKS)
        if (a.peer_up != nullptr) {  // fused halo: boundary-plane launch with peer stores (plain kernels)
            if (odd) k_aa_odd<Q, OP, T, FM, FORCE, true><<<grid, block, 0, s>>>(a, static_cast<T *>(f));
            else k_aa_even<Q, OP, T, (FM != FM_NONE), FORCE, true><<<grid, block, 0, s>>>(a, static_cast<T *>(f));
            return;
        }
    if (odd) {
        if (staged_launch<Q, OP, T, FM, FORCE, SM_AA_ODD>(a, f, f, (int)grid.z, s)) return;
    } else {
        if (staged_launch<Q, OP, T, (FM == FM_NONE ? FM_NONE : FM == FM_LINKS ? FM_LINKS : FM_BULK), FORCE, SM_AA_EVEN>(
                a, f, f, (int)grid.z, s))
            return;
    }
    if constexpr (FM == FM_NONE && sizeof(T) == 4 && Q == 19) {
        // even step: two cells per thread (periodic fp32 D3Q19 on the plain path; C2 0.944 -> 0.964 of copy BW,
        // profiles/r03e; the odd step keeps one cell per thread: both two-cell 0.951); LBM_AA_X2=0 disables it
        static const bool x2 = [] {
            const char *e = getenv("LBM_AA_X2");
            return e ? atoi(e) != 0 : true;
        }();
        if (x2 && !odd && a.flat_hi == 0 && block.x >= 32 && block.x % 32 == 0) {
            const unsigned w = (unsigned)(a.x1 - a.x0);
            const dim3 g2((w + 2 * block.x - 1) / (2 * block.x), grid.y, grid.z);
            k_aa_even_x2<Q, OP, T, FORCE><<<g2, block, 0, s>>>(a, static_cast<T *>(f));
            return;
        }
    }
    if (odd)
        k_aa_odd<Q, OP, T, FM, FORCE><<<grid, block, 0, s>>>(a, static_cast<T *>(f));
    else  // the even step is in place: walls are skipped, near-wall cells need nothing special (FM_LINKS:
          // they fill the wall slots of their links)
        k_aa_even<Q, OP, T, (FM != FM_NONE), FORCE, false, (FM == FM_LINKS)><<<grid, block, 0, s>>>(a, static_cast<T *>(f));
}

template <int Q, int OP, typename T, bool FORCE>
void aa_edge_launcher(const StepArgs &a, const void *src, void *f, const uint32_t *cells, uint32_t n, cudaStream_t s) {
    (void)src;
    if (n == 0) return;
    if (a.peer_up != nullptr)
        k_aa_odd_edges<Q, OP, T, FORCE, true><<<(n + 127) / 128, 128, 0, s>>>(a, static_cast<T *>(f), cells, n);
    else
        k_aa_odd_edges<Q, OP, T, FORCE, false><<<(n + 127) / 128, 128, 0, s>>>(a, static_cast<T *>(f), cells, n);
}

template <int Q, int OP, typename T, int FM, bool FORCE>
void push_launcher(const StepArgs &a, const void *src, void *dst, dim3 grid, dim3 block, cudaStream_t s) {
    if constexpr (FM != FM_INLINE)
        if (a.peer_up != nullptr) {  // fused halo: boundary-plane launch with peer stores (plain kernels)
            k_push<Q, OP, T, FM, FORCE, true><<<grid, block, 0, s>>>(a, static_cast<const T *>(src), static_cast<T *>(dst));
            return;
        }
    if (staged_launch<Q, OP, T, FM, FORCE, SM_PUSH>(a, src, dst, (int)grid.z, s)) return;
    k_push<Q, OP, T, FM, FORCE, false><<<grid, block, 0, s>>>(a, static_cast<const T *>(src), static_cast<T *>(dst));
}

template <int Q, int OP, typename T, bool FORCE>
void push_edge_launcher(const StepArgs &a, const void *src, void *dst, const uint32_t *cells, uint32_t n, cudaStream_t s) {
    if (n == 0) return;
    const unsigned b = (n + 127) / 128;
    if (a.peer_up != nullptr)
        k_push_edges<Q, OP, T, FORCE, true><<<b, 128, 0, s>>>(a, static_cast<const T *>(src), static_cast<T *>(dst), cells, n);
    else
        k_push_edges<Q, OP, T, FORCE, false><<<b, 128, 0, s>>>(a, static_cast<const T *>(src), static_cast<T *>(dst), cells, n);
}

template <int Q, int OP, typename T, bool FLAGS, bool FORCE>
void collide_launcher(const StepArgs &a, void *f, int, dim3 grid, dim3 block, cudaStream_t s) {
    k_collide<Q, OP, T, FLAGS, FORCE><<<grid, block, 0, s>>>(a, static_cast<T *>(f));
}

template <int Q, int OP, typename T, int FM, bool FORCE>
void eso_launcher(const StepArgs &a, void *f, int odd, dim3 grid, dim3 block, cudaStream_t s) {
    if constexpr (FM != FM_INLINE)
        if (a.peer_up != nullptr) {  // fused halo: boundary-plane launch with peer stores (plain kernels)
            if (odd) k_eso<Q, OP, T, FM, FORCE, true, true><<<grid, block, 0, s>>>(a, static_cast<T *>(f));
            else k_eso<Q, OP, T, FM, FORCE, false, true><<<grid, block, 0, s>>>(a, static_cast<T *>(f));
            return;
        }
    if (odd ? staged_launch<Q, OP, T, FM, FORCE, SM_ESO_ODD>(a, f, f, (int)grid.z, s)
            : staged_launch<Q, OP, T, FM, FORCE, SM_ESO_EVEN>(a, f, f, (int)grid.z, s))
        return;
    if (odd) k_eso<Q, OP, T, FM, FORCE, true><<<grid, block, 0, s>>>(a, static_cast<T *>(f));
    else k_eso<Q, OP, T, FM, FORCE, false><<<grid, block, 0, s>>>(a, static_cast<T *>(f));
}

// EdgeLaunch has no parity argument; for EsoTwist the caller (runtime.cu) marks the odd step by a
// non-null `src` (the kernel itself only uses `f`).
template <int Q, int OP, typename T, bool FORCE>
void eso_edge_launcher(const StepArgs &a, const void *src, void *f, const uint32_t *cells, uint32_t n, cudaStream_t s) {
    if (n == 0) return;
    const bool odd = src != nullptr;  // runtime passes a non-null marker for odd steps
    const unsigned b = (n + 127) / 128;
    T *ff = static_cast<T *>(f);
    if (a.peer_up != nullptr) {
        if (odd) k_eso_edges<Q, OP, T, FORCE, true, true><<<b, 128, 0, s>>>(a, ff, cells, n);
        else k_eso_edges<Q, OP, T, FORCE, false, true><<<b, 128, 0, s>>>(a, ff, cells, n);
    } else {
        if (odd) k_eso_edges<Q, OP, T, FORCE, true, false><<<b, 128, 0, s>>>(a, ff, cells, n);
        else k_eso_edges<Q, OP, T, FORCE, false, false><<<b, 128, 0, s>>>(a, ff, cells, n);
    }
}

template <int Q, int OP, typename T, int FM, bool FORCE, bool AA>
int persistent_launcher(const StepArgs &a, void *A, void *B, int phase, int nsteps, cudaStream_t s) {
    auto kern = k_persistent<Q, OP, T, FM, FORCE, AA>;
    // co-resident CTA count: an occupancy result of the current device, cached per device ordinal
    static int coresident_of[kMaxDevices] = {};
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev < 0 || dev >= kMaxDevices) return -1;
    int &coresident = coresident_of[dev];
    if (coresident == 0) {
        int per_sm = 0, sms = 0;
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, 256, 0);
        coresident = per_sm * sms;
    }
    const int64_t ncell = (int64_t)a.geo.nx * a.geo.ny * a.geo.nz;
    // cells per thread: a few cells per thread keeps the grid (and so the grid barrier) small
    static const int cpt = [] {
        const char *e = getenv("LBM_PERSIST_CELLS_PER_THREAD");
        return e ? atoi(e) : 1;
    }();
    int64_t grid = (ncell + 256 * (int64_t)cpt - 1) / (256 * (int64_t)cpt);
    if (grid > coresident) grid = coresident;
    if (grid < 1) return -1;
    T *pa = static_cast<T *>(A), *pb = static_cast<T *>(B);
    void *args[] = {const_cast<StepArgs *>(&a), &pa, &pb, &phase, &nsteps};
    return cudaLaunchCooperativeKernel((const void *)kern, dim3((unsigned)grid), dim3(256), args, 0, s) == cudaSuccess ? 0 : -1;
}

template <int Q, int OP, typename T, bool FORCE>
void pick_persistent(int fm, Kernels &k) {
    if constexpr (op_eq(OP) != EQ_COMPRESSIBLE) {  // small-domain persistent kernels: base equilibrium only
        (void)fm, (void)k;
        return;
    } else {
    if (fm == FM_NONE) {  // (FM_FACES handles: the persistent kernels test the flag field inline)
        k.persist_pull = &persistent_launcher<Q, OP, T, FM_NONE, FORCE, false>;
        k.persist_aa = &persistent_launcher<Q, OP, T, FM_NONE, FORCE, true>;
    } else {
        k.persist_pull = &persistent_launcher<Q, OP, T, FM_INLINE, FORCE, false>;
        k.persist_aa = &persistent_launcher<Q, OP, T, FM_INLINE, FORCE, true>;
    }
    }
}

// Face-aligned-wall kernels (FM_FACES) are instantiated for the TRT/SRT class (the runtime selects them
// for the D3Q19 fp64 pull kernels, where they measured faster than the split and index-list modes)
template <int OP>
constexpr bool faces_supported() {
    constexpr int c = op_class(op_base(OP));
    return c == OP_SRT || c == OP_TRT;
}

template <int Q, int OP, typename T, bool FORCE>
PullLaunch pick_pull_fm(int fm) {
    if constexpr (faces_supported<OP>())
        if (fm == FM_FACES) return &pull_launcher<Q, OP, T, FM_FACES, FORCE>;
    if (fm == FM_FACES) return nullptr;
    switch (fm) {
        case FM_INLINE: return &pull_launcher<Q, OP, T, FM_INLINE, FORCE>;
        case FM_BULK: return &pull_launcher<Q, OP, T, FM_BULK, FORCE>;
        case FM_LINKS: return &pull_launcher<Q, OP, T, FM_LINKS, FORCE>;
        default: return &pull_launcher<Q, OP, T, FM_NONE, FORCE>;
    }
}

template <int Q, int OP, typename T, bool FORCE>
PullLaunch pick_push_fm(int fm) {
    if (fm == FM_FACES || fm == FM_LINKS) return nullptr;  // face-aligned walls / in-kernel links: pull and AA only
    switch (fm) {
        case FM_INLINE: return &push_launcher<Q, OP, T, FM_INLINE, FORCE>;
        case FM_BULK: return &push_launcher<Q, OP, T, FM_BULK, FORCE>;
        default: return &push_launcher<Q, OP, T, FM_NONE, FORCE>;
    }
}

template <int Q, int OP, typename T, bool FORCE>
AALaunch pick_eso_fm(int fm) {
    if (fm == FM_FACES || fm == FM_LINKS) return nullptr;  // face-aligned walls / in-kernel links: pull and AA only
    switch (fm) {
        case FM_INLINE: return &eso_launcher<Q, OP, T, FM_INLINE, FORCE>;
        case FM_BULK: return &eso_launcher<Q, OP, T, FM_BULK, FORCE>;
        default: return &eso_launcher<Q, OP, T, FM_NONE, FORCE>;
    }
}

template <int Q, int OP, typename T, bool FORCE>
AALaunch pick_aa_fm(int fm) {
    if constexpr (faces_supported<OP>())
        if (fm == FM_FACES) return &aa_launcher<Q, OP, T, FM_FACES, FORCE>;
    if (fm == FM_FACES) return nullptr;
    switch (fm) {
        case FM_INLINE: return &aa_launcher<Q, OP, T, FM_INLINE, FORCE>;
        case FM_BULK: return &aa_launcher<Q, OP, T, FM_BULK, FORCE>;
        case FM_LINKS: return &aa_launcher<Q, OP, T, FM_LINKS, FORCE>;
        default: return &aa_launcher<Q, OP, T, FM_NONE, FORCE>;
    }
}

// FORCE variants are instantiated only for operators with a forcing term (SRT/TRT).
template <int Q, int OP, typename T, bool WITH_FORCE>
Kernels pick(int fm, bool force) {
    Kernels k;
    if constexpr (WITH_FORCE) {
        if (force) {
            k.pull = pick_pull_fm<Q, OP, T, true>(fm);
            k.aa = pick_aa_fm<Q, OP, T, true>(fm);
            k.pull_edges = &pull_edge_launcher<Q, OP, T, true>;
            k.aa_edges = &aa_edge_launcher<Q, OP, T, true>;
            k.eso = pick_eso_fm<Q, OP, T, true>(fm);
            k.eso_edges = &eso_edge_launcher<Q, OP, T, true>;
            k.push = pick_push_fm<Q, OP, T, true>(fm);
            k.push_edges = &push_edge_launcher<Q, OP, T, true>;
            k.collide = fm == FM_NONE ? &collide_launcher<Q, OP, T, false, true> : &collide_launcher<Q, OP, T, true, true>;
            pick_persistent<Q, OP, T, true>(fm, k);
            return k;
        }
    } else {
        if (force) return k;  // not instantiated
    }
    k.pull = pick_pull_fm<Q, OP, T, false>(fm);
    k.aa = pick_aa_fm<Q, OP, T, false>(fm);
    k.pull_edges = &pull_edge_launcher<Q, OP, T, false>;
    k.aa_edges = &aa_edge_launcher<Q, OP, T, false>;
    k.eso = pick_eso_fm<Q, OP, T, false>(fm);
    k.eso_edges = &eso_edge_launcher<Q, OP, T, false>;
    k.push = pick_push_fm<Q, OP, T, false>(fm);
    k.push_edges = &push_edge_launcher<Q, OP, T, false>;
    k.collide = fm == FM_NONE ? &collide_launcher<Q, OP, T, false, false> : &collide_launcher<Q, OP, T, true, false>;
    pick_persistent<Q, OP, T, false>(fm, k);
    return k;
}

// (Q, dtype) dispatch of one operator over the stencils it is instantiated for
template <int OP, bool WITH_FORCE, bool Q19, bool Q27>
Kernels select_op(int Q, int dtype, int fm, bool force) {
    if constexpr (Q19)
        if (Q == 19) return dtype == 0 ? pick<19, OP, double, WITH_FORCE>(fm, force) : pick<19, OP, float, WITH_FORCE>(fm, force);
    if constexpr (Q27)
        if (Q == 27) return dtype == 0 ? pick<27, OP, double, WITH_FORCE>(fm, force) : pick<27, OP, float, WITH_FORCE>(fm, force);
    return Kernels{};
}

}  // namespace lbm
