// staged.cuh — TMA-staged persistent update kernels (bulk kernels of the pull, AA and EsoTwist
// patterns).
//
// The plain kernels (kernels.cuh) keep every population load of a cell in registers until it
// arrives, so the bytes a SM has in flight are bounded by registers x occupancy; the heavy
// operators (MRT, cumulant, KBC) need 80-170 registers per thread and fall short of the ~50 KB per
// SM that Little's law asks for at HBM3e bandwidth. Here the loads are
// decoupled from registers. A persistent CTA = BT consumer threads + one producer warp walks tiles
// of H full x-rows of one plane. Full rows are contiguous in the [q][z][y][x] layout, so for every
// direction q the producer issues ONE 1-D bulk copy (cp.async.bulk, the TMA engine; two when the
// y-shift wraps) of the shifted source rows into a shared-memory ring of nstages stages, arming the
// stage's "full" mbarrier with expect_tx; consumer warps wait on it, gather their Q values from
// shared memory (the x-shift and the periodic x-wrap are index arithmetic inside the staged row),
// release the stage on its "empty" mbarrier, collide in registers and store straight to global
// memory. Warp specialisation keeps the copy issue off the consumers' critical path: one warp
// issues about one bulk copy per ~125 cycles, so copies are kept >= 2 KB (scripts/tma_probe.cu).
//
//   pull: plane q of src, row (y - cy, z - cz), element x - cx; store dst[x](q)
//   AA even: plane q of f, row (y, z), element x; store f[x](qbar)
//   AA odd             : plane qbar of f, row (y - cy, z - cz), element x - cx; store f[x + c](q)
//   EsoTwist: slot q (even) / qbar (odd) of location x - c^+; store at x + c^- (slot
//                        qbar / q)
//
// In-place safety (AA, EsoTwist): every slot a cell reads in a step is written in that step by the
// same cell only, and a CTA prefetches only rows of its own future tiles, so the early reads of the
// prefetch never see another cell's write of this step. Bulk copies need 16-byte aligned addresses
// and sizes: the launcher uses this path only when nx * sizeof(T) % 16 == 0 (then every row start
// is aligned); flag rows are staged too when nx % 16 == 0.
#pragma once
#include "kernels.cuh"

namespace lbm {

enum SMode { SM_PULL = 0, SM_AA_EVEN = 1, SM_AA_ODD = 2, SM_ESO_EVEN = 3, SM_ESO_ODD = 4, SM_PUSH = 5 };
// arriving population q of cell x is read from location x - rshift(c_q) (componentwise) ...
__host__ __device__ constexpr int rshift(int mode, int c) {
    return (mode == SM_AA_EVEN || mode == SM_PUSH) ? 0 : (mode == SM_ESO_EVEN || mode == SM_ESO_ODD) ? (c > 0 ? c : 0) : c;
}
// ... in slot src_slot (EsoTwist: P:875-891, kernels.cuh eso_cell)
template <int Q>
__host__ __device__ constexpr int src_slot(int mode, int q) {
    return (mode == SM_AA_ODD || mode == SM_ESO_ODD) ? Stencil<Q>::opp(q) : q;
}

#ifndef LBM_STAGED_BT
#define LBM_STAGED_BT 256
#endif
constexpr int kStagedBT = LBM_STAGED_BT;

// Consumer threads per CTA. A CTA of 9 warps puts 3 warps on one of the 4 SM sub-partitions, whose 16K
// registers then cap every thread at 168; the D3Q27 KBC needs more (it spilled ~160 B per thread at 168),
// so it runs 7 consumer warps + the producer (8 warps, 2 per sub-partition: up to 255 registers).
// (LBM_STAGED_BT224_F64 = build variant for sweeps: every fp64 staged kernel with 7 consumer warps)
template <int Q, int OPX, typename T>
struct StagedBT {
    static constexpr int OP = op_class(op_base(OPX));
#ifdef LBM_STAGED_BT224_F64
    static constexpr int value = sizeof(T) == 8 ? 224 : kStagedBT;
#else
    static constexpr int value = (sizeof(T) == 8 && Q == 27 && (OP == OP_KBC || OP == OP_KBC_EXACT)) ? 224 : kStagedBT;
#endif
};

// registers: 65536 / (BT * minBlocks); the heavy fp64 operators get more room
template <int Q, int OPX, typename T>
struct StagedMinBlocks {
    static constexpr int OP = op_class(op_base(OPX));
    static constexpr bool heavy = sizeof(T) == 8 && (OP == OP_MRT || OP == OP_CUMULANT || OP == OP_KBC || OP == OP_KBC_EXACT || OP == OP_SMAGORINSKY || Q == 27);
#ifdef LBM_STAGED_MINB
    static constexpr int value = LBM_STAGED_MINB;
#else
    static constexpr int value = (StagedBT<Q, OPX, T>::value >= 224 ? 1 : 2) * (heavy ? 1 : 2);
#endif
};

__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint64_t *b, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_fence_init() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
__device__ __forceinline__ void mbar_expect_tx(uint64_t *b, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *b, uint32_t parity) {
    uint32_t done;
    do {
        asm volatile(
            "{\n\t.reg .pred p;\n\t"
            "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
            "selp.u32 %0, 1, 0, p;\n\t}"
            : "=r"(done)
            : "r"(smem_u32(b)), "r"(parity)
            : "memory");
    } while (!done);
}
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, uint32_t bytes, uint64_t *bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(smem_u32(dst)),
                 "l"(src), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t *b) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}

// Tile = hl (<= H) consecutive full x-rows y0 .. y0+hl-1 of one storage plane zs. Full rows are
// contiguous in the [q][z][y][x] layout, so the source rows of a direction are one bulk copy (two
// when the y-shift wraps around the domain), and the periodic x-wrap is an index wrap inside the
// staged row: no halo pads, no extra copies.
struct Tile {
    int y0, hl, zs;
};

__device__ __forceinline__ Tile tile_of(const StepArgs &a, int t, int H) {
    const int nyt = (a.geo.ny + H - 1) / H;
    Tile tl;
    const int p = t / nyt;
    tl.y0 = (t - p * nyt) * H;
    tl.hl = min(H, a.geo.ny - tl.y0);
    tl.zs = a.z_begin + p * a.z_step + a.geo.g;
    return tl;
}

// Producer warp: bulk copies of tile `tl` into stage `buf` ([Q][H*nx] elements, + the tile's own flag
// rows after them in bulk wall mode), completion on `bar`.
template <int Q, typename T, int FM, int MODE>
__device__ __forceinline__ void stage_issue(const StepArgs &a, const T *f, const Tile &tl, int H, T *buf, uint64_t *bar,
                                            int lane) {
    using S = Stencil<Q>;
    const int nx = a.geo.nx, ny = a.geo.ny;
    const uint32_t row_bytes = (uint32_t)nx * sizeof(T);
    const uint32_t per_q = (uint32_t)tl.hl * row_bytes;
    // flag rows staged too (bulk copies need 16-byte rows and a 16-byte aligned flag base; the host side
    // checks the base, flags_staged())
    const bool sflags = (FM == FM_BULK || FM == FM_LINKS) && nx % 16 == 0 && a.stage_flags;
    const uint32_t flag_bytes = sflags ? (uint32_t)tl.hl * (uint32_t)nx : 0u;
    if (lane == 0) mbar_expect_tx(bar, per_q * Q + flag_bytes);
    __syncwarp();
    for (int q = lane; q < Q; q += 32) {
        const int P = src_slot<Q>(MODE, q);
        int ys = tl.y0 - rshift(MODE, S::cy(q));
        ys = ys < 0 ? ys + ny : (ys >= ny ? ys - ny : ys);
        int zz = tl.zs - rshift(MODE, S::cz(q));
        if (!a.geo.g) zz = zz < 0 ? zz + a.geo.nz : (zz >= a.geo.nz ? zz - a.geo.nz : zz);
        LBM_ASSERT(zz >= 0 && zz < a.geo.nz + 2 * a.geo.g && ys >= 0 && ys < ny && tl.hl >= 1 && tl.hl <= H);
        const T *plane = f + (int64_t)P * a.geo.Sq + (int64_t)zz * ny * nx;
        T *dst = buf + (int64_t)q * H * nx;
        const int n1 = min(tl.hl, ny - ys);  // rows before the y-wrap
        bulk_g2s(dst, plane + (int64_t)ys * nx, (uint32_t)n1 * row_bytes, bar);
        if (n1 < tl.hl) bulk_g2s(dst + (int64_t)n1 * nx, plane, (uint32_t)(tl.hl - n1) * row_bytes, bar);
    }
    if (sflags && lane == 31)
        bulk_g2s(reinterpret_cast<uint8_t *>(buf + (int64_t)Q * H * nx),
                 a.flags + ((int64_t)tl.zs * ny + tl.y0) * nx, flag_bytes, bar);
}

template <int Q, int OP, typename T, int FM, bool FORCE, int MODE>
__global__ void __launch_bounds__(StagedBT<Q, OP, T>::value + 32, (StagedMinBlocks<Q, OP, T>::value))
    k_staged(const StepArgs a, const T *src, T *dst, int nplanes, int H, int nstages, int stage_elems) {
    using S = Stencil<Q>;
    constexpr int BT = StagedBT<Q, OP, T>::value;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    uint64_t *full = reinterpret_cast<uint64_t *>(smem_raw);  // [nstages]: tile bytes landed
    uint64_t *empty = full + 8;                                 // [nstages]: consumer warps done with it
    T *stages = reinterpret_cast<T *>(smem_raw + 128);
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int nx = a.geo.nx;
    const int ntiles = ((a.geo.ny + H - 1) / H) * nplanes;
    if (tid == 0) {
        for (int s = 0; s < nstages; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], BT / 32);
        }
        mbar_fence_init();
    }
    __syncthreads();
    if (warp == BT / 32) {
        // producer warp: refill a stage as soon as every consumer warp is done with it
        int it = 0;
        for (int t = blockIdx.x; t < ntiles; t += gridDim.x, ++it) {
            const int stage = it % nstages;
            if (it >= nstages) mbar_wait(&empty[stage], (uint32_t)(((it / nstages) - 1) & 1));
            stage_issue<Q, T, FM, MODE>(a, src, tile_of(a, t, H), H, stages + (int64_t)stage * stage_elems, &full[stage], lane);
        }
        return;
    }
    const Rates<T> r = load_rates<T>(a);
    const int64_t Sq = a.geo.Sq;
    const int rowlen = H * nx;  // elements per q in a stage
    const bool sflags = (FM == FM_BULK || FM == FM_LINKS) && nx % 16 == 0 && a.stage_flags;
    int it = 0;
    for (int t = blockIdx.x; t < ntiles; t += gridDim.x, ++it) {
        const int stage = it % nstages;
        const Tile tl = tile_of(a, t, H);
        const T *buf = stages + (int64_t)stage * stage_elems;
        const uint8_t *fl = reinterpret_cast<const uint8_t *>(buf + (int64_t)Q * rowlen);
        mbar_wait(&full[stage], (uint32_t)((it / nstages) & 1));
        const int ncell = tl.hl * nx;
        int h = tid / nx, x = tid - (tid / nx) * nx;
        for (int c = tid; c < ncell; c += BT) {
            const int hc = h, xc = x;
            x += BT;
            while (x >= nx) {
                x -= nx;
                ++h;
            }
            uint8_t own = 0;
            if (FM == FM_BULK || FM == FM_LINKS) {
                // FM_BULK: walls and near-wall cells belong to the edge kernel (AA even: only walls are skipped;
                // the even step is local, so near-wall cells need nothing special there). FM_LINKS: walls are
                // skipped, near-wall cells store their links after the collision.
                own = sflags ? fl[c]
                             : a.flags[((uint32_t)tl.zs * (uint32_t)a.geo.ny + (uint32_t)(tl.y0 + hc)) * (uint32_t)nx +
                                       (uint32_t)xc];
                if ((FM == FM_LINKS || MODE == SM_AA_EVEN) ? (own & 3) != 0 : own != 0) continue;
            }
            const int xm = xc == 0 ? nx - 1 : xc - 1, xp = xc == nx - 1 ? 0 : xc + 1;
            T g[Q];
#pragma unroll
            for (int q = 0; q < Q; ++q) {
                const int sx = rshift(MODE, S::cx(q));
                const int xs = sx == 0 ? xc : (sx > 0 ? xm : xp);
                g[q] = buf[q * rowlen + hc * nx + xs];
            }
            collide<Q, OP, T, FORCE>(g, r);
            const int y = tl.y0 + hc;
            const uint32_t self = ((uint32_t)tl.zs * (uint32_t)a.geo.ny + (uint32_t)y) * (uint32_t)nx + (uint32_t)xc;
            LBM_ASSERT((int64_t)self < Sq && y < a.geo.ny && (a.geo.g ? (tl.zs >= 1 && tl.zs <= a.geo.nz) : tl.zs < a.geo.nz));
            if constexpr (MODE == SM_PULL) {
#pragma unroll
                for (int q = 0; q < Q; ++q) dst[q * Sq + self] = g[q];
            } else if constexpr (MODE == SM_AA_EVEN) {
#pragma unroll
                for (int q = 0; q < Q; ++q) dst[S::opp(q) * Sq + self] = g[q];
            } else if constexpr (MODE == SM_PUSH) {  // collide-stream-push into the second array
                const Nbr n = neighbours(a.geo, xc, y, tl.zs);
#pragma unroll
                for (int q = 0; q < Q; ++q) dst[q * Sq + nb_off(a.geo, n, S::cx(q), S::cy(q), S::cz(q))] = g[q];
            } else if constexpr (MODE == SM_ESO_EVEN || MODE == SM_ESO_ODD) {
                // departing q at x + c_q^- (slot qbar after the even step, q after the odd one)
                const Nbr n = neighbours(a.geo, xc, y, tl.zs);
#pragma unroll
                for (int q = 0; q < Q; ++q)
                    dst[(MODE == SM_ESO_ODD ? q : S::opp(q)) * Sq + nb_off(a.geo, n, cneg(S::cx(q)), cneg(S::cy(q)), cneg(S::cz(q)))] =
                        g[q];
            } else {
                const Nbr n = neighbours(a.geo, xc, y, tl.zs);
#pragma unroll
                for (int q = 0; q < Q; ++q) dst[q * Sq + nb_off(a.geo, n, S::cx(q), S::cy(q), S::cz(q))] = g[q];
            }
            if constexpr (FM == FM_LINKS && (MODE == SM_PULL || MODE == SM_AA_EVEN || MODE == SM_AA_ODD)) {
                if (own & 0x80) {  // the link stores of kernels.cuh FM_LINKS
                    const uint64_t m = a.lmask[self];
                    const Nbr n = neighbours(a.geo, xc, y, tl.zs);
#pragma unroll
                    for (int q = 0; q < Q; ++q) {
                        if (!((m >> q) & 1)) continue;
                        const T v = link_value<Q, T>(a, m, g, q);
                        if constexpr (MODE == SM_PULL) dst[q * Sq + nb_off(a.geo, n, -S::cx(q), -S::cy(q), -S::cz(q))] = v;
                        else if constexpr (MODE == SM_AA_EVEN)
                            dst[S::opp(q) * Sq + nb_off(a.geo, n, -S::cx(q), -S::cy(q), -S::cz(q))] = v;
                        else dst[q * Sq + self] = v;
                    }
                }
            }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[stage]);  // this warp is done with the stage
    }
}

// Host side: persistent grid of (co-resident CTAs); stage = H full rows per direction (+ flag rows),
// H chosen so that a stage stays below ~48 KB; nstages stages.
int staged_nstages();  // LBM_STAGES (default 2), k_misc.cu
int staged_path();     // 0 auto, 1 plain, 2 staged (lbm_set_kernel_path / LBM_KERNEL_PATH)

// Auto policy, from B200 sweeps: the staged kernels win for the register-heavy
// operators (MRT, KBC, Smagorinsky; the cumulant in the AA pattern), the plain kernels for TRT/SRT
// (already at copy bandwidth) and the cumulant pull kernel. The exact (Newton) KBC is FP64-ALU bound:
// the plain kernel with the full register file wins (D3Q27 1.65 vs 0.94 GLUPS, staged spills).
template <int Q, int OPX, int MODE>
constexpr bool staged_auto() {
    constexpr int OP = op_class(op_base(OPX));
    // generated D3Q27 SRT/TRT: the CSE'd code needs more registers than the plain kernels' cap
    // (AA 512^3 fp64: plain 0.86, staged 0.92 of copy BW; hand-written TRT plain 0.97)
    constexpr bool gen27 = Q == 27 && (op_base(OPX) == OP_GEN_SRT || op_base(OPX) == OP_GEN_TRT);
    // cumulant: staged for AA / EsoTwist (in place), plain for the two-array pull and push kernels
    // (C3 push: plain 0.906 vs staged 0.857 of copy BW; scripts/gpu_path_sweep.sh). The unit-rate D3Q27
    // cumulant (C3's rates, ~650 instead of 1135 FP64 operations) runs plain in every pattern (AA 512^3:
    // 1.004 vs 0.906; C3 cavity AA + index lists 0.930 vs 0.879; EsoTwist 0.844 vs 0.831; scripts/gpu_r02i.sh)
    constexpr bool cum_unit = op_base(OPX) == OP_CUMULANT_UNIT;
    // the shear-only weighted MRT (C2's rates) runs plain too: AA 512^3 fp64 0.996 vs 0.942 staged; C2 fp32
    // 0.918 vs 0.912 (scripts/gpu_r02q.sh)
    constexpr bool mrt_shear = op_base(OPX) == OP_MRT_SHEAR;
    return (OP == OP_MRT && !mrt_shear) || OP == OP_MRT_ROWS || OP == OP_KBC || OP == OP_SMAGORINSKY ||
           (OP == OP_CUMULANT && !cum_unit && MODE != SM_PULL && MODE != SM_PUSH) || gen27;
}

template <int Q, int OP, typename T, int FM, bool FORCE, int MODE>
bool staged_launch(const StepArgs &a, const void *src, void *dst, int nplanes, cudaStream_t s) {
    if constexpr (FM != FM_NONE && FM != FM_BULK && FM != FM_LINKS) {  // inline walls (low-level ABI): plain kernels only
        (void)a, (void)src, (void)dst, (void)nplanes, (void)s;
        return false;
    } else {
    constexpr int BT = StagedBT<Q, OP, T>::value;
    const int path = staged_path();
    // (AA with the split flag mode ran staged for the TRT class until the plain AA kernels issued their
    // population loads ahead of the flag test: Fig. 8 walled channel plain 0.869 vs staged 0.831 of copy BW)
    if (path == 1 || (path == 0 && !staged_auto<Q, OP, MODE>())) return false;
    const int64_t row_bytes = (int64_t)a.geo.nx * (int64_t)sizeof(T);
    if (row_bytes % 16 != 0) return false;
    if ((reinterpret_cast<uintptr_t>(src) | reinterpret_cast<uintptr_t>(dst)) % 16 != 0) return false;
    const int nst = staged_nstages();
    int H = (int)((48 * 1024) / (Q * row_bytes));
    if (H < 1) H = 1;
    if (H > a.geo.ny) H = a.geo.ny;
    // flag rows are staged by bulk copy only from a 16-byte aligned flag base (a caller's flags pointer in
    // the low-level ABI may be any torch view); otherwise consumers read the flag byte from global memory
    StepArgs b = a;
    b.stage_flags = (FM == FM_BULK || FM == FM_LINKS) && a.geo.nx % 16 == 0 && reinterpret_cast<uintptr_t>(a.flags) % 16 == 0;
    const int64_t stage_bytes = ((int64_t)Q * H * row_bytes + (b.stage_flags ? (int64_t)H * a.geo.nx : 0) + 127) / 128 * 128;
    const size_t smem = 128 + (size_t)nst * stage_bytes;
    if (smem > 227 * 1024) return false;
    auto kern = k_staged<Q, OP, T, FM, FORCE, MODE>;
    int dev = 0;
    cudaGetDevice(&dev);
    // the shared-memory attribute is per device: cache the largest size set, per device ordinal
    static size_t smem_set[kMaxDevices] = {};
    if (dev < 0 || dev >= kMaxDevices) return false;
    if (smem > smem_set[dev]) {
        if (cudaFuncSetAttribute((const void *)kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
            return false;
        smem_set[dev] = smem;
    }
    int per_sm = 0, sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, BT + 32, smem) != cudaSuccess || per_sm < 1) return false;
    const int64_t ntiles = (int64_t)((a.geo.ny + H - 1) / H) * nplanes;
    if (ntiles <= 0) return true;
    const int64_t cores = (int64_t)per_sm * sms;
    const int grid = (int)(ntiles < cores ? ntiles : cores);
    kern<<<grid, BT + 32, smem, s>>>(b, static_cast<const T *>(src), static_cast<T *>(dst), nplanes, H, nst,
                                     (int)(stage_bytes / (int64_t)sizeof(T)));
    return true;
    }
}

}  // namespace lbm
