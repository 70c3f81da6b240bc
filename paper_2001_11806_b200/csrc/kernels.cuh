// kernels.cuh — sm_100a kernels of the fused LB time step (templates; instantiated per op in
// k_*.cu so the heavy variants compile in parallel).
//
// Data layout: SoA, element (q, zs, y, x) at q*Sq + (zs*ny + y)*nx + x,
// zs = z + g the storage plane (g = 1 ghost plane per z side in slab mode, else 0), x fastest.
// One thread per cell along x; a block spans an x-row segment (BX threads) times BY rows; the
// grid covers (x-blocks, y-blocks, z planes). Every population is read once and written once
// per step: 2*q*sizeof(T) bytes per fluid cell, + 1 B of flag near walls.
#pragma once
#include <cassert>
#include <cstdint>
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include "collide.cuh"
#include "stencil.cuh"

// Minimum resident 256-thread blocks per SM requested from ptxas; it caps registers per thread
// (2 -> 128, 3 -> 80, 4 -> 64, 6 -> 40) and so sets how many population loads are in flight per SM.
// Measured on B200 (scripts/gpu_sweep.sh): D3Q19 TRT fp64 3 (c4 1.03 of copy
// BW, c1 0.98), D3Q19 TRT fp32 6 (c1 0.92), D3Q27 cumulant fp64 3 (c3 0.67), MRT fp32 AA 3 (c2
// 0.75); other families use the largest value without register spills. Exception: the exact (Newton)
// KBC is FP64-latency bound; 2 CTAs of 128 registers (small spills) beat 1 CTA of 255 registers
// without spills (D3Q19 4.77 vs 3.14 GLUPS, D3Q27 2.76 vs 2.08). LBM_MINB_OVERRIDE_* exist
// for sweeps only.
namespace lbm {

template <int Q, int OPX, typename T>
struct MinBlocks {
    static constexpr int OP = op_class(op_base(OPX));  // the equilibrium variant bits do not change the cap
    static constexpr bool f64 = sizeof(T) == 8;
    // OP: 0 SRT, 1 TRT, 2 MRT, 3 cumulant, 4 identity, 5 Smagorinsky, 6 KBC, 7 KBC exact, 8 MRT rows
    static constexpr int pull_default =
        f64 ? ((OP == 2 || OP == 5 || OP == 6 || OP == 7 || (Q == 27 && OP <= 1)) ? 2 : 3)
            : ((OP <= 1 || OP == 4 || OP == 5) ? (Q == 19 ? 6 : 4) : 3);
    static constexpr int aa_default = f64 ? 2 : ((OP == 2 || OP == 6 || (Q == 19 && (OP <= 1 || OP == 5))) ? 3 : 2);
#ifdef LBM_MINB_OVERRIDE_PULL
    static constexpr int pull = LBM_MINB_OVERRIDE_PULL;
#else
    static constexpr int pull = pull_default;
#endif
#ifdef LBM_MINB_OVERRIDE_AA
    static constexpr int aa = LBM_MINB_OVERRIDE_AA;
#else
    static constexpr int aa = aa_default;
#endif
};

struct Geo {
    int nx, ny, nz;  // local interior extent
    int g;           // ghost planes per z side (0: z wraps locally)
    int64_t Sq;      // elements per q plane = nx*ny*(nz+2g)
};

struct StepArgs {
    Geo geo;
    int z_begin;  // first local plane (interior index) of this launch
    int z_step;   // plane stride between blockIdx.z values (boundary-plane launches use nz-1)
    double rates[16];              // per operator (include/lbm.h); 15 per-moment MRT rates
    double F[3];
    double uw[3];                  // UBB wall velocity; rho_w = 1 (G8)
    const uint8_t *flags;          // storage-indexed (with ghost planes) or nullptr; bits 0-1 = type
                                   // (0 fluid, 1 no-slip, 2 UBB), bit 7 = fluid cell with a non-fluid
                                   // neighbour (only such cells read neighbour flags)
    void *peer_up;                 // fused halo (boundary launch only): base of the up neighbour's
    void *peer_down;               // dst array / down neighbour's dst array (NVLink LSA pointers)
    int stage_flags;               // staged kernels (set by the launcher): flag rows moved by bulk copy
    // FM_FACES (face-aligned walls): wall type of the faces -x, +x, -y, +y, -z, +z (0 none, 1 no-slip,
    // 2 UBB; a cell on several wall faces takes the first in this order), global z of interior plane 0
    // and the global nz
    int8_t face[6];
    int zg0, nzg;
    // FM_LINKS (in-kernel index-list boundaries): per storage cell, bit q = the cell x - c_q is a wall whose
    // slot x streams from (the link (b = x - c_q, q) of LBM_BOUNDARY_LINKS), bit 32 + q = that wall is UBB;
    // read by near-wall fluid cells only
    const uint64_t *lmask;
    // launch box of the plain update kernels (local x, y): the bounding box of the non-wall cells (walls on
    // the domain faces get no threads at all), or the whole plane
    int x0, x1, y0, y1;
    // flat rows (flat_hi > 0; box of full x-rows whose nx leaves idle lanes at the row end, e.g. the
    // 300 x 100 x 100 domain of Fig. 7 / 8): the threads of a plane index the contiguous cells
    // [flat_lo, flat_hi) = [y0 nx, y1 nx) linearly from flat_start = flat_lo rounded down to 32, so warps
    // stay full across row ends and keep their 32-cell alignment in the plane; flat_magic = 2^32 / nx + 1
    int flat_lo, flat_hi, flat_start;
    unsigned flat_magic;
};

// this thread's cell of the launch box; false outside it
__device__ __forceinline__ bool box_cell(const StepArgs &a, int &x, int &y) {
    if (a.flat_hi > 0) {  // (256, 1, 1) blocks over the rows' cells
        const unsigned i = (unsigned)a.flat_start + blockIdx.x * blockDim.x + threadIdx.x;
        if (i < (unsigned)a.flat_lo || i >= (unsigned)a.flat_hi) return false;
        unsigned r = __umulhi(i, a.flat_magic);  // i / nx or one more
        if (r * (unsigned)a.geo.nx > i) --r;
        y = (int)r;
        x = (int)(i - r * (unsigned)a.geo.nx);
        return true;
    }
    x = a.x0 + (int)(blockIdx.x * blockDim.x + threadIdx.x);
    y = a.y0 + (int)(blockIdx.y * blockDim.y + threadIdx.y);
    return x < a.x1 && y < a.y1;
}

constexpr int kMaxDevices = 64;  // per-device caches of launch attributes and occupancy

template <typename T>
__device__ __forceinline__ Rates<T> load_rates(const StepArgs &a) {
    Rates<T> r;
#pragma unroll
    for (int i = 0; i < 16; ++i) r.r[i] = T(a.rates[i]);
#pragma unroll
    for (int i = 0; i < 3; ++i) r.F[i] = T(a.F[i]);
    return r;
}

template <typename T>
__device__ __forceinline__ T ldg_stream(const T *p) {
    return __ldg(p);
}

// The flag-reading kernels (FM_LINKS, FM_BULK) issue the population loads before they test the cell's flag
// byte, so the two memory latencies overlap instead of adding up. ptxas sinks loads below a branch whose
// other side does not use them (even loads from volatile asm), so the early exit consumes them: an XOR of
// their bit patterns guards a store into a scratch word of the library that nothing reads.
__device__ __forceinline__ uint64_t bits_of(double v) { return (uint64_t)__double_as_longlong(v); }
__device__ __forceinline__ uint64_t bits_of(float v) { return (uint64_t)__float_as_uint(v); }
static __device__ unsigned long long g_lbm_sink;  // one per translation unit (no relocatable device code)
template <int Q, typename T>
__device__ __forceinline__ void keep_loads(const T (&g)[Q]) {
    uint64_t x = 0;
#pragma unroll
    for (int q = 0; q < Q; ++q) x ^= bits_of(g[q]);
    if (x == 0x5bd1e9955bd1e995ull) g_lbm_sink = x;
}

// Neighbour coordinates for a cell: index arrays [c+1] -> coordinate of the cell at offset c.
struct Nbr {
    int xs[3], ys[3], zs[3];
};

// Debug builds (-DLBM_BOUNDS_CHECK, `build.build(defines=["LBM_BOUNDS_CHECK"])`) assert that every
// cell an update kernel touches lies inside the storage of its slab (compute-sanitizer is not
// available on the GPU pool; the GPU tests run once against this variant).
#ifdef LBM_BOUNDS_CHECK
#define LBM_ASSERT(c) assert(c)
#else
#define LBM_ASSERT(c) ((void)0)
#endif

// Fused halo: a thread that stored into a neighbour's window over NVLink makes those stores visible at
// system scope before it exits; the next step's LSA gate (k_fused.cu) then orders them before every
// rank's next reads. (Kernel completion alone is not specified to order peer-GPU stores for readers on
// the other GPU; the fence makes the release explicit, and costs only the two boundary planes.)
template <bool PEER>
__device__ __forceinline__ void peer_fence() {
    if constexpr (PEER) __threadfence_system();
}

__device__ __forceinline__ Nbr neighbours(const Geo &g, int x, int y, int zs) {
    LBM_ASSERT(x >= 0 && x < g.nx && y >= 0 && y < g.ny);
    LBM_ASSERT(g.g ? (zs >= 1 && zs <= g.nz) : (zs >= 0 && zs < g.nz));  // only interior planes update
    Nbr n;
    n.xs[1] = x;
    n.xs[0] = (x == 0) ? g.nx - 1 : x - 1;
    n.xs[2] = (x == g.nx - 1) ? 0 : x + 1;
    n.ys[1] = y;
    n.ys[0] = (y == 0) ? g.ny - 1 : y - 1;
    n.ys[2] = (y == g.ny - 1) ? 0 : y + 1;
    n.zs[1] = zs;
    if (g.g) {
        n.zs[0] = zs - 1;
        n.zs[2] = zs + 1;
    } else {
        n.zs[0] = (zs == 0) ? g.nz - 1 : zs - 1;
        n.zs[2] = (zs == g.nz - 1) ? 0 : zs + 1;
    }
    return n;
}

// in-plane offset (cells) of the neighbour at offset (dx,dy,dz)
__device__ __forceinline__ uint32_t nb_off(const Geo &g, const Nbr &n, int dx, int dy, int dz) {
    return ((uint32_t)n.zs[dz + 1] * (uint32_t)g.ny + (uint32_t)n.ys[dy + 1]) * (uint32_t)g.nx + (uint32_t)n.xs[dx + 1];
}

// =======================================================================================
// Wall handling modes of the update kernels (flags = storage-indexed flag bytes):
//   FM_NONE   no flag field (periodic / walls absent);
//   FM_INLINE every cell reads its flag, wall cells return, near-wall cells (bit 7) resolve the
//             directions that come from a wall in the same kernel (low-level ABI);
//   FM_BULK   the bulk kernel of the split: cells with any flag bit (walls and near-wall cells)
//             return after one 1-byte read, so the kernel runs the periodic fast path;
//   FM_EDGE   the boundary kernel of the split: processes only the near-wall fluid cells given by
//             an index list (the GPU form of the paper's separate boundary kernels);
//   FM_FACES  face-aligned walls (every wall cell lies on a domain face, e.g. the channel and cavity of
//             C1/C3, detected from the flag field at create): wall and near-wall cells are recognised from
//             their coordinates, no flag read and no separate boundary launch; the same substitutions.
//   FM_LINKS  index-list boundaries folded into the update (LBM_BOUNDARY_LINKS, pull and AA): every cell
//             reads its flag byte (wall cells return), the gathers are unconditional (the wall slots hold
//             the bounced values), and a near-wall fluid cell writes, after its collision, the wall slots of
//             its links that the next stream reads — the link kernel's work without its launch
//             and without re-reading the fluid slots:
//               pull    dst[x - c_q](q)  = f*_qbar(x) + t_q   (= link mode 0 before the next step)
//               AA even a[x - c_q](qbar) = f*_qbar(x) + t_q   (= link mode 1)
//               AA odd  a[x](q)          = f*_qbar(x) + t_q   (= link mode 2: x's push toward the wall)
//             for every link (b = x - c_q, q) in the cell's mask (StepArgs::lmask), t_q the UBB term. Each such
//             slot is read by x alone, and no other cell writes it in that step.
// =======================================================================================
enum FMode { FM_NONE = 0, FM_INLINE = 1, FM_BULK = 2, FM_EDGE = 3, FM_FACES = 4, FM_LINKS = 5 };

// UBB term 6 w_q rho_w c_q.u_w (rho_w = 1, G8) in the storage precision
template <int Q, typename T>
__device__ __forceinline__ T ubb_term(const StepArgs &a, int q) {
    using S = Stencil<Q>;
    const double cu = S::cx(q) * a.uw[0] + S::cy(q) * a.uw[1] + S::cz(q) * a.uw[2];
    return T(6.0 * S::w(q) * cu);
}

// FM_LINKS: the value the link (x - c_q, q) of a near-wall cell stores, f*_qbar(x) + t_q, rounded like the
// link kernel's load + add (an add that is never contracted with the collision's last product)
__device__ __forceinline__ double add_rn(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ float add_rn(float a, float b) { return __fadd_rn(a, b); }
template <int Q, typename T>
__device__ __forceinline__ T link_value(const StepArgs &a, uint64_t m, const T (&g)[Q], int q) {
    using S = Stencil<Q>;
    return ((m >> (32 + q)) & 1) ? add_rn(g[S::opp(q)], ubb_term<Q, T>(a, q)) : g[S::opp(q)];
}

// FM_FACES: wall type of the cell at (x, y, global z), 0 for fluid (coordinates one step outside the
// domain belong to a periodic axis: never a wall)
__device__ __forceinline__ int face_wall(const StepArgs &a, int x, int y, int zg) {
    if (a.face[0] && x == 0) return a.face[0];
    if (a.face[1] && x == a.geo.nx - 1) return a.face[1];
    if (a.face[2] && y == 0) return a.face[2];
    if (a.face[3] && y == a.geo.ny - 1) return a.face[3];
    if (a.face[4] && zg == 0) return a.face[4];
    if (a.face[5] && zg == a.nzg - 1) return a.face[5];
    return 0;
}
// FM_FACES: a fluid cell with a wall among its neighbours (next to a wall face)
__device__ __forceinline__ bool near_face(const StepArgs &a, int x, int y, int zg) {
    return (a.face[0] && x == 1) || (a.face[1] && x == a.geo.nx - 2) || (a.face[2] && y == 1) ||
           (a.face[3] && y == a.geo.ny - 2) || (a.face[4] && zg == 1) || (a.face[5] && zg == a.nzg - 2);
}

// =======================================================================================
// Fused stream-pull-collide, two arrays: dst = C(S(src)) at one fluid cell.
// =======================================================================================
template <int Q, int OP, typename T, int FM, bool FORCE, bool PEER>
__device__ __forceinline__ void pull_cell(const StepArgs &a, const T *__restrict__ src, T *__restrict__ dst, int x, int y,
                                          int zs) {
    using S = Stencil<Q>;
    const Nbr n = neighbours(a.geo, x, y, zs);
    const uint32_t self = nb_off(a.geo, n, 0, 0, 0);
    const int64_t Sq = a.geo.Sq;
    bool edge = FM == FM_EDGE;
    int zg = 0;
    // inline walls with the gather-then-fix-up strategy (below): the own flag is tested after the gathers for
    // the D3Q19 fp64 kernels (C1 inline 0.991 -> 1.009); the D3Q27 cumulant pull kernel spills with the live
    // flag at its 80-register cap (C3 inline 0.755 -> 0.663) and keeps the flag-first order
    constexpr bool kInlineLate = FM == FM_INLINE && sizeof(T) == 8 && Q == 19;
    if (FM == FM_INLINE && !kInlineLate) {
        const uint8_t own = a.flags[self];
        if (own & 3) return;  // wall cells are not updated
        edge = (own & 0x80) != 0;
    } else if (FM == FM_BULK) {
        // walls, and near-wall cells (done by the edge kernel); flag first: for the pull kernels the
        // load-first order measured no better (C3 split 0.83 either way) and the fp32 kernel pays for the
        // live flag (C1 fp32 split 0.933 -> 0.913)
        if (a.flags[self] != 0) return;
    } else if (FM == FM_FACES) {
        zg = a.zg0 + zs - a.geo.g;
        if (face_wall(a, x, y, zg)) return;
        edge = near_face(a, x, y, zg);
    }
    // FM_LINKS: the flag byte is tested after the gathers are issued (every cell's storage exists), so the
    // population loads do not wait for the flag load
    const uint8_t own_l = (FM == FM_LINKS || kInlineLate) ? a.flags[self] : 0;
    // wall type of the cell x - c_q (the source of direction q)
    auto wall_src = [&](int q) -> int {
        if constexpr (FM == FM_FACES) return face_wall(a, x - S::cx(q), y - S::cy(q), zg - S::cz(q));
        else return a.flags[nb_off(a.geo, n, -S::cx(q), -S::cy(q), -S::cz(q))] & 3;
    };
    // Two strategies for near-wall cells in the inline mode, chosen per kernel family from B200
    // measurements: gather-then-fix-up (fp64 and the cumulant: all Q loads
    // issue back to back — the neighbour's storage always exists, wall or not — and the wall
    // directions are replaced afterwards) and branch-per-direction (fp32 TRT at 40 registers).
    constexpr bool kWalls = FM == FM_INLINE || FM == FM_EDGE || FM == FM_FACES;
    constexpr bool kFixup = kWalls && (sizeof(T) == 8 || op_class(op_base(OP)) == OP_CUMULANT) &&
                            (FM == FM_INLINE || FM == FM_FACES);
    T g[Q];
    if constexpr (kWalls && !kFixup) {
#pragma unroll
        for (int q = 0; q < Q; ++q) {
            const uint32_t o = nb_off(a.geo, n, -S::cx(q), -S::cy(q), -S::cz(q));
            if (edge) {
                const int fl = wall_src(q);
                if (fl == 0) {
                    g[q] = ldg_stream(src + q * Sq + o);
                } else {
                    T v = ldg_stream(src + S::opp(q) * Sq + self);
                    if (fl == 2) {
                        const double cu = S::cx(q) * a.uw[0] + S::cy(q) * a.uw[1] + S::cz(q) * a.uw[2];
                        v += T(6.0 * S::w(q) * cu);
                    }
                    g[q] = v;
                }
            } else {
                g[q] = ldg_stream(src + q * Sq + o);
            }
        }
    } else {
#pragma unroll
        for (int q = 0; q < Q; ++q)
            g[q] = ldg_stream(src + q * Sq + nb_off(a.geo, n, -S::cx(q), -S::cy(q), -S::cz(q)));
    }
    if (FM == FM_LINKS || kInlineLate) {
        if (own_l & 3) {  // wall cells are not updated
            keep_loads<Q, T>(g);
            return;
        }
        edge = (own_l & 0x80) != 0;
    }
    if (kFixup && edge) {
#pragma unroll
        for (int q = 0; q < Q; ++q) {
            const int fl = wall_src(q);
            if (fl != 0) {
                T v = ldg_stream(src + S::opp(q) * Sq + self);
                if (fl == 2) {
                    const double cu = S::cx(q) * a.uw[0] + S::cy(q) * a.uw[1] + S::cz(q) * a.uw[2];
                    v += T(6.0 * S::w(q) * cu);
                }
                g[q] = v;
            }
        }
    }
    const Rates<T> r = load_rates<T>(a);
    collide<Q, OP, T, FORCE>(g, r);
#pragma unroll
    for (int q = 0; q < Q; ++q) dst[q * Sq + self] = g[q];
    if (FM == FM_LINKS && edge) {
        const uint64_t m = a.lmask[self];
#pragma unroll
        for (int q = 0; q < Q; ++q)
            if ((m >> q) & 1) dst[q * Sq + nb_off(a.geo, n, -S::cx(q), -S::cy(q), -S::cz(q))] = link_value<Q, T>(a, m, g, q);
    }
    if (PEER) {
        // fused halo: the crossing populations of the boundary planes also go straight into the
        // neighbours' ghost planes (top plane, c_z = +1 -> up's plane 0; bottom, c_z = -1 -> down's nz+1)
        const uint32_t inplane = (uint32_t)y * (uint32_t)a.geo.nx + (uint32_t)x;
        const int64_t plane = (int64_t)a.geo.nx * a.geo.ny;
        if (zs == a.geo.nz) {
            T *up = static_cast<T *>(a.peer_up);
#pragma unroll
            for (int q = 0; q < Q; ++q)
                if (S::cz(q) == 1) up[q * Sq + inplane] = g[q];
        }
        if (zs == 1) {
            T *dn = static_cast<T *>(a.peer_down);
#pragma unroll
            for (int q = 0; q < Q; ++q)
                if (S::cz(q) == -1) dn[q * Sq + (a.geo.nz + 1) * plane + inplane] = g[q];
        }
    }
}

// One thread per cell along x; planes z = z_begin + blockIdx.z * z_step (interior indices).
template <int Q, int OP, typename T, int FM, bool FORCE, bool PEER = false>
__global__ void __launch_bounds__(256, (MinBlocks<Q, OP, T>::pull)) k_pull(const StepArgs a, const T *__restrict__ src, T *__restrict__ dst) {
    int x, y;
    if (!box_cell(a, x, y)) return;
    const int zs = a.z_begin + (int)blockIdx.z * a.z_step + a.geo.g;
    pull_cell<Q, OP, T, FM, FORCE, PEER>(a, src, dst, x, y, zs);
    peer_fence<PEER>();
}

// Near-wall fluid cells from a list of storage cell indices (one thread per listed cell).
template <int Q, int OP, typename T, bool FORCE, bool PEER = false>
__global__ void __launch_bounds__(128) k_pull_edges(const StepArgs a, const T *__restrict__ src, T *__restrict__ dst,
                                                   const uint32_t *__restrict__ cells, uint32_t n) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const uint32_t c = cells[i];
    LBM_ASSERT((int64_t)c < a.geo.Sq);
    const uint32_t plane = (uint32_t)a.geo.nx * (uint32_t)a.geo.ny;
    const int zs = (int)(c / plane);
    const uint32_t r = c - (uint32_t)zs * plane;
    pull_cell<Q, OP, T, FM_EDGE, FORCE, PEER>(a, src, dst, (int)(r % (uint32_t)a.geo.nx), (int)(r / (uint32_t)a.geo.nx), zs);
    peer_fence<PEER>();
}

// =======================================================================================
// AA pattern, one array, periodic (no flags, no ghosts).
// even: read a[x](q), collide, write a[x](qbar)   (in-place, reversed storage)
// odd : read a[x - c_q](qbar), collide, write a[x + c_q](q)
// =======================================================================================
// Fused AA halo (PEER): the boundary planes' even step also stores the slots the neighbours' odd step
// pulls across the face into their ghost planes (top plane, slots with c_z = -1 -> up's plane 0;
// bottom plane, slots with c_z = +1 -> down's plane nz+1), and the odd step stores its pushes across
// the face straight into the neighbours' interior planes (top plane, c_z = +1 -> up's plane 1; bottom
// plane, c_z = -1 -> down's plane nz), through NCCL LSA pointers of the single array. These are the
// fill and return phases of the NCCL path without a pack, a send/recv or a masked unpack (a wall
// target never receives a push: the odd step's wall rule keeps that value in the cell's own slot).
template <int Q, int OP, typename T, bool FLAGS, bool FORCE, bool PEER = false, bool LINKS = false>
__device__ __forceinline__ void aa_even_cell(const StepArgs &a, T *__restrict__ f, int x, int y, int zs) {
    using S = Stencil<Q>;
    const uint32_t self = ((uint32_t)zs * (uint32_t)a.geo.ny + (uint32_t)y) * (uint32_t)a.geo.nx + (uint32_t)x;
    const int64_t Sq = a.geo.Sq;
    const uint8_t own = FLAGS ? a.flags[self] : 0;
    T g[Q];
#pragma unroll
    for (int q = 0; q < Q; ++q) g[q] = f[q * Sq + self];
    if (own & 3) {  // wall cells are not updated (tested after the loads are issued)
        keep_loads<Q, T>(g);
        return;
    }
    const Rates<T> r = load_rates<T>(a);
    collide<Q, OP, T, FORCE>(g, r);
#pragma unroll
    for (int q = 0; q < Q; ++q) f[S::opp(q) * Sq + self] = g[q];
    if (LINKS && (own & 0x80)) {  // FM_LINKS: fill the wall slots the odd step streams from
        const uint64_t m = a.lmask[self];
        const Nbr n = neighbours(a.geo, x, y, zs);
#pragma unroll
        for (int q = 0; q < Q; ++q)
            if ((m >> q) & 1) f[S::opp(q) * Sq + nb_off(a.geo, n, -S::cx(q), -S::cy(q), -S::cz(q))] = link_value<Q, T>(a, m, g, q);
    }
    if (PEER) {
        const uint32_t inplane = (uint32_t)y * (uint32_t)a.geo.nx + (uint32_t)x;
        const int64_t plane = (int64_t)a.geo.nx * a.geo.ny;
        if (zs == a.geo.nz) {  // slot qbar with c_qbar,z = -1, i.e. c_q,z = +1
            T *up = static_cast<T *>(a.peer_up);
#pragma unroll
            for (int q = 0; q < Q; ++q)
                if (S::cz(q) == 1) up[S::opp(q) * Sq + inplane] = g[q];
        }
        if (zs == 1) {
            T *dn = static_cast<T *>(a.peer_down);
#pragma unroll
            for (int q = 0; q < Q; ++q)
                if (S::cz(q) == -1) dn[S::opp(q) * Sq + (a.geo.nz + 1) * plane + inplane] = g[q];
        }
    }
}

template <int Q, int OP, typename T, bool FLAGS, bool FORCE, bool PEER = false, bool LINKS = false>
__global__ void __launch_bounds__(256, (MinBlocks<Q, OP, T>::aa)) k_aa_even(const StepArgs a, T *__restrict__ f) {
    int x, y;
    if (!box_cell(a, x, y)) return;
    aa_even_cell<Q, OP, T, FLAGS, FORCE, PEER, LINKS>(a, f, x, y, a.z_begin + (int)blockIdx.z * a.z_step + a.geo.g);
    peer_fence<PEER>();
}

template <int Q, int OP, typename T, int FM, bool FORCE, bool PEER = false>
__device__ __forceinline__ void aa_odd_cell(const StepArgs &a, T *__restrict__ f, int x, int y, int zs) {
    using S = Stencil<Q>;
    const Nbr n = neighbours(a.geo, x, y, zs);
    const int64_t Sq = a.geo.Sq;
    bool edge = FM == FM_EDGE;
    const uint32_t self = nb_off(a.geo, n, 0, 0, 0);
    int zg = 0;
    if (FM == FM_FACES) {
        zg = a.zg0 + zs - a.geo.g;
        if (face_wall(a, x, y, zg)) return;
        edge = near_face(a, x, y, zg);
    }
    const uint8_t own_l = (FM == FM_LINKS || FM == FM_BULK || FM == FM_INLINE) ? a.flags[self] : 0;  // tested after the gathers
    // wall type of the cell x + s c_q (s = -1: the source of q, s = +1: the target of q's push)
    auto wall_at = [&](int q, int sgn) -> int {
        if constexpr (FM == FM_FACES) return face_wall(a, x + sgn * S::cx(q), y + sgn * S::cy(q), zg + sgn * S::cz(q));
        else return a.flags[nb_off(a.geo, n, sgn * S::cx(q), sgn * S::cy(q), sgn * S::cz(q))] & 3;
    };
    // unconditional gather (loads issue back to back), wall directions fixed up in near-wall cells
    T g[Q];
#pragma unroll
    for (int q = 0; q < Q; ++q) g[q] = f[S::opp(q) * Sq + nb_off(a.geo, n, -S::cx(q), -S::cy(q), -S::cz(q))];
    if (FM == FM_BULK && own_l != 0) {  // walls and near-wall cells (the edge kernel)
        keep_loads<Q, T>(g);
        return;
    }
    if (FM == FM_LINKS || FM == FM_INLINE) {
        if (own_l & 3) {
            keep_loads<Q, T>(g);
            return;
        }
        edge = (own_l & 0x80) != 0;
    }
    uint32_t wallmask = 0;  // bit q: x - c_q is a wall (x + c_q for the opposite direction)
    if (FM != FM_LINKS && edge) {  // (FM_LINKS: the even step filled the wall slots)
#pragma unroll
        for (int q = 0; q < Q; ++q) {
            const int fl = wall_at(q, -1);
            if (fl != 0) {
                wallmask |= 1u << q;
                T v = f[q * Sq + self];
                if (fl == 2) v += ubb_term<Q, T>(a, q);
                g[q] = v;
            }
        }
    }
    const Rates<T> r = load_rates<T>(a);
    collide<Q, OP, T, FORCE>(g, r);
    if (PEER && (zs == a.geo.nz || zs == 1)) {
        // pushes across the face go straight to the neighbour's interior plane (in-plane target wraps)
        const int64_t plane = (int64_t)a.geo.nx * a.geo.ny;
#pragma unroll
        for (int q = 0; q < Q; ++q) {
            const int dz = S::cz(q);
            if (dz == 0 || (dz == 1) != (zs == a.geo.nz)) continue;
            if (edge && (wallmask & (1u << S::opp(q)))) continue;  // toward a wall: kept locally below
            const uint32_t inplane = (uint32_t)n.ys[S::cy(q) + 1] * (uint32_t)a.geo.nx + (uint32_t)n.xs[S::cx(q) + 1];
            if (dz == 1) static_cast<T *>(a.peer_up)[q * Sq + plane + inplane] = g[q];
            else static_cast<T *>(a.peer_down)[q * Sq + a.geo.nz * plane + inplane] = g[q];
        }
    }
    if (FM == FM_LINKS || !edge) {
#pragma unroll
        for (int q = 0; q < Q; ++q) f[q * Sq + nb_off(a.geo, n, S::cx(q), S::cy(q), S::cz(q))] = g[q];
        if (FM == FM_LINKS && edge) {  // x's pushes toward walls also return into its own slots
            const uint64_t m = a.lmask[self];
#pragma unroll
            for (int q = 0; q < Q; ++q)
                if ((m >> q) & 1) f[q * Sq + self] = link_value<Q, T>(a, m, g, q);
        }
    } else {
#pragma unroll
        for (int q = 0; q < Q; ++q) {
            const uint32_t o = nb_off(a.geo, n, S::cx(q), S::cy(q), S::cz(q));
            if (wallmask & (1u << S::opp(q))) {  // x + c_q is a wall: returns next step as qbar
                const int fl = wall_at(q, +1);
                T v = g[q];
                if (fl == 2) v += ubb_term<Q, T>(a, S::opp(q));
                f[S::opp(q) * Sq + self] = v;
            } else {
                f[q * Sq + o] = g[q];
            }
        }
    }
}

// Walls in the odd step (the pull rules of a3 expressed in AA slots): a population that
// would come from a wall cell x - c_q is the cell's own bounced C_qbar(x), which the even step left
// in a[x](q) (+ UBB term of q); a population leaving toward a wall x + c_q returns next step as qbar
// and is stored directly in a[x](qbar) (+ UBB term of qbar).
template <int Q, int OP, typename T, int FM, bool FORCE, bool PEER = false>
__global__ void __launch_bounds__(256, (MinBlocks<Q, OP, T>::aa)) k_aa_odd(const StepArgs a, T *__restrict__ f) {
    int x, y;
    if (!box_cell(a, x, y)) return;
    const int zs = a.z_begin + (int)blockIdx.z * a.z_step + a.geo.g;
    aa_odd_cell<Q, OP, T, FM, FORCE, PEER>(a, f, x, y, zs);
    peer_fence<PEER>();
}

// Two cells per thread in the AA even step (periodic, no flags, no peer stores): lane l of warp w of an
// x-block updates the cells x_A = x0 + 64 w + l and x_B = x_A + 32, so both are 128-byte coalesced and the
// thread issues 2 Q loads back to back (twice the bytes in flight per warp of the one-cell kernel; ncu of
// C2's even step: 3.22 -> 3.08 ms, DRAM 77 -> 81 % of peak). The same scheme in the odd step (shared row
// bases, per-cell x neighbours) measured slower than one cell per thread (3.44 -> 3.53 ms, more integer
// instructions at 16 instead of 24 warps per SM) and is not used.
template <int Q>
struct MinBlocksX2 {
    static constexpr int aa = Q == 19 ? 2 : 1;
};

__device__ __forceinline__ bool box_cell_x2(const StepArgs &a, int &x, int &y) {
    const int bx = (int)blockDim.x;
    x = a.x0 + (int)blockIdx.x * 2 * bx + ((int)threadIdx.x >> 5) * 64 + ((int)threadIdx.x & 31);
    y = a.y0 + (int)(blockIdx.y * blockDim.y + threadIdx.y);
    return x < a.x1 && y < a.y1;
}

template <int Q, int OP, typename T, bool FORCE>
__global__ void __launch_bounds__(256, MinBlocksX2<Q>::aa) k_aa_even_x2(const StepArgs a, T *__restrict__ f) {
    using S = Stencil<Q>;
    int x, y;
    if (!box_cell_x2(a, x, y)) return;
    const bool hasB = x + 32 < a.x1;
    const int zs = a.z_begin + (int)blockIdx.z * a.z_step + a.geo.g;
    const uint32_t self = ((uint32_t)zs * (uint32_t)a.geo.ny + (uint32_t)y) * (uint32_t)a.geo.nx + (uint32_t)x;
    const int64_t Sq = a.geo.Sq;
    T g[Q], h[Q];
#pragma unroll
    for (int q = 0; q < Q; ++q) {
        const T *p = f + q * Sq + self;
        g[q] = p[0];
        h[q] = hasB ? p[32] : T(0);
    }
    const Rates<T> r = load_rates<T>(a);
    collide<Q, OP, T, FORCE>(g, r);
#pragma unroll
    for (int q = 0; q < Q; ++q) f[S::opp(q) * Sq + self] = g[q];
    if (hasB) {
        collide<Q, OP, T, FORCE>(h, r);
#pragma unroll
        for (int q = 0; q < Q; ++q) f[S::opp(q) * Sq + self + 32] = h[q];
    }
}

template <int Q, int OP, typename T, bool FORCE, bool PEER = false>
__global__ void __launch_bounds__(128) k_aa_odd_edges(const StepArgs a, T *__restrict__ f, const uint32_t *__restrict__ cells,
                                                     uint32_t n) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const uint32_t c = cells[i];
    LBM_ASSERT((int64_t)c < a.geo.Sq);
    const uint32_t plane = (uint32_t)a.geo.nx * (uint32_t)a.geo.ny;
    const int zs = (int)(c / plane);
    const uint32_t r = c - (uint32_t)zs * plane;
    aa_odd_cell<Q, OP, T, FM_EDGE, FORCE, PEER>(a, f, (int)(r % (uint32_t)a.geo.nx), (int)(r / (uint32_t)a.geo.nx), zs);
    peer_fence<PEER>();
}

// =======================================================================================
// EsoTwist (Fig. 4), one array. Populations live on their links: the one travelling from
// y to y + c_q at location y + c_q^- (componentwise min(c, 0)), i.e. x - c_q^+ seen from the
// arriving cell x. Both parities touch the same locations of a cell (itself and its neighbours in
// negative directions) and differ only in the slot, the "twist" that replaces EsoTwist's pointer
// swap by an even and an odd kernel:
//   even: read arriving q at (x - c_q^+, q),    write departing q at (x + c_q^-, qbar)
//   odd : read arriving q at (x - c_q^+, qbar), write departing q at (x + c_q^-, q)
// Walls: a departing population toward a wall returns as qbar next step; it goes, plus the UBB term of
// qbar, into the other slot of the same location (the one the next step reads). Reads need no rule.
// Every slot a cell touches belongs to one of its links, so cells are independent (in place).
// =======================================================================================
__host__ __device__ constexpr int cpos(int c) { return c > 0 ? c : 0; }
__host__ __device__ constexpr int cneg(int c) { return c < 0 ? c : 0; }

// Fused EsoTwist halo (PEER, boundary planes): the regular departing writes that the neighbours read
// next step are also stored into their copy of the location — top plane, c_z = +1 -> up's lower ghost;
// bottom plane, c_z = -1 (written into our lower ghost) -> down's top plane. Bounce writes stay local.
// Within a step the neighbour touches the other slot of those locations (the twist), so only the
// per-step LSA barrier is needed.
template <int Q, int OP, typename T, int FM, bool FORCE, bool ODD, bool PEER = false>
__device__ __forceinline__ void eso_cell(const StepArgs &a, T *__restrict__ f, int x, int y, int zs) {
    using S = Stencil<Q>;
    const Nbr n = neighbours(a.geo, x, y, zs);
    const int64_t Sq = a.geo.Sq;
    bool edge = FM == FM_EDGE;
    const uint32_t self = nb_off(a.geo, n, 0, 0, 0);
    if (FM == FM_INLINE) {
        const uint8_t own = a.flags[self];
        if (own & 3) return;
        edge = (own & 0x80) != 0;
    }
    const uint8_t own_b = FM == FM_BULK ? a.flags[self] : 0;  // tested after the loads are issued (as the AA kernels)
    T g[Q];
#pragma unroll
    for (int q = 0; q < Q; ++q)
        g[q] = f[(ODD ? S::opp(q) : q) * Sq + nb_off(a.geo, n, -cpos(S::cx(q)), -cpos(S::cy(q)), -cpos(S::cz(q)))];
    if (FM == FM_BULK && own_b != 0) {  // walls and near-wall cells (the edge kernel)
        keep_loads<Q, T>(g);
        return;
    }
    const Rates<T> r = load_rates<T>(a);
    collide<Q, OP, T, FORCE>(g, r);
#pragma unroll
    for (int q = 0; q < Q; ++q) {
        const uint32_t loc = nb_off(a.geo, n, cneg(S::cx(q)), cneg(S::cy(q)), cneg(S::cz(q)));
        if (edge) {
            const uint8_t fl = a.flags[nb_off(a.geo, n, S::cx(q), S::cy(q), S::cz(q))] & 3;
            if (fl != 0) {  // toward a wall: back as qbar next step, into the other slot
                T v = g[q];
                if (fl == 2) v += ubb_term<Q, T>(a, S::opp(q));
                f[(ODD ? S::opp(q) : q) * Sq + loc] = v;
                continue;
            }
        }
        f[(ODD ? q : S::opp(q)) * Sq + loc] = g[q];
        if (PEER && S::cz(q) != 0 && (S::cz(q) == 1) == (zs == a.geo.nz) && (zs == a.geo.nz || zs == 1)) {
            const uint32_t inplane =
                (uint32_t)n.ys[cneg(S::cy(q)) + 1] * (uint32_t)a.geo.nx + (uint32_t)n.xs[cneg(S::cx(q)) + 1];
            const int64_t slot = (int64_t)(ODD ? q : S::opp(q)) * Sq;
            if (S::cz(q) == 1) static_cast<T *>(a.peer_up)[slot + inplane] = g[q];  // up's plane 0
            else static_cast<T *>(a.peer_down)[slot + (int64_t)a.geo.nz * a.geo.nx * a.geo.ny + inplane] = g[q];
        }
    }
}

template <int Q, int OP, typename T, int FM, bool FORCE, bool ODD, bool PEER = false>
__global__ void __launch_bounds__(256, (MinBlocks<Q, OP, T>::aa)) k_eso(const StepArgs a, T *f) {
    int x, y;
    if (!box_cell(a, x, y)) return;
    eso_cell<Q, OP, T, FM, FORCE, ODD, PEER>(a, f, x, y, a.z_begin + (int)blockIdx.z * a.z_step + a.geo.g);
    peer_fence<PEER>();
}

template <int Q, int OP, typename T, bool FORCE, bool ODD, bool PEER = false>
__global__ void __launch_bounds__(128) k_eso_edges(const StepArgs a, T *f, const uint32_t *__restrict__ cells, uint32_t n) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const uint32_t c = cells[i];
    LBM_ASSERT((int64_t)c < a.geo.Sq);
    const uint32_t plane = (uint32_t)a.geo.nx * (uint32_t)a.geo.ny;
    const int zs = (int)(c / plane);
    const uint32_t r = c - (uint32_t)zs * plane;
    eso_cell<Q, OP, T, FM_EDGE, FORCE, ODD, PEER>(a, f, (int)(r % (uint32_t)a.geo.nx), (int)(r / (uint32_t)a.geo.nx), zs);
    peer_fence<PEER>();
}

// =======================================================================================
// Fused collide-stream-push, two arrays: dst[x + c_q](q) = C(src[x])_q, the push state
// F(n) = (S o C)^n f0 (G11). Reads are aligned (own cell), stores shifted. Walls (pull rule O6 in push
// form): a population leaving toward a wall x + c_q comes back as qbar: dst[x](qbar) = C_q + UBB term
// of qbar. Fused halo (PEER, boundary planes): pushes across the face also go straight into the
// neighbour's interior plane of its dst array. Collide-only: the same cell update without
// streaming, in place (k_collide).
// =======================================================================================
template <int Q, int OP, typename T, int FM, bool FORCE, bool PEER = false>
__device__ __forceinline__ void push_cell(const StepArgs &a, const T *__restrict__ src, T *__restrict__ dst, int x, int y,
                                          int zs) {
    using S = Stencil<Q>;
    const Nbr n = neighbours(a.geo, x, y, zs);
    const int64_t Sq = a.geo.Sq;
    bool edge = FM == FM_EDGE;
    const uint32_t self = nb_off(a.geo, n, 0, 0, 0);
    if (FM == FM_INLINE) {
        const uint8_t own = a.flags[self];
        if (own & 3) return;
        edge = (own & 0x80) != 0;
    } else if (FM == FM_BULK) {
        if (a.flags[self] != 0) return;
    }
    T g[Q];
#pragma unroll
    for (int q = 0; q < Q; ++q) g[q] = ldg_stream(src + q * Sq + self);
    const Rates<T> r = load_rates<T>(a);
    collide<Q, OP, T, FORCE>(g, r);
    const int64_t plane = (int64_t)a.geo.nx * a.geo.ny;
#pragma unroll
    for (int q = 0; q < Q; ++q) {
        const uint32_t o = nb_off(a.geo, n, S::cx(q), S::cy(q), S::cz(q));
        if (edge) {
            const uint8_t fl = a.flags[o] & 3;
            if (fl != 0) {  // toward a wall: bounced into the cell's own slot qbar
                T v = g[q];
                if (fl == 2) v += ubb_term<Q, T>(a, S::opp(q));
                dst[S::opp(q) * Sq + self] = v;
                continue;
            }
        }
        dst[q * Sq + o] = g[q];
        if (PEER && S::cz(q) != 0 && (S::cz(q) == 1) == (zs == a.geo.nz) && (zs == a.geo.nz || zs == 1)) {
            const uint32_t inplane = (uint32_t)n.ys[S::cy(q) + 1] * (uint32_t)a.geo.nx + (uint32_t)n.xs[S::cx(q) + 1];
            if (S::cz(q) == 1) static_cast<T *>(a.peer_up)[q * Sq + plane + inplane] = g[q];
            else static_cast<T *>(a.peer_down)[q * Sq + a.geo.nz * plane + inplane] = g[q];
        }
    }
}

template <int Q, int OP, typename T, int FM, bool FORCE, bool PEER = false>
__global__ void __launch_bounds__(256, (MinBlocks<Q, OP, T>::aa)) k_push(const StepArgs a, const T *__restrict__ src,
                                                                          T *__restrict__ dst) {
    int x, y;
    if (!box_cell(a, x, y)) return;
    push_cell<Q, OP, T, FM, FORCE, PEER>(a, src, dst, x, y, a.z_begin + (int)blockIdx.z * a.z_step + a.geo.g);
    peer_fence<PEER>();
}

template <int Q, int OP, typename T, bool FORCE, bool PEER = false>
__global__ void __launch_bounds__(128) k_push_edges(const StepArgs a, const T *__restrict__ src, T *__restrict__ dst,
                                                   const uint32_t *__restrict__ cells, uint32_t n) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const uint32_t c = cells[i];
    LBM_ASSERT((int64_t)c < a.geo.Sq);
    const uint32_t plane = (uint32_t)a.geo.nx * (uint32_t)a.geo.ny;
    const int zs = (int)(c / plane);
    const uint32_t r = c - (uint32_t)zs * plane;
    push_cell<Q, OP, T, FM_EDGE, FORCE, PEER>(a, src, dst, (int)(r % (uint32_t)a.geo.nx), (int)(r / (uint32_t)a.geo.nx), zs);
    peer_fence<PEER>();
}

// collision only, in place (same slot), fluid cells of the launched planes
template <int Q, int OP, typename T, bool FLAGS, bool FORCE>
__global__ void __launch_bounds__(256, (MinBlocks<Q, OP, T>::aa)) k_collide(const StepArgs a, T *__restrict__ f) {
    using S = Stencil<Q>;
    int x, y;
    if (!box_cell(a, x, y)) return;
    const int zs = a.z_begin + (int)blockIdx.z * a.z_step + a.geo.g;
    const uint32_t self = ((uint32_t)zs * (uint32_t)a.geo.ny + (uint32_t)y) * (uint32_t)a.geo.nx + (uint32_t)x;
    const int64_t Sq = a.geo.Sq;
    if (FLAGS && (a.flags[self] & 3)) return;
    T g[Q];
#pragma unroll
    for (int q = 0; q < Q; ++q) g[q] = f[q * Sq + self];
    const Rates<T> r = load_rates<T>(a);
    collide<Q, OP, T, FORCE>(g, r);
#pragma unroll
    for (int q = 0; q < Q; ++q) f[q * Sq + self] = g[q];
    (void)sizeof(S);
}

// =======================================================================================
// Persistent multi-step kernel for small single-slab domains (launch-bound otherwise, e.g. the
// 32^3 config 0): one cooperative launch runs all n steps of an lbm_step call, cells grid-strided,
// with a grid-wide barrier between steps instead of a kernel boundary. Walls are handled inline.
// =======================================================================================
template <int Q, int OP, typename T, int FM, bool FORCE, bool AA>
__global__ void __launch_bounds__(256) k_persistent(const StepArgs a, T *A, T *B, int phase, int nsteps) {
    cooperative_groups::grid_group grid = cooperative_groups::this_grid();
    const int64_t ncell = (int64_t)a.geo.nx * a.geo.ny * a.geo.nz;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int t = 0; t < nsteps; ++t) {
        const int p = (phase + t) & 1;
        for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < ncell; i += stride) {
            const int x = (int)(i % a.geo.nx);
            const int y = (int)((i / a.geo.nx) % a.geo.ny);
            const int zs = (int)(i / ((int64_t)a.geo.nx * a.geo.ny));
            if constexpr (AA) {
                if (p == 0) aa_even_cell<Q, OP, T, (FM != FM_NONE), FORCE>(a, A, x, y, zs);
                else aa_odd_cell<Q, OP, T, FM, FORCE>(a, A, x, y, zs);
            } else {
                pull_cell<Q, OP, T, FM, FORCE, false>(a, p ? B : A, p ? A : B, x, y, zs);
            }
        }
        grid.sync();
    }
}

// =======================================================================================
// Initialisation: equilibrium of (rho, u) per interior cell, written to planes [zlo, zhi) of
// the storage (ghost planes included when their global z is available, i.e. random init).
// =======================================================================================
struct InitArgs {
    Geo geo;
    int64_t nx_g, ny_g, nz_g;  // global lattice
    int64_t z0;                // global z of local interior plane 0
    int zlo, zhi;              // storage planes to write
    const double *rho;         // interior cells (mode 0)
    const double *u;           // component d of cell i at u[d * ustride + i]
    int64_t ustride;
    int mode;                  // 0 = arrays, 1 = random (G13)
    uint64_t seed;
    double rho_amp, u_amp, profile_amp;
    int profile;
    int product_eq;            // cumulant: product equilibrium (G2)
    int eq_kind;               // EQ_* of collide.cuh (SRT/TRT/MRT): Eq. (3) rho0 = rho / rho0 = 1 / moment-matched
    int eso;                   // EsoTwist storage: f_q(x) goes to location x - c_q^+ (slot q)
};

__device__ __forceinline__ uint64_t splitmix64(uint64_t k) {
    uint64_t z = k + 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}
// U(a, b) = a + (b - a) r, r = top 53 bits * 2^-53, no FMA contraction (matches the host generator)
__device__ __forceinline__ double uniform_g13(uint64_t seed, uint64_t ig, int k, double a, double b) {
    const uint64_t key = (seed << 40) ^ (4ull * ig + (uint64_t)k);
    const double r = (double)(splitmix64(key) >> 11) * 0x1p-53;
    return __dadd_rn(a, __dmul_rn(__dsub_rn(b, a), r));
}

template <int Q, typename T>
__global__ void k_init(const InitArgs a, T *__restrict__ f0, T *__restrict__ f1) {
    using S = Stencil<Q>;
    const int x = blockIdx.x * blockDim.x + threadIdx.x;
    const int y = blockIdx.y * blockDim.y + threadIdx.y;
    if (x >= a.geo.nx || y >= a.geo.ny) return;
    const int zs = a.zlo + (int)blockIdx.z;
    if (zs >= a.zhi) return;
    const int zl = zs - a.geo.g;  // local interior index (may be -1 or nz for ghosts)
    double rho, ux, uy, uz;
    if (a.mode == 0) {
        const int64_t i = ((int64_t)zl * a.geo.ny + y) * a.geo.nx + x;
        rho = a.rho[i];
        ux = a.u[i];
        uy = a.u[a.ustride + i];
        uz = a.u[2 * a.ustride + i];
    } else {
        int64_t zg = a.z0 + zl;
        zg = ((zg % a.nz_g) + a.nz_g) % a.nz_g;
        const uint64_t ig = (uint64_t)x + (uint64_t)a.nx_g * ((uint64_t)y + (uint64_t)a.ny_g * (uint64_t)zg);
        rho = (a.rho_amp != 0.0) ? __dadd_rn(1.0, uniform_g13(a.seed, ig, 0, -a.rho_amp, a.rho_amp)) : 1.0;
        ux = (a.u_amp != 0.0) ? uniform_g13(a.seed, ig, 1, -a.u_amp, a.u_amp) : 0.0;
        uy = (a.u_amp != 0.0) ? uniform_g13(a.seed, ig, 2, -a.u_amp, a.u_amp) : 0.0;
        uz = (a.u_amp != 0.0) ? uniform_g13(a.seed, ig, 3, -a.u_amp, a.u_amp) : 0.0;
        if (a.profile == 1) {
            const double s = sin(__ddiv_rn(__dmul_rn(2.0 * 3.141592653589793, (double)zg), (double)a.nz_g));
            ux = __dadd_rn(__dmul_rn(a.profile_amp, s), ux);
        }
    }
    const uint32_t self0 = ((uint32_t)zs * (uint32_t)a.geo.ny + (uint32_t)y) * (uint32_t)a.geo.nx + (uint32_t)x;
    Nbr nb;
    if (a.eso) nb = neighbours(a.geo, x, y, zs);
    auto addr = [&](int q) -> uint32_t {
        return a.eso ? nb_off(a.geo, nb, -cpos(S::cx(q)), -cpos(S::cy(q)), -cpos(S::cz(q))) : self0;
    };
    const double drho = rho - 1.0;
    const double uu15 = 1.5 * (ux * ux + uy * uy + uz * uz);
#pragma unroll
    for (int q = 0; q < Q; ++q) {
        double gq;
        if (a.product_eq && Q == 19) {
            gq = 0.0;  // written below from the Maxwellian basis moments
        } else if (a.product_eq) {
            double v = rho;
            const double uc[3] = {ux, uy, uz};
            const int c[3] = {S::cx(q), S::cy(q), S::cz(q)};
#pragma unroll
            for (int d = 0; d < 3; ++d)
                v *= (c[d] == 0) ? (2.0 / 3.0 - uc[d] * uc[d]) : 0.5 * (1.0 / 3.0 + uc[d] * uc[d] + c[d] * uc[d]);
            gq = v - S::w(q);
        } else {
            const double cu = S::cx(q) * ux + S::cy(q) * uy + S::cz(q) * uz;
            const double rho0 = a.eq_kind == EQ_INCOMPRESSIBLE ? 1.0 : rho;
            gq = S::w(q) * drho + S::w(q) * rho0 * (3.0 * cu + 4.5 * cu * cu - uu15);
            if (a.eq_kind == EQ_MOMENT_MATCHED) gq += mm_delta<Q, double>(q, rho, ux, uy, uz);
        }
        if (a.product_eq && Q == 19) continue;
        f0[q * a.geo.Sq + addr(q)] = T(gq);
        if (f1) f1[q * a.geo.Sq + addr(q)] = T(gq);
    }
    if (Q == 19 && a.product_eq) {
        // D3Q19 cumulant fixed point: basis moments = untruncated Maxwellian moments rho prod mu_e(u)
        double M[27], f[19];
        const double uc[3] = {ux, uy, uz};
#pragma unroll
        for (int t = 0; t < 27; ++t) {
            const int e[3] = {t / 9, (t / 3) % 3, t % 3};
            double v = rho;
#pragma unroll
            for (int d = 0; d < 3; ++d) v *= e[d] == 0 ? 1.0 : e[d] == 1 ? uc[d] : (1.0 / 3.0 + uc[d] * uc[d]);
            M[t] = v;
        }
        d3q19_from_raw<double>(M, f);
#pragma unroll
        for (int q = 0; q < 19; ++q) {
            const double gq = f[q] - Stencil<19>::w(q);
            f0[q * a.geo.Sq + addr(q)] = T(gq);
            if (f1) f1[q * a.geo.Sq + addr(q)] = T(gq);
        }
    }
}

// =======================================================================================
// Readout: canonical populations / macroscopic values of interior cells.
// For AA with odd parity the state is gathered: F_q(y) = a[y - c_q](qbar).
// =======================================================================================
struct ReadArgs {
    Geo geo;
    int aa_odd;      // 1: AA array after an odd number of steps
    int raw;         // 1: stored values, no +w, no gather
    double fsign;    // +1 pre-collision state, -1 post-collision (pull)
    double F[3];
    const uint8_t *flags;  // AA odd gather with walls (same rule as k_aa_odd's reads)
    double uw[3];
    int incompressible;    // u = (j +- F/2) / rho0 with rho0 = 1 instead of rho
    int eso;               // EsoTwist storage: F_q(x) = f(x - c_q^+)(eso_odd ? qbar : q)
    int eso_odd;
};

template <int Q, typename T>
__device__ __forceinline__ T read_canonical(const ReadArgs &a, const T *f, int x, int y, int zs, int q) {
    using S = Stencil<Q>;
    const uint32_t self = ((uint32_t)zs * (uint32_t)a.geo.ny + (uint32_t)y) * (uint32_t)a.geo.nx + (uint32_t)x;
    if (a.eso && !a.raw) {
        const Nbr n = neighbours(a.geo, x, y, zs);
        return f[(a.eso_odd ? S::opp(q) : q) * a.geo.Sq + nb_off(a.geo, n, -cpos(S::cx(q)), -cpos(S::cy(q)), -cpos(S::cz(q)))];
    }
    if (a.aa_odd && !a.raw) {
        const Nbr n = neighbours(a.geo, x, y, zs);
        const uint32_t o = nb_off(a.geo, n, -S::cx(q), -S::cy(q), -S::cz(q));
        if (a.flags && (a.flags[self] & 0x80)) {
            const uint8_t fl = a.flags[o] & 3;
            if (fl != 0) {
                const double cu = S::cx(q) * a.uw[0] + S::cy(q) * a.uw[1] + S::cz(q) * a.uw[2];
                return f[q * a.geo.Sq + self] + (fl == 2 ? T(6.0 * S::w(q) * cu) : T(0));
            }
        }
        return f[S::opp(q) * a.geo.Sq + o];
    }
    return f[q * a.geo.Sq + self];
}

template <int Q, typename T>
__global__ void k_get_pops(const ReadArgs a, const T *__restrict__ f, double *__restrict__ out) {
    using S = Stencil<Q>;
    const int x = blockIdx.x * blockDim.x + threadIdx.x;
    const int y = blockIdx.y * blockDim.y + threadIdx.y;
    if (x >= a.geo.nx || y >= a.geo.ny) return;
    const int zl = blockIdx.z;
    const int zs = zl + a.geo.g;
    const int64_t nc = (int64_t)a.geo.nx * a.geo.ny * a.geo.nz;
    const int64_t i = ((int64_t)zl * a.geo.ny + y) * a.geo.nx + x;
#pragma unroll
    for (int q = 0; q < Q; ++q) {
        const double v = (double)read_canonical<Q, T>(a, f, x, y, zs, q);
        out[q * nc + i] = a.raw ? v : v + S::w(q);
    }
}

template <int Q, typename T>
__global__ void k_get_at(const ReadArgs a, const T *__restrict__ f, const int64_t *__restrict__ cells, int64_t n,
                         int64_t first, int64_t last, double *__restrict__ out) {
    using S = Stencil<Q>;
    const int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (k >= n) return;
    const int64_t c = cells[k];
    if (c < first || c >= last) return;  // another slab's cell
    const int64_t i = c - first;
    const int x = (int)(i % a.geo.nx);
    const int y = (int)((i / a.geo.nx) % a.geo.ny);
    const int zl = (int)(i / ((int64_t)a.geo.nx * a.geo.ny));
#pragma unroll
    for (int q = 0; q < Q; ++q) {
        const double v = (double)read_canonical<Q, T>(a, f, x, y, zl + a.geo.g, q);
        out[q * n + k] = a.raw ? v : v + S::w(q);
    }
}

template <int Q, typename T>
__global__ void k_set_pops(const ReadArgs a, T *__restrict__ f, const double *__restrict__ in) {
    using S = Stencil<Q>;
    const int x = blockIdx.x * blockDim.x + threadIdx.x;
    const int y = blockIdx.y * blockDim.y + threadIdx.y;
    if (x >= a.geo.nx || y >= a.geo.ny) return;
    const int zl = blockIdx.z;
    const uint32_t self = ((uint32_t)(zl + a.geo.g) * (uint32_t)a.geo.ny + (uint32_t)y) * (uint32_t)a.geo.nx + (uint32_t)x;
    const int64_t nc = (int64_t)a.geo.nx * a.geo.ny * a.geo.nz;
    const int64_t i = ((int64_t)zl * a.geo.ny + y) * a.geo.nx + x;
    const bool eso = a.eso && !a.raw;
    Nbr n;
    if (eso) n = neighbours(a.geo, x, y, zl + a.geo.g);
#pragma unroll
    for (int q = 0; q < Q; ++q) {
        const double v = in[q * nc + i];
        const int64_t addr = eso ? (int64_t)(a.eso_odd ? S::opp(q) : q) * a.geo.Sq +
                                       nb_off(a.geo, n, -cpos(S::cx(q)), -cpos(S::cy(q)), -cpos(S::cz(q)))
                                 : (int64_t)q * a.geo.Sq + self;
        f[addr] = a.raw ? T(v) : T(v - S::w(q));
    }
}

template <int Q, typename T>
__global__ void k_macro(const ReadArgs a, const T *__restrict__ f, double *__restrict__ rho_out, double *__restrict__ u_out) {
    using S = Stencil<Q>;
    const int x = blockIdx.x * blockDim.x + threadIdx.x;
    const int y = blockIdx.y * blockDim.y + threadIdx.y;
    if (x >= a.geo.nx || y >= a.geo.ny) return;
    const int zl = blockIdx.z;
    const int zs = zl + a.geo.g;
    double drho = 0, jx = 0, jy = 0, jz = 0;
#pragma unroll
    for (int q = 0; q < Q; ++q) {
        const double v = (double)read_canonical<Q, T>(a, f, x, y, zs, q);
        drho += v;
        jx += S::cx(q) * v;
        jy += S::cy(q) * v;
        jz += S::cz(q) * v;
    }
    const double rho = 1.0 + drho;
    const double rho0 = a.incompressible ? 1.0 : rho;
    const int64_t nc = (int64_t)a.geo.nx * a.geo.ny * a.geo.nz;
    const int64_t i = ((int64_t)zl * a.geo.ny + y) * a.geo.nx + x;
    rho_out[i] = rho;
    u_out[i] = (jx + a.fsign * 0.5 * a.F[0]) / rho0;
    u_out[nc + i] = (jy + a.fsign * 0.5 * a.F[1]) / rho0;
    u_out[2 * nc + i] = (jz + a.fsign * 0.5 * a.F[2]) / rho0;
}

// =======================================================================================
// Halo: pack the crossing populations of storage plane zs (canonical order: q ascending over
// {q : c_qz = dir}, then y, then x) into a contiguous buffer, and the inverse.
// =======================================================================================
template <int Q, typename T, typename OutT>
__global__ void k_pack(const Geo geo, const T *__restrict__ f, int zs, int dir, OutT *__restrict__ out) {
    const int64_t plane = (int64_t)geo.nx * geo.ny;
    const int64_t n = plane * Stencil<Q>::kCross;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const int k = (int)(i / plane);
        const int64_t r = i - k * plane;
        const int q = crossing_dir<Q>(dir, k);
        LBM_ASSERT(q >= 0 && zs >= 0 && zs < geo.nz + 2 * geo.g);
        out[i] = OutT(f[q * geo.Sq + zs * plane + r]);
    }
}

template <int Q, typename T>
__global__ void k_unpack(const Geo geo, T *__restrict__ f, int zs, int dir, const T *__restrict__ in) {
    const int64_t plane = (int64_t)geo.nx * geo.ny;
    const int64_t n = plane * Stencil<Q>::kCross;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const int k = (int)(i / plane);
        const int64_t r = i - k * plane;
        const int q = crossing_dir<Q>(dir, k);
        LBM_ASSERT(q >= 0 && zs >= 0 && zs < geo.nz + 2 * geo.g);
        f[q * geo.Sq + zs * plane + r] = in[i];
    }
}

// AA return of ghost-plane writes with walls: population q arriving in storage plane zs was
// produced by the cell one step against c_q (in the neighbour's slab). If that cell is a wall the
// value is not in the buffer (the receiving cell bounced it locally), so it is skipped.
template <int Q, typename T>
__global__ void k_unpack_masked(const Geo geo, T *__restrict__ f, int zs, int dir, const T *__restrict__ in,
                                const uint8_t *__restrict__ flags) {
    using S = Stencil<Q>;
    const int64_t plane = (int64_t)geo.nx * geo.ny;
    const int64_t n = plane * S::kCross;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const int k = (int)(i / plane);
        const int64_t r = i - k * plane;
        const int q = crossing_dir<Q>(dir, k);
        const int x = (int)(r % geo.nx), y = (int)(r / geo.nx);
        const int xs = (x - S::cx(q) + geo.nx) % geo.nx, ys = (y - S::cy(q) + geo.ny) % geo.ny;
        const int64_t src = (int64_t)(zs - S::cz(q)) * plane + (int64_t)ys * geo.nx + xs;
        LBM_ASSERT(q >= 0 && zs >= 0 && zs < geo.nz + 2 * geo.g && zs - S::cz(q) >= 0 && zs - S::cz(q) < geo.nz + 2 * geo.g);
        if ((flags[src] & 3) == 0) f[q * geo.Sq + zs * plane + r] = in[i];
    }
}

// =======================================================================================
// Index-list boundary handling: one entry per boundary link (wall cell b, direction q
// pointing from b to the fluid cell x = b + c_q, per-link UBB term 6 w_q rho_w c_q.u_w, 0 for
// no-slip). The separate boundary kernel prepares the wall cell's slot that the flag-free update
// kernel streams from:
//   mode 0, pull, before the step:    src[b](q)    = src[x](qbar) + term
//   mode 1, AA, after the even step:  a[b](qbar)   = a[x](q) + term     (read by x in the odd step)
//   mode 2, AA, after the odd step:   a[x](q)      = a[b](qbar) + term  (x's push toward b, bounced)
//   EsoTwist (G23; the link's populations live at L = b + c_q^- = x - c_q^+, passed in `fluid`): x's
//   departing qbar (toward b) was written at (L, q) after an even step and at (L, qbar) after an odd one;
//   the next step reads x's arriving q at the other slot of L:
//   mode 3, EsoTwist, after even:     a[L](qbar)   = a[L](q) + term
//   mode 4, EsoTwist, after odd:      a[L](q)      = a[L](qbar) + term
// Every slot is written by one link and read by no other link of the same launch.
// =======================================================================================
struct LinkArgs {
    int64_t Sq;
    const uint32_t *wall, *fluid;  // storage cell indices (EsoTwist: `fluid` holds the link location L)
    const uint8_t *dir;            // q
    const double *term;            // per-link UBB term
    uint32_t n;
    int mode;
};

template <int Q, typename T>
__global__ void k_links(const LinkArgs a, T *__restrict__ f) {
    using S = Stencil<Q>;
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= a.n) return;
    const int q = a.dir[i];
    const int qb = S::opp(q);
    const int64_t b = a.wall[i], x = a.fluid[i];
    LBM_ASSERT(b < a.Sq && x < a.Sq && q > 0 && q < Q);
    const T t = T(a.term[i]);
    if (a.mode == 0) f[q * a.Sq + b] = f[qb * a.Sq + x] + t;
    else if (a.mode == 1) f[qb * a.Sq + b] = f[q * a.Sq + x] + t;
    else if (a.mode == 2) f[q * a.Sq + x] = f[qb * a.Sq + b] + t;
    else if (a.mode == 3) f[qb * a.Sq + x] = f[q * a.Sq + x] + t;
    else f[q * a.Sq + x] = f[qb * a.Sq + x] + t;
}

// EsoTwist exchange with walls: slot r of location L (storage plane zs) was written by the cell that
// produced the population stored there — L + c_r^+ after an even step (departing rbar, slot r), L - c_r^-
// after an odd one (departing r). If that cell is a wall, nothing was produced (the receiving side keeps
// its own bounced value in that slot), so the entry is skipped.
template <int Q, typename T>
__global__ void k_unpack_masked_eso(const Geo geo, T *__restrict__ f, int zs, int dir, const T *__restrict__ in,
                                    const uint8_t *__restrict__ flags, int parity_done) {
    using S = Stencil<Q>;
    const int64_t plane = (int64_t)geo.nx * geo.ny;
    const int64_t n = plane * S::kCross;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const int k = (int)(i / plane);
        const int64_t r = i - k * plane;
        const int q = crossing_dir<Q>(dir, k);
        const int x = (int)(r % geo.nx), y = (int)(r / geo.nx);
        const int ox = parity_done ? -cneg(S::cx(q)) : cpos(S::cx(q));
        const int oy = parity_done ? -cneg(S::cy(q)) : cpos(S::cy(q));
        const int oz = parity_done ? -cneg(S::cz(q)) : cpos(S::cz(q));
        const int xs = (x + ox + geo.nx) % geo.nx, ys = (y + oy + geo.ny) % geo.ny;
        const int64_t src = (int64_t)(zs + oz) * plane + (int64_t)ys * geo.nx + xs;
        LBM_ASSERT(q >= 0 && zs + oz >= 0 && zs + oz < geo.nz + 2 * geo.g);
        if ((flags[src] & 3) == 0) f[q * geo.Sq + zs * plane + r] = in[i];
    }
}

// =======================================================================================
// Roofline probe "copy-q" (the B200 analogue of the paper's copy-19 / update-19 probes, Table III,
// P:1083-1127): every cell copies its q populations from src to dst with the LB access pattern but no
// collision — gathered from x - c_q (periodic) when `shifted`, else from x — so its bandwidth is the
// ceiling for the update kernels' memory streams.
// =======================================================================================
template <int Q, typename T, bool SHIFTED>
__global__ void __launch_bounds__(256) k_copyq(const Geo g, const T *__restrict__ src, T *__restrict__ dst) {
    using S = Stencil<Q>;
    const int x = blockIdx.x * blockDim.x + threadIdx.x;
    const int y = blockIdx.y * blockDim.y + threadIdx.y;
    if (x >= g.nx || y >= g.ny) return;
    const int zs = blockIdx.z;
    const Nbr n = neighbours(g, x, y, zs);
    const uint32_t self = nb_off(g, n, 0, 0, 0);
    T v[Q];
#pragma unroll
    for (int q = 0; q < Q; ++q)
        v[q] = __ldg(src + q * g.Sq + (SHIFTED ? nb_off(g, n, -S::cx(q), -S::cy(q), -S::cz(q)) : self));
#pragma unroll
    for (int q = 0; q < Q; ++q) dst[q * g.Sq + self] = v[q];
}

// In-place probe "update-q" (the analogue of the paper's update-19 probe, Table III): the
// AA-pattern access streams of one array without collision. Even (SHIFTED = false): read f[x](q), write
// f[x](qbar); odd (SHIFTED = true): read f[x - c_q](qbar), write f[x + c_q](q). Ceiling of the in-place
// (AA / EsoTwist) update kernels, as copy-q is of the two-array ones.
template <int Q, typename T, bool SHIFTED>
__global__ void __launch_bounds__(256) k_updateq(const Geo g, T *__restrict__ f) {
    using S = Stencil<Q>;
    const int x = blockIdx.x * blockDim.x + threadIdx.x;
    const int y = blockIdx.y * blockDim.y + threadIdx.y;
    if (x >= g.nx || y >= g.ny) return;
    const int zs = blockIdx.z;
    const Nbr n = neighbours(g, x, y, zs);
    const uint32_t self = nb_off(g, n, 0, 0, 0);
    T v[Q];
#pragma unroll
    for (int q = 0; q < Q; ++q)
        v[q] = f[(SHIFTED ? S::opp(q) : q) * g.Sq + (SHIFTED ? nb_off(g, n, -S::cx(q), -S::cy(q), -S::cz(q)) : self)];
#pragma unroll
    for (int q = 0; q < Q; ++q)
        f[(SHIFTED ? q : S::opp(q)) * g.Sq + (SHIFTED ? nb_off(g, n, S::cx(q), S::cy(q), S::cz(q)) : self)] = v[q];
}

// ALU ceiling probe: independent fused multiply-add chains (8 per thread, no memory traffic) on a full
// grid; 2 FLOP per FMA. Measures the DFMA / FFMA throughput the ALU-bound operators are judged against.
template <typename T>
__global__ void __launch_bounds__(256) k_fma_probe(T a, T b, int iters, T *__restrict__ sink) {
    T x0 = T(threadIdx.x) * T(1e-3), x1 = x0 + T(1), x2 = x0 + T(2), x3 = x0 + T(3), x4 = x0 + T(4), x5 = x0 + T(5),
      x6 = x0 + T(6), x7 = x0 + T(7);
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int k = 0; k < 16; ++k) {
            x0 = fma(x0, a, b); x1 = fma(x1, a, b); x2 = fma(x2, a, b); x3 = fma(x3, a, b);
            x4 = fma(x4, a, b); x5 = fma(x5, a, b); x6 = fma(x6, a, b); x7 = fma(x7, a, b);
        }
    }
    const T r = ((x0 + x1) + (x2 + x3)) + ((x4 + x5) + (x6 + x7));
    if (r == T(-1.2345)) sink[threadIdx.x] = r;  // never true for the probe's inputs; keeps the chains live
}

// =======================================================================================
// Flag preprocessing and diagnostics
// =======================================================================================
// out = in | 0x80 for fluid cells with a non-fluid cell among their 26 neighbours (x, y wrap; z wraps
// without ghost planes; ghost planes themselves are never updated)
__global__ void k_mark_near_wall(const Geo geo, int nplanes, const uint8_t *__restrict__ in, uint8_t *__restrict__ out);

template <typename T>
__global__ void k_nan_check(const T *__restrict__ f, int64_t n, int *__restrict__ flag) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const T v = f[i];
        if (v != v) {
            *flag = 1;
            return;
        }
    }
}

}  // namespace lbm
