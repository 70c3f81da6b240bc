// runtime.cu — C-ABI runtime of the LB library (include/lbm.h): configuration validation,
// device allocation, flag preprocessing, the time-step scheduler (single slab, loopback slabs,
// NCCL slabs with halo exchange overlapped with the interior update), CUDA-graph capture,
// readout and error handling. No C++ exception crosses the ABI.
#include <cuda_runtime.h>
#include <nccl.h>
#include <nvtx3/nvToolsExt.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <memory>
#include <new>
#include <string>
#include <vector>

#include "../../include/lbm.h"
#include "dispatch.h"
#include "fused.h"

using namespace lbm;

namespace {

struct Slab {
    int64_t z0 = 0;       // global z of local interior plane 0
    int nz = 0;           // interior planes
    void *pdf[2] = {nullptr, nullptr};
    uint8_t *flags = nullptr;    // storage-indexed, with ghost planes
    uint32_t *edges = nullptr;   // storage indices of near-wall fluid cells (split wall mode)
    std::vector<int64_t> edge_off;  // edges of storage plane zs: [edge_off[zs], edge_off[zs+1])
    // index-list boundaries (LBM_BOUNDARY_LINKS): device arrays + host copies for queries
    uint32_t *link_wall = nullptr, *link_fluid = nullptr;
    uint8_t *link_dir = nullptr;
    double *link_term = nullptr;
    std::vector<uint32_t> h_link_wall;
    std::vector<uint8_t> h_link_dir, h_link_type;
    // in-kernel links (FM_LINKS): per storage cell link mask (kernels.cuh StepArgs::lmask), and the residual
    // list of the links the update kernels cannot store (wall cell in a ghost plane: the exchange overwrites
    // it), run by the link kernel at the usual points; primed = the wall slots match the current state
    uint64_t *lmask = nullptr;
    uint32_t *res_wall = nullptr, *res_fluid = nullptr;
    uint8_t *res_dir = nullptr;
    double *res_term = nullptr;
    uint32_t n_res = 0;
    std::vector<uint32_t> h_res_idx;  // positions of the residual links in the full list
    bool links_primed = false;
    void *halo[4] = {nullptr, nullptr, nullptr, nullptr};  // packed mode: send up, send down, recv below, recv above
    int cur = 0;          // index of the array holding the current state (pull)
    int zlo = 0, zhi = 0; // interior planes [zlo, zhi) holding non-wall cells (launch trimming)
    bool own_pdf[2] = {true, true}, own_flags = true, own_halo = true;  // false: borrowed (lbm_config.*_dev)
};

struct Timing {
    bool on = false;
    std::vector<cudaEvent_t> ev;  // pairs
    // phase timeline of the last timed decomposed step (lbm_step_phases_ms): boundary planes, exchange
    // (comm stream with NCCL, compute stream otherwise), interior planes; begin/end events
    cudaEvent_t ph[6] = {nullptr, nullptr, nullptr, nullptr, nullptr, nullptr};
    bool ph_valid = false;
};

// NVTX ranges around the phases of a step (visible in an nsys / ncu timeline; no-ops without a tool)
struct NvtxRange {
    explicit NvtxRange(const char *name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
};

}  // namespace

struct lbm_handle_s {
    lbm_config cfg{};
    int Q = 19, dtype = 0, esize = 8, op = 0;
    int g = 0;  // ghost planes per side
    int64_t nx = 0, ny = 0, nzg = 0;
    std::vector<Slab> slabs;
    cudaStream_t stream = nullptr, comm_stream = nullptr;
    bool own_stream = false;
    cudaEvent_t ev_bnd = nullptr, ev_x = nullptr;
    ncclComm_t comm = nullptr;
    int rank = 0, nranks = 1, up = 0, down = 0;
    bool use_nccl = false;  // nranks > 1, or the 1-rank self-exchange variant
    bool have_flags = false, have_force = false;
    Kernels kern;  // kernels of the configured operator and wall mode
    StepArgs base{};
    int64_t steps = 0;
    int aa_parity = 0;
    cudaGraphExec_t graph = nullptr;
    int graph_parity = -1;
    int graph_path = -1;  // kernel path (lbm_set_kernel_path) the graph was captured with
    int64_t launches = 0;
    int *d_nanflag = nullptr;
    double *scratch = nullptr;
    size_t scratch_bytes = 0;
    // asynchronous host I/O (LBM_HOST_ASYNC): double-buffered device staging of rho/u, uploads on h2d_stream
    // and downloads on d2h_stream (PCIe is full duplex) overlapped with the compute stream
    struct AsyncIO {
        bool ready = false;
        cudaStream_t h2d = nullptr, d2h = nullptr;
        double *in[2] = {nullptr, nullptr}, *out[2] = {nullptr, nullptr};
        cudaEvent_t in_ready[2] = {nullptr, nullptr}, in_free[2] = {nullptr, nullptr};
        cudaEvent_t out_ready[2] = {nullptr, nullptr}, out_free[2] = {nullptr, nullptr};
        int in_k = 0, out_k = 0;
    } aio;
    Timing timing;
    bool fused = false;       // halo through NVLink peer stores (LBM_HALO_FUSED)
    bool links = false;       // index-list boundaries: flag-free update kernels + link kernel
    bool links_fused = false; // index lists folded into the pull / AA update kernels (FM_LINKS)
    Kernels kern_links;       // links_fused: the flag-free kernels of the plain index-list mode (per-link velocities)
    bool inline_bc = false;   // compiled-in boundaries: every cell tests its neighbours' flags, no edge kernel
    bool faces = false;       // face-aligned walls (FM_FACES): walls recognised from coordinates, no edge kernel
    int links_pending = -1;   // fused halo + index lists: deferred link fix of the last step (parity | array << 1)
    int8_t base_face[6] = {0, 0, 0, 0, 0, 0};  // FM_FACES wall types (detect_faces)
    FusedState fst;
    std::string err;
    dim3 block;
};

namespace {

thread_local std::string g_create_error;

int fail(lbm_handle h, int code, const std::string &msg) {
    if (h) h->err = msg;
    else g_create_error = msg;
    return code;
}

#define CUDA_TRY(h, expr)                                                                     \
    do {                                                                                      \
        cudaError_t _e = (expr);                                                              \
        if (_e != cudaSuccess)                                                                \
            return fail((h), _e == cudaErrorMemoryAllocation ? LBM_EOOM : LBM_ECUDA,          \
                        std::string(#expr) + ": " + cudaGetErrorString(_e));                  \
    } while (0)

#define NCCL_TRY(h, expr)                                                                     \
    do {                                                                                      \
        ncclResult_t _r = (expr);                                                             \
        if (_r != ncclSuccess) return fail((h), LBM_ENCCL, std::string(#expr) + ": " + ncclGetErrorString(_r)); \
    } while (0)

int crossing(int Q, int dir, int *out) {
    int n = 0;
    for (int q = 0; q < Q; ++q)
        if (kC27[q][2] == dir) out[n++] = q;
    return n;
}

bool two_arrays(const lbm_handle_s *h) { return h->cfg.pattern == LBM_PULL || h->cfg.pattern == LBM_PUSH; }
int cur_array(const lbm_handle_s *h, const Slab &s) { return two_arrays(h) ? s.cur : 0; }

Geo geo_of(const lbm_handle_s *h, const Slab &s) {
    Geo g;
    g.nx = (int)h->nx;
    g.ny = (int)h->ny;
    g.nz = s.nz;
    g.g = h->g;
    g.Sq = (int64_t)h->nx * h->ny * (s.nz + 2 * h->g);
    return g;
}

// grid of the plain update kernels: the launch box (StepArgs x0..x1, y0..y1) times the planes
dim3 box_grid(const StepArgs &a, dim3 block, int nplanes);
dim3 grid_for(const lbm_handle_s *h, int nplanes) { return box_grid(h->base, h->block, nplanes); }

// contiguous plane ranges (z_step 1) lose their leading / trailing planes without non-wall cells; false if
// nothing is left
bool trim_planes(const Slab &s, int &z_begin, int &nplanes, int z_step) {
    if (z_step != 1 && nplanes != 1) return nplanes > 0;
    const int lo = std::max(z_begin, s.zlo), hi = std::min(z_begin + nplanes, s.zhi);
    if (hi <= lo) return false;
    z_begin = lo;
    nplanes = hi - lo;
    return true;
}

size_t plane_bytes(const lbm_handle_s *h) { return (size_t)h->nx * h->ny * h->esize; }

char *qplane(const lbm_handle_s *h, const Slab &s, int arr, int q, int zs) {
    const Geo g = geo_of(h, s);
    return static_cast<char *>(s.pdf[arr]) + ((size_t)q * g.Sq + (size_t)zs * h->nx * h->ny) * h->esize;
}

// ---- kernel launch helpers (counted, optionally timed) ------------------------------
void tbegin(lbm_handle_s *h, cudaStream_t s) {
    if (!h->timing.on) return;
    cudaEvent_t e;
    cudaEventCreate(&e);
    cudaEventRecord(e, s);
    h->timing.ev.push_back(e);
}
void tend(lbm_handle_s *h, cudaStream_t s) { tbegin(h, s); }

// Split wall mode: the near-wall cells of the planes a bulk launch covered (interior indices
// z_begin + k * z_step, k < nplanes), one edge-list launch per contiguous run of planes.
void launch_edges(lbm_handle_s *h, Slab &s, const StepArgs &a, EdgeLaunch fn, const void *src, void *dst, int z_begin,
                  int nplanes, int z_step, cudaStream_t st) {
    if (!s.edges || !fn || h->links || h->inline_bc || h->faces) return;  // links: flag-free; inline / faces: no edge pass
    auto run = [&](int zlo, int zhi) {  // interior planes [zlo, zhi)
        const int64_t b = s.edge_off[zlo + h->g], e = s.edge_off[zhi + h->g];
        if (e <= b) return;
        tbegin(h, st);
        fn(a, src, dst, s.edges + b, (uint32_t)(e - b), st);
        tend(h, st);
        h->launches++;
    };
    if (z_step == 1) run(z_begin, z_begin + nplanes);
    else
        for (int k = 0; k < nplanes; ++k) run(z_begin + k * z_step, z_begin + k * z_step + 1);
}

// index-list boundary kernel (mode 0: pull, before the step; 1: AA after even; 2: AA after odd;
// 3 / 4: EsoTwist after even / odd)
// In-kernel links (links_fused): only the residual list, unless `full` (priming the wall slots).
void launch_links_fix(lbm_handle_s *h, Slab &s, void *f, int mode, cudaStream_t st, bool full = false) {
    if (!h->links || s.h_link_wall.empty()) return;
    const bool res = h->links_fused && !full;
    if (res && s.n_res == 0) return;
    LinkArgs a;
    a.Sq = geo_of(h, s).Sq;
    a.wall = res ? s.res_wall : s.link_wall;
    a.fluid = res ? s.res_fluid : s.link_fluid;
    a.dir = res ? s.res_dir : s.link_dir;
    a.term = res ? s.res_term : s.link_term;
    a.n = res ? s.n_res : (uint32_t)s.h_link_wall.size();
    a.mode = mode;
    tbegin(h, st);
    launch_links(h->Q, h->dtype, a, f, st);
    tend(h, st);
    h->launches++;
}

void launch_pull_range(lbm_handle_s *h, Slab &s, int z_begin, int nplanes, int z_step, cudaStream_t st,
                       bool peer_stores = false) {
    if (nplanes <= 0 || !trim_planes(s, z_begin, nplanes, z_step)) return;
    StepArgs a = h->base;
    a.geo = geo_of(h, s);
    a.z_begin = z_begin;
    a.z_step = z_step;
    a.flags = s.flags;
    a.lmask = s.lmask;
    a.zg0 = (int)s.z0;
    if (peer_stores) {  // fused halo: LSA bases of the neighbours' dst array (1 - cur)
        a.peer_up = h->fst.bases[2 * (1 - s.cur) + 0];
        a.peer_down = h->fst.bases[2 * (1 - s.cur) + 1];
    }
    tbegin(h, st);
    h->kern.pull(a, s.pdf[s.cur], s.pdf[1 - s.cur], grid_for(h, nplanes), h->block, st);
    tend(h, st);
    h->launches++;
    launch_edges(h, s, a, h->kern.pull_edges, s.pdf[s.cur], s.pdf[1 - s.cur], z_begin, nplanes, z_step, st);
}

void launch_push_range(lbm_handle_s *h, Slab &s, int z_begin, int nplanes, int z_step, cudaStream_t st,
                       bool peer_stores = false) {
    if (nplanes <= 0 || !trim_planes(s, z_begin, nplanes, z_step)) return;
    StepArgs a = h->base;
    a.geo = geo_of(h, s);
    a.z_begin = z_begin;
    a.z_step = z_step;
    a.flags = s.flags;
    if (peer_stores) {  // LSA bases of the neighbours' dst array (1 - cur)
        a.peer_up = h->fst.bases[2 * (1 - s.cur) + 0];
        a.peer_down = h->fst.bases[2 * (1 - s.cur) + 1];
    }
    tbegin(h, st);
    h->kern.push(a, s.pdf[s.cur], s.pdf[1 - s.cur], grid_for(h, nplanes), h->block, st);
    tend(h, st);
    h->launches++;
    launch_edges(h, s, a, h->kern.push_edges, s.pdf[s.cur], s.pdf[1 - s.cur], z_begin, nplanes, z_step, st);
}

void launch_eso_range(lbm_handle_s *h, Slab &s, int odd, int z_begin, int nplanes, int z_step, cudaStream_t st,
                      bool peer_stores = false) {
    if (nplanes <= 0 || !trim_planes(s, z_begin, nplanes, z_step)) return;
    StepArgs a = h->base;
    a.geo = geo_of(h, s);
    a.z_begin = z_begin;
    a.z_step = z_step;
    a.flags = s.flags;
    if (peer_stores) {
        a.peer_up = h->fst.bases[0];
        a.peer_down = h->fst.bases[1];
    }
    tbegin(h, st);
    h->kern.eso(a, s.pdf[0], odd, grid_for(h, nplanes), h->block, st);
    tend(h, st);
    h->launches++;
    // near-wall cells (split wall mode); a non-null src marks the odd parity for the edge launcher
    launch_edges(h, s, a, h->kern.eso_edges, odd ? s.pdf[0] : nullptr, s.pdf[0], z_begin, nplanes, z_step, st);
}

void launch_aa_range(lbm_handle_s *h, Slab &s, int odd, int z_begin, int nplanes, int z_step, cudaStream_t st,
                     bool peer_stores = false) {
    if (nplanes <= 0 || !trim_planes(s, z_begin, nplanes, z_step)) return;
    StepArgs a = h->base;
    a.geo = geo_of(h, s);
    a.z_begin = z_begin;
    a.z_step = z_step;
    a.flags = s.flags;
    a.lmask = s.lmask;
    a.zg0 = (int)s.z0;
    if (peer_stores) {  // fused halo: LSA bases of the neighbours' single array
        a.peer_up = h->fst.bases[0];
        a.peer_down = h->fst.bases[1];
    }
    tbegin(h, st);
    h->kern.aa(a, s.pdf[0], odd, grid_for(h, nplanes), h->block, st);
    tend(h, st);
    h->launches++;
    if (odd) launch_edges(h, s, a, h->kern.aa_edges, nullptr, s.pdf[0], z_begin, nplanes, z_step, st);
}

// Halo exchange phases. Each phase moves, per slab, one set of crossing slots through face A
// (sent up, received from below) and one through face B (sent down, received from above):
//   pull           : A = c_z=+1 slots of the top plane   -> lower ghost;  B = c_z=-1 of plane 1 -> upper ghost
//   AA ghost fill  : A = c_z=-1 slots of the top plane   -> lower ghost;  B = c_z=+1 of plane 1 -> upper ghost
//                    (after the even step: the odd step pulls a[x - c_q](qbar) across the face)
//   AA return      : A = c_z=+1 slots of the upper ghost -> plane 1;      B = c_z=-1 of the lower ghost -> plane nz
//                    (after the odd step: its pushes a[x + c_q](q) that landed in ghost planes go home;
//                    with walls only where the producing cell is fluid)
//   EsoTwist       : after every step, A = the slots the next step's plane-1 cells read from below, of the
//                    top plane -> lower ghost (slot set c_z(slot) = -1 after even steps, +1 after odd),
//                    B = the slots the plane-1 cells wrote into the lower ghost -> the down neighbour's top
//                    plane (c_z(slot) = +1 after even, -1 after odd). With walls both are masked by the
//                    cell that produced the slot (EsoTwist rule: L + c^+ after even, L - c^- after odd).
struct Phase {
    int dirA, sendA, recvA, dirB, sendB, recvB;
    bool masked;
    int eso_parity = -1;  // EsoTwist exchange: parity of the step just done (selects the producer rule)
};
Phase phase_pull(int nz) { return {+1, nz, 0, -1, 1, nz + 1, false}; }
Phase phase_aa_fill(int nz) { return {-1, nz, 0, +1, 1, nz + 1, false}; }
Phase phase_aa_return(int nz, bool masked) { return {+1, nz + 1, 1, -1, 0, nz, masked}; }
Phase phase_eso(int nz, int parity_done, bool masked) {
    const int d = parity_done ? 1 : -1;
    return {d, nz, 0, -d, 0, nz, masked, parity_done};
}

// Zero-copy schedule of a phase (posting order inside one NCCL group). Per peer pair the sends of
// one side and the receives of the other are posted in the same order, so NCCL matches them even
// when the up and down neighbours are the same rank (P = 2).
struct HaloOp {
    int kind, peer, q, zs;  // kind 0 = send, 1 = recv
};

std::vector<HaloOp> phase_schedule(int Q, const Phase &ph, int up, int down) {
    int qa[9], qb[9];
    const int na = crossing(Q, ph.dirA, qa), nb = crossing(Q, ph.dirB, qb);
    std::vector<HaloOp> ops;
    for (int k = 0; k < na; ++k) ops.push_back({0, up, qa[k], ph.sendA});
    for (int k = 0; k < na; ++k) ops.push_back({1, down, qa[k], ph.recvA});
    for (int k = 0; k < nb; ++k) ops.push_back({0, down, qb[k], ph.sendB});
    for (int k = 0; k < nb; ++k) ops.push_back({1, up, qb[k], ph.recvB});
    return ops;
}

std::vector<HaloOp> halo_schedule(int Q, int nz, int up, int down) { return phase_schedule(Q, phase_pull(nz), up, down); }

void unpack_face(lbm_handle_s *h, const Slab &d, int arr, int zs, int dir, const void *buf, bool masked, cudaStream_t st,
                 int eso_parity = -1) {
    const Geo g = geo_of(h, d);
    if (masked && eso_parity >= 0) launch_unpack_masked_eso(h->Q, h->dtype, g, d.pdf[arr], zs, dir, buf, d.flags, eso_parity, st);
    else if (masked) launch_unpack_masked(h->Q, h->dtype, g, d.pdf[arr], zs, dir, buf, d.flags, st);
    else launch_unpack(h->Q, h->dtype, g, d.pdf[arr], zs, dir, buf, st);
    h->launches++;
}

// ---- halo exchange ------------------------------------------------------------------
// arr(slab) selects the array of each slab the phase works on (pull: the freshly written one).
template <typename ArrSel>
int exchange_loopback(lbm_handle_s *h, const Phase &ph0, ArrSel arr, cudaStream_t st) {
    const int P = (int)h->slabs.size();
    const bool packed = h->cfg.halo_mode == LBM_HALO_PACKED || ph0.masked;
    if (packed) {
        for (int r = 0; r < P; ++r) {
            Slab &s = h->slabs[r];
            Slab &su = h->slabs[(r + 1) % P];
            Slab &sd = h->slabs[(r - 1 + P) % P];
            const Phase ph = ph0;
            launch_pack(h->Q, h->dtype, geo_of(h, s), s.pdf[arr(s)], ph.sendA, ph.dirA, s.halo[0], false, st);
            unpack_face(h, su, arr(su), ph.recvA, ph.dirA, s.halo[0], ph.masked, st, ph.eso_parity);
            launch_pack(h->Q, h->dtype, geo_of(h, s), s.pdf[arr(s)], ph.sendB, ph.dirB, s.halo[1], false, st);
            unpack_face(h, sd, arr(sd), ph.recvB, ph.dirB, s.halo[1], ph.masked, st, ph.eso_parity);
            h->launches += 2;
        }
        return LBM_OK;
    }
    // zero-copy: execute the same per-rank schedule NCCL uses; the k-th send of slab r to peer p
    // is matched with the k-th receive of p from r (NCCL's in-order matching per peer pair)
    std::vector<std::vector<HaloOp>> sched(P);
    for (int r = 0; r < P; ++r) sched[r] = phase_schedule(h->Q, ph0, (r + 1) % P, (r - 1 + P) % P);
    for (int r = 0; r < P; ++r) {
        for (int p = 0; p < P; ++p) {
            std::vector<const HaloOp *> sends, recvs;
            for (const HaloOp &op : sched[r])
                if (op.kind == 0 && op.peer == p) sends.push_back(&op);
            for (const HaloOp &op : sched[p])
                if (op.kind == 1 && op.peer == r) recvs.push_back(&op);
            if (sends.size() != recvs.size()) return fail(h, LBM_EINVAL, "halo schedule mismatch");
            Slab &s = h->slabs[r];
            Slab &d = h->slabs[p];
            for (size_t k = 0; k < sends.size(); ++k)
                CUDA_TRY(h, cudaMemcpyAsync(qplane(h, d, arr(d), recvs[k]->q, recvs[k]->zs),
                                            qplane(h, s, arr(s), sends[k]->q, sends[k]->zs), plane_bytes(h),
                                            cudaMemcpyDeviceToDevice, st));
        }
    }
    return LBM_OK;
}

int exchange_nccl(lbm_handle_s *h, const Phase &ph, int arr, cudaStream_t st) {
    Slab &s = h->slabs[0];
    const ncclDataType_t dt = h->dtype == 0 ? ncclDouble : ncclFloat;
    const size_t plane = (size_t)h->nx * h->ny;
    const size_t ncross = h->Q == 19 ? 5 : 9;
    const Geo g = geo_of(h, s);
    if (h->cfg.halo_mode == LBM_HALO_PACKED || ph.masked) {
        launch_pack(h->Q, h->dtype, g, s.pdf[arr], ph.sendA, ph.dirA, s.halo[0], false, st);
        launch_pack(h->Q, h->dtype, g, s.pdf[arr], ph.sendB, ph.dirB, s.halo[1], false, st);
        h->launches += 2;
        NCCL_TRY(h, ncclGroupStart());
        NCCL_TRY(h, ncclSend(s.halo[0], plane * ncross, dt, h->up, h->comm, st));
        NCCL_TRY(h, ncclRecv(s.halo[2], plane * ncross, dt, h->down, h->comm, st));
        NCCL_TRY(h, ncclSend(s.halo[1], plane * ncross, dt, h->down, h->comm, st));
        NCCL_TRY(h, ncclRecv(s.halo[3], plane * ncross, dt, h->up, h->comm, st));
        NCCL_TRY(h, ncclGroupEnd());
        unpack_face(h, s, arr, ph.recvA, ph.dirA, s.halo[2], ph.masked, st, ph.eso_parity);
        unpack_face(h, s, arr, ph.recvB, ph.dirB, s.halo[3], ph.masked, st, ph.eso_parity);
    } else {
        // zero-copy: each crossing population's plane is one contiguous nx*ny run
        NCCL_TRY(h, ncclGroupStart());
        for (const HaloOp &op : phase_schedule(h->Q, ph, h->up, h->down)) {
            if (op.kind == 0) NCCL_TRY(h, ncclSend(qplane(h, s, arr, op.q, op.zs), plane, dt, op.peer, h->comm, st));
            else NCCL_TRY(h, ncclRecv(qplane(h, s, arr, op.q, op.zs), plane, dt, op.peer, h->comm, st));
        }
        NCCL_TRY(h, ncclGroupEnd());
    }
    return LBM_OK;
}

// exchange the CURRENT pull state's ghost planes (after init / set_populations), ordered on stream
int exchange_current(lbm_handle_s *h) {
    // AA needs ghosts only before odd steps; EsoTwist initialises its lower ghost slots itself
    if (h->g == 0 || h->cfg.pattern != LBM_PULL) return LBM_OK;
    const Phase ph = phase_pull(h->slabs[0].nz);
    if (h->use_nccl) return exchange_nccl(h, ph, h->slabs[0].cur, h->stream);
    return exchange_loopback(h, ph, [](const Slab &s) { return s.cur; }, h->stream);
}

// the bulk update of planes z_begin + k * z_step (k < nplanes) in the configured pattern
void launch_update(lbm_handle_s *h, Slab &s, int odd, int z_begin, int nplanes, int z_step, cudaStream_t st, bool peer) {
    switch (h->cfg.pattern) {
        case LBM_PUSH: launch_push_range(h, s, z_begin, nplanes, z_step, st, peer); break;
        case LBM_ESOTWIST: launch_eso_range(h, s, odd, z_begin, nplanes, z_step, st, peer); break;
        case LBM_AA: launch_aa_range(h, s, odd, z_begin, nplanes, z_step, st, peer); break;
        default: launch_pull_range(h, s, z_begin, nplanes, z_step, st, peer); break;
    }
}

// index-list boundaries: pull fixes the wall slots it is about to stream from (before the step, after
// the previous exchange); AA (after even: pre-odd, after odd: post-odd), EsoTwist (the arriving slot of
// the link location from the departing one, by parity) and push fix after the step's exchange.
// `written` = the array the step wrote (push: the fresh array; AA / EsoTwist: the single one).
void links_before_step(lbm_handle_s *h, Slab &s, cudaStream_t st) {
    if (h->cfg.pattern == LBM_PULL) launch_links_fix(h, s, s.pdf[s.cur], 0, st);
}
void links_fix_step(lbm_handle_s *h, Slab &s, int odd, int written, cudaStream_t st) {
    if (h->cfg.pattern == LBM_AA) launch_links_fix(h, s, s.pdf[0], odd ? 2 : 1, st);
    else if (h->cfg.pattern == LBM_ESOTWIST) launch_links_fix(h, s, s.pdf[0], odd ? 4 : 3, st);
    else if (h->cfg.pattern == LBM_PUSH) launch_links_fix(h, s, s.pdf[written], 2, st);
}
void links_after_step(lbm_handle_s *h, Slab &s, int odd, cudaStream_t st) { links_fix_step(h, s, odd, 1 - s.cur, st); }
// Fused halo: a step's link fix must follow the neighbours' peer stores of that step, i.e. the next LSA
// gate; it is deferred to after the next step's gate, or to the closing gate at the end of lbm_step.
// In-kernel links: before the first step after the state was set from outside (init, set, load), the wall
// slots the next step streams from are filled from the full list (pull: mode 0; AA before an odd step: mode
// 1; before an even step nothing is read from walls). Outside any graph capture (lbm_step's entry).
void links_prime(lbm_handle_s *h, cudaStream_t st) {
    if (!h->links_fused) return;
    for (Slab &s : h->slabs) {
        if (s.links_primed) continue;
        if (h->cfg.pattern == LBM_PULL) launch_links_fix(h, s, s.pdf[s.cur], 0, st, true);
        else if (h->aa_parity) launch_links_fix(h, s, s.pdf[0], 1, st, true);
        s.links_primed = true;
    }
}
void links_unprime(lbm_handle_s *h) {
    for (Slab &s : h->slabs) s.links_primed = false;
}

void links_deferred(lbm_handle_s *h, Slab &s, cudaStream_t st) {
    if (h->links_pending < 0) return;
    links_fix_step(h, s, h->links_pending & 1, h->links_pending >> 1, st);
    h->links_pending = -1;
}

void toggle_state(lbm_handle_s *h) {
    if (two_arrays(h))
        for (Slab &s : h->slabs) s.cur ^= 1;
    else
        h->aa_parity ^= 1;
}

// the exchange phase that follows a step of the configured pattern (odd = parity of that step)
Phase step_phase(const lbm_handle_s *h, int odd) {
    const int nz = h->slabs[0].nz;
    switch (h->cfg.pattern) {
        case LBM_PUSH: return phase_aa_return(nz, h->have_flags);  // pushes that landed in ghost planes go home
        case LBM_ESOTWIST: return phase_eso(nz, odd, h->have_flags);
        case LBM_AA: return odd ? phase_aa_return(nz, h->have_flags) : phase_aa_fill(nz);
        default: return phase_pull(nz);
    }
}

// ---- one time step ------------------------------------------------------------------
// Decomposed steps run the boundary planes first, then exchange (NCCL: on the comm stream while the
// interior planes update on the compute stream; loopback: device copies; fused: the boundary-plane
// kernels store into the neighbours' planes after an LSA barrier); the next step waits for it.
// phase event k of the timeline (timing mode only; k: 0/1 boundary, 2/3 exchange, 4/5 interior)
void mark(lbm_handle_s *h, int k, cudaStream_t st) {
    if (!h->timing.on) return;
    if (!h->timing.ph[k]) cudaEventCreate(&h->timing.ph[k]);
    cudaEventRecord(h->timing.ph[k], st);
    if (k == 5) h->timing.ph_valid = true;
}

int step_once(lbm_handle_s *h) {
    cudaStream_t st = h->stream;
    const int odd = h->aa_parity;
    if (h->g == 0) {
        NvtxRange r("lbm.step");
        Slab &s = h->slabs[0];
        links_before_step(h, s, st);
        launch_update(h, s, odd, 0, s.nz, 1, st, false);
        links_after_step(h, s, odd, st);
        toggle_state(h);
        return LBM_OK;
    }
    const bool single = !two_arrays(h);  // the exchanged array: the single one, or the freshly written one
    const Phase ph = step_phase(h, odd);
    auto bnd = [&](Slab &s, bool peer) {
        NvtxRange r("lbm.boundary_planes");
        launch_update(h, s, odd, 0, 2, s.nz - 1, st, peer);
    };
    auto inner = [&](Slab &s) {
        NvtxRange r("lbm.interior");
        launch_update(h, s, odd, 1, s.nz - 2, 1, st, false);
    };
    if (!h->use_nccl) {
        // loopback slabs on one GPU, one stream: boundary planes, exchange, interior
        for (Slab &s : h->slabs) links_before_step(h, s, st);
        mark(h, 0, st);
        for (Slab &s : h->slabs) bnd(s, false);
        mark(h, 1, st);
        mark(h, 2, st);
        int rc;
        {
            NvtxRange r("lbm.exchange");
            rc = single ? exchange_loopback(h, ph, [](const Slab &) { return 0; }, st)
                        : exchange_loopback(h, ph, [](const Slab &s) { return 1 - s.cur; }, st);
        }
        if (rc) return rc;
        mark(h, 3, st);
        mark(h, 4, st);
        for (Slab &s : h->slabs) inner(s);
        mark(h, 5, st);
        for (Slab &s : h->slabs) links_after_step(h, s, odd, st);
        toggle_state(h);
        return LBM_OK;
    }
    Slab &s = h->slabs[0];
    if (h->fused) {
        // gate (LSA barrier: every rank finished the previous step, so the stores into our planes are
        // done and the slots we overwrite are no longer read) -> the previous step's deferred link fix
        // (index lists with AA / EsoTwist / push) -> boundary planes with peer stores -> interior planes;
        // one stream, no send/recv
        mark(h, 2, st);
        {
            NvtxRange r("lbm.lsa_gate");
            fused_gate(h->fst, st);
        }
        mark(h, 3, st);
        h->launches++;
        links_deferred(h, s, st);
        links_before_step(h, s, st);
        mark(h, 0, st);
        bnd(s, true);
        mark(h, 1, st);
        mark(h, 4, st);
        inner(s);
        mark(h, 5, st);
        if (h->links && h->cfg.pattern != LBM_PULL) h->links_pending = odd | ((1 - s.cur) << 1);
        toggle_state(h);
        return LBM_OK;
    }
    links_before_step(h, s, st);
    mark(h, 0, st);
    bnd(s, false);
    mark(h, 1, st);
    CUDA_TRY(h, cudaEventRecord(h->ev_bnd, st));
    CUDA_TRY(h, cudaStreamWaitEvent(h->comm_stream, h->ev_bnd, 0));
    mark(h, 2, h->comm_stream);
    int rc;
    {
        NvtxRange r("lbm.exchange");
        rc = exchange_nccl(h, ph, single ? 0 : 1 - s.cur, h->comm_stream);
    }
    if (rc) return rc;
    mark(h, 3, h->comm_stream);
    CUDA_TRY(h, cudaEventRecord(h->ev_x, h->comm_stream));
    mark(h, 4, st);
    inner(s);
    mark(h, 5, st);
    CUDA_TRY(h, cudaStreamWaitEvent(st, h->ev_x, 0));  // the next step's boundary planes need the exchange
    links_after_step(h, s, odd, st);
    toggle_state(h);
    return LBM_OK;
}

bool graph_ok(const lbm_handle_s *h) { return h->cfg.use_graph == 1 && h->g == 0 && h->slabs.size() == 1 && !h->timing.on; }
bool persistent_ok(const lbm_handle_s *h) {
    return h->cfg.use_graph == 2 && !h->links && (h->cfg.pattern == LBM_PULL || h->cfg.pattern == LBM_AA) && h->g == 0 && h->slabs.size() == 1 && h->kern.persist_pull && h->kern.persist_aa;
}

int run_graph_cycle(lbm_handle_s *h) {
    // one cycle = two steps (pull: src->dst->src; AA: even+odd), replayed; state returns to the same slots
    // re-capture when the parity or the process-wide kernel path changed since the capture
    if (!h->graph || h->graph_parity != (!two_arrays(h) ? h->aa_parity : h->slabs[0].cur) ||
        h->graph_path != lbm::staged_path()) {
        if (h->graph) {
            cudaGraphExecDestroy(h->graph);
            h->graph = nullptr;
        }
        cudaGraph_t gr;
        const int par = !two_arrays(h) ? h->aa_parity : h->slabs[0].cur;
        CUDA_TRY(h, cudaStreamBeginCapture(h->stream, cudaStreamCaptureModeThreadLocal));
        const int64_t l0 = h->launches;
        step_once(h);
        step_once(h);
        cudaError_t e = cudaStreamEndCapture(h->stream, &gr);
        if (e != cudaSuccess) return fail(h, LBM_ECUDA, std::string("graph capture: ") + cudaGetErrorString(e));
        CUDA_TRY(h, cudaGraphInstantiate(&h->graph, gr, 0));
        cudaGraphDestroy(gr);
        h->launches = l0;  // the capture did not launch
        h->graph_parity = par;
        h->graph_path = lbm::staged_path();
    }
    CUDA_TRY(h, cudaGraphLaunch(h->graph, h->stream));
    h->launches += 2;
    return LBM_OK;
}

int validate(const lbm_config *c) {
    if (!c) return fail(nullptr, LBM_EINVAL, "null config");
    if (c->stencil != 19 && c->stencil != 27) return fail(nullptr, LBM_EINVAL, "stencil must be 19 or 27");
    if (c->collision < 0 || c->collision > LBM_GEN_SMAGORINSKY) return fail(nullptr, LBM_EINVAL, "bad collision");
    if (c->dtype != LBM_F64 && c->dtype != LBM_F32) return fail(nullptr, LBM_EINVAL, "bad dtype");
    if (c->pattern < LBM_PULL || c->pattern > LBM_PUSH) return fail(nullptr, LBM_EINVAL, "bad pattern");
    const int need[] = {1, 2, 1, 1, 0, 2, 1, 1, 1, 2, 1, 2};
    const int need_n = (c->collision == LBM_MRT && c->n_row_rates == 15) ? 0 : need[c->collision];
    if (c->n_rates < need_n || c->n_rates > 8) return fail(nullptr, LBM_EINVAL, "wrong number of rates");
    for (int i = 0; i < c->n_rates; ++i)
        if (!(c->rates[i] > 0.0 && c->rates[i] < 2.0)) return fail(nullptr, LBM_EINVAL, "relaxation rate outside (0, 2)");
    for (int d = 0; d < 3; ++d)
        if (c->global[d] < 1) return fail(nullptr, LBM_EINVAL, "empty lattice");
    if (c->nranks < 1 || c->rank < 0 || c->rank >= c->nranks) return fail(nullptr, LBM_EINVAL, "bad rank/nranks");
    if (c->n_local_slabs < 0) return fail(nullptr, LBM_EINVAL, "bad n_local_slabs");
    if (c->nranks > 1 && c->n_local_slabs > 1) return fail(nullptr, LBM_EINVAL, "loopback slabs require nranks == 1");
    const int P = c->nranks > 1 ? c->nranks : (c->n_local_slabs > 1 ? c->n_local_slabs : 1);
    if (c->global[2] % P != 0) return fail(nullptr, LBM_EINVAL, "nz % nranks != 0");
    if (P > 1 && c->global[2] / P < 2) return fail(nullptr, LBM_EINVAL, "slabs need at least 2 planes");
    if (c->nranks > 1 && !c->nccl_id) return fail(nullptr, LBM_EINVAL, "nranks > 1 needs an nccl_id");
    if (c->halo_mode == LBM_HALO_FUSED && c->nranks == 1 && !c->nccl_self)
        return fail(nullptr, LBM_EUNSUPPORTED, "fused halo needs NCCL ranks (or nccl_self)");
    if (c->halo_mode < 0 || c->halo_mode > 2) return fail(nullptr, LBM_EINVAL, "bad halo_mode");
    if (c->nccl_self && (c->nranks != 1 || c->n_local_slabs > 1 || c->global[2] < 2))
        return fail(nullptr, LBM_EINVAL, "nccl_self needs nranks == 1, one slab and nz >= 2");
    const int64_t planes = c->global[2] / P + (P > 1 ? 2 : 0);
    if ((double)c->global[0] * c->global[1] * planes >= 2147483647.0)
        return fail(nullptr, LBM_EINVAL, "slab too large for 32-bit in-plane offsets (split it over more slabs)");
    const bool force = c->force[0] != 0 || c->force[1] != 0 || c->force[2] != 0;
    if (c->collision == LBM_MRT && c->stencil != 19)
        return fail(nullptr, LBM_EUNSUPPORTED, "MRT is implemented for D3Q19 (D3Q27: LBM_GEN_MRT)");
    if (force && c->collision != LBM_SRT && c->collision != LBM_TRT)
        return fail(nullptr, LBM_EUNSUPPORTED, "forcing is implemented for SRT/TRT");
    if (c->n_row_rates != 0 && c->n_row_rates != 15) return fail(nullptr, LBM_EINVAL, "n_row_rates must be 0 or 15");
    if (c->n_row_rates == 15) {
        if (c->collision != LBM_MRT) return fail(nullptr, LBM_EINVAL, "per-moment rates are for LBM_MRT");
        for (int i = 0; i < 15; ++i)
            if (!(c->row_rates[i] > 0.0 && c->row_rates[i] < 2.0))
                return fail(nullptr, LBM_EINVAL, "relaxation rate outside (0, 2)");
        if (c->equilibrium != LBM_EQ_COMPRESSIBLE)
            return fail(nullptr, LBM_EUNSUPPORTED, "per-moment MRT rates use the compressible equilibrium");
    }
    if (c->boundary_mode != LBM_BOUNDARY_FLAGS && c->boundary_mode != LBM_BOUNDARY_LINKS &&
        c->boundary_mode != LBM_BOUNDARY_INLINE)
        return fail(nullptr, LBM_EINVAL, "bad boundary_mode");
    if (c->boundary_mode == LBM_BOUNDARY_INLINE && c->halo_mode == LBM_HALO_FUSED && (c->nranks > 1 || c->nccl_self))
        return fail(nullptr, LBM_EUNSUPPORTED, "compiled-in (inline) boundaries use the NCCL or loopback halo");
    if (c->equilibrium < LBM_EQ_COMPRESSIBLE || c->equilibrium > LBM_EQ_MOMENT_MATCHED)
        return fail(nullptr, LBM_EINVAL, "bad equilibrium");
    // borrowed device buffers (lbm_config.pdf_dev / flags_dev / halo_dev)
    const bool two = c->pattern == LBM_PULL || c->pattern == LBM_PUSH;
    const bool borrowed = c->pdf_dev[0] || c->pdf_dev[1] || c->flags_dev || c->halo_dev;
    if (borrowed) {
        if (c->n_local_slabs > 1) return fail(nullptr, LBM_EUNSUPPORTED, "borrowed device buffers need one slab per process");
        if (c->halo_mode == LBM_HALO_FUSED && (c->nranks > 1 || c->nccl_self))
            return fail(nullptr, LBM_EUNSUPPORTED, "the fused halo owns its arrays (NCCL symmetric windows)");
        if (two ? (c->pdf_dev[0] == nullptr) != (c->pdf_dev[1] == nullptr) : c->pdf_dev[1] != nullptr)
            return fail(nullptr, LBM_EINVAL, "pdf_dev: give both arrays for PULL/PUSH, one (pdf_dev[0]) for AA/EsoTwist");
        if (c->flags_dev && !c->flags) return fail(nullptr, LBM_EINVAL, "flags_dev without a flag field");
        if (c->halo_dev && !(c->nranks > 1 || c->nccl_self))
            return fail(nullptr, LBM_EINVAL, "halo_dev without a decomposition");
        for (const void *p : {(const void *)c->pdf_dev[0], (const void *)c->pdf_dev[1], (const void *)c->flags_dev,
                              (const void *)c->halo_dev})
            if (reinterpret_cast<uintptr_t>(p) % 16 != 0) return fail(nullptr, LBM_EINVAL, "borrowed buffer not 16-byte aligned");
    }
    if (c->equilibrium != LBM_EQ_COMPRESSIBLE && c->collision != LBM_SRT && c->collision != LBM_TRT &&
        c->collision != LBM_MRT && c->collision != LBM_IDENTITY &&
        !((c->collision == LBM_GEN_SRT || c->collision == LBM_GEN_TRT) && c->equilibrium == LBM_EQ_INCOMPRESSIBLE))
        return fail(nullptr, LBM_EUNSUPPORTED, "equilibrium variants are implemented for SRT/TRT/MRT (generated: incompressible SRT/TRT)");
    // a non-periodic axis must carry wall cells on both faces
    for (int d = 0; d < 3; ++d) {
        if (c->periodic[d]) continue;
        if (!c->flags) return fail(nullptr, LBM_EINVAL, "non-periodic axis without a flag field");
        const int64_t n[3] = {c->global[0], c->global[1], c->global[2]};
        for (int side = 0; side < 2; ++side) {
            const int64_t fix = side ? n[d] - 1 : 0;
            const int a1 = (d + 1) % 3, a2 = (d + 2) % 3;
            for (int64_t i = 0; i < n[a1]; ++i)
                for (int64_t j = 0; j < n[a2]; ++j) {
                    int64_t co[3];
                    co[d] = fix;
                    co[a1] = i;
                    co[a2] = j;
                    if (c->flags[co[0] + n[0] * (co[1] + n[1] * co[2])] == 0)
                        return fail(nullptr, LBM_EINVAL, "non-periodic axis has fluid cells on its face");
                }
        }
    }
    return LBM_OK;
}

// Face-aligned walls (FM_FACES): every non-fluid cell lies on a face of a non-periodic axis, each such
// face carries one wall type, and a cell on several wall faces has the type of the first face in the
// order -x, +x, -y, +y, -z, +z (the channel of C1, the cavity of C3 with its NoSlip lid edges, G9). Then
// the update kernels recognise wall and near-wall cells from coordinates. O(cells) host check at create.
bool detect_faces(const lbm_config *c, int8_t face[6]) {
    const int64_t n[3] = {c->global[0], c->global[1], c->global[2]};
    for (int f = 0; f < 6; ++f) face[f] = 0;
    bool any = false;
    for (int d = 0; d < 3; ++d) {
        if (c->periodic[d]) continue;
        if (n[d] < 3) return false;
        for (int side = 0; side < 2; ++side) {
            int64_t co[3] = {n[0] / 2, n[1] / 2, n[2] / 2};
            co[d] = side ? n[d] - 1 : 0;
            const uint8_t t = c->flags[co[0] + n[0] * (co[1] + n[1] * co[2])];
            if (t != LBM_FLAG_NOSLIP && t != LBM_FLAG_UBB) return false;
            face[2 * d + side] = (int8_t)t;
            any = true;
        }
    }
    if (!any) return false;
    for (int64_t z = 0; z < n[2]; ++z)
        for (int64_t y = 0; y < n[1]; ++y)
            for (int64_t x = 0; x < n[0]; ++x) {
                const int64_t co[3] = {x, y, z};
                int expect = 0;
                for (int f = 0; f < 6 && !expect; ++f)
                    if (face[f] && co[f / 2] == ((f & 1) ? n[f / 2] - 1 : 0)) expect = face[f];
                if (c->flags[x + n[0] * (y + n[1] * z)] != expect) return false;
            }
    return true;
}

// per-link UBB terms 6 w_q rho_w c_q.u_w (rho_w = 1, G8) from per-link wall velocities uw[3*i+d];
// no-slip links get 0
int upload_link_terms(lbm_handle h, Slab &s, const double *uw) {
    const size_t n = s.h_link_wall.size();
    std::vector<double> term(n, 0.0);
    for (size_t i = 0; i < n; ++i) {
        if (s.h_link_type[i] != LBM_FLAG_UBB) continue;
        const int q = s.h_link_dir[i];
        const double w = h->Q == 19 ? Stencil<19>::w(q) : Stencil<27>::w(q);
        const double cu = kC27[q][0] * uw[3 * i] + kC27[q][1] * uw[3 * i + 1] + kC27[q][2] * uw[3 * i + 2];
        term[i] = 6.0 * w * cu;
    }
    if (n) CUDA_TRY(h, cudaMemcpy(s.link_term, term.data(), n * sizeof(double), cudaMemcpyHostToDevice));
    if (s.n_res) {
        std::vector<double> rt(s.n_res);
        for (uint32_t i = 0; i < s.n_res; ++i) rt[i] = term[s.h_res_idx[i]];
        CUDA_TRY(h, cudaMemcpy(s.res_term, rt.data(), s.n_res * sizeof(double), cudaMemcpyHostToDevice));
    }
    return LBM_OK;
}

// Thread block of the plain update kernels: 256 threads as bx x-cells times 256/bx rows, with bx the
// largest of 256, 128, 64, 32 that wastes the fewest idle lanes at the row end (nx = 384 -> 128 x 2,
// nx = 300 -> 64 x 4 instead of 256 + a mostly idle block); the register caps of the kernels assume
// 256-thread blocks. bx_req > 0 forces the x extent.
dim3 block_for(int64_t nx, int64_t ny, int bx_req) {
    int bx = bx_req;
    if (bx <= 0) {
        int64_t best = -1;
        for (int c = 256; c >= 32; c /= 2) {
            const int64_t waste = (nx + c - 1) / c * c - nx;
            if (best < 0 || waste < best) {
                best = waste;
                bx = c;
            }
        }
    }
    if (bx > nx) bx = (int)((nx + 31) / 32 * 32);
    if (bx > 256) bx = 256;
    int by = 256 / bx;
    if (by > ny) by = (int)ny;
    if (by < 1) by = 1;
    return dim3(bx, by, 1);
}

// Flat rows (kernels.cuh box_cell): a launch box of full x-rows whose row end leaves idle lanes in every block
// shape (nx = 300: 20 of 320 thread slots, in CTAs that hold their registers until the full warps finish) is
// indexed linearly over the rows' contiguous cells by (256, 1, 1) blocks; LBM_FLAT=0 keeps the 2-D blocks.
// Sets a.flat_* and `block` and returns true if the box a.x0..a.y1 qualifies.
bool flat_rows(StepArgs &a, dim3 &block, int64_t nx, int64_t ny) {
    const char *env = std::getenv("LBM_FLAT");
    if ((env && env[0] == '0') || a.x0 != 0 || a.x1 != (int)nx || nx < 2 || nx % block.x == 0 || nx * ny >= (int64_t)1 << 30 || a.y1 <= a.y0)
        return false;
    a.flat_lo = a.y0 * (int)nx;
    a.flat_hi = a.y1 * (int)nx;
    a.flat_start = a.flat_lo / 32 * 32;
    a.flat_magic = (unsigned)(((uint64_t)1 << 32) / (uint64_t)nx + 1);
    block = dim3(256, 1, 1);
    return true;
}

// grid of one plain update launch over the box of `a` (2-D blocks or flat rows) times the planes
dim3 box_grid(const StepArgs &a, dim3 block, int nplanes) {
    if (a.flat_hi > 0) return dim3((unsigned)((a.flat_hi - a.flat_start + 255) / 256), 1u, (unsigned)nplanes);
    const int64_t bx = a.x1 - a.x0, by = a.y1 - a.y0;
    return dim3((unsigned)((bx + block.x - 1) / block.x), (unsigned)((by + block.y - 1) / block.y), (unsigned)nplanes);
}

// staging buffers and streams of LBM_HOST_ASYNC, created on first use (4 doubles per local cell, x 4)
int ensure_async(lbm_handle h) {
    auto &a = h->aio;
    if (a.ready) return LBM_OK;
    int64_t cells = 0;
    for (const Slab &s : h->slabs) cells += (int64_t)h->nx * h->ny * s.nz;
    const size_t bytes = (size_t)cells * 4 * sizeof(double);
    CUDA_TRY(h, cudaStreamCreateWithFlags(&a.h2d, cudaStreamNonBlocking));
    CUDA_TRY(h, cudaStreamCreateWithFlags(&a.d2h, cudaStreamNonBlocking));
    for (int k = 0; k < 2; ++k) {
        CUDA_TRY(h, cudaMalloc(&a.in[k], bytes));
        CUDA_TRY(h, cudaMalloc(&a.out[k], bytes));
        for (cudaEvent_t *e : {&a.in_ready[k], &a.in_free[k], &a.out_ready[k], &a.out_free[k]})
            CUDA_TRY(h, cudaEventCreateWithFlags(e, cudaEventDisableTiming));
    }
    a.ready = true;
    return LBM_OK;
}

void free_async(lbm_handle h) {
    auto &a = h->aio;
    if (a.h2d) cudaStreamSynchronize(a.h2d);
    if (a.d2h) cudaStreamSynchronize(a.d2h);
    for (int k = 0; k < 2; ++k) {
        if (a.in[k]) cudaFree(a.in[k]);
        if (a.out[k]) cudaFree(a.out[k]);
        for (cudaEvent_t e : {a.in_ready[k], a.in_free[k], a.out_ready[k], a.out_free[k]})
            if (e) cudaEventDestroy(e);
    }
    if (a.h2d) cudaStreamDestroy(a.h2d);
    if (a.d2h) cudaStreamDestroy(a.d2h);
    a = lbm_handle_s::AsyncIO{};
}

int ensure_scratch(lbm_handle h, size_t bytes) {
    if (h->scratch_bytes >= bytes) return LBM_OK;
    if (h->scratch) cudaFree(h->scratch);
    h->scratch = nullptr;
    h->scratch_bytes = 0;
    CUDA_TRY(h, cudaMalloc(&h->scratch, bytes));
    h->scratch_bytes = bytes;
    return LBM_OK;
}

int64_t local_cells(const lbm_handle_s *h) {
    int64_t n = 0;
    for (const Slab &s : h->slabs) n += (int64_t)h->nx * h->ny * s.nz;
    return n;
}

}  // namespace

// =========================================================================================
// C ABI
// =========================================================================================
namespace lbm {
Kernels select_kernels(int collision, int Q, int dtype, int fm, bool force, int eq) {
    if (eq == EQ_MOMENT_MATCHED && Q == 27) eq = EQ_COMPRESSIBLE;  // identical for D3Q27
    if (eq != EQ_COMPRESSIBLE) {
        if (collision == LBM_SRT || collision == LBM_TRT) return select_trt_eq(Q, dtype, fm, force, eq);
        if (collision == LBM_MRT) return select_mrt_eq(Q, dtype, fm, force, eq);
        if (collision == LBM_GEN_SRT || collision == LBM_GEN_TRT) return select_generated(collision, Q, dtype, fm, force, eq);
        if (collision != LBM_IDENTITY) return Kernels{};
    }
    switch (collision) {
        case OP_MRT_ROWS: return eq == EQ_COMPRESSIBLE ? select_mrt_rows(Q, dtype, fm, force) : Kernels{};
        case LBM_SRT:
        case LBM_TRT: return select_trt(Q, dtype, fm, force);
        case LBM_MRT: return select_mrt(Q, dtype, fm, force);
        case LBM_CUMULANT: return select_cumulant(Q, dtype, fm, force);
        case OP_CUMULANT_UNIT: return select_cumulant_unit(Q, dtype, fm, force);
        case OP_MRT_SHEAR: return select_mrt_shear(Q, dtype, fm, force);
        case LBM_SMAGORINSKY: return select_smagorinsky(Q, dtype, fm, force);
        case LBM_KBC: return select_kbc(Q, dtype, fm, force);
        case LBM_KBC_EXACT: return select_kbc_exact(Q, dtype, fm, force);
        case LBM_GEN_SRT:
        case LBM_GEN_TRT:
        case LBM_GEN_MRT:
        case LBM_GEN_SMAGORINSKY: return select_generated(collision, Q, dtype, fm, force, eq);
        default: return select_identity(Q, dtype, fm, force);
    }
}
}  // namespace lbm

extern "C" {

void lbm_config_default(lbm_config *c) {
    std::memset(c, 0, sizeof(*c));
    c->stencil = LBM_D3Q19;
    c->collision = LBM_SRT;
    c->dtype = LBM_F64;
    c->pattern = LBM_PULL;
    c->n_rates = 1;
    c->rates[0] = 1.8;
    c->global[0] = c->global[1] = c->global[2] = 32;
    c->periodic[0] = c->periodic[1] = c->periodic[2] = 1;
    c->nranks = 1;
    c->n_local_slabs = 1;
}

const char *lbm_version(void) { return "b200-lbm 0.2 (sm_100a)"; }

int64_t lbm_boundary_links(lbm_handle h, int64_t *cells, int32_t *dirs, int32_t *types, int64_t cap) {
    if (!h) return LBM_EINVAL;
    if (!h->links) return 0;
    int64_t n = 0;
    for (const Slab &s : h->slabs) n += (int64_t)s.h_link_wall.size();
    if (cap < n && (cells || dirs || types)) return fail(h, LBM_EINVAL, "link buffer too small");
    int64_t i = 0;
    const int64_t plane = h->nx * h->ny;
    for (const Slab &s : h->slabs)
        for (size_t k = 0; k < s.h_link_wall.size(); ++k, ++i) {
            if (cells) {  // storage index -> global linear index (ghost planes map to the neighbour's planes)
                const int64_t b = s.h_link_wall[k], zs = b / plane;
                const int64_t zg = ((s.z0 + zs - h->g) % h->nzg + h->nzg) % h->nzg;
                cells[i] = zg * plane + (b - zs * plane);
            }
            if (dirs) dirs[i] = s.h_link_dir[k];
            if (types) types[i] = s.h_link_type[k];
        }
    return n;
}

int lbm_set_link_velocities(lbm_handle h, const double *uw, int64_t n) {
    if (!h || !uw) return LBM_EINVAL;
    if (!h->links) return fail(h, LBM_EINVAL, "no index-list boundaries (boundary_mode != LBM_BOUNDARY_LINKS)");
    int64_t total = 0;
    for (const Slab &s : h->slabs) total += (int64_t)s.h_link_wall.size();
    if (n != total) return fail(h, LBM_EINVAL, "link count mismatch");
    CUDA_TRY(h, cudaStreamSynchronize(h->stream));  // the terms may be in use by queued link kernels
    if (h->links_fused) {
        // per-link velocities: the in-kernel stores use one wall velocity; from here on the separate link
        // kernel with the full list runs (same state invariants: the wall slots hold the same values)
        h->links_fused = false;
        h->kern = h->kern_links;
        if (h->graph) {
            cudaGraphExecDestroy(h->graph);
            h->graph = nullptr;
        }
    }
    int64_t off = 0;
    for (Slab &s : h->slabs) {
        const int rc = upload_link_terms(h, s, uw + 3 * off);
        if (rc) return rc;
        off += (int64_t)s.h_link_wall.size();
    }
    return LBM_OK;
}

int lbm_probe_copy(int32_t stencil, int32_t dtype, int32_t shifted, int64_t nx, int64_t ny, int64_t nz, int32_t reps,
                   int32_t device, double *gbs_out) {
    if ((stencil != 19 && stencil != 27) || (dtype != LBM_F64 && dtype != LBM_F32) || nx < 1 || ny < 1 || nz < 1 ||
        reps < 1 || !gbs_out || (double)nx * ny * nz >= 2147483647.0 || nx > 2147483647 / 256)
        return LBM_EINVAL;
    if (cudaSetDevice(device) != cudaSuccess) return LBM_ECUDA;
    Geo g;
    g.nx = (int)nx;
    g.ny = (int)ny;
    g.nz = (int)nz;
    g.g = 0;
    g.Sq = nx * ny * nz;
    const size_t es = dtype == LBM_F64 ? 8 : 4;
    const size_t bytes = (size_t)g.Sq * stencil * es;
    void *a = nullptr, *b = nullptr;
    if (cudaMalloc(&a, bytes) != cudaSuccess) return LBM_EOOM;
    if (cudaMalloc(&b, bytes) != cudaSuccess) {
        cudaFree(a);
        return LBM_EOOM;
    }
    cudaStream_t s;
    cudaEvent_t e0, e1;
    cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaMemsetAsync(a, 0, bytes, s);
    cudaMemsetAsync(b, 0, bytes, s);
    for (int w = 0; w < 2; ++w) launch_copyq(stencil, dtype, shifted != 0, g, w ? b : a, w ? a : b, s);  // warm-up
    cudaEventRecord(e0, s);
    for (int r = 0; r < reps; ++r) launch_copyq(stencil, dtype, shifted != 0, g, (r & 1) ? b : a, (r & 1) ? a : b, s);
    cudaEventRecord(e1, s);
    const cudaError_t err = cudaEventSynchronize(e1);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaStreamDestroy(s);
    cudaFree(a);
    cudaFree(b);
    if (err != cudaSuccess || ms <= 0.f) return LBM_ECUDA;
    *gbs_out = 2.0 * (double)bytes * reps / (ms * 1e-3) / 1e9;
    return LBM_OK;
}

int lbm_probe_update(int32_t stencil, int32_t dtype, int32_t mode, int64_t nx, int64_t ny, int64_t nz, int32_t reps,
                     int32_t device, double *gbs_out) {
    if ((stencil != 19 && stencil != 27) || (dtype != LBM_F64 && dtype != LBM_F32) || mode < 0 || mode > 2 || nx < 1 ||
        ny < 1 || nz < 1 || reps < 1 || !gbs_out || (double)nx * ny * nz >= 2147483647.0 || nx > 2147483647 / 256)
        return LBM_EINVAL;
    if (cudaSetDevice(device) != cudaSuccess) return LBM_ECUDA;
    Geo g;
    g.nx = (int)nx;
    g.ny = (int)ny;
    g.nz = (int)nz;
    g.g = 0;
    g.Sq = nx * ny * nz;
    const size_t es = dtype == LBM_F64 ? 8 : 4;
    const size_t bytes = (size_t)g.Sq * stencil * es;
    void *a = nullptr;
    if (cudaMalloc(&a, bytes) != cudaSuccess) return LBM_EOOM;
    cudaStream_t s;
    cudaEvent_t e0, e1;
    cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaMemsetAsync(a, 0, bytes, s);
    // mode 0: even pattern only, 1: odd pattern only, 2: alternating even/odd (the AA pair)
    auto odd_of = [&](int r) { return mode == 2 ? (r & 1) != 0 : mode == 1; };
    for (int w = 0; w < 2; ++w) launch_updateq(stencil, dtype, odd_of(w), g, a, s);
    cudaEventRecord(e0, s);
    for (int r = 0; r < reps; ++r) launch_updateq(stencil, dtype, odd_of(r), g, a, s);
    cudaEventRecord(e1, s);
    const cudaError_t err = cudaEventSynchronize(e1);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaStreamDestroy(s);
    cudaFree(a);
    if (err != cudaSuccess || ms <= 0.f) return LBM_ECUDA;
    *gbs_out = 2.0 * (double)bytes * reps / (ms * 1e-3) / 1e9;
    return LBM_OK;
}

int lbm_probe_fma(int32_t dtype, int32_t device, double *tflops_out) {
    if ((dtype != LBM_F64 && dtype != LBM_F32) || !tflops_out) return LBM_EINVAL;
    if (cudaSetDevice(device) != cudaSuccess) return LBM_ECUDA;
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
    const int blocks = sms * 8, iters = dtype == LBM_F64 ? 2048 : 8192;  // 8 x 256 threads per SM
    void *sink = nullptr;
    if (cudaMalloc(&sink, 256 * 8) != cudaSuccess) return LBM_EOOM;
    cudaStream_t s;
    cudaEvent_t e0, e1;
    cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    launch_fma_probe(dtype, blocks, iters / 8, sink, s);  // warm-up
    cudaEventRecord(e0, s);
    const int reps = 5;
    for (int r = 0; r < reps; ++r) launch_fma_probe(dtype, blocks, iters, sink, s);
    cudaEventRecord(e1, s);
    const cudaError_t err = cudaEventSynchronize(e1);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaStreamDestroy(s);
    cudaFree(sink);
    if (err != cudaSuccess || ms <= 0.f) return LBM_ECUDA;
    const double fmas = (double)blocks * 256 * iters * 16 * 8 * reps;
    *tflops_out = 2.0 * fmas / (ms * 1e-3) / 1e12;
    return LBM_OK;
}

int lbm_set_kernel_path(int32_t path) {
    if (path < LBM_PATH_AUTO || path > LBM_PATH_STAGED) return LBM_EINVAL;
    lbm::set_staged_path(path);
    return LBM_OK;
}
int32_t lbm_get_kernel_path(void) { return lbm::staged_path(); }

const char *lbm_strerror(int s) {
    switch (s) {
        case LBM_OK: return "ok";
        case LBM_EINVAL: return "invalid argument";
        case LBM_EUNSUPPORTED: return "unsupported configuration";
        case LBM_ECUDA: return "CUDA error";
        case LBM_ENCCL: return "NCCL error";
        case LBM_ENAN: return "NaN in populations";
        case LBM_EOOM: return "out of device memory";
        default: return "unknown status";
    }
}

const char *lbm_last_error(lbm_handle h) { return h ? h->err.c_str() : g_create_error.c_str(); }


static int kernel_args_common(const lbm_kernel_args *k, StepArgs &a, bool aa) {
    if (!k || (k->stencil != 19 && k->stencil != 27) || k->collision < 0 || k->collision > LBM_GEN_SMAGORINSKY ||
        (k->dtype != LBM_F64 && k->dtype != LBM_F32) || !k->dst || (!aa && !k->src) || k->ghost < 0 || k->ghost > 1 ||
        k->equilibrium < LBM_EQ_COMPRESSIBLE || k->equilibrium > LBM_EQ_MOMENT_MATCHED)
        return LBM_EINVAL;
    if (k->shape[0] < 1 || k->shape[1] < 1 || k->shape[2] < 1 || k->z_begin < 0 || k->z_end > k->shape[2] ||
        k->z_begin > k->z_end)
        return LBM_EINVAL;
    if ((double)k->shape[0] * k->shape[1] * (k->shape[2] + 2 * k->ghost) >= 2147483647.0) return LBM_EINVAL;
    if (aa && k->ghost) return LBM_EUNSUPPORTED;
    std::memset(&a, 0, sizeof(a));
    a.geo.nx = (int)k->shape[0];
    a.geo.ny = (int)k->shape[1];
    a.geo.nz = (int)k->shape[2];
    a.geo.g = k->ghost;
    a.geo.Sq = k->shape[0] * k->shape[1] * (k->shape[2] + 2 * k->ghost);
    a.z_begin = (int)k->z_begin;
    a.z_step = 1;
    a.x0 = 0;
    a.x1 = (int)k->shape[0];
    a.y0 = 0;
    a.y1 = (int)k->shape[1];
    for (int i = 0; i < 8; ++i) a.rates[i] = k->rates[i];
    if (k->collision == LBM_SRT) a.rates[1] = a.rates[0];
    if (k->collision == LBM_MRT || k->collision == LBM_GEN_MRT)
        for (int i = 0; i < 4; ++i)
            if (a.rates[i] == 0.0) a.rates[i] = 1.0;
    if (k->collision == LBM_CUMULANT)
        for (int i = 1; i < 6; ++i)
            if (a.rates[i] == 0.0) a.rates[i] = 1.0;
    for (int d = 0; d < 3; ++d) {
        a.F[d] = k->force[d];
        a.uw[d] = k->ubb_velocity[d];
    }
    a.flags = k->flags;
    return LBM_OK;
}

static dim3 kernel_block(int64_t nx, int64_t ny) { return block_for(nx, ny, 0); }

int lbm_kernel_pull(const lbm_kernel_args *k) {
    StepArgs a;
    int rc = kernel_args_common(k, a, false);
    if (rc) return rc;
    const bool flags = k->flags != nullptr;
    const bool force = k->force[0] != 0 || k->force[1] != 0 || k->force[2] != 0;
    const PullLaunch fn = select_kernels(k->collision, k->stencil, k->dtype, flags ? FM_INLINE : FM_NONE, force, k->equilibrium).pull;
    if (!fn) return LBM_EUNSUPPORTED;
    if (k->z_end == k->z_begin) return LBM_OK;
    dim3 b = kernel_block(k->shape[0], k->shape[1]);
    flat_rows(a, b, k->shape[0], k->shape[1]);
    const dim3 grid = box_grid(a, b, (int)(k->z_end - k->z_begin));
    fn(a, k->src, k->dst, grid, b, static_cast<cudaStream_t>(k->stream));
    return cudaGetLastError() == cudaSuccess ? LBM_OK : LBM_ECUDA;
}

int lbm_kernel_aa(const lbm_kernel_args *k, int32_t odd) {
    StepArgs a;
    int rc = kernel_args_common(k, a, true);
    if (rc) return rc;
    const bool flags = k->flags != nullptr;
    const bool force = k->force[0] != 0 || k->force[1] != 0 || k->force[2] != 0;
    const AALaunch fn = select_kernels(k->collision, k->stencil, k->dtype, flags ? FM_INLINE : FM_NONE, force, k->equilibrium).aa;
    if (!fn) return LBM_EUNSUPPORTED;
    if (k->z_end == k->z_begin) return LBM_OK;
    dim3 b = kernel_block(k->shape[0], k->shape[1]);
    flat_rows(a, b, k->shape[0], k->shape[1]);
    const dim3 grid = box_grid(a, b, (int)(k->z_end - k->z_begin));
    fn(a, k->dst, odd ? 1 : 0, grid, b, static_cast<cudaStream_t>(k->stream));
    return cudaGetLastError() == cudaSuccess ? LBM_OK : LBM_ECUDA;
}

int lbm_kernel_push(const lbm_kernel_args *k) {
    StepArgs a;
    int rc = kernel_args_common(k, a, false);
    if (rc) return rc;
    const bool flags = k->flags != nullptr;
    const bool force = k->force[0] != 0 || k->force[1] != 0 || k->force[2] != 0;
    const PullLaunch fn = select_kernels(k->collision, k->stencil, k->dtype, flags ? FM_INLINE : FM_NONE, force, k->equilibrium).push;
    if (!fn) return LBM_EUNSUPPORTED;
    if (k->z_end == k->z_begin) return LBM_OK;
    dim3 b = kernel_block(k->shape[0], k->shape[1]);
    flat_rows(a, b, k->shape[0], k->shape[1]);
    const dim3 grid = box_grid(a, b, (int)(k->z_end - k->z_begin));
    fn(a, k->src, k->dst, grid, b, static_cast<cudaStream_t>(k->stream));
    return cudaGetLastError() == cudaSuccess ? LBM_OK : LBM_ECUDA;
}

int lbm_kernel_collide(const lbm_kernel_args *k) {
    StepArgs a;
    int rc = kernel_args_common(k, a, true);
    if (rc) return rc;
    const bool flags = k->flags != nullptr;
    const bool force = k->force[0] != 0 || k->force[1] != 0 || k->force[2] != 0;
    const AALaunch fn = select_kernels(k->collision, k->stencil, k->dtype, flags ? FM_INLINE : FM_NONE, force, k->equilibrium).collide;
    if (!fn) return LBM_EUNSUPPORTED;
    if (k->z_end == k->z_begin) return LBM_OK;
    dim3 b = kernel_block(k->shape[0], k->shape[1]);
    flat_rows(a, b, k->shape[0], k->shape[1]);
    const dim3 grid = box_grid(a, b, (int)(k->z_end - k->z_begin));
    fn(a, k->dst, 0, grid, b, static_cast<cudaStream_t>(k->stream));
    return cudaGetLastError() == cudaSuccess ? LBM_OK : LBM_ECUDA;
}

int lbm_prepare_flags(const uint8_t *host_flags, int64_t nx, int64_t ny, int64_t nplanes, int32_t ghost,
                      uint8_t *device_out, void *stream) {
    if (!host_flags || !device_out || nx < 1 || ny < 1 || nplanes < 1 || ghost < 0 || ghost > 1) return LBM_EINVAL;
    const size_t cells = (size_t)nx * ny * nplanes;
    uint8_t *tmp = nullptr;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    if (cudaMalloc(&tmp, cells) != cudaSuccess) return LBM_EOOM;
    Geo g;
    g.nx = (int)nx;
    g.ny = (int)ny;
    g.nz = (int)(nplanes - 2 * ghost);
    g.g = ghost;
    g.Sq = (int64_t)cells;
    if (cudaMemcpyAsync(tmp, host_flags, cells, cudaMemcpyHostToDevice, st) != cudaSuccess) {
        cudaFree(tmp);
        return LBM_ECUDA;
    }
    launch_mark_near_wall(g, (int)nplanes, tmp, device_out, st);
    const cudaError_t e = cudaStreamSynchronize(st);
    cudaFree(tmp);
    return e == cudaSuccess ? LBM_OK : LBM_ECUDA;
}

int lbm_buffer_sizes(const lbm_config *cfg, int64_t out[3]) {
    if (!out) return LBM_EINVAL;
    const int rc = validate(cfg);
    if (rc) return rc;
    const int P = cfg->nranks > 1 ? cfg->nranks : (cfg->n_local_slabs > 1 ? cfg->n_local_slabs : 1);
    const bool exch = P > 1 || cfg->nccl_self;
    const int64_t g = exch ? 1 : 0;
    const int64_t planes = cfg->global[2] / P + 2 * g;
    const int64_t esize = cfg->dtype == LBM_F64 ? 8 : 4;
    const int64_t plane = cfg->global[0] * cfg->global[1];
    out[0] = plane * planes * cfg->stencil * esize;
    out[1] = cfg->flags ? plane * planes : 0;
    out[2] = exch ? 4 * plane * (cfg->stencil == 19 ? 5 : 9) * esize : 0;
    return LBM_OK;
}

int lbm_slab_plan(int64_t nz, int32_t nranks, int32_t rank, int64_t out[4]) {
    if (nranks < 1 || rank < 0 || rank >= nranks || nz % nranks != 0 || (nranks > 1 && nz / nranks < 2)) return LBM_EINVAL;
    const int64_t nzl = nz / nranks;
    out[0] = rank * nzl;
    out[1] = nzl;
    out[2] = (rank - 1 + nranks) % nranks;
    out[3] = (rank + 1) % nranks;
    return LBM_OK;
}

int lbm_crossing_directions(int32_t stencil, int32_t dir, int32_t *q_out) {
    if ((stencil != 19 && stencil != 27) || (dir != 1 && dir != -1)) return LBM_EINVAL;
    int tmp[9];
    const int n = crossing(stencil, dir, tmp);
    for (int i = 0; i < n; ++i) q_out[i] = tmp[i];
    return n;
}

int lbm_halo_schedule(int32_t stencil, int64_t nz_local, int32_t rank, int32_t nranks, int32_t *out, int32_t cap) {
    return lbm_halo_schedule_phase(stencil, LBM_PHASE_PULL, nz_local, rank, nranks, out, cap);
}

int lbm_halo_schedule_phase(int32_t stencil, int32_t phase, int64_t nz_local, int32_t rank, int32_t nranks, int32_t *out,
                            int32_t cap) {
    if ((stencil != 19 && stencil != 27) || nranks < 1 || rank < 0 || rank >= nranks || nz_local < 2 || !out ||
        phase < LBM_PHASE_PULL || phase > LBM_PHASE_ESO_AFTER_ODD)
        return LBM_EINVAL;
    const int nz = (int)nz_local;
    const Phase ph = phase == LBM_PHASE_PULL ? phase_pull(nz)
                   : phase == LBM_PHASE_AA_FILL ? phase_aa_fill(nz)
                   : phase == LBM_PHASE_AA_RETURN ? phase_aa_return(nz, false)
                   : phase_eso(nz, phase == LBM_PHASE_ESO_AFTER_ODD, false);
    const auto ops = phase_schedule(stencil, ph, (rank + 1) % nranks, (rank - 1 + nranks) % nranks);
    if ((int)ops.size() > cap) return LBM_EINVAL;
    for (size_t i = 0; i < ops.size(); ++i) {
        out[4 * i + 0] = ops[i].kind;
        out[4 * i + 1] = ops[i].peer;
        out[4 * i + 2] = ops[i].q;
        out[4 * i + 3] = ops[i].zs;
    }
    return (int)ops.size();
}

int lbm_stencil_table(int32_t stencil, int32_t *c_out, double *w_out) {
    if (stencil != 19 && stencil != 27) return LBM_EINVAL;
    for (int q = 0; q < stencil; ++q) {
        for (int d = 0; d < 3; ++d) c_out[3 * q + d] = kC27[q][d];
        w_out[q] = stencil == 19 ? Stencil<19>::w(q) : Stencil<27>::w(q);
    }
    return stencil;
}

int lbm_nccl_unique_id(uint8_t out[128]) {
    ncclUniqueId id;
    if (ncclGetUniqueId(&id) != ncclSuccess) return LBM_ENCCL;
    static_assert(sizeof(id) == 128, "ncclUniqueId is 128 bytes");
    std::memcpy(out, &id, 128);
    return LBM_OK;
}

int lbm_create(const lbm_config *cfg, lbm_handle *out) {
    if (!out) return LBM_EINVAL;
    *out = nullptr;
    int rc = validate(cfg);
    if (rc) return rc;
    std::unique_ptr<lbm_handle_s> hp(new (std::nothrow) lbm_handle_s());
    if (!hp) return LBM_EOOM;
    lbm_handle h = hp.get();
    h->cfg = *cfg;
    h->cfg.flags = nullptr;
    h->cfg.nccl_id = nullptr;
    h->Q = cfg->stencil;
    h->dtype = cfg->dtype;
    h->esize = cfg->dtype == LBM_F64 ? 8 : 4;
    h->op = cfg->collision;
    h->nx = cfg->global[0];
    h->ny = cfg->global[1];
    h->nzg = cfg->global[2];
    h->rank = cfg->nranks > 1 ? cfg->rank : 0;
    h->nranks = cfg->nranks;
    const int P = cfg->nranks > 1 ? cfg->nranks : (cfg->n_local_slabs > 1 ? cfg->n_local_slabs : 1);
    h->use_nccl = cfg->nranks > 1 || cfg->nccl_self;
    h->fused = h->use_nccl && cfg->halo_mode == LBM_HALO_FUSED;
    h->g = (P > 1 || h->use_nccl) ? 1 : 0;
    h->have_flags = cfg->flags != nullptr;
    h->have_force = cfg->force[0] != 0 || cfg->force[1] != 0 || cfg->force[2] != 0;
    h->links = cfg->boundary_mode == LBM_BOUNDARY_LINKS && h->have_flags;
    // index lists folded into the pull / AA update kernels (FM_LINKS); the fused halo keeps the link kernel.
    // Default where it measured at least as fast as the separate link kernel (B200, gpurun_out/r02v): fp64
    // except the D3Q27 AA kernels (Fig. 8 D3Q19 TRT AA 0.876 vs 0.862 of copy BW; C3 D3Q27 cumulant pull 0.950
    // vs 0.947; C3 AA 0.871 vs 0.935; C1 fp32 pull, issue-bound, 0.86 vs 0.965). LBM_LINKS_FUSED=1 / 0 forces.
    const char *lf_env = std::getenv("LBM_LINKS_FUSED");
    const bool lf_pref = cfg->dtype == LBM_F64 && !(cfg->stencil == 27 && cfg->pattern == LBM_AA);
    h->links_fused = h->links && !h->fused && (cfg->pattern == LBM_PULL || cfg->pattern == LBM_AA) &&
                     (lf_env ? lf_env[0] == '1' : lf_pref);
    h->inline_bc = cfg->boundary_mode == LBM_BOUNDARY_INLINE && h->have_flags;

    // kernel selection (SRT = TRT with equal rates); index-list boundaries run the flag-free kernels;
    // flag boundaries on face-aligned walls run the FM_FACES kernels where they measured fastest on the
    // B200: D3Q19 SRT/TRT fp64 pull (C1 fp64 1.024 of copy BW vs 1.008 split / 1.009 index lists). For
    // fp32 (issue-bound: the coordinate tests cost 0.95 -> 0.86), the cumulant (the inline fix-up of the
    // near-wall cells: C3 0.87 vs 0.94 index lists) and the AA odd step (Fig. 8 0.79 vs 0.81 staged split)
    // the split / index-list kernels stay. LBM_FACES=1 / 0 forces it on / off.
    const char *faces_env = std::getenv("LBM_FACES");
    const bool face_op = cfg->collision == LBM_SRT || cfg->collision == LBM_TRT ||
                         ((cfg->collision == LBM_GEN_SRT || cfg->collision == LBM_GEN_TRT) && cfg->stencil == 19);
    const bool face_pref = cfg->stencil == 19 && cfg->dtype == LBM_F64 && cfg->pattern == LBM_PULL;
    const bool face_force = faces_env && faces_env[0] == '1';
    h->faces = cfg->boundary_mode == LBM_BOUNDARY_FLAGS && h->have_flags && face_op &&
               (cfg->pattern == LBM_PULL || cfg->pattern == LBM_AA) && (face_pref || face_force) &&
               !(faces_env && faces_env[0] == '0') && detect_faces(cfg, h->base_face);
    const int fm_bulk = !h->have_flags ? FM_NONE : h->links ? (h->links_fused ? FM_LINKS : FM_NONE)
                      : h->inline_bc ? FM_INLINE : h->faces ? FM_FACES : FM_BULK;
    const bool per_row = cfg->collision == LBM_MRT && cfg->n_row_rates == 15;
    // D3Q27 cumulant whose bulk and higher-order rates are all 1 (C3, G7): the specialised kernels that
    // skip the relaxations with factor 1 - omega = 0 (collide_cumulant27_unit)
    bool unit_rates = cfg->collision == LBM_CUMULANT && cfg->stencil == 27 && cfg->equilibrium == LBM_EQ_COMPRESSIBLE &&
                      std::getenv("LBM_CUMULANT_GENERAL") == nullptr;
    for (int i = 1; i < 6 && unit_rates; ++i) unit_rates = i >= cfg->n_rates || cfg->rates[i] == 1.0;
    // D3Q19 weighted MRT with bulk / order-3 / order-4 rates 1 (C2): only the shear group relaxes
    // (collide_mrt_shear, the G6 closed form)
    bool shear_only = cfg->collision == LBM_MRT && !per_row && cfg->stencil == 19 &&
                      cfg->equilibrium == LBM_EQ_COMPRESSIBLE && std::getenv("LBM_MRT_GENERAL") == nullptr;
    for (int i = 1; i < 4 && shear_only; ++i) shear_only = i >= cfg->n_rates || cfg->rates[i] == 1.0;
    const int kcoll = per_row ? (int)OP_MRT_ROWS : unit_rates ? (int)OP_CUMULANT_UNIT
                    : shear_only ? (int)OP_MRT_SHEAR : cfg->collision;
    const bool force = h->have_force;
    if (cfg->pattern == LBM_PULL || cfg->pattern == LBM_PUSH) {
        h->kern = select_kernels(kcoll, h->Q, h->dtype, fm_bulk, force, cfg->equilibrium);
        if (!(cfg->pattern == LBM_PUSH ? (void *)h->kern.push : (void *)h->kern.pull)) return fail(nullptr, LBM_EUNSUPPORTED, "no kernel instantiated for this combination");
    } else {
        h->kern = select_kernels(kcoll, h->Q, h->dtype, fm_bulk, force, cfg->equilibrium);
        if (!(cfg->pattern == LBM_ESOTWIST ? (void *)h->kern.eso : (void *)h->kern.aa))
            return fail(nullptr, LBM_EUNSUPPORTED, "no kernel instantiated for this combination");
    }
    if (h->links_fused) {
        // the flag-free kernels of the separate link kernel mode, for lbm_set_link_velocities
        h->kern_links = select_kernels(kcoll, h->Q, h->dtype, FM_NONE, force, cfg->equilibrium);
        if (!(cfg->pattern == LBM_PULL ? (void *)h->kern_links.pull : (void *)h->kern_links.aa))
            return fail(nullptr, LBM_EUNSUPPORTED, "no kernel instantiated for this combination");
    }
    // rates into the kernel argument block
    StepArgs &b = h->base;
    std::memset(&b, 0, sizeof(b));
    for (int i = 0; i < 8; ++i) b.rates[i] = cfg->rates[i];
    if (per_row)
        for (int i = 0; i < 15; ++i) b.rates[i] = cfg->row_rates[i];
    if (cfg->collision == LBM_SRT) b.rates[1] = b.rates[0];
    if ((cfg->collision == LBM_MRT && !per_row) || cfg->collision == LBM_GEN_MRT)
        for (int i = cfg->n_rates; i < 4; ++i) b.rates[i] = 1.0;
    if (cfg->collision == LBM_CUMULANT)
        for (int i = cfg->n_rates; i < 6; ++i) b.rates[i] = 1.0;  // higher orders default to 1 (G7)
    for (int d = 0; d < 3; ++d) {
        b.F[d] = cfg->force[d];
        b.uw[d] = cfg->ubb_velocity[d];
    }
    for (int f = 0; f < 6; ++f) b.face[f] = h->faces ? h->base_face[f] : 0;
    b.nzg = (int)h->nzg;
    // launch box: the bounding box of the non-wall cells of the flag field (walls on the domain faces get no
    // threads; LBM_BOX=0 launches the whole plane), interior planes with non-wall cells per slab below
    b.x0 = 0;
    b.x1 = (int)h->nx;
    b.y0 = 0;
    b.y1 = (int)h->ny;
    std::vector<char> plane_fluid(h->nzg, 1);
    const char *box_env = std::getenv("LBM_BOX");
    // (not for the inline mode: Fig. 8 inline 0.867 -> 0.842 with the box, three repetitions each; walled
    // configs otherwise +0.4 to +0.8 %: C1 fp32 0.960 -> 0.968, C3-AA links 0.935 -> 0.943; scripts/gpu_r02z10.sh)
    if (h->have_flags && !h->inline_bc && !(box_env && box_env[0] == '0')) {
        int64_t x0 = h->nx, x1 = -1, y0 = h->ny, y1 = -1;
        const int64_t pl = h->nx * h->ny;
        for (int64_t z = 0; z < h->nzg; ++z) {
            bool any = false;
            for (int64_t y = 0; y < h->ny; ++y) {
                const uint8_t *row = cfg->flags + z * pl + y * h->nx;
                int64_t first = -1, last = -1;
                for (int64_t x = 0; x < h->nx; ++x)
                    if ((row[x] & 3) == 0) {
                        if (first < 0) first = x;
                        last = x;
                    }
                if (first < 0) continue;
                any = true;
                x0 = std::min(x0, first);
                x1 = std::max(x1, last);
                y0 = std::min(y0, y);
                y1 = std::max(y1, y);
            }
            plane_fluid[z] = any;
        }
        if (x1 >= 0) {
            // x starts on a 32-cell boundary: a warp's 32 cells keep their aligned 128 / 256 B segments (a box
            // starting at x = 1 misaligned every warp of the C3 cavity: 0.95 -> 0.90 of copy BW)
            b.x0 = (int)(x0 / 32 * 32);
            b.x1 = (int)x1 + 1;
            b.y0 = (int)y0;
            b.y1 = (int)y1 + 1;
        }
    }
    h->block = cfg->block_x > 0 ? block_for(h->nx, h->ny, cfg->block_x) : block_for(h->nx, h->ny, 0);
    if (cfg->block_x <= 0) flat_rows(b, h->block, h->nx, h->ny);  // (a forced block_x keeps the 2-D blocks)

    CUDA_TRY(nullptr, cudaSetDevice(cfg->device));
    if (cfg->stream) {
        h->stream = static_cast<cudaStream_t>(cfg->stream);
    } else {
        CUDA_TRY(nullptr, cudaStreamCreateWithFlags(&h->stream, cudaStreamNonBlocking));
        h->own_stream = true;
    }
    hp.release();  // from here on, lbm_destroy cleans up
    auto bail = [&](int code) {
        std::string m = h->err;
        lbm_destroy(h);
        g_create_error = m;
        return code;
    };
    // the comm stream gets the highest priority: the NCCL kernels of the halo exchange are scheduled on SMs as
    // soon as interior-update blocks retire instead of queueing behind the whole interior launch
    int prio_lo = 0, prio_hi = 0;
    cudaDeviceGetStreamPriorityRange(&prio_lo, &prio_hi);
    if (cudaStreamCreateWithPriority(&h->comm_stream, cudaStreamNonBlocking, prio_hi) != cudaSuccess ||
        cudaEventCreateWithFlags(&h->ev_bnd, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&h->ev_x, cudaEventDisableTiming) != cudaSuccess) {
        h->err = "stream/event creation failed";
        return bail(LBM_ECUDA);
    }
    if (per_row && mrt_rows_upload() != 0) {
        h->err = "per-moment MRT rows: constant upload failed";
        return bail(LBM_ECUDA);
    }
    if (cudaMalloc(&h->d_nanflag, sizeof(int)) != cudaSuccess) {
        h->err = "cudaMalloc nan flag";
        return bail(LBM_EOOM);
    }

    // slabs
    const int nloc = cfg->nranks > 1 ? 1 : P;
    const int64_t nzl = h->nzg / P;
    h->slabs.resize(nloc);
    for (int i = 0; i < nloc; ++i) {
        Slab &s = h->slabs[i];
        const int slab_index = cfg->nranks > 1 ? cfg->rank : i;
        s.z0 = slab_index * nzl;
        s.nz = (int)nzl;
        s.zlo = 0;  // first / last interior planes with non-wall cells
        while (s.zlo < s.nz && !plane_fluid[s.z0 + s.zlo]) ++s.zlo;
        s.zhi = s.nz;
        while (s.zhi > s.zlo && !plane_fluid[s.z0 + s.zhi - 1]) --s.zhi;
        const Geo g = geo_of(h, s);
        const size_t bytes = (size_t)g.Sq * h->Q * h->esize;
        for (int a = 0; a < (two_arrays(h) ? 2 : 1); ++a) {
            if (h->fused) break;  // allocated in NCCL symmetric memory below
            if (cfg->pdf_dev[a]) {  // borrowed (e.g. a torch tensor): used in place, never freed
                s.pdf[a] = cfg->pdf_dev[a];
                s.own_pdf[a] = false;
            } else if (cudaMalloc(&s.pdf[a], bytes) != cudaSuccess) {
                h->err = "cudaMalloc populations (" + std::to_string(bytes) + " B)";
                return bail(LBM_EOOM);
            }
            cudaMemsetAsync(s.pdf[a], 0, bytes, h->stream);
        }
        if (h->g) {
            const size_t hb = (size_t)h->nx * h->ny * (h->Q == 19 ? 5 : 9) * h->esize;
            for (int k = 0; k < 4; ++k) {
                if (cfg->halo_dev) {
                    s.halo[k] = static_cast<char *>(cfg->halo_dev) + k * hb;
                    s.own_halo = false;
                } else if (cudaMalloc(&s.halo[k], hb) != cudaSuccess) {
                    h->err = "cudaMalloc halo";
                    return bail(LBM_EOOM);
                }
            }
        }
        if (h->have_flags) {
            const int nplanes = s.nz + 2 * h->g;
            const size_t cells = (size_t)h->nx * h->ny * nplanes;
            std::vector<uint8_t> hf(cells);
            for (int zs = 0; zs < nplanes; ++zs) {
                int64_t zg = s.z0 + zs - h->g;
                zg = ((zg % h->nzg) + h->nzg) % h->nzg;
                std::memcpy(&hf[(size_t)zs * h->nx * h->ny], cfg->flags + (size_t)zg * h->nx * h->ny, (size_t)h->nx * h->ny);
            }
            uint8_t *tmp = nullptr;
            if (cfg->flags_dev) {
                s.flags = cfg->flags_dev;
                s.own_flags = false;
            } else if (cudaMalloc(&s.flags, cells) != cudaSuccess) {
                h->err = "cudaMalloc flags";
                return bail(LBM_EOOM);
            }
            if (cudaMalloc(&tmp, cells) != cudaSuccess) {
                h->err = "cudaMalloc flags";
                return bail(LBM_EOOM);
            }
            cudaMemcpy(tmp, hf.data(), cells, cudaMemcpyHostToDevice);
            launch_mark_near_wall(g, nplanes, tmp, s.flags, h->stream);
            cudaStreamSynchronize(h->stream);
            cudaFree(tmp);
            // near-wall fluid cells of the interior planes, in storage order, for the edge kernels
            cudaMemcpy(hf.data(), s.flags, cells, cudaMemcpyDeviceToHost);
            std::vector<uint32_t> list;
            s.edge_off.assign(nplanes + 1, 0);
            const size_t plane = (size_t)h->nx * h->ny;
            for (int zs = 0; zs < nplanes; ++zs) {
                s.edge_off[zs] = (int64_t)list.size();
                if (zs >= h->g && zs < h->g + s.nz)
                    for (size_t i = 0; i < plane; ++i)
                        if (hf[zs * plane + i] == 0x80) list.push_back((uint32_t)(zs * plane + i));
            }
            s.edge_off[nplanes] = (int64_t)list.size();
            if (!list.empty()) {
                if (cudaMalloc(&s.edges, list.size() * sizeof(uint32_t)) != cudaSuccess) {
                    h->err = "cudaMalloc edge list";
                    return bail(LBM_EOOM);
                }
                cudaMemcpy(s.edges, list.data(), list.size() * sizeof(uint32_t), cudaMemcpyHostToDevice);
            }
            if (h->links) {
                // one entry per boundary link: wall cell b (any storage plane, ghosts included), direction q
                // with b + c_q a fluid cell of this slab's interior (x, y wrap; z wraps without ghost planes),
                // grouped by direction q, storage order of b within a direction, so that consecutive threads of
                // the link kernel touch consecutive cells of one q-plane. A link is listed by the
                // slab owning its fluid cell.
                std::vector<uint32_t> lf, walls;
                for (size_t b = 0; b < (size_t)nplanes * plane; ++b)
                    if (hf[b] & 3) walls.push_back((uint32_t)b);
                for (int q = 1; q < h->Q; ++q)
                    for (const uint32_t b : walls) {
                        const int64_t zs = b / plane, y = (b % plane) / h->nx, x = b % h->nx;
                        int64_t zz = zs + kC27[q][2];
                        if (h->g == 0) zz = (zz + s.nz) % s.nz;
                        else if (zz < h->g || zz >= h->g + s.nz) continue;  // fluid cell not in this slab
                        const int64_t xx = (x + kC27[q][0] + h->nx) % h->nx, yy = (y + kC27[q][1] + h->ny) % h->ny;
                        const size_t nb = ((size_t)zz * h->ny + yy) * h->nx + xx;
                        if (hf[nb] & 3) continue;
                        s.h_link_wall.push_back(b);
                        if (cfg->pattern == LBM_ESOTWIST) {
                            // EsoTwist: the link's populations live at L = b + c_q^- (= x - c_q^+, G23), the
                            // location the fix works on (x, y wrap; z stays inside the storage planes)
                            int64_t lz = zs + (kC27[q][2] < 0 ? kC27[q][2] : 0);
                            if (h->g == 0) lz = (lz + s.nz) % s.nz;
                            const int64_t lx = (x + (kC27[q][0] < 0 ? -1 : 0) + h->nx) % h->nx;
                            const int64_t ly = (y + (kC27[q][1] < 0 ? -1 : 0) + h->ny) % h->ny;
                            lf.push_back((uint32_t)(((size_t)lz * h->ny + ly) * h->nx + lx));
                        } else {
                            lf.push_back((uint32_t)nb);
                        }
                        s.h_link_dir.push_back((uint8_t)q);
                        s.h_link_type.push_back(hf[b] & 3);
                    }
                const size_t n = s.h_link_wall.size();
                if (n) {
                    if (cudaMalloc(&s.link_wall, n * 4) != cudaSuccess || cudaMalloc(&s.link_fluid, n * 4) != cudaSuccess ||
                        cudaMalloc(&s.link_dir, n) != cudaSuccess || cudaMalloc(&s.link_term, n * 8) != cudaSuccess) {
                        h->err = "cudaMalloc link list";
                        return bail(LBM_EOOM);
                    }
                    cudaMemcpy(s.link_wall, s.h_link_wall.data(), n * 4, cudaMemcpyHostToDevice);
                    cudaMemcpy(s.link_fluid, lf.data(), n * 4, cudaMemcpyHostToDevice);
                    cudaMemcpy(s.link_dir, s.h_link_dir.data(), n, cudaMemcpyHostToDevice);
                    if (h->links_fused) {
                        // per-cell link masks of the links whose wall cell is in this slab's interior (the
                        // update kernels store them); the others (wall in a ghost plane) stay in a residual list
                        std::vector<uint64_t> mask(cells, 0);
                        std::vector<uint32_t> rw, rf;
                        std::vector<uint8_t> rd;
                        for (size_t i = 0; i < n; ++i) {
                            const int64_t zb = s.h_link_wall[i] / (int64_t)plane;
                            const int q = s.h_link_dir[i];
                            if (h->g == 0 || (zb >= h->g && zb < h->g + s.nz)) {
                                mask[lf[i]] |= 1ull << q;
                                if (s.h_link_type[i] == LBM_FLAG_UBB) mask[lf[i]] |= 1ull << (32 + q);
                            } else {
                                s.h_res_idx.push_back((uint32_t)i);
                                rw.push_back(s.h_link_wall[i]);
                                rf.push_back(lf[i]);
                                rd.push_back((uint8_t)q);
                            }
                        }
                        s.n_res = (uint32_t)rw.size();
                        if (cudaMalloc(&s.lmask, cells * sizeof(uint64_t)) != cudaSuccess) {
                            h->err = "cudaMalloc link masks";
                            return bail(LBM_EOOM);
                        }
                        cudaMemcpy(s.lmask, mask.data(), cells * sizeof(uint64_t), cudaMemcpyHostToDevice);
                        if (s.n_res) {
                            const size_t r = s.n_res;
                            if (cudaMalloc(&s.res_wall, r * 4) != cudaSuccess || cudaMalloc(&s.res_fluid, r * 4) != cudaSuccess ||
                                cudaMalloc(&s.res_dir, r) != cudaSuccess || cudaMalloc(&s.res_term, r * 8) != cudaSuccess) {
                                h->err = "cudaMalloc residual link list";
                                return bail(LBM_EOOM);
                            }
                            cudaMemcpy(s.res_wall, rw.data(), r * 4, cudaMemcpyHostToDevice);
                            cudaMemcpy(s.res_fluid, rf.data(), r * 4, cudaMemcpyHostToDevice);
                            cudaMemcpy(s.res_dir, rd.data(), r, cudaMemcpyHostToDevice);
                        }
                    }
                    std::vector<double> uw(3 * n);
                    for (size_t i = 0; i < n; ++i)
                        for (int d = 0; d < 3; ++d) uw[3 * i + d] = cfg->ubb_velocity[d];
                    upload_link_terms(h, s, uw.data());
                }
            }
        }
    }
    if (h->use_nccl) {
        int64_t plan[4];
        lbm_slab_plan(h->nzg, cfg->nranks, h->rank, plan);
        h->down = (int)plan[2];
        h->up = (int)plan[3];
        ncclUniqueId id;
        if (cfg->nranks > 1) {
            std::memcpy(&id, cfg->nccl_id, sizeof(id));
        } else if (ncclGetUniqueId(&id) != ncclSuccess) {  // 1-rank self-exchange communicator
            h->err = "ncclGetUniqueId failed";
            return bail(LBM_ENCCL);
        }
        ncclResult_t r = ncclCommInitRank(&h->comm, cfg->nranks, id, h->rank);
        if (r != ncclSuccess) {
            h->err = std::string("ncclCommInitRank: ") + ncclGetErrorString(r);
            return bail(LBM_ENCCL);
        }
        if (h->fused) {
            Slab &s = h->slabs[0];
            const size_t bytes = (size_t)geo_of(h, s).Sq * h->Q * h->esize;
            for (int a = 0; a < (two_arrays(h) ? 2 : 1); ++a) {
                if ((r = ncclMemAlloc(&s.pdf[a], bytes)) != ncclSuccess) {
                    h->err = std::string("ncclMemAlloc populations: ") + ncclGetErrorString(r);
                    return bail(LBM_EOOM);
                }
                cudaMemsetAsync(s.pdf[a], 0, bytes, h->stream);
            }
            std::string err;
            if (fused_setup(h->comm, s.pdf[0], s.pdf[1], bytes, h->up, h->down, &h->fst, h->stream, err)) {
                h->err = "fused halo: " + err;
                return bail(LBM_ENCCL);
            }
        }
    }
    cudaError_t e = cudaStreamSynchronize(h->stream);
    if (e != cudaSuccess) {
        h->err = std::string("create: ") + cudaGetErrorString(e);
        return bail(LBM_ECUDA);
    }
    *out = h;
    return LBM_OK;
}

int lbm_destroy(lbm_handle h) {
    if (!h) return LBM_OK;
    if (h->stream) cudaStreamSynchronize(h->stream);
    if (h->comm_stream) cudaStreamSynchronize(h->comm_stream);
    free_async(h);
    if (h->graph) cudaGraphExecDestroy(h->graph);
    if (h->fused && h->comm) fused_teardown(h->comm, &h->fst);
    for (Slab &s : h->slabs) {
        for (int a = 0; a < 2; ++a)
            if (s.pdf[a] && s.own_pdf[a]) {
                if (h->fused) ncclMemFree(s.pdf[a]);
                else cudaFree(s.pdf[a]);
            }
        if (s.own_halo)
            for (void *p : s.halo) if (p) cudaFree(p);
        if (s.flags && s.own_flags) cudaFree(s.flags);
        if (s.edges) cudaFree(s.edges);
        for (void *p : {(void *)s.link_wall, (void *)s.link_fluid, (void *)s.link_dir, (void *)s.link_term, (void *)s.lmask,
                        (void *)s.res_wall, (void *)s.res_fluid, (void *)s.res_dir, (void *)s.res_term})
            if (p) cudaFree(p);
    }
    if (h->comm) ncclCommDestroy(h->comm);
    for (cudaEvent_t e : h->timing.ev) cudaEventDestroy(e);
    for (cudaEvent_t e : h->timing.ph) if (e) cudaEventDestroy(e);
    if (h->ev_bnd) cudaEventDestroy(h->ev_bnd);
    if (h->ev_x) cudaEventDestroy(h->ev_x);
    if (h->comm_stream) cudaStreamDestroy(h->comm_stream);
    if (h->own_stream && h->stream) cudaStreamDestroy(h->stream);
    if (h->d_nanflag) cudaFree(h->d_nanflag);
    if (h->scratch) cudaFree(h->scratch);
    delete h;
    return LBM_OK;
}

int lbm_detect_faces(const lbm_config *cfg, int8_t face_out[6]) {
    if (!cfg || !face_out) return LBM_EINVAL;
    const int rc = validate(cfg);
    if (rc) return rc;
    if (!cfg->flags) return 0;
    return detect_faces(cfg, face_out) ? 1 : 0;
}

int lbm_boundary_impl(lbm_handle h) {
    if (!h) return LBM_EINVAL;
    if (!h->have_flags) return LBM_IMPL_NONE;
    if (h->links) return h->links_fused ? LBM_IMPL_LINKS_FUSED : LBM_IMPL_LINKS;
    if (h->inline_bc) return LBM_IMPL_INLINE;
    return h->faces ? LBM_IMPL_FACES : LBM_IMPL_SPLIT;
}

int lbm_local_extent(lbm_handle h, int64_t out[4]) {
    if (!h || !out) return LBM_EINVAL;
    int64_t nz = 0;
    for (const Slab &s : h->slabs) nz += s.nz;
    out[0] = h->slabs[0].z0;
    out[1] = nz;
    out[2] = h->nx;
    out[3] = h->ny;
    return LBM_OK;
}

static int init_common(lbm_handle h, InitArgs &a, const double *rho, const double *u, int where) {
    const int64_t cells = local_cells(h);
    const double *drho = rho, *du = u;
    int async_k = -1;
    if (a.mode == 0) {
        if (!rho || !u) return fail(h, LBM_EINVAL, "null rho/u");
        if (where == LBM_HOST_ASYNC) {
            // upload on the h2d stream into a staging buffer no earlier init still reads; the compute stream
            // waits for the upload only (earlier steps and downloads keep running)
            int rc = ensure_async(h);
            if (rc) return rc;
            auto &io = h->aio;
            async_k = io.in_k;
            io.in_k ^= 1;
            CUDA_TRY(h, cudaStreamWaitEvent(io.h2d, io.in_free[async_k], 0));
            CUDA_TRY(h, cudaMemcpyAsync(io.in[async_k], rho, cells * sizeof(double), cudaMemcpyHostToDevice, io.h2d));
            CUDA_TRY(h, cudaMemcpyAsync(io.in[async_k] + cells, u, 3 * cells * sizeof(double), cudaMemcpyHostToDevice, io.h2d));
            CUDA_TRY(h, cudaEventRecord(io.in_ready[async_k], io.h2d));
            CUDA_TRY(h, cudaStreamWaitEvent(h->stream, io.in_ready[async_k], 0));
            drho = io.in[async_k];
            du = io.in[async_k] + cells;
        } else if (where == LBM_HOST) {
            int rc = ensure_scratch(h, (size_t)cells * 4 * sizeof(double));
            if (rc) return rc;
            CUDA_TRY(h, cudaMemcpyAsync(h->scratch, rho, cells * sizeof(double), cudaMemcpyHostToDevice, h->stream));
            CUDA_TRY(h, cudaMemcpyAsync(h->scratch + cells, u, 3 * cells * sizeof(double), cudaMemcpyHostToDevice, h->stream));
            drho = h->scratch;
            du = h->scratch + cells;
        }
    }
    int64_t off = 0;
    for (Slab &s : h->slabs) {
        InitArgs b = a;
        b.geo = geo_of(h, s);
        b.z0 = s.z0;
        b.nx_g = h->nx;
        b.ny_g = h->ny;
        b.nz_g = h->nzg;
        b.product_eq = h->op == LBM_CUMULANT;
        b.eq_kind = h->cfg.equilibrium;
        b.eso = h->cfg.pattern == LBM_ESOTWIST;
        if (a.mode == 0) {
            // the arrays cover the concatenated local slabs; ghost planes are filled by exchange
            b.rho = drho + off;
            b.u = du + off;
            b.ustride = cells;
            b.zlo = h->g;
            b.zhi = h->g + s.nz;
        } else if (b.eso) {
            b.zlo = h->g;  // EsoTwist: each interior cell writes its arriving populations (lower ghost included)
            b.zhi = h->g + s.nz;
        } else {
            b.zlo = 0;  // random init is keyed by the global index: ghost planes computed directly
            b.zhi = s.nz + 2 * h->g;
        }
        off += (int64_t)h->nx * h->ny * s.nz;
        const dim3 grid((unsigned)((h->nx + 31) / 32), (unsigned)((h->ny + 7) / 8), (unsigned)(b.zhi - b.zlo));
        launch_init(h->Q, h->dtype, b, s.pdf[0], s.pdf[1], grid, dim3(32, 8, 1), h->stream);
        h->launches++;
        s.cur = 0;
    }
    h->steps = 0;
    h->aa_parity = 0;
    h->links_pending = -1;
    links_unprime(h);
    if (a.mode == 0 && h->g) {
        int rc = exchange_current(h);
        if (rc) return rc;
        for (Slab &s : h->slabs)
            if (s.pdf[1]) {
                const Geo g = geo_of(h, s);
                CUDA_TRY(h, cudaMemcpyAsync(s.pdf[1], s.pdf[0], (size_t)g.Sq * h->Q * h->esize, cudaMemcpyDeviceToDevice, h->stream));
            }
    }
    if (async_k >= 0) {  // the staging buffer is free again once the init kernels have read it; no host wait
        CUDA_TRY(h, cudaEventRecord(h->aio.in_free[async_k], h->stream));
        return LBM_OK;
    }
    CUDA_TRY(h, cudaStreamSynchronize(h->stream));
    return LBM_OK;
}

int lbm_init_equilibrium(lbm_handle h, const double *rho, const double *u, int32_t where) {
    if (!h) return LBM_EINVAL;
    InitArgs a;
    std::memset(&a, 0, sizeof(a));
    a.mode = 0;
    return init_common(h, a, rho, u, where);
}

int lbm_init_random(lbm_handle h, uint64_t seed, double rho_amp, double u_amp, int32_t profile, double profile_amp) {
    if (!h) return LBM_EINVAL;
    InitArgs a;
    std::memset(&a, 0, sizeof(a));
    a.mode = 1;
    a.seed = seed;
    a.rho_amp = rho_amp;
    a.u_amp = u_amp;
    a.profile = profile;
    a.profile_amp = profile_amp;
    return init_common(h, a, nullptr, nullptr, LBM_DEVICE);
}

static int nccl_async_status(lbm_handle h);

int lbm_step(lbm_handle h, int64_t n) {
    if (!h || n < 0) return LBM_EINVAL;
    cudaError_t pending = cudaGetLastError();
    if (pending != cudaSuccess) return fail(h, LBM_ECUDA, std::string("pending: ") + cudaGetErrorString(pending));
    if (int rc = nccl_async_status(h)) return rc;
    if (h->timing.on) {
        for (cudaEvent_t e : h->timing.ev) cudaEventDestroy(e);
        h->timing.ev.clear();
    }
    if (n > 0) links_prime(h, h->stream);
    int64_t done = 0;
    const int every = h->cfg.check_nan_every;
    while (done < n) {
        int64_t chunk = n - done;
        if (every > 0) {
            const int64_t to_check = every - (h->steps % every);
            if (chunk > to_check) chunk = to_check;
        }
        int64_t i = 0;
        if (persistent_ok(h) && chunk > 0) {
            // one cooperative launch runs the whole chunk (grid-wide barrier between steps)
            Slab &s = h->slabs[0];
            StepArgs a = h->base;
            a.geo = geo_of(h, s);
            a.z_begin = 0;
            a.z_step = 1;
            a.flags = s.flags;
            const bool aa = h->cfg.pattern == LBM_AA;
            const int phase = aa ? h->aa_parity : s.cur;
            tbegin(h, h->stream);
            const int rc = (aa ? h->kern.persist_aa : h->kern.persist_pull)(a, s.pdf[0], aa ? nullptr : s.pdf[1], phase,
                                                                          (int)chunk, h->stream);
            tend(h, h->stream);
            if (rc) return fail(h, LBM_ECUDA, "persistent cooperative launch failed");
            h->launches++;
            if (chunk & 1) {
                if (aa) h->aa_parity ^= 1;
                else s.cur ^= 1;
            }
            i = chunk;
        }
        if (graph_ok(h)) {
            for (; i + 2 <= chunk; i += 2) {  // a two-step cycle returns the state to the same slots
                int rc = run_graph_cycle(h);
                if (rc) return rc;
            }
        }
        for (; i < chunk; ++i) {
            int rc = step_once(h);
            if (rc) return rc;
        }
        done += chunk;
        h->steps += chunk;
        if (every > 0 && h->steps % every == 0) {
            CUDA_TRY(h, cudaMemsetAsync(h->d_nanflag, 0, sizeof(int), h->stream));
            for (Slab &s : h->slabs) {
                const Geo g = geo_of(h, s);
                launch_nan_check(h->dtype, s.pdf[cur_array(h, s)], g.Sq * h->Q, h->d_nanflag, h->stream);
            }
            int flag = 0;
            CUDA_TRY(h, cudaMemcpyAsync(&flag, h->d_nanflag, sizeof(int), cudaMemcpyDeviceToHost, h->stream));
            CUDA_TRY(h, cudaStreamSynchronize(h->stream));
            if (flag) return fail(h, LBM_ENAN, "NaN detected after step " + std::to_string(h->steps));
        }
    }
    if (h->fused && h->links_pending >= 0) {  // closing gate: the state of the call is complete on return
        fused_gate(h->fst, h->stream);
        h->launches++;
        links_deferred(h, h->slabs[0], h->stream);
    }
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return fail(h, LBM_ECUDA, std::string("launch: ") + cudaGetErrorString(e));
    return LBM_OK;
}

// Asynchronous NCCL failures (a peer died, a network/NVLink error): ncclCommGetAsyncError reports them
// without blocking; surfaced at lbm_step and lbm_sync as LBM_ENCCL.
static int nccl_async_status(lbm_handle h) {
    if (!h->comm) return LBM_OK;
    ncclResult_t async = ncclSuccess;
    NCCL_TRY(h, ncclCommGetAsyncError(h->comm, &async));
    if (async != ncclSuccess && async != ncclInProgress)
        return fail(h, LBM_ENCCL, std::string("NCCL asynchronous error: ") + ncclGetErrorString(async));
    return LBM_OK;
}

int lbm_sync(lbm_handle h) {
    if (!h) return LBM_EINVAL;
    CUDA_TRY(h, cudaStreamSynchronize(h->stream));
    CUDA_TRY(h, cudaStreamSynchronize(h->comm_stream));
    if (h->aio.ready) {
        CUDA_TRY(h, cudaStreamSynchronize(h->aio.h2d));
        CUDA_TRY(h, cudaStreamSynchronize(h->aio.d2h));
    }
    CUDA_TRY(h, cudaGetLastError());
    return nccl_async_status(h);
}

int lbm_step_phases_ms(lbm_handle h, double out[6]) {
    if (!h || !out) return LBM_EINVAL;
    if (!h->timing.ph_valid) return fail(h, LBM_EINVAL, "no timed decomposed step (lbm_kernel_time_ms(h, NULL, NULL) first)");
    CUDA_TRY(h, cudaStreamSynchronize(h->stream));
    CUDA_TRY(h, cudaStreamSynchronize(h->comm_stream));
    for (int k = 0; k < 6; ++k) {
        float t = 0.f;
        CUDA_TRY(h, cudaEventElapsedTime(&t, h->timing.ph[0], h->timing.ph[k]));
        out[k] = t;
    }
    return LBM_OK;
}

// ---- checkpoint / resume ---------------------------------------------------------------
int64_t lbm_state_bytes(lbm_handle h) {
    if (!h) return LBM_EINVAL;
    int64_t n = 0;
    for (const Slab &s : h->slabs) n += geo_of(h, s).Sq * h->Q * h->esize;
    return n;
}

int lbm_save_state(lbm_handle h, void *out, int32_t where, int64_t *steps_done) {
    if (!h || !out) return LBM_EINVAL;
    if (where == LBM_HOST_ASYNC) where = LBM_HOST;  // synchronous call
    const cudaMemcpyKind kind = where == LBM_HOST ? cudaMemcpyDeviceToHost : cudaMemcpyDeviceToDevice;
    char *dst = static_cast<char *>(out);
    for (Slab &s : h->slabs) {
        const size_t b = (size_t)geo_of(h, s).Sq * h->Q * h->esize;
        CUDA_TRY(h, cudaMemcpyAsync(dst, s.pdf[cur_array(h, s)], b, kind, h->stream));
        dst += b;
    }
    CUDA_TRY(h, cudaStreamSynchronize(h->stream));
    if (steps_done) *steps_done = h->steps;
    return LBM_OK;
}

int lbm_load_state(lbm_handle h, const void *in, int32_t where, int64_t steps_done) {
    if (!h || !in || steps_done < 0) return LBM_EINVAL;
    if (where == LBM_HOST_ASYNC) where = LBM_HOST;  // synchronous call
    const cudaMemcpyKind kind = where == LBM_HOST ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToDevice;
    const char *src = static_cast<const char *>(in);
    for (Slab &s : h->slabs) {
        const size_t b = (size_t)geo_of(h, s).Sq * h->Q * h->esize;
        s.cur = 0;
        CUDA_TRY(h, cudaMemcpyAsync(s.pdf[0], src, b, kind, h->stream));
        if (two_arrays(h)) CUDA_TRY(h, cudaMemcpyAsync(s.pdf[1], s.pdf[0], b, cudaMemcpyDeviceToDevice, h->stream));
        src += b;
    }
    h->steps = steps_done;
    h->aa_parity = two_arrays(h) ? 0 : (int)(steps_done & 1);
    h->links_pending = -1;
    links_unprime(h);
    CUDA_TRY(h, cudaStreamSynchronize(h->stream));
    return LBM_OK;
}

int64_t lbm_steps_done(lbm_handle h) { return h ? h->steps : -1; }
int64_t lbm_launch_count(lbm_handle h) { return h ? h->launches : -1; }

int lbm_kernel_time_ms(lbm_handle h, double *ms, int64_t *launches) {
    if (!h) return LBM_EINVAL;
    if (!ms) {  // toggle: lbm_kernel_time_ms(h, NULL, NULL) switches timing on for subsequent steps
        h->timing.on = true;
        return LBM_OK;
    }
    CUDA_TRY(h, cudaStreamSynchronize(h->stream));
    double tot = 0;
    int64_t n = 0;
    for (size_t i = 0; i + 1 < h->timing.ev.size(); i += 2) {
        float t = 0;
        CUDA_TRY(h, cudaEventElapsedTime(&t, h->timing.ev[i], h->timing.ev[i + 1]));
        tot += t;
        ++n;
    }
    *ms = tot;
    if (launches) *launches = n;
    return LBM_OK;
}

static int read_common(lbm_handle h, ReadArgs &r, int raw, const Slab &s) {
    r.raw = raw;
    r.aa_odd = (h->cfg.pattern == LBM_AA) && h->aa_parity;
    r.eso = h->cfg.pattern == LBM_ESOTWIST;
    r.eso_odd = h->aa_parity;
    r.fsign = h->cfg.pattern == LBM_PULL ? -1.0 : 1.0;  // push / AA / EsoTwist hold pre-collision states
    r.incompressible = h->cfg.equilibrium == LBM_EQ_INCOMPRESSIBLE;
    for (int d = 0; d < 3; ++d) {
        r.F[d] = h->cfg.force[d];
        r.uw[d] = h->cfg.ubb_velocity[d];
    }
    r.geo = geo_of(h, s);
    r.flags = h->links ? nullptr : s.flags;  // link mode: the wall slots hold the bounced values
    return LBM_OK;
}

int lbm_get_populations(lbm_handle h, double *out, int32_t where, int32_t raw) {
    if (!h || !out) return LBM_EINVAL;
    if (where == LBM_HOST_ASYNC) where = LBM_HOST;  // synchronous call
    const int64_t cells = local_cells(h);
    double *dst = out;
    if (where == LBM_HOST) {
        int rc = ensure_scratch(h, (size_t)cells * h->Q * sizeof(double));
        if (rc) return rc;
        dst = h->scratch;
    }
    int64_t off = 0;
    for (Slab &s : h->slabs) {
        ReadArgs r;
        std::memset(&r, 0, sizeof(r));
        read_common(h, r, raw, s);
        r.geo = geo_of(h, s);
        const int64_t sc = (int64_t)h->nx * h->ny * s.nz;
        const void *f = s.pdf[cur_array(h, s)];
        double *tmp = dst;
        if (h->slabs.size() > 1) {  // per-slab block then scatter into [q][cells]
            int rc = ensure_scratch(h, (size_t)cells * h->Q * sizeof(double) * 2);
            if (rc) return rc;
            if (where == LBM_HOST) dst = h->scratch;
            tmp = h->scratch + (size_t)cells * h->Q;
        }
        launch_get_pops(h->Q, h->dtype, r, f, tmp, dim3((unsigned)((h->nx + 31) / 32), (unsigned)((h->ny + 7) / 8), (unsigned)s.nz),
                        dim3(32, 8, 1), h->stream);
        if (h->slabs.size() > 1)
            for (int q = 0; q < h->Q; ++q)
                CUDA_TRY(h, cudaMemcpyAsync(dst + (size_t)q * cells + off, tmp + (size_t)q * sc, sc * sizeof(double),
                                            cudaMemcpyDeviceToDevice, h->stream));
        off += sc;
    }
    if (where == LBM_HOST)
        CUDA_TRY(h, cudaMemcpyAsync(out, dst, (size_t)cells * h->Q * sizeof(double), cudaMemcpyDeviceToHost, h->stream));
    CUDA_TRY(h, cudaStreamSynchronize(h->stream));
    return LBM_OK;
}

int lbm_get_populations_at(lbm_handle h, const int64_t *cells, int64_t n, double *out) {
    if (!h || !cells || !out || n < 0) return LBM_EINVAL;
    if (n == 0) return LBM_OK;
    const int64_t total = local_cells(h);
    for (int64_t k = 0; k < n; ++k)
        if (cells[k] < 0 || cells[k] >= total) return fail(h, LBM_EINVAL, "cell index out of range");
    const size_t ib = ((size_t)n * sizeof(int64_t) + 255) / 256 * 256;
    int rc = ensure_scratch(h, ib + (size_t)n * h->Q * sizeof(double));
    if (rc) return rc;
    int64_t *didx = reinterpret_cast<int64_t *>(h->scratch);
    double *dout = reinterpret_cast<double *>(reinterpret_cast<char *>(h->scratch) + ib);
    CUDA_TRY(h, cudaMemcpyAsync(didx, cells, n * sizeof(int64_t), cudaMemcpyHostToDevice, h->stream));
    int64_t first = 0;
    for (Slab &s : h->slabs) {
        ReadArgs r;
        std::memset(&r, 0, sizeof(r));
        read_common(h, r, 0, s);
        r.geo = geo_of(h, s);
        const int64_t sc = (int64_t)h->nx * h->ny * s.nz;
        launch_get_at(h->Q, h->dtype, r, s.pdf[cur_array(h, s)], didx, n, first, first + sc, dout, h->stream);
        first += sc;
    }
    CUDA_TRY(h, cudaMemcpyAsync(out, dout, (size_t)n * h->Q * sizeof(double), cudaMemcpyDeviceToHost, h->stream));
    CUDA_TRY(h, cudaStreamSynchronize(h->stream));
    return LBM_OK;
}

int lbm_set_populations(lbm_handle h, const double *in, int32_t where, int32_t raw) {
    if (!h || !in) return LBM_EINVAL;
    if (where == LBM_HOST_ASYNC) where = LBM_HOST;  // synchronous call
    const int64_t cells = local_cells(h);
    int rc = ensure_scratch(h, (size_t)cells * h->Q * sizeof(double) * 2);
    if (rc) return rc;
    const double *src = in;
    if (where == LBM_HOST) {
        CUDA_TRY(h, cudaMemcpyAsync(h->scratch, in, (size_t)cells * h->Q * sizeof(double), cudaMemcpyHostToDevice, h->stream));
        src = h->scratch;
    }
    int64_t off = 0;
    h->aa_parity = 0;
    h->links_pending = -1;
    links_unprime(h);
    for (Slab &s : h->slabs) {
        ReadArgs r;
        std::memset(&r, 0, sizeof(r));
        read_common(h, r, raw, s);
        r.aa_odd = 0;
        r.geo = geo_of(h, s);
        const int64_t sc = (int64_t)h->nx * h->ny * s.nz;
        double *tmp = h->scratch + (size_t)cells * h->Q;
        for (int q = 0; q < h->Q; ++q)
            CUDA_TRY(h, cudaMemcpyAsync(tmp + (size_t)q * sc, src + (size_t)q * cells + off, sc * sizeof(double),
                                        cudaMemcpyDeviceToDevice, h->stream));
        s.cur = 0;
        launch_set_pops(h->Q, h->dtype, r, s.pdf[0], tmp, dim3((unsigned)((h->nx + 31) / 32), (unsigned)((h->ny + 7) / 8), (unsigned)s.nz),
                        dim3(32, 8, 1), h->stream);
        if (s.pdf[1]) {
            const Geo g = geo_of(h, s);
            CUDA_TRY(h, cudaMemcpyAsync(s.pdf[1], s.pdf[0], (size_t)g.Sq * h->Q * h->esize, cudaMemcpyDeviceToDevice, h->stream));
        }
        off += sc;
    }
    rc = exchange_current(h);
    if (rc) return rc;
    CUDA_TRY(h, cudaStreamSynchronize(h->stream));
    return LBM_OK;
}

int lbm_get_macroscopic(lbm_handle h, double *rho, double *u, int32_t where) {
    if (!h || !rho || !u) return LBM_EINVAL;
    const int64_t cells = local_cells(h);
    if (where == LBM_HOST_ASYNC && h->slabs.size() == 1) {
        // macro kernel on the compute stream into a staging buffer whose previous download finished, then the
        // download on the d2h stream; returns without waiting (outputs valid after lbm_sync)
        int rc = ensure_async(h);
        if (rc) return rc;
        auto &io = h->aio;
        const int k = io.out_k;
        io.out_k ^= 1;
        Slab &s = h->slabs[0];
        ReadArgs r;
        std::memset(&r, 0, sizeof(r));
        read_common(h, r, 0, s);
        r.geo = geo_of(h, s);
        CUDA_TRY(h, cudaStreamWaitEvent(h->stream, io.out_free[k], 0));
        launch_macro(h->Q, h->dtype, r, s.pdf[cur_array(h, s)], io.out[k], io.out[k] + cells,
                     dim3((unsigned)((h->nx + 31) / 32), (unsigned)((h->ny + 7) / 8), (unsigned)s.nz), dim3(32, 8, 1), h->stream);
        CUDA_TRY(h, cudaEventRecord(io.out_ready[k], h->stream));
        CUDA_TRY(h, cudaStreamWaitEvent(io.d2h, io.out_ready[k], 0));
        CUDA_TRY(h, cudaMemcpyAsync(rho, io.out[k], cells * sizeof(double), cudaMemcpyDeviceToHost, io.d2h));
        CUDA_TRY(h, cudaMemcpyAsync(u, io.out[k] + cells, 3 * cells * sizeof(double), cudaMemcpyDeviceToHost, io.d2h));
        CUDA_TRY(h, cudaEventRecord(io.out_free[k], io.d2h));
        return LBM_OK;
    }
    if (where == LBM_HOST_ASYNC) where = LBM_HOST;  // several local slabs: synchronous gather
    double *drho = rho, *du = u;
    if (where == LBM_HOST || h->slabs.size() > 1) {
        int rc = ensure_scratch(h, (size_t)cells * 4 * sizeof(double) * 2);
        if (rc) return rc;
        drho = h->scratch;
        du = h->scratch + cells;
    }
    int64_t off = 0;
    for (Slab &s : h->slabs) {
        ReadArgs r;
        std::memset(&r, 0, sizeof(r));
        read_common(h, r, 0, s);
        r.geo = geo_of(h, s);
        const int64_t sc = (int64_t)h->nx * h->ny * s.nz;
        const void *f = s.pdf[cur_array(h, s)];
        double *tr = h->slabs.size() > 1 ? h->scratch + 4 * cells : drho;
        double *tu = h->slabs.size() > 1 ? h->scratch + 5 * cells : du;
        launch_macro(h->Q, h->dtype, r, f, tr, tu, dim3((unsigned)((h->nx + 31) / 32), (unsigned)((h->ny + 7) / 8), (unsigned)s.nz),
                     dim3(32, 8, 1), h->stream);
        if (h->slabs.size() > 1) {
            CUDA_TRY(h, cudaMemcpyAsync(drho + off, tr, sc * sizeof(double), cudaMemcpyDeviceToDevice, h->stream));
            for (int d = 0; d < 3; ++d)
                CUDA_TRY(h, cudaMemcpyAsync(du + (size_t)d * cells + off, tu + (size_t)d * sc, sc * sizeof(double),
                                            cudaMemcpyDeviceToDevice, h->stream));
        }
        off += sc;
    }
    if (where == LBM_HOST) {
        CUDA_TRY(h, cudaMemcpyAsync(rho, drho, cells * sizeof(double), cudaMemcpyDeviceToHost, h->stream));
        CUDA_TRY(h, cudaMemcpyAsync(u, du, 3 * cells * sizeof(double), cudaMemcpyDeviceToHost, h->stream));
    } else if (h->slabs.size() > 1) {
        CUDA_TRY(h, cudaMemcpyAsync(rho, drho, cells * sizeof(double), cudaMemcpyDeviceToDevice, h->stream));
        CUDA_TRY(h, cudaMemcpyAsync(u, du, 3 * cells * sizeof(double), cudaMemcpyDeviceToDevice, h->stream));
    }
    CUDA_TRY(h, cudaStreamSynchronize(h->stream));
    return LBM_OK;
}

int lbm_pack_face(lbm_handle h, int64_t z, int32_t dir, double *out, int32_t where) {
    if (!h || !out || (dir != 1 && dir != -1)) return LBM_EINVAL;
    if (where == LBM_HOST_ASYNC) where = LBM_HOST;  // synchronous call
    // z is a local interior plane across the concatenated slabs
    int64_t zz = z;
    Slab *sp = nullptr;
    for (Slab &s : h->slabs) {
        if (zz < s.nz) {
            sp = &s;
            break;
        }
        zz -= s.nz;
    }
    if (!sp || zz < 0) return fail(h, LBM_EINVAL, "plane out of range");
    if (h->cfg.pattern == LBM_AA && h->aa_parity) return fail(h, LBM_EUNSUPPORTED, "pack_face on an odd AA state");
    if (h->cfg.pattern == LBM_ESOTWIST) return fail(h, LBM_EUNSUPPORTED, "pack_face on an EsoTwist state");
    const size_t n = (size_t)h->nx * h->ny * (h->Q == 19 ? 5 : 9);
    double *dst = out;
    if (where == LBM_HOST) {
        int rc = ensure_scratch(h, n * sizeof(double));
        if (rc) return rc;
        dst = h->scratch;
    }
    launch_pack(h->Q, h->dtype, geo_of(h, *sp), sp->pdf[cur_array(h, *sp)], (int)zz + h->g, dir, dst, true,
                h->stream);
    if (where == LBM_HOST) CUDA_TRY(h, cudaMemcpyAsync(out, dst, n * sizeof(double), cudaMemcpyDeviceToHost, h->stream));
    CUDA_TRY(h, cudaStreamSynchronize(h->stream));
    return LBM_OK;
}

}  // extern "C"
