// k_fused.cu — fused halo exchange over NVLink peer memory (NCCL 2.28 device API).
//
// The population arrays live in NCCL symmetric memory windows. The boundary-plane launch of
// k_pull (AA: k_aa_even / k_aa_odd, kernels.cuh) stores the populations that cross a z face both into its own array and, through LSA
// (load/store accessible) pointers, straight into the neighbour's ghost plane of the same array
// — no pack kernel, no send/recv, the transfer overlaps the collision math thread by thread
// (P:1067-1071 for the exchange it replaces). A one-CTA gate kernel at the
// start of every step runs an LSA barrier: a rank passes it only when every rank has finished the
// previous step (so the ghosts it is about to read are complete, and the ghosts it is about to
// overwrite are no longer read).
#include <nccl.h>
#include <nccl_device.h>

#include <string>

#include "dispatch.h"
#include "fused.h"

namespace lbm {

__global__ void k_lsa_peer_bases(ncclWindow_t w0, ncclWindow_t w1, int up, int down, void **out) {
    out[0] = ncclGetLsaPointer(w0, 0, up);
    out[1] = ncclGetLsaPointer(w0, 0, down);
    out[2] = w1 ? ncclGetLsaPointer(w1, 0, up) : nullptr;  // single-array patterns register one window
    out[3] = w1 ? ncclGetLsaPointer(w1, 0, down) : nullptr;
}

__global__ void k_lsa_gate(ncclDevComm comm) {
    __threadfence_system();  // previous kernels' peer stores are performed before we arrive
    ncclLsaBarrierSession<ncclCoopCta> bar(ncclCoopCta(), comm, ncclTeamTagLsa(), 0);
    bar.sync(ncclCoopCta(), cuda::memory_order_acq_rel);
}

struct FusedImpl {
    ncclDevComm dev{};
    bool have_dev = false;
    ncclWindow_t win[2] = {nullptr, nullptr};
};

int fused_setup(ncclComm_t comm, void *pdf0, void *pdf1, size_t bytes, int up_world, int down_world, FusedState *st,
                cudaStream_t s, std::string &err) {
    FusedImpl *im = new FusedImpl();
    st->impl = im;
    const ncclTeam_t world = ncclTeamWorld(comm);
    const int up = ncclTeamRankToLsa(comm, world, up_world);
    const int down = ncclTeamRankToLsa(comm, world, down_world);
    if (up < 0 || down < 0) {
        err = "fused halo needs the neighbours in the same NVLink (LSA) domain";
        return -1;
    }
    ncclResult_t r;
    if ((r = ncclCommWindowRegister(comm, pdf0, bytes, &im->win[0], NCCL_WIN_COLL_SYMMETRIC)) != ncclSuccess ||
        (pdf1 && (r = ncclCommWindowRegister(comm, pdf1, bytes, &im->win[1], NCCL_WIN_COLL_SYMMETRIC)) != ncclSuccess)) {
        err = std::string("ncclCommWindowRegister: ") + ncclGetErrorString(r);
        return -1;
    }
    ncclDevCommRequirements reqs{};
    reqs.lsaBarrierCount = 1;
    if ((r = ncclDevCommCreate(comm, &reqs, &im->dev)) != ncclSuccess) {
        err = std::string("ncclDevCommCreate: ") + ncclGetErrorString(r);
        return -1;
    }
    im->have_dev = true;
    void **d = nullptr;
    if (cudaMalloc(&d, 4 * sizeof(void *)) != cudaSuccess) {
        err = "cudaMalloc peer bases";
        return -1;
    }
    k_lsa_peer_bases<<<1, 1, 0, s>>>(im->win[0], im->win[1], up, down, d);
    cudaMemcpyAsync(st->bases, d, 4 * sizeof(void *), cudaMemcpyDeviceToHost, s);
    const cudaError_t e = cudaStreamSynchronize(s);
    cudaFree(d);
    if (e != cudaSuccess) {
        err = std::string("peer bases: ") + cudaGetErrorString(e);
        return -1;
    }
    return 0;
}

void fused_gate(const FusedState &st, cudaStream_t s) {
    const FusedImpl *im = static_cast<const FusedImpl *>(st.impl);
    k_lsa_gate<<<1, 32, 0, s>>>(im->dev);
}

void fused_teardown(ncclComm_t comm, FusedState *st) {
    FusedImpl *im = static_cast<FusedImpl *>(st->impl);
    if (!im) return;
    if (im->have_dev) ncclDevCommDestroy(comm, &im->dev);
    for (ncclWindow_t w : im->win)
        if (w) ncclCommWindowDeregister(comm, w);
    delete im;
    st->impl = nullptr;
}

}  // namespace lbm
