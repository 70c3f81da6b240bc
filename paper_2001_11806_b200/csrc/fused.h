// fused.h — host interface of the fused (NVLink peer-store) halo exchange, k_fused.cu.
#pragma once
#include <cuda_runtime.h>
#include <nccl.h>

#include <string>

namespace lbm {

struct FusedState {
    void *impl = nullptr;                              // NCCL device communicator + windows
    void *bases[4] = {nullptr, nullptr, nullptr, nullptr};  // LSA base of array 0 up/down, array 1 up/down
};

// Registers the population arrays (allocated with ncclMemAlloc, `bytes` each, same size on every
// rank; pdf1 = nullptr for the single-array AA pattern) as symmetric windows, creates a device communicator with one LSA barrier and resolves the
// neighbours' window base pointers. Collective over the communicator. Returns 0 or -1 (err set).
int fused_setup(ncclComm_t comm, void *pdf0, void *pdf1, size_t bytes, int up_world, int down_world, FusedState *st,
                cudaStream_t s, std::string &err);
// One-CTA LSA barrier kernel run at the start of every fused step.
void fused_gate(const FusedState &st, cudaStream_t s);
void fused_teardown(ncclComm_t comm, FusedState *st);

}  // namespace lbm
