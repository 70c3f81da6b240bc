// tma_probe.cu — microbenchmark (not product code): read bandwidth of 1-D bulk copies
// (cp.async.bulk + mbarrier) into shared memory vs copy size and pipeline depth, and the same
// with per-thread 16-byte cp.async (LDGSTS), to size the staged update kernels.
// Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o tma_probe scripts/tma_probe.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t su32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

// Each CTA streams `per_cta` chunks of `bytes` through `depth` stages; warp 0 issues (one copy per lane
// for `copies_per_stage` copies), the other warps wait on the stage barrier and touch one word.
__global__ void bulk_probe(const char *src, size_t total, int bytes, int copies, int depth, int iters, int *sink) {
    extern __shared__ __align__(128) unsigned char sm[];
    uint64_t *full = (uint64_t *)sm;
    uint64_t *empty = full + 16;
    char *buf = (char *)(sm + 256);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
    if (threadIdx.x == 0) {
        for (int s = 0; s < depth; ++s) {
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&full[s])));
            asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(&empty[s])), "r"(nw - 1));
        }
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    __syncthreads();
    const size_t stage_bytes = (size_t)bytes * copies;
    if (warp == nw - 1) {
        for (int it = 0; it < iters; ++it) {
            const int s = it % depth;
            if (it >= depth) {
                uint32_t ok;
                do {
                    asm volatile("{.reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0,1,0,p;}"
                                 : "=r"(ok) : "r"(su32(&empty[s])), "r"((uint32_t)(((it / depth) - 1) & 1)) : "memory");
                } while (!ok);
            }
            if (lane == 0)
                asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&full[s])), "r"((uint32_t)stage_bytes) : "memory");
            __syncwarp();
            for (int c = lane; c < copies; c += 32) {
                size_t off = (((size_t)(blockIdx.x + (size_t)it * gridDim.x) * copies + c) * bytes) % (total - bytes);
                off &= ~(size_t)127;
                asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                                 su32(buf + s * stage_bytes + (size_t)c * bytes)),
                             "l"(src + off), "r"(bytes), "r"(su32(&full[s]))
                             : "memory");
            }
        }
        return;
    }
    int acc = 0;
    for (int it = 0; it < iters; ++it) {
        const int s = it % depth;
        uint32_t ok;
        do {
            asm volatile("{.reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0,1,0,p;}"
                         : "=r"(ok) : "r"(su32(&full[s])), "r"((uint32_t)((it / depth) & 1)) : "memory");
        } while (!ok);
        acc += buf[s * stage_bytes + threadIdx.x * 4];
        __syncwarp();
        if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(&empty[s])) : "memory");
    }
    if (acc == 12345) *sink = acc;
}

// per-thread 16-byte cp.async, each warp owns its stage ring (no CTA barrier)
__global__ void ldgsts_probe(const char *src, size_t total, int bytes, int copies, int depth, int iters, int *sink) {
    extern __shared__ __align__(128) unsigned char sm[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
    const size_t stage_bytes = (size_t)bytes * copies;
    char *ring = (char *)sm + (size_t)warp * depth * stage_bytes;
    int acc = 0;
    const int gw = blockIdx.x * nw + warp, GW = gridDim.x * nw;
    auto issue = [&](int it) {
        const int s = it % depth;
        for (int c = 0; c < copies; ++c) {
            size_t off = (((size_t)(gw + (size_t)it * GW) * copies + c) * bytes) % (total - bytes);
            off &= ~(size_t)127;
            for (int k = lane * 16; k < bytes; k += 512)
                asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(su32(ring + s * stage_bytes + (size_t)c * bytes + k)),
                             "l"(src + off + k) : "memory");
        }
        asm volatile("cp.async.commit_group;" ::: "memory");
    };
    for (int it = 0; it < depth - 1 && it < iters; ++it) issue(it);
    for (int it = 0; it < iters; ++it) {
        if (it + depth - 1 < iters) issue(it + depth - 1);
        else asm volatile("cp.async.commit_group;" ::: "memory");
        asm volatile("cp.async.wait_group %0;" ::"n"(3) : "memory");  // depth 4
        __syncwarp();
        acc += ring[(it % depth) * stage_bytes + lane * 4];
        __syncwarp();
    }
    if (acc == 12345) *sink = acc;
}

int main() {
    const size_t total = (size_t)8 << 30;
    char *src;
    int *sink;
    cudaMalloc(&src, total);
    cudaMalloc(&sink, 4);
    cudaMemset(src, 1, total);
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaFuncSetAttribute(bulk_probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
    cudaFuncSetAttribute(ldgsts_probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
    printf("bulk: bytes copies depth ctas/SM threads -> GB/s\n");
    int sizes[] = {256, 512, 1024, 2048, 4096, 8192};
    for (int bytes : sizes)
        for (int copies : {8, 19})
            for (int depth : {2, 4})
                for (int cps : {1, 2, 4}) {
                    size_t smem = 256 + (size_t)bytes * copies * depth;
                    if (smem * cps > 220 * 1024) continue;
                    int iters = (int)((2ull << 30) / ((size_t)bytes * copies * sms * cps));
                    if (iters < 8) iters = 8;
                    bulk_probe<<<sms * cps, 160, smem>>>(src, total, bytes, copies, depth, iters, sink);
                    cudaEventRecord(a);
                    bulk_probe<<<sms * cps, 160, smem>>>(src, total, bytes, copies, depth, iters, sink);
                    cudaEventRecord(b);
                    cudaEventSynchronize(b);
                    float ms;
                    cudaEventElapsedTime(&ms, a, b);
                    double gb = (double)bytes * copies * iters * sms * cps / 1e9;
                    printf("bulk %5d %3d %d %d 160 -> %8.1f GB/s  (%s)\n", bytes, copies, depth, cps, gb / (ms * 1e-3),
                           cudaGetErrorString(cudaGetLastError()));
                }
    printf("ldgsts (per-warp rings, depth 4): bytes copies warps/CTA ctas/SM -> GB/s\n");
    for (int bytes : {128, 256, 512})
        for (int copies : {19})
            for (int nw : {4, 8})
                for (int cps : {1, 2, 4}) {
                    const int depth = 4;
                    size_t smem = (size_t)bytes * copies * depth * nw;
                    if (smem * cps > 220 * 1024) continue;
                    int iters = (int)((2ull << 30) / ((size_t)bytes * copies * sms * cps * nw));
                    if (iters < 8) iters = 8;
                    ldgsts_probe<<<sms * cps, nw * 32, smem>>>(src, total, bytes, copies, depth, iters, sink);
                    cudaEventRecord(a);
                    ldgsts_probe<<<sms * cps, nw * 32, smem>>>(src, total, bytes, copies, depth, iters, sink);
                    cudaEventRecord(b);
                    cudaEventSynchronize(b);
                    float ms;
                    cudaEventElapsedTime(&ms, a, b);
                    double gb = (double)bytes * copies * iters * sms * cps * nw / 1e9;
                    printf("ldgsts %4d %3d %d %d -> %8.1f GB/s  (%s)\n", bytes, copies, nw, cps, gb / (ms * 1e-3),
                           cudaGetErrorString(cudaGetLastError()));
                }
    return 0;
}
