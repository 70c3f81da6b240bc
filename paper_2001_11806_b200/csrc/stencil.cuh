// stencil.cuh — D3Q19 / D3Q27 velocity sets for the device kernels.
//
// Direction order G10 (ABI): index 0 = centre, then by |c|_1, then lexicographic on
// (cx, cy, cz) with -1 < 0 < 1. D3Q27 = D3Q19 + the 8 corners at 19..26. Weights: D3Q19
// 1/3, 1/18, 1/36; D3Q27 8/27, 2/27, 1/54, 1/216; cs^2 = 1/3.
#pragma once
#include <cstdint>

namespace lbm {

__host__ __device__ constexpr int kC27[27][3] = {
    {0, 0, 0},                                                                      // 0
    {-1, 0, 0}, {0, -1, 0}, {0, 0, -1}, {0, 0, 1}, {0, 1, 0}, {1, 0, 0},            // 1..6
    {-1, -1, 0}, {-1, 0, -1}, {-1, 0, 1}, {-1, 1, 0}, {0, -1, -1}, {0, -1, 1},       // 7..12
    {0, 1, -1}, {0, 1, 1}, {1, -1, 0}, {1, 0, -1}, {1, 0, 1}, {1, 1, 0},            // 13..18
    {-1, -1, -1}, {-1, -1, 1}, {-1, 1, -1}, {-1, 1, 1},                              // 19..22
    {1, -1, -1}, {1, -1, 1}, {1, 1, -1}, {1, 1, 1}};                                 // 23..26

template <int Q>
struct Stencil {
    static_assert(Q == 19 || Q == 27, "D3Q19 or D3Q27");
    __host__ __device__ static constexpr int cx(int q) { return kC27[q][0]; }
    __host__ __device__ static constexpr int cy(int q) { return kC27[q][1]; }
    __host__ __device__ static constexpr int cz(int q) { return kC27[q][2]; }
    __host__ __device__ static constexpr int c2(int q) { return cx(q) * cx(q) + cy(q) * cy(q) + cz(q) * cz(q); }
    // opposite direction: i -> 7 - i on 1..6, 25 - i on 7..18, 45 - i on 19..26
    __host__ __device__ static constexpr int opp(int q) {
        return q == 0 ? 0 : (q <= 6 ? 7 - q : (q <= 18 ? 25 - q : 45 - q));
    }
    __host__ __device__ static constexpr double w(int q) {
        return Q == 19 ? (c2(q) == 0 ? 1.0 / 3.0 : c2(q) == 1 ? 1.0 / 18.0 : 1.0 / 36.0)
                       : (c2(q) == 0 ? 8.0 / 27.0 : c2(q) == 1 ? 2.0 / 27.0 : c2(q) == 2 ? 1.0 / 54.0 : 1.0 / 216.0);
    }
    // number of directions crossing a z face (c_z = +1 or -1)
    static constexpr int kCross = (Q == 19) ? 5 : 9;
};

// The q-th direction with c_z == dir (ascending q); used by halo pack/unpack and NCCL planes.
template <int Q>
__host__ __device__ constexpr int crossing_dir(int dir, int k) {
    int n = 0;
    for (int q = 0; q < Q; ++q) {
        if (kC27[q][2] == dir) {
            if (n == k) return q;
            ++n;
        }
    }
    return -1;
}

}  // namespace lbm
