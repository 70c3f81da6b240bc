// k_mrt.cu — weighted-orthogonal MRT instantiations (D3Q19; fp64 and fp32; no force).
#include "k_pull_inst.cuh"

namespace lbm {

PullLaunch select_pull_mrt(int Q, int dtype, bool flags, bool force) {
    if (Q != 19) return nullptr;
    return dtype == 0 ? pick_pull_noforce<19, OP_MRT, double>(flags, force) : pick_pull_noforce<19, OP_MRT, float>(flags, force);
}

AALaunch select_aa_mrt(int Q, int dtype, bool force) {
    if (Q != 19 || force) return nullptr;
    return dtype == 0 ? &aa_launcher<19, OP_MRT, double, false> : &aa_launcher<19, OP_MRT, float, false>;
}

}  // namespace lbm
