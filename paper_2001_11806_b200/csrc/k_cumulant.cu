// k_cumulant.cu — D3Q27 cumulant instantiations (fp64 and fp32; no force).
#include "k_pull_inst.cuh"

namespace lbm {

PullLaunch select_pull_cumulant(int Q, int dtype, bool flags, bool force) {
    if (Q != 27) return nullptr;
    return dtype == 0 ? pick_pull_noforce<27, OP_CUMULANT, double>(flags, force)
                      : pick_pull_noforce<27, OP_CUMULANT, float>(flags, force);
}

AALaunch select_aa_cumulant(int Q, int dtype, bool force) {
    if (Q != 27 || force) return nullptr;
    return dtype == 0 ? &aa_launcher<27, OP_CUMULANT, double, false> : &aa_launcher<27, OP_CUMULANT, float, false>;
}

}  // namespace lbm
