// k_identity.cu — IDENTITY (no collision) instantiations: pure data movement for the bit-exact
// streaming / boundary / AA-slot / halo tests.
#include "k_pull_inst.cuh"

namespace lbm {

PullLaunch select_pull_identity(int Q, int dtype, bool flags, bool force) {
    (void)force;
    if (Q == 19) return dtype == 0 ? pick_pull_noforce<19, OP_IDENTITY, double>(flags, false)
                                   : pick_pull_noforce<19, OP_IDENTITY, float>(flags, false);
    if (Q == 27) return dtype == 0 ? pick_pull_noforce<27, OP_IDENTITY, double>(flags, false)
                                   : pick_pull_noforce<27, OP_IDENTITY, float>(flags, false);
    return nullptr;
}

AALaunch select_aa_identity(int Q, int dtype, bool force) {
    (void)force;
    if (Q == 19) return dtype == 0 ? &aa_launcher<19, OP_IDENTITY, double, false> : &aa_launcher<19, OP_IDENTITY, float, false>;
    if (Q == 27) return dtype == 0 ? &aa_launcher<27, OP_IDENTITY, double, false> : &aa_launcher<27, OP_IDENTITY, float, false>;
    return nullptr;
}

}  // namespace lbm
