// k_identity.cu — IDENTITY (no collision) instantiations: pure data movement for the bit-exact
// streaming / boundary / AA-slot / halo tests.
#include "k_pull_inst.cuh"

namespace lbm {

PullLaunch select_pull_identity(int Q, int dtype, bool flags, bool force) {
    (void)force;
    return select_pull_op<OP_IDENTITY, false, true, true>(Q, dtype, flags, false);
}

AALaunch select_aa_identity(int Q, int dtype, bool flags, bool force) {
    (void)force;
    return select_aa_op<OP_IDENTITY, false, true, true>(Q, dtype, flags, false);
}

}  // namespace lbm
