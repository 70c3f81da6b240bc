// k_identity.cu — IDENTITY (no collision) instantiations: pure data movement for the bit-exact
// streaming / boundary / AA-slot / halo tests.
#include "k_pull_inst.cuh"

namespace lbm {

Kernels select_identity(int Q, int dtype, int fm, bool force) {
    (void)force;
    return select_op<OP_IDENTITY, false, true, true>(Q, dtype, fm, false);
}
}  // namespace lbm
