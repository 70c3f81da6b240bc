// k_cumulant.cu — D3Q27 cumulant instantiations (fp64 and fp32; no force; pull and AA).
#include "k_pull_inst.cuh"

namespace lbm {

PullLaunch select_pull_cumulant(int Q, int dtype, bool flags, bool force) {
    return select_pull_op<OP_CUMULANT, false, false, true>(Q, dtype, flags, force);
}

AALaunch select_aa_cumulant(int Q, int dtype, bool flags, bool force) {
    return select_aa_op<OP_CUMULANT, false, false, true>(Q, dtype, flags, force);
}

}  // namespace lbm
