// k_mrt.cu — weighted-orthogonal MRT instantiations (D3Q19; fp64 and fp32; no force; pull and AA).
#include "k_pull_inst.cuh"

namespace lbm {

PullLaunch select_pull_mrt(int Q, int dtype, bool flags, bool force) {
    return select_pull_op<OP_MRT, false, true, false>(Q, dtype, flags, force);
}

AALaunch select_aa_mrt(int Q, int dtype, bool flags, bool force) {
    return select_aa_op<OP_MRT, false, true, false>(Q, dtype, flags, force);
}

}  // namespace lbm
