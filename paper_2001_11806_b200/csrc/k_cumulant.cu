// k_cumulant.cu — D3Q27 cumulant instantiations (fp64 and fp32; no force; pull and AA).
#include "k_pull_inst.cuh"

namespace lbm {

Kernels select_cumulant(int Q, int dtype, int fm, bool force) {
    if (Q == 19) return select_cumulant19(Q, dtype, fm, force);
    return select_op<OP_CUMULANT, false, false, true>(Q, dtype, fm, force);
}
}  // namespace lbm
