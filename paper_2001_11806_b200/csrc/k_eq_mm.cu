// k_eq_mm.cu — moment-matched D3Q19 equilibrium variants (Maxwellian moments truncated at 2nd order,
// P:361-375; for D3Q27 the runtime uses the Eq. (3) kernels, which are identical):
// SRT/TRT (+ Guo) and weighted MRT; fp64 and fp32; pull and AA; every wall mode.
#include "k_pull_inst.cuh"

namespace lbm {

Kernels select_trt_mm(int Q, int dtype, int fm, bool force) {
    return select_op<op_with_eq(OP_TRT, EQ_MOMENT_MATCHED), true, true, false>(Q, dtype, fm, force);
}
Kernels select_mrt_mm(int Q, int dtype, int fm, bool force) {
    return select_op<op_with_eq(OP_MRT, EQ_MOMENT_MATCHED), false, true, false>(Q, dtype, fm, force);
}
}  // namespace lbm
