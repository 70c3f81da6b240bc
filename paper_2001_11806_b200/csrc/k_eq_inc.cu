// k_eq_inc.cu — incompressible-equilibrium variants (Eq. (3) with rho0 = 1): SRT/TRT (+ Guo)
// for D3Q19 and D3Q27, weighted MRT for D3Q19; fp64 and fp32; pull and AA; every wall mode.
#include "k_pull_inst.cuh"

namespace lbm {

Kernels select_trt_eq(int Q, int dtype, int fm, bool force, int eq) {
    if (eq == EQ_INCOMPRESSIBLE) return select_op<op_with_eq(OP_TRT, EQ_INCOMPRESSIBLE), true, true, true>(Q, dtype, fm, force);
    if (eq == EQ_MOMENT_MATCHED) return select_trt_mm(Q, dtype, fm, force);
    return Kernels{};
}
Kernels select_mrt_eq(int Q, int dtype, int fm, bool force, int eq) {
    if (eq == EQ_INCOMPRESSIBLE) return select_op<op_with_eq(OP_MRT, EQ_INCOMPRESSIBLE), false, true, false>(Q, dtype, fm, force);
    if (eq == EQ_MOMENT_MATCHED) return select_mrt_mm(Q, dtype, fm, force);
    return Kernels{};
}
}  // namespace lbm
