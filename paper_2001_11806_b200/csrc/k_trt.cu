// k_trt.cu — SRT/TRT (+ Guo) instantiations: D3Q19 and D3Q27, fp64 and fp32, with/without flags
// and force, pull and AA. SRT is launched as TRT with omega_e = omega_o.
#include "k_pull_inst.cuh"

namespace lbm {

PullLaunch select_pull_trt(int Q, int dtype, bool flags, bool force) {
    return select_pull_op<OP_TRT, true, true, true>(Q, dtype, flags, force);
}

AALaunch select_aa_trt(int Q, int dtype, bool flags, bool force) {
    return select_aa_op<OP_TRT, true, true, true>(Q, dtype, flags, force);
}

}  // namespace lbm
