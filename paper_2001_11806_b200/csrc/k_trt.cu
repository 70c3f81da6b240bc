// k_trt.cu — SRT/TRT (+ Guo) instantiations: D3Q19 and D3Q27, fp64 and fp32, pull and AA, every wall mode,
// with and without force. SRT is launched as TRT with omega_e = omega_o.
#include "k_pull_inst.cuh"

namespace lbm {

Kernels select_trt(int Q, int dtype, int fm, bool force) { return select_op<OP_TRT, true, true, true>(Q, dtype, fm, force); }
}  // namespace lbm
