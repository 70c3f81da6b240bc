// k_les.cu — locally varying relaxation rates: Smagorinsky SRT (D3Q19 and D3Q27) and
// the entropic KBC operator (D3Q19); fp64 and fp32; pull and AA; no force.
#include "k_pull_inst.cuh"

namespace lbm {

Kernels select_smagorinsky(int Q, int dtype, int fm, bool force) {
    return select_op<OP_SMAGORINSKY, false, true, true>(Q, dtype, fm, force);
}
Kernels select_kbc(int Q, int dtype, int fm, bool force) {
    if (Q == 27) return select_kbc27(Q, dtype, fm, force);
    return select_op<OP_KBC, false, true, false>(Q, dtype, fm, force);
}
}  // namespace lbm
