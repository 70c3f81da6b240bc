// k_les.cu — locally varying relaxation rates: Smagorinsky SRT (D3Q19 and D3Q27) and
// the entropic KBC operator (D3Q19); fp64 and fp32; pull and AA; no force.
#include "k_pull_inst.cuh"

namespace lbm {

PullLaunch select_pull_smagorinsky(int Q, int dtype, bool flags, bool force) {
    return select_pull_op<OP_SMAGORINSKY, false, true, true>(Q, dtype, flags, force);
}
AALaunch select_aa_smagorinsky(int Q, int dtype, bool flags, bool force) {
    return select_aa_op<OP_SMAGORINSKY, false, true, true>(Q, dtype, flags, force);
}
PullLaunch select_pull_kbc(int Q, int dtype, bool flags, bool force) {
    return select_pull_op<OP_KBC, false, true, false>(Q, dtype, flags, force);
}
AALaunch select_aa_kbc(int Q, int dtype, bool flags, bool force) {
    return select_aa_op<OP_KBC, false, true, false>(Q, dtype, flags, force);
}

}  // namespace lbm
