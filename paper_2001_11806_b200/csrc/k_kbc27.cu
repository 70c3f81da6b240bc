// k_kbc27.cu — KBC entropic operator on D3Q27: fp64 and fp32, pull and
// AA, no force.
#include "k_pull_inst.cuh"

namespace lbm {

Kernels select_kbc27(int Q, int dtype, int fm, bool force) { return select_op<OP_KBC, false, false, true>(Q, dtype, fm, force); }
}  // namespace lbm
