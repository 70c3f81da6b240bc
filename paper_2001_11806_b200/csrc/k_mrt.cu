// k_mrt.cu — weighted-orthogonal MRT instantiations (D3Q19; fp64 and fp32; no force; pull and AA).
#include "k_pull_inst.cuh"

namespace lbm {

Kernels select_mrt(int Q, int dtype, int fm, bool force) { return select_op<OP_MRT, false, true, false>(Q, dtype, fm, force); }
}  // namespace lbm
