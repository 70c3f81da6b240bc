// k_cumulant19.cu — D3Q19 cumulant instantiations (fp64 and fp32; no force; pull and AA).
#include "k_pull_inst.cuh"

namespace lbm {

Kernels select_cumulant19(int Q, int dtype, int fm, bool force) { return select_op<OP_CUMULANT, false, true, false>(Q, dtype, fm, force); }
}  // namespace lbm
