// k_inst.cu — one kernel family per object file: the pull / AA / EsoTwist / staged / edge / persistent
// launchers of one (operator, stencil, dtype). build.py compiles this file once per entry of its
// INSTANCES table with -DLBM_INST_NAME=<function> -DLBM_INST_OP=<op | eq << 4> -DLBM_INST_Q=<19|27>
// -DLBM_INST_T=<double|float> -DLBM_INST_FORCE=<0|1> (FORCE: the Guo-forced variants are
// instantiated too), so the heavy template instantiations compile in parallel; k_select.cu maps the
// run-time (collision, equilibrium, stencil, dtype) to these functions.
#include "k_pull_inst.cuh"

#ifndef LBM_INST_NAME
#error "k_inst.cu is compiled by build.py with the LBM_INST_* definitions"
#endif

namespace lbm {

Kernels LBM_INST_NAME(int fm, bool force) { return pick<LBM_INST_Q, LBM_INST_OP, LBM_INST_T, (LBM_INST_FORCE != 0)>(fm, force); }

}  // namespace lbm
