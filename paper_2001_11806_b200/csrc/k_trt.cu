// k_trt.cu — SRT/TRT (+ Guo) instantiations: D3Q19 and D3Q27, fp64 and fp32, with/without flags
// and force. SRT is launched as TRT with omega_e = omega_o.
#include "k_pull_inst.cuh"

namespace lbm {

PullLaunch select_pull_trt(int Q, int dtype, bool flags, bool force) {
    if (Q == 19) return dtype == 0 ? pick_pull<19, OP_TRT, double>(flags, force) : pick_pull<19, OP_TRT, float>(flags, force);
    if (Q == 27) return dtype == 0 ? pick_pull<27, OP_TRT, double>(flags, force) : pick_pull<27, OP_TRT, float>(flags, force);
    return nullptr;
}

AALaunch select_aa_trt(int Q, int dtype, bool force) {
    if (Q == 19) {
        if (dtype == 0) return force ? &aa_launcher<19, OP_TRT, double, true> : &aa_launcher<19, OP_TRT, double, false>;
        return force ? &aa_launcher<19, OP_TRT, float, true> : &aa_launcher<19, OP_TRT, float, false>;
    }
    if (Q == 27) {
        if (dtype == 0) return force ? &aa_launcher<27, OP_TRT, double, true> : &aa_launcher<27, OP_TRT, double, false>;
        return force ? &aa_launcher<27, OP_TRT, float, true> : &aa_launcher<27, OP_TRT, float, false>;
    }
    return nullptr;
}

}  // namespace lbm
