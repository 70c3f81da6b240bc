// k_select.cu — run-time selection of the kernel families compiled from k_inst.cu (one object per
// (operator, equilibrium, stencil, dtype), see build.py INSTANCES).
#include "dispatch.h"

namespace lbm {

Kernels inst_trt19d(int fm, bool force);
Kernels inst_trt19f(int fm, bool force);
Kernels inst_trt27d(int fm, bool force);
Kernels inst_trt27f(int fm, bool force);
Kernels inst_mrt19d(int fm, bool force);
Kernels inst_mrt19f(int fm, bool force);
Kernels inst_cum19d(int fm, bool force);
Kernels inst_cum19f(int fm, bool force);
Kernels inst_cum27d(int fm, bool force);
Kernels inst_cum27f(int fm, bool force);
Kernels inst_cumu27d(int fm, bool force);
Kernels inst_cumu27f(int fm, bool force);
Kernels inst_mrts19d(int fm, bool force);
Kernels inst_mrts19f(int fm, bool force);
Kernels inst_ident19d(int fm, bool force);
Kernels inst_ident19f(int fm, bool force);
Kernels inst_ident27d(int fm, bool force);
Kernels inst_ident27f(int fm, bool force);
Kernels inst_smag19d(int fm, bool force);
Kernels inst_smag19f(int fm, bool force);
Kernels inst_smag27d(int fm, bool force);
Kernels inst_smag27f(int fm, bool force);
Kernels inst_kbc19d(int fm, bool force);
Kernels inst_kbc19f(int fm, bool force);
Kernels inst_kbc27d(int fm, bool force);
Kernels inst_kbc27f(int fm, bool force);
Kernels inst_gsrt19d(int fm, bool force);
Kernels inst_gsrt19f(int fm, bool force);
Kernels inst_gsrt27d(int fm, bool force);
Kernels inst_gsrt27f(int fm, bool force);
Kernels inst_gtrt19d(int fm, bool force);
Kernels inst_gtrt19f(int fm, bool force);
Kernels inst_gtrt27d(int fm, bool force);
Kernels inst_gtrt27f(int fm, bool force);
Kernels inst_gmrt19d(int fm, bool force);
Kernels inst_gmrt19f(int fm, bool force);
Kernels inst_gmrt27d(int fm, bool force);
Kernels inst_gmrt27f(int fm, bool force);
Kernels inst_gsmag19d(int fm, bool force);
Kernels inst_gsmag19f(int fm, bool force);
Kernels inst_gsmag27d(int fm, bool force);
Kernels inst_gsmag27f(int fm, bool force);
Kernels inst_gsrt_inc19d(int fm, bool force);
Kernels inst_gsrt_inc19f(int fm, bool force);
Kernels inst_gsrt_inc27d(int fm, bool force);
Kernels inst_gsrt_inc27f(int fm, bool force);
Kernels inst_gtrt_inc19d(int fm, bool force);
Kernels inst_gtrt_inc19f(int fm, bool force);
Kernels inst_gtrt_inc27d(int fm, bool force);
Kernels inst_gtrt_inc27f(int fm, bool force);
Kernels inst_kbcx19d(int fm, bool force);
Kernels inst_kbcx19f(int fm, bool force);
Kernels inst_kbcx27d(int fm, bool force);
Kernels inst_kbcx27f(int fm, bool force);
Kernels inst_trt_inc19d(int fm, bool force);
Kernels inst_trt_inc19f(int fm, bool force);
Kernels inst_trt_inc27d(int fm, bool force);
Kernels inst_trt_inc27f(int fm, bool force);
Kernels inst_mrt_inc19d(int fm, bool force);
Kernels inst_mrt_inc19f(int fm, bool force);
Kernels inst_trt_mm19d(int fm, bool force);
Kernels inst_trt_mm19f(int fm, bool force);
Kernels inst_mrt_mm19d(int fm, bool force);
Kernels inst_mrt_mm19f(int fm, bool force);

Kernels select_trt(int Q, int dtype, int fm, bool force) {
    if (Q == 19) return dtype == 0 ? inst_trt19d(fm, force) : inst_trt19f(fm, force);
    if (Q == 27) return dtype == 0 ? inst_trt27d(fm, force) : inst_trt27f(fm, force);
    return Kernels{};
}
Kernels select_mrt(int Q, int dtype, int fm, bool force) {
    if (Q == 19) return dtype == 0 ? inst_mrt19d(fm, force) : inst_mrt19f(fm, force);
    return Kernels{};
}
Kernels select_cumulant(int Q, int dtype, int fm, bool force) {
    if (Q == 19) return dtype == 0 ? inst_cum19d(fm, force) : inst_cum19f(fm, force);
    if (Q == 27) return dtype == 0 ? inst_cum27d(fm, force) : inst_cum27f(fm, force);
    return Kernels{};
}
Kernels select_mrt_shear(int Q, int dtype, int fm, bool force) {
    if (Q == 19) return dtype == 0 ? inst_mrts19d(fm, force) : inst_mrts19f(fm, force);
    return Kernels{};
}
Kernels select_cumulant_unit(int Q, int dtype, int fm, bool force) {
    if (Q == 27) return dtype == 0 ? inst_cumu27d(fm, force) : inst_cumu27f(fm, force);
    return Kernels{};
}
Kernels select_identity(int Q, int dtype, int fm, bool force) {
    force = false;
    if (Q == 19) return dtype == 0 ? inst_ident19d(fm, force) : inst_ident19f(fm, force);
    if (Q == 27) return dtype == 0 ? inst_ident27d(fm, force) : inst_ident27f(fm, force);
    return Kernels{};
}
Kernels select_smagorinsky(int Q, int dtype, int fm, bool force) {
    if (Q == 19) return dtype == 0 ? inst_smag19d(fm, force) : inst_smag19f(fm, force);
    if (Q == 27) return dtype == 0 ? inst_smag27d(fm, force) : inst_smag27f(fm, force);
    return Kernels{};
}
Kernels select_kbc(int Q, int dtype, int fm, bool force) {
    if (Q == 19) return dtype == 0 ? inst_kbc19d(fm, force) : inst_kbc19f(fm, force);
    if (Q == 27) return dtype == 0 ? inst_kbc27d(fm, force) : inst_kbc27f(fm, force);
    return Kernels{};
}
Kernels select_generated(int op, int Q, int dtype, int fm, bool force, int eq) {
    force = false;
    const bool d = dtype == 0;
    if (eq == EQ_INCOMPRESSIBLE) {
        if (op == OP_GEN_SRT) {
            if (Q == 19) return d ? inst_gsrt_inc19d(fm, force) : inst_gsrt_inc19f(fm, force);
            if (Q == 27) return d ? inst_gsrt_inc27d(fm, force) : inst_gsrt_inc27f(fm, force);
        } else if (op == OP_GEN_TRT) {
            if (Q == 19) return d ? inst_gtrt_inc19d(fm, force) : inst_gtrt_inc19f(fm, force);
            if (Q == 27) return d ? inst_gtrt_inc27d(fm, force) : inst_gtrt_inc27f(fm, force);
        }
        return Kernels{};
    }
    if (eq != EQ_COMPRESSIBLE) return Kernels{};
    if (op == OP_GEN_SMAGORINSKY) {
        if (Q == 19) return d ? inst_gsmag19d(fm, force) : inst_gsmag19f(fm, force);
        if (Q == 27) return d ? inst_gsmag27d(fm, force) : inst_gsmag27f(fm, force);
    } else if (op == OP_GEN_SRT) {
        if (Q == 19) return d ? inst_gsrt19d(fm, force) : inst_gsrt19f(fm, force);
        if (Q == 27) return d ? inst_gsrt27d(fm, force) : inst_gsrt27f(fm, force);
    } else if (op == OP_GEN_TRT) {
        if (Q == 19) return d ? inst_gtrt19d(fm, force) : inst_gtrt19f(fm, force);
        if (Q == 27) return d ? inst_gtrt27d(fm, force) : inst_gtrt27f(fm, force);
    } else if (op == OP_GEN_MRT) {
        if (Q == 19) return d ? inst_gmrt19d(fm, force) : inst_gmrt19f(fm, force);
        if (Q == 27) return d ? inst_gmrt27d(fm, force) : inst_gmrt27f(fm, force);
    }
    return Kernels{};
}
Kernels select_kbc_exact(int Q, int dtype, int fm, bool force) {
    if (Q == 19) return dtype == 0 ? inst_kbcx19d(fm, force) : inst_kbcx19f(fm, force);
    if (Q == 27) return dtype == 0 ? inst_kbcx27d(fm, force) : inst_kbcx27f(fm, force);
    return Kernels{};
}
Kernels select_trt_eq(int Q, int dtype, int fm, bool force, int eq) {
    if (eq == EQ_INCOMPRESSIBLE) {
        if (Q == 19) return dtype == 0 ? inst_trt_inc19d(fm, force) : inst_trt_inc19f(fm, force);
        if (Q == 27) return dtype == 0 ? inst_trt_inc27d(fm, force) : inst_trt_inc27f(fm, force);
    } else if (eq == EQ_MOMENT_MATCHED) {
        if (Q == 19) return dtype == 0 ? inst_trt_mm19d(fm, force) : inst_trt_mm19f(fm, force);
    }
    return Kernels{};
}
Kernels select_mrt_eq(int Q, int dtype, int fm, bool force, int eq) {
    if (eq == EQ_INCOMPRESSIBLE) {
        if (Q == 19) return dtype == 0 ? inst_mrt_inc19d(fm, force) : inst_mrt_inc19f(fm, force);
    } else if (eq == EQ_MOMENT_MATCHED) {
        if (Q == 19) return dtype == 0 ? inst_mrt_mm19d(fm, force) : inst_mrt_mm19f(fm, force);
    }
    return Kernels{};
}

}  // namespace lbm
