#!/bin/bash
# Final round-2 pass after the C2 even-step change: whole GPU suite, smoke, bounds-check suite, then the
# evidence profile (bench lines, launch list, ncu full captures) into gpurun_out/r02zz.
O=gpurun_out/r02zz; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q --durations=20 > $O/gpu_tests.log 2>&1; echo "rc=$?" >> $O/gpu_tests.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "rc=$?" >> $O/smoke.log
python -c "
from paper_2001_11806_b200 import build
build.build(defines=['LBM_BOUNDS_CHECK'], out='paper_2001_11806_b200/variants/liblbm_b200_bounds.so')
" > $O/bounds_build.log 2>&1
LBM_B200_LIB=$PWD/paper_2001_11806_b200/variants/liblbm_b200_bounds.so timeout 1500 python -m pytest tests -m gpu -q > $O/gpu_tests_bounds_check.log 2>&1; echo "rc=$?" >> $O/gpu_tests_bounds_check.log
OUT=$O bash scripts/gpu_r02zz_profile.sh
