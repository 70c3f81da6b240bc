# Bounds-check build (LBM_BOUNDS_CHECK: every population / flag / link index asserted in the kernels) with the
# flat-row launch indexing: whole GPU suite through it
O=gpurun_out/r03k; mkdir -p $O
python -c "
from paper_2001_11806_b200 import build
build.build(defines=['LBM_BOUNDS_CHECK'], out='paper_2001_11806_b200/variants/liblbm_b200_bounds.so')
" > $O/bounds_build.log 2>&1
LBM_B200_LIB=$PWD/paper_2001_11806_b200/variants/liblbm_b200_bounds.so timeout 1500 python -m pytest tests -m gpu -q > $O/gpu_tests_bounds_check.log 2>&1; echo "rc=$?" >> $O/gpu_tests_bounds_check.log
