# Round 2 pass c: runtime subsystems (resume, phase timeline), borrowed buffers, configs; then the whole GPU
# suite against the LBM_BOUNDS_CHECK build (built here on the box: the variant does not fit the snapshot).
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_runtime.py tests/test_gpu_parity.py -m gpu -q -k "resume or phase or borrowed or low_level" > gpurun_out/r02c_runtime.log 2>&1; echo "rc=$?" >> gpurun_out/r02c_runtime.log
timeout 900 python -m pytest tests/test_gpu_configs.py -m gpu -q -k viscosity > gpurun_out/r02c_nu.log 2>&1; echo "rc=$?" >> gpurun_out/r02c_nu.log
python -c "
from paper_2001_11806_b200 import build
build.build(defines=['LBM_BOUNDS_CHECK'], out='paper_2001_11806_b200/variants/liblbm_b200_bounds.so')
" > gpurun_out/r02c_bounds_build.log 2>&1
LBM_B200_LIB=$PWD/paper_2001_11806_b200/variants/liblbm_b200_bounds.so timeout 2400 python -m pytest tests -m gpu -q --durations=10 > gpurun_out/r02c_bounds_check.log 2>&1; echo "rc=$?" >> gpurun_out/r02c_bounds_check.log
