# Link / resume / config GPU tests after removing the coordinate-link kernels.
O=gpurun_out/r02z5; mkdir -p $O
timeout 1800 python -m pytest tests/test_gpu_parity.py tests/test_gpu_runtime.py -m gpu -q -k "link or lk or resume" > $O/tests.log 2>&1; echo "rc=$?" >> $O/tests.log
