mkdir -p gpurun_out
timeout 900 python scripts/diag_nu.py > gpurun_out/r02b_nu.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -k "low_level or borrowed" > gpurun_out/r02b_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r02b_tests.log
