# Round 2, first GPU pass: the new full-step-count config tests, then the whole GPU suite, then the default bench.
mkdir -p gpurun_out
nproc > gpurun_out/r02a_host.txt; grep -m1 "model name" /proc/cpuinfo >> gpurun_out/r02a_host.txt
timeout 1500 python -m pytest tests/test_gpu_configs.py -m gpu -q --durations=20 > gpurun_out/r02a_configs.log 2>&1; echo "rc=$?" >> gpurun_out/r02a_configs.log
timeout 1500 python -m pytest tests -m gpu -q -x --durations=15 --ignore=tests/test_gpu_configs.py > gpurun_out/r02a_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r02a_tests.log
timeout 600 python bench.py > gpurun_out/r02a_bench.json 2> gpurun_out/r02a_bench.err
