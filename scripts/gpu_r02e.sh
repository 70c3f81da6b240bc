mkdir -p gpurun_out
for c in op_kbc27 op_kbc op_kbc_exact op_kbc27_exact; do
  LBM_KERNEL_PATH=staged timeout 300 python bench.py --config $c --steps 20 --warmup 3 --no-probe --no-cpu-baseline --e2e-reps 0 > gpurun_out/r02e_${c}.json 2> gpurun_out/r02e_${c}.err
done
timeout 900 python -m pytest tests -m gpu -q -k "kbc or index_list or link" > gpurun_out/r02e_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r02e_tests.log
