mkdir -p gpurun_out
timeout 600 python scripts/probes.py > gpurun_out/r02d_probes.json 2> gpurun_out/r02d_probes.err
timeout 900 python -m pytest tests -m gpu -q -k "kbc" > gpurun_out/r02d_kbc_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r02d_kbc_tests.log
for c in op_kbc27 op_kbc op_kbc_exact op_kbc27_exact; do
  timeout 300 python bench.py --config $c --steps 20 --warmup 3 --no-probe --no-cpu-baseline --e2e-reps 0 > gpurun_out/r02d_${c}.json 2> gpurun_out/r02d_${c}.err
done
for c in op_kbc_exact op_kbc27_exact; do
  LBM_KERNEL_PATH=staged timeout 300 python bench.py --config $c --steps 20 --warmup 3 --no-probe --no-cpu-baseline --e2e-reps 0 > gpurun_out/r02d_${c}_staged.json 2> gpurun_out/r02d_${c}_staged.err
done
