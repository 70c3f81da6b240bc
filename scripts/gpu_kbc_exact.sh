set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "kbc or abi" > gpurun_out/kx_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/kx_tests.log
for c in op_kbc op_kbc_exact op_kbc27 op_kbc27_exact; do
  for p in auto plain staged; do
    LBM_KERNEL_PATH=$p timeout 300 python bench.py --config $c --steps 20 --warmup 3 --no-probe > gpurun_out/kx_${c}_$p.json 2> gpurun_out/kx_${c}_$p.err
  done
done
