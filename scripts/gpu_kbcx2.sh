mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -k "kbc" > gpurun_out/kx2_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/kx2_tests.log
for c in op_kbc_exact op_kbc27_exact; do
  timeout 300 python bench.py --config $c --steps 20 --warmup 3 --no-probe > gpurun_out/kx2_${c}.json 2> gpurun_out/kx2_${c}.err
done
