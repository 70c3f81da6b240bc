mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -k "cum" > gpurun_out/cu2_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/cu2_tests.log
for c in op_cumulant27 c3_aa_links c3_aa eso_c3 push_c3 c3 c3_periodic; do
  timeout 300 python bench.py --config $c --steps 20 --warmup 3 --no-probe > gpurun_out/cu2_${c}.json 2> gpurun_out/cu2_${c}.err
done
