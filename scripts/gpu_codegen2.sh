mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "gen_ or generated" > gpurun_out/cg2_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/cg2_tests.log
for c in op_gen_srt27 op_gen_trt op_gen_mrt c4_gen; do
  timeout 300 python bench.py --config $c --steps 20 --warmup 3 --no-probe > gpurun_out/cg2_${c}.json 2> gpurun_out/cg2_${c}.err
done
