# GPU check of the generated operators: parity tests + bench lines (plain/staged/auto paths)
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "gen_ or generated or abi" > gpurun_out/cg_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/cg_tests.log
for c in c4 c4_gen c2 c2_gen op_trt op_gen_trt op_mrt op_gen_mrt op_gen_srt27 op_smagorinsky op_gen_smagorinsky; do
  timeout 300 python bench.py --config $c --steps 20 --warmup 3 --no-probe > gpurun_out/cg_${c}.json 2> gpurun_out/cg_${c}.err
done
for c in c4_gen c2_gen op_gen_srt27; do
  for p in plain staged; do
    LBM_KERNEL_PATH=$p timeout 300 python bench.py --config $c --steps 20 --warmup 3 --no-probe > gpurun_out/cg_${c}_$p.json 2> gpurun_out/cg_${c}_$p.err
  done
done
