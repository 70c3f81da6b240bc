# D3Q27 TRT-class kernels: plain vs staged (auto-policy input), AA and pull; then the full GPU suite
mkdir -p gpurun_out
for c in op_trt27 op_srt27 op_gen_srt27 fig7_trt_aa_q27; do
  for p in plain staged; do
    LBM_KERNEL_PATH=$p timeout 300 python bench.py --config $c --steps 20 --warmup 3 --no-probe > gpurun_out/q27_${c}_$p.json 2> gpurun_out/q27_${c}_$p.err
  done
done
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/q27_gpu_tests.log 2>&1; echo "rc=$?" >> gpurun_out/q27_gpu_tests.log
