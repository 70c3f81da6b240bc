# Round 2 pass g: staged pull / AA-odd kernels resolve near-wall cells inline (no edge launch): tests of the
# flag paths, then the walled bench lines plain vs staged, and the ALU-bound lines with the alu block.
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py -m gpu -q -k "aa or staged or channel or cavity or obst or c1 or c3 or walls" > gpurun_out/r02g_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r02g_tests.log
for c in fig8_channel_flags c3_aa fig8_channel_links c3_aa_links c1_f64_flags c1_f32_flags c3_flags op_cumulant27 op_kbc_exact op_kbc27_exact op_kbc27 c2; do
  timeout 300 python bench.py --config $c --steps 20 --warmup 3 --no-cpu-baseline --e2e-reps 0 > gpurun_out/r02g_${c}.json 2> gpurun_out/r02g_${c}.err
done
for c in fig8_channel_flags c3_aa c1_f64_flags; do
  LBM_KERNEL_PATH=staged timeout 300 python bench.py --config $c --steps 20 --warmup 3 --no-probe --no-cpu-baseline --e2e-reps 0 > gpurun_out/r02g_${c}_staged.json 2> gpurun_out/r02g_${c}_staged.err
done
