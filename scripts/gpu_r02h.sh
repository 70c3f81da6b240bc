# Round 2 pass h: the unit-rate D3Q27 cumulant kernels (C3's rates): tests, bench lines, FLOP counts.
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py -m gpu -q -k "cumulant or c3 or cum" > gpurun_out/r02h_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r02h_tests.log
for c in c3 c3_aa c3_aa_links c3_flags op_cumulant27 eso_c3 push_c3 fig8_channel_flags; do
  timeout 300 python bench.py --config $c --steps 20 --warmup 3 --no-cpu-baseline --e2e-reps 0 > gpurun_out/r02h_${c}.json 2> gpurun_out/r02h_${c}.err
done
for c in c3 op_cumulant27; do
  LBM_CUMULANT_GENERAL=1 timeout 300 python bench.py --config $c --steps 20 --warmup 3 --no-probe --no-cpu-baseline --e2e-reps 0 > gpurun_out/r02h_${c}_general.json 2> gpurun_out/r02h_${c}_general.err
  LBM_KERNEL_PATH=staged timeout 300 python bench.py --config $c --steps 20 --warmup 3 --no-probe --no-cpu-baseline --e2e-reps 0 > gpurun_out/r02h_${c}_staged.json 2> gpurun_out/r02h_${c}_staged.err
  LBM_KERNEL_PATH=plain timeout 300 python bench.py --config $c --steps 20 --warmup 3 --no-probe --no-cpu-baseline --e2e-reps 0 > gpurun_out/r02h_${c}_plain.json 2> gpurun_out/r02h_${c}_plain.err
done
MET=smsp__sass_thread_inst_executed_op_dadd_pred_on.sum,smsp__sass_thread_inst_executed_op_dmul_pred_on.sum,smsp__sass_thread_inst_executed_op_dfma_pred_on.sum,smsp__sass_thread_inst_executed_op_fadd_pred_on.sum,smsp__sass_thread_inst_executed_op_fmul_pred_on.sum,smsp__sass_thread_inst_executed_op_ffma_pred_on.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active,gpu__time_duration.sum
for c in c3 c3_aa_links op_cumulant27; do
  timeout 600 ncu --metrics $MET --clock-control none -k regex:"k_(staged|pull|aa|eso|push)" -s 2 -c 2 --csv --log-file gpurun_out/r02h_${c}_alu.csv python bench.py --config $c --steps 2 --warmup 1 --no-probe --no-cpu-baseline --e2e-reps 0 > /dev/null 2> gpurun_out/r02h_${c}_alu.err
done
