# Round 2 pass f: whole GPU suite (new tests included), smoke, FLOP counts of the ALU-heavy update kernels,
# then the whole suite against the LBM_BOUNDS_CHECK build.
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q --durations=25 > gpurun_out/r02f_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r02f_tests.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02f_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/r02f_smoke.log
MET=smsp__sass_thread_inst_executed_op_dadd_pred_on.sum,smsp__sass_thread_inst_executed_op_dmul_pred_on.sum,smsp__sass_thread_inst_executed_op_dfma_pred_on.sum,smsp__sass_thread_inst_executed_op_fadd_pred_on.sum,smsp__sass_thread_inst_executed_op_fmul_pred_on.sum,smsp__sass_thread_inst_executed_op_ffma_pred_on.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active,gpu__time_duration.sum
for c in c4 c2 c3 c3_aa_links op_cumulant27 op_cumulant19 op_kbc op_kbc27 op_kbc_exact op_kbc27_exact op_mrt op_smagorinsky op_trt; do
  timeout 600 ncu --metrics $MET --clock-control none -k regex:"k_(staged|pull|aa|eso|push)" -s 2 -c 2 --csv --log-file gpurun_out/r02f_${c}_alu.csv python bench.py --config $c --steps 2 --warmup 1 --no-probe --no-cpu-baseline --e2e-reps 0 > /dev/null 2> gpurun_out/r02f_${c}_alu.err
done
python -c "
from paper_2001_11806_b200 import build
build.build(defines=['LBM_BOUNDS_CHECK'], out='paper_2001_11806_b200/variants/liblbm_b200_bounds.so')
" > gpurun_out/r02f_bounds_build.log 2>&1
LBM_B200_LIB=$PWD/paper_2001_11806_b200/variants/liblbm_b200_bounds.so timeout 2400 python -m pytest tests -m gpu -q --durations=10 > gpurun_out/r02f_bounds_check.log 2>&1; echo "rc=$?" >> gpurun_out/r02f_bounds_check.log
