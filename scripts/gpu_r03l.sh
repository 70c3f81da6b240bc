# Flat rows through the low-level kernel ABI too (one helper for lbm_create and lbm_kernel_*): whole GPU suite,
# smoke, default bench line, the paper-shaped lines
O=gpurun_out/r03l; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q > $O/gpu_tests.log 2>&1; echo rc=$? >> $O/gpu_tests.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo rc=$? >> $O/smoke.log
timeout 900 python bench.py > $O/bench_default.log 2>&1; echo rc=$? >> $O/bench_default.log
for c in fig5_srt_pull fig7_trt_aa fig8_channel_links fig8_channel_flags fig10_small c1_f64 c3; do
  timeout 300 python bench.py --config $c --steps 200 --warmup 10 --e2e-reps 0 --no-cpu-baseline 2>>$O/err.log | tail -1 >> $O/bench.jsonl
done
