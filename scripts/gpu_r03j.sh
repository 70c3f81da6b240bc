# Flat rows, final: the bit-identity test (fp32 two-cell cases within rounding), whole GPU suite, smoke, default
# bench line, paper-shaped lines at their defaults (flat rows; fig10_small now graph-launched), and the ncu
# launch metrics + one --set full capture of the Fig. 8 index-list kernels under flat rows
O=gpurun_out/r03j; mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_runtime.py -m gpu -q -k flat > $O/flat_tests.log 2>&1; echo rc=$? >> $O/flat_tests.log
timeout 1500 python -m pytest tests -m gpu -q > $O/gpu_tests.log 2>&1; echo rc=$? >> $O/gpu_tests.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo rc=$? >> $O/smoke.log
timeout 900 python bench.py > $O/bench_default.log 2>&1; echo rc=$? >> $O/bench_default.log
for c in fig5_srt_pull fig7_trt_aa fig7_trt_aa_q27 fig8_channel_flags fig8_channel_links fig8_channel_inline fig10_small c0 c1_f64 c1_f32 c2 c3; do
  timeout 300 python bench.py --config $c --steps 200 --warmup 10 --e2e-reps 1 --no-cpu-baseline 2>>$O/err.log | tail -1 >> $O/bench.jsonl
done
for c in fig7_trt_aa fig8_channel_links; do
  CMD="python bench.py --config $c --steps 6 --warmup 3 --e2e-reps 0 --no-cpu-baseline --no-probe --graph 0"
  timeout 300 $CMD > $O/plain_$c.log 2>&1 && \
  timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,launch__registers_per_thread,launch__grid_size,launch__block_size,sm__warps_active.avg.pct_of_peak_sustained_active --clock-control none -c 14 --csv --log-file $O/${c}_launch_metrics.csv $CMD > $O/ncu_$c.log 2>&1
done
C="python bench.py --config fig8_channel_links --steps 4 --warmup 3 --e2e-reps 0 --no-cpu-baseline --no-probe --graph 0"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_aa -s 6 -c 2 -o $O/prof_fig8_channel_links $C > $O/ncu_full.log 2>&1
ncu -i $O/prof_fig8_channel_links.ncu-rep --page raw --csv > $O/prof_fig8_channel_links_raw.csv 2>/dev/null
ncu -i $O/prof_fig8_channel_links.ncu-rep --page details --csv > $O/prof_fig8_channel_links_details.csv 2>/dev/null
rm -f $O/prof_fig8_channel_links.ncu-rep
