# Launch lists (kernel durations) of the Fig. 7 periodic AA run and the Fig. 8 channel runs, plain launches
O=gpurun_out/r03g; mkdir -p $O
for c in fig7_trt_aa fig8_channel_links fig8_channel_flags; do
  CMD="python bench.py --config $c --steps 6 --warmup 3 --e2e-reps 0 --no-cpu-baseline --no-probe --graph 0"
  timeout 300 $CMD > $O/plain_$c.log 2>&1 && \
  timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__warps_active.avg.pct_of_peak_sustained_active,launch__registers_per_thread,launch__grid_size,launch__block_size --clock-control none -c 60 --csv --log-file $O/launches_$c.csv $CMD > $O/ncu_$c.log 2>&1
  echo "$c=$?" >> $O/status.txt
done
