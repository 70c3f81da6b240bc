#!/bin/bash
# bench every BASELINE config on one B200 + ncu evidence for the default (c4) workload
set -u
O=gpurun_out
mkdir -p $O
timeout 600 python bench.py > $O/bench_c4_default.log 2>&1; echo "c4=$?" >> $O/status.txt
for c in c0 c1_f64 c1_f32 c2 c3; do
  timeout 300 python bench.py --config $c --steps 100 --warmup 5 --e2e-reps 1 --no-cpu-baseline > $O/bench_$c.log 2>&1; echo "$c=$?" >> $O/status.txt
done
CMD="python bench.py --steps 5 --warmup 3 --e2e-reps 0 --no-cpu-baseline"
timeout 300 $CMD > $O/plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv --log-file $O/launches.csv $CMD > $O/ncu_launch.log 2>&1; echo "launches=$?" >> $O/status.txt
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_pull -s 3 -c 1 -o $O/prof_c4 $CMD > $O/ncu_full.log 2>&1; echo "ncufull=$?" >> $O/status.txt
cat $O/status.txt
