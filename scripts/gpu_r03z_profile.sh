#!/bin/bash
# Final-kernel evidence for the default (C4) command after the flat-rows change: launch list and one
# ncu --set full capture of the dominant kernel. Each ncu command runs only after the same command
# exited 0 without ncu.
set -u
O=${OUT:-gpurun_out/r03z}; mkdir -p $O
CMD="python bench.py --steps 5 --warmup 3 --e2e-reps 0 --no-cpu-baseline"
timeout 300 $CMD > $O/plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv --log-file $O/launches_c4.csv $CMD > $O/ncu_launch.log 2>&1
echo "launches=$?" >> $O/status.txt
C="python bench.py --config c4 --steps 4 --warmup 3 --e2e-reps 0 --no-cpu-baseline --no-probe --graph 0"
timeout 300 $C > $O/plain_c4.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_ -s 3 -c 1 -o $O/prof_c4 $C > $O/ncu_c4.log 2>&1
echo "prof_c4=$?" >> $O/status.txt
ncu -i $O/prof_c4.ncu-rep --page raw --csv > $O/prof_c4_raw.csv 2>/dev/null
ncu -i $O/prof_c4.ncu-rep --page details --csv > $O/prof_c4_details.csv 2>/dev/null
rm -f $O/prof_c4.ncu-rep
cat $O/status.txt
