#!/bin/bash
# ncu --set full of the dominant kernel of one bench config: plain run first, then ncu.
# usage: scripts/gpu_profile.sh <config> <kernel-regex> <skip> <count> [extra bench args]
set -u
c=$1; k=$2; s=$3; n=$4; shift 4
O=gpurun_out
mkdir -p $O
CMD="python bench.py --config $c --steps 4 --warmup 3 --e2e-reps 0 --no-cpu-baseline $*"
timeout 300 $CMD > $O/plain_$c.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:$k -s $s -c $n -o $O/prof_$c $CMD > $O/ncu_$c.log 2>&1
echo "$c profile rc=$?" >> $O/status.txt
