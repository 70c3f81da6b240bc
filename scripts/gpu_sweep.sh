#!/bin/bash
# A/B sweep of library build variants (paper_2001_11806_b200/variants/*.so) over bench configs.
# usage: scripts/gpu_sweep.sh "<configs>" "<variants>" [extra bench args]
set -u
O=gpurun_out; mkdir -p $O
CFGS=$1; VARS=$2; shift 2
for v in $VARS; do
  for c in $CFGS; do
    if [ "$v" = "default" ]; then lib=""; else lib="$PWD/paper_2001_11806_b200/variants/liblbm_$v.so"; fi
    LBM_B200_LIB=$lib timeout 300 python bench.py --config $c --steps 50 --warmup 5 --e2e-reps 0 --no-cpu-baseline "$@" 2>&1 \
      | python -c "import sys,json
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); r=d['roofline']; print('$v $c', round(d['value']), 'MLUPS', round(r['achieved']), 'GB/s', round(r['frac'],3), d['clocks']['sm_mhz'])
    elif 'Error' in l or 'error' in l: print('$v $c ERR', l.strip()[:200])" >> $O/sweep.txt
  done
done
