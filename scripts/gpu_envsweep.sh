#!/bin/bash
# A/B sweep of runtime switches (env assignments) over bench configs.
# usage: scripts/gpu_envsweep.sh "<configs>" "<env-set> <env-set> ..." [extra bench args]
#   env-set: comma-separated assignments, e.g. LBM_STAGED=0 or LBM_STAGED=1,LBM_STAGES=3
set -u
O=gpurun_out; mkdir -p $O
CFGS=$1; SETS=$2; shift 2
for e in $SETS; do
  for c in $CFGS; do
    env $(echo $e | tr ',' ' ') timeout 300 python bench.py --config $c --steps 50 --warmup 5 --e2e-reps 0 --no-cpu-baseline "$@" 2>&1 \
      | python -c "import sys,json
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); r=d['roofline']; print('$e $c', round(d['value']), 'MLUPS', round(r['achieved']), 'GB/s', round(r['frac'],3), d['clocks']['sm_mhz'], d['clocks']['reasons'])
    elif 'Error' in l or 'error' in l: print('$e $c ERR', l.strip()[:200])" >> $O/envsweep.txt
  done
done
cat $O/envsweep.txt
