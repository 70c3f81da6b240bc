# Flat rows: diagnostic of the one bit-identity failure (fp32 AA channel with index-list boundaries), and the
# small-domain launch modes (persistent kernel vs CUDA graph vs plain launches) of fig10_small and c0
O=gpurun_out/r03i; mkdir -p $O
timeout 600 python scripts/diag_flat.py > $O/diag.log 2>&1; echo rc=$? >> $O/diag.log
B="python bench.py --steps 200 --warmup 10 --e2e-reps 0 --no-cpu-baseline --no-probe"
for r in 1 2; do
  for g in 2 1 0; do
    for c in fig10_small c0; do
      timeout 300 $B --config $c --graph $g 2>>$O/err.log | tail -1 | sed "s/^{/{\"graph\": $g, /" >> $O/bench.jsonl
    done
  done
done
