# fp32 on the Fig. 7 domain: flat rows (one-cell even step) vs 2-D blocks (two-cell even step, --block-x 64 or
# LBM_FLAT=0), three alternating repetitions; and the same for the fp32 TRT pull kernel via c1-like pull? (AA only here)
O=gpurun_out/r03n; mkdir -p $O
B="python bench.py --steps 400 --warmup 20 --e2e-reps 0 --no-cpu-baseline --no-probe --config fig7_mrt_aa_f32"
for r in 1 2 3; do
  timeout 300 $B 2>>$O/err.log | tail -1 | sed 's/^{/{"mode": "flat", /' >> $O/bench.jsonl
  LBM_FLAT=0 timeout 300 $B 2>>$O/err.log | tail -1 | sed 's/^{/{"mode": "box_x2", /' >> $O/bench.jsonl
  LBM_FLAT=0 LBM_AA_X2=0 timeout 300 $B 2>>$O/err.log | tail -1 | sed 's/^{/{"mode": "box_onecell", /' >> $O/bench.jsonl
done
