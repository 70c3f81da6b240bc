# C2: two cells per thread in both AA steps (LBM_AA_X2=1), in the even step only (2), in neither (0);
# three alternating repetitions on one box
O=gpurun_out/r03e; mkdir -p $O
B="python bench.py --steps 100 --warmup 5 --e2e-reps 0 --no-cpu-baseline --no-probe --config c2"
for r in 1 2 3; do
for m in 1 2 0; do
  LBM_AA_X2=$m timeout 300 $B > $O/c2_m${m}_r$r.json 2> $O/c2_m${m}_r$r.err
done
done
