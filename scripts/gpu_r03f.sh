# Even-step two-cell kernels for every fp32 D3Q19 periodic AA operator on the plain path: AA tests, then
# c2 / eq_inc_c2 / c2_gen with and without (LBM_AA_X2=0), two alternating repetitions
O=gpurun_out/r03f; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "aa or c2" > $O/gpu_tests.log 2>&1; echo rc=$? >> $O/gpu_tests.log
B="python bench.py --steps 100 --warmup 5 --e2e-reps 0 --no-cpu-baseline --no-probe"
for r in 1 2; do
for c in c2 eq_inc_c2 c2_gen; do
  timeout 300 $B --config $c > $O/${c}_x2_r$r.json 2> $O/${c}_x2_r$r.err
  LBM_AA_X2=0 timeout 300 $B --config $c > $O/${c}_x1_r$r.json 2> $O/${c}_x1_r$r.err
done
done
