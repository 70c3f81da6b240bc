# Two cells per thread for the periodic fp32 D3Q19 AA kernels (C2): parity suite, then C2 / eq_inc_c2 with and
# without (LBM_AA_X2=0), three alternating repetitions.
O=gpurun_out/r03a; mkdir -p $O
timeout 900 python -m pytest tests -m gpu -x -q > $O/gpu_tests.log 2>&1; echo rc=$? >> $O/gpu_tests.log
B="python bench.py --steps 100 --warmup 5 --e2e-reps 0 --no-cpu-baseline --no-probe"
for r in 1 2 3; do
for c in c2 eq_inc_c2; do
  LBM_AA_X2=1 timeout 300 $B --config $c > $O/${c}_x2_r$r.json 2> $O/${c}_x2_r$r.err
  LBM_AA_X2=0 timeout 300 $B --config $c > $O/${c}_x1_r$r.json 2> $O/${c}_x1_r$r.err
done
done
