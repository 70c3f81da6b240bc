# Asynchronous-copy (cp.async) persistent AA kernels, LBM_AA_ASYNC=1: AA parity tests through them, then
# C2 / op_trt (fp64 AA 512^3) / fig7 (fp64 AA 300x100x100) with and without, two alternating repetitions
O=gpurun_out/r03d; mkdir -p $O
LBM_AA_ASYNC=1 timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "aa" > $O/gpu_tests.log 2>&1; echo rc=$? >> $O/gpu_tests.log
B="python bench.py --steps 100 --warmup 5 --e2e-reps 0 --no-cpu-baseline --no-probe"
for r in 1 2; do
for c in c2 op_trt fig7_trt_aa; do
  LBM_AA_ASYNC=1 timeout 300 $B --config $c > $O/${c}_async_r$r.json 2> $O/${c}_async_r$r.err
  LBM_AA_ASYNC=0 timeout 300 $B --config $c > $O/${c}_base_r$r.json 2> $O/${c}_base_r$r.err
done
done
