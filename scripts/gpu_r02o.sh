mkdir -p gpurun_out/r02o
O=gpurun_out/r02o
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_runtime.py -m gpu -q -k "graph or phase or nccl_self or resume" > $O/tests.log 2>&1; echo "rc=$?" >> $O/tests.log
timeout 900 python bench.py > $O/bench_default.json 2> $O/bench_default.err
for c in c1_f64 c1_f32 c2 c3 c3_aa_links; do
  timeout 300 python bench.py --config $c --steps 50 --warmup 5 --no-cpu-baseline --e2e-reps 2 > $O/${c}.json 2> $O/${c}.err
done
for hm in 0 2; do
  timeout 300 python bench.py --config c4 --nccl-self 1 --halo-mode $hm --steps 30 --warmup 5 --e2e-reps 0 --no-cpu-baseline --no-probe > $O/self_c4_h$hm.json 2> $O/self_c4_h$hm.err
done
