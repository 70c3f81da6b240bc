mkdir -p gpurun_out/r02m
O=gpurun_out/r02m
timeout 900 python -m pytest tests/test_gpu_runtime.py -m gpu -q -k "async or resume" > $O/tests.log 2>&1; echo "rc=$?" >> $O/tests.log
timeout 900 python bench.py > $O/bench_default.json 2> $O/bench_default.err
for c in c1_f64 c2 c3; do
  timeout 300 python bench.py --config $c --steps 50 --warmup 5 --no-probe --no-cpu-baseline > $O/${c}.json 2> $O/${c}.err
done
