# EsoTwist split-mode kernels with loads ahead of the flag test: eso tests + eso config lines.
O=gpurun_out/r02z6; mkdir -p $O
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_runtime.py -m gpu -q -k "eso" > $O/tests.log 2>&1; echo "rc=$?" >> $O/tests.log
B="python bench.py --steps 50 --warmup 5 --e2e-reps 0 --no-cpu-baseline --no-probe"
for c in eso_c3 eso_c4 eso_c2; do
  timeout 300 $B --config $c > $O/$c.json 2> $O/$c.err
done
