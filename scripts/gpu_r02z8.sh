# Inline kernels after restricting the late own-flag test to D3Q19 fp64.
O=gpurun_out/r02z8; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -k "inline or low_level" > $O/tests.log 2>&1; echo "rc=$?" >> $O/tests.log
B="python bench.py --steps 50 --warmup 5 --e2e-reps 0 --no-cpu-baseline --no-probe"
for c in fig8_channel_inline c3_inline c1_f64_inline; do
  timeout 300 $B --config $c > $O/$c.json 2> $O/$c.err
done
