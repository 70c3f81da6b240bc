# Inline (compiled-in) boundary kernels with the own flag tested after the gathers: tests + inline config lines.
O=gpurun_out/r02z7; mkdir -p $O
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py -m gpu -q -k "inline or low_level or persistent or parity_vs_oracle or c0" > $O/tests.log 2>&1; echo "rc=$?" >> $O/tests.log
B="python bench.py --steps 50 --warmup 5 --e2e-reps 0 --no-cpu-baseline --no-probe"
for c in fig8_channel_inline c3_inline c1_f64_inline c0; do
  timeout 300 $B --config $c > $O/$c.json 2> $O/$c.err
done
