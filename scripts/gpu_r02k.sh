mkdir -p gpurun_out/r02k
O=gpurun_out/r02k
timeout 1200 python -m pytest tests/test_gpu_parity.py -m gpu -q -k "face or persistent or link or channel or cavity" > $O/tests.log 2>&1; echo "rc=$?" >> $O/tests.log
for c in c1_f64 c1_f64_flags c1_f64_links c1_f64_inline c1_f32 c3 c3_aa fig8_channel_flags; do
  timeout 300 python bench.py --config $c --steps 50 --warmup 5 --no-probe --no-cpu-baseline --e2e-reps 0 > $O/${c}.json 2> $O/${c}.err
done
