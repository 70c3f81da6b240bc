# Whole GPU suite after the in-kernel links / flag-after-load AA changes, smoke, and the walled-config bench lines.
O=gpurun_out/r02w; mkdir -p $O
timeout 1800 python -m pytest tests -m gpu -q > $O/gpu_tests.log 2>&1; echo "rc=$?" >> $O/gpu_tests.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "rc=$?" >> $O/smoke.log
B="python bench.py --steps 50 --warmup 5 --e2e-reps 1 --no-cpu-baseline"
for c in fig8_channel_flags fig8_channel_links fig8_channel_inline c3 c3_aa c3_aa_links c3_flags c1_f32 c1_f32_flags c1_f64 fig7_trt_aa op_kbc27 c4; do
  timeout 300 $B --config $c > $O/$c.json 2> $O/$c.err
done
