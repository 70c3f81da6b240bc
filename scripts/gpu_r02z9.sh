# Launch box (bounding box of the non-wall cells) + plane trimming: whole GPU suite, then the walled configs
# with the box vs without (LBM_BOX=0).
O=gpurun_out/r02z9; mkdir -p $O
timeout 2400 python -m pytest tests -m gpu -q -x > $O/gpu_tests.log 2>&1; echo "rc=$?" >> $O/gpu_tests.log
B="python bench.py --steps 50 --warmup 5 --e2e-reps 0 --no-cpu-baseline --no-probe"
for c in fig8_channel_links fig8_channel_flags fig8_channel_inline c3 c3_aa_links c3_aa c3_flags c1_f64 c1_f32 eso_c3; do
  timeout 300 $B --config $c > $O/$c.json 2> $O/$c.err
  LBM_BOX=0 timeout 300 $B --config $c > $O/${c}_nobox.json 2> $O/${c}_nobox.err
done
