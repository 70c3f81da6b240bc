# Launch box with a warp-aligned x start: walled configs, box vs no box, three alternating repetitions.
O=gpurun_out/r02z10; mkdir -p $O
B="python bench.py --steps 50 --warmup 5 --e2e-reps 0 --no-cpu-baseline --no-probe"
for r in 1 2 3; do
for c in fig8_channel_links fig8_channel_inline c3 c3_flags c3_aa_links c1_f32; do
  timeout 300 $B --config $c > $O/${c}_r$r.json 2> $O/${c}_r$r.err
  LBM_BOX=0 timeout 300 $B --config $c > $O/${c}_nobox_r$r.json 2> $O/${c}_nobox_r$r.err
done
done
