# In-kernel links on face-aligned walls (FM_FACEL): link/face tests, then the walled configs with the coordinate
# form vs the mask form (LBM_LINKS_FACES=0) vs the separate link kernel (LBM_LINKS_FUSED=0).
O=gpurun_out/r02z4; mkdir -p $O
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_runtime.py tests/test_gpu_configs.py -m gpu -q \
  -k "link or lk or resume or face or c1_full or c3_cavity" > $O/tests.log 2>&1; echo "rc=$?" >> $O/tests.log
B="python bench.py --steps 50 --warmup 5 --e2e-reps 0 --no-cpu-baseline --no-probe"
for c in fig8_channel_links c3 c3_aa_links c1_f32; do
  timeout 300 $B --config $c > $O/$c.json 2> $O/$c.err
  LBM_LINKS_FACES=0 LBM_LINKS_FUSED=1 timeout 300 $B --config $c > $O/${c}_mask.json 2> $O/${c}_mask.err
  LBM_LINKS_FUSED=0 timeout 300 $B --config $c > $O/${c}_sep.json 2> $O/${c}_sep.err
done
for c in c1_f64; do
  timeout 300 $B --config $c > $O/$c.json 2> $O/$c.err
  timeout 300 $B --config c1_f64_links > $O/${c}_links.json 2> $O/${c}_links.err
done
