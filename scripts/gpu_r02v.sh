# In-kernel links (FM_LINKS) and flag-after-load plain kernels (FM_BULK): tests, then bench lines of the walled
# configs: in-kernel links vs the separate link kernel (LBM_LINKS_FUSED=0), split flags plain vs staged.
O=gpurun_out/r02v; mkdir -p $O
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_runtime.py -m gpu -q \
  -k "link or lk or resume or parity_vs_oracle or staged_and_plain or graph or low_level or face or inline" > $O/tests.log 2>&1; echo "rc=$?" >> $O/tests.log
B="python bench.py --steps 50 --warmup 5 --e2e-reps 0 --no-cpu-baseline --no-probe"
for c in fig8_channel_links c3 c3_aa_links c1_f32 fig8_channel_flags c3_flags c1_f32_flags c3_aa; do
  timeout 300 $B --config $c > $O/$c.json 2> $O/$c.err
  LBM_KERNEL_PATH=plain timeout 300 $B --config $c > $O/${c}_plain.json 2> $O/${c}_plain.err
  LBM_KERNEL_PATH=staged timeout 300 $B --config $c > $O/${c}_staged.json 2> $O/${c}_staged.err
done
for c in fig8_channel_links c3 c3_aa_links c1_f32; do
  LBM_LINKS_FUSED=0 timeout 300 $B --config $c > $O/${c}_sep.json 2> $O/${c}_sep.err
done
