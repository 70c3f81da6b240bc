# In-kernel index-list boundaries (FM_LINKS): link-related GPU tests, then bench lines of the walled configs
# with the in-kernel links against the separate link kernel (LBM_LINKS_FUSED=0), plain and staged paths.
O=gpurun_out/r02u; mkdir -p $O
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_runtime.py tests/test_gpu_configs.py -m gpu -q -x \
  -k "link or resume or lk or c1_full or c3_cavity" > $O/tests.log 2>&1; echo "rc=$?" >> $O/tests.log
B="python bench.py --steps 50 --warmup 5 --e2e-reps 0 --no-cpu-baseline --no-probe"
for c in fig8_channel_links c3 c3_aa_links c1_f32; do
  timeout 300 $B --config $c > $O/$c.json 2> $O/$c.err
  LBM_LINKS_FUSED=0 timeout 300 $B --config $c > $O/${c}_sep.json 2> $O/${c}_sep.err
  LBM_KERNEL_PATH=staged timeout 300 $B --config $c > $O/${c}_staged.json 2> $O/${c}_staged.err
done
L="python bench.py --steps 4 --warmup 3 --e2e-reps 0 --no-cpu-baseline --no-probe"
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 40 --csv --log-file $O/launch_fig8_links.csv $L --config fig8_channel_links > $O/ncu_fig8.log 2>&1
