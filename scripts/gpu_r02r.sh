mkdir -p gpurun_out/r02r
O=gpurun_out/r02r
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py -m gpu -q -k "mrt or c2" > $O/tests.log 2>&1; echo "rc=$?" >> $O/tests.log
for c in c2 op_mrt eso_c2 fig10_small eq_inc_c2 c2_gen; do
  timeout 300 python bench.py --config $c --steps 50 --warmup 5 --no-cpu-baseline --e2e-reps 2 > $O/${c}.json 2> $O/${c}.err
done
for c in c2 eso_c2; do
  LBM_KERNEL_PATH=staged timeout 300 python bench.py --config $c --steps 50 --warmup 5 --no-cpu-baseline --no-probe --e2e-reps 0 > $O/${c}_staged.json 2> $O/${c}_staged.err
done
