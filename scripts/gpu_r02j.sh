# FM_FACES (face-aligned walls): tests, then the walled bench lines.
mkdir -p gpurun_out/r02j
O=gpurun_out/r02j
timeout 1200 python -m pytest tests/test_gpu_parity.py -m gpu -q -k "face or link or aa_slots or streaming or obstacles or cavity or channel" > $O/tests.log 2>&1; echo "rc=$?" >> $O/tests.log
for c in c1_f64_flags c1_f32_flags c3_flags c3_aa fig8_channel_flags c1_f64 c1_f32 c3 c3_aa_links; do
  timeout 300 python bench.py --config $c --steps 30 --warmup 3 --no-probe --no-cpu-baseline --e2e-reps 0 > $O/${c}.json 2> $O/${c}.err
done
for c in c1_f64_flags c3_flags c3_aa fig8_channel_flags; do
  LBM_FACES=0 timeout 300 python bench.py --config $c --steps 30 --warmup 3 --no-probe --no-cpu-baseline --e2e-reps 0 > $O/${c}_nofaces.json 2> $O/${c}_nofaces.err
done
