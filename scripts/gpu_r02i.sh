# Kernel-path sweep for the unit-rate D3Q27 cumulant (AA / EsoTwist / push patterns, flags and links).
mkdir -p gpurun_out
for c in c3_aa c3_aa_links eso_c3 op_cumulant27 push_c3; do
  for p in plain staged; do
    LBM_KERNEL_PATH=$p timeout 300 python bench.py --config $c --steps 20 --warmup 3 --no-probe --no-cpu-baseline --e2e-reps 0 > gpurun_out/r02i_${c}_${p}.json 2> gpurun_out/r02i_${c}_${p}.err
  done
done
