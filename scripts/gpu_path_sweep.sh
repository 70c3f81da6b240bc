# plain vs staged for the walled / non-BASELINE workloads (auto-policy inputs)
mkdir -p gpurun_out
for c in c3_flags c3_aa eso_c3 push_c3 c1_f32_flags push_c4 eso_c4; do
  for p in plain staged; do
    LBM_KERNEL_PATH=$p timeout 300 python bench.py --config $c --steps 20 --warmup 3 --no-probe > gpurun_out/ps_${c}_$p.json 2>&1
  done
done
