mkdir -p gpurun_out
for c in op_kbc_exact op_kbc27_exact; do
  LBM_B200_LIB=$PWD/paper_2001_11806_b200/liblbm_b200_aa2.so LBM_KERNEL_PATH=plain timeout 300 python bench.py --config $c --steps 20 --warmup 3 --no-probe > gpurun_out/aa2_${c}.json 2> gpurun_out/aa2_${c}.err
done
