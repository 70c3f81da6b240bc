mkdir -p gpurun_out
for c in op_cumulant27 c3_aa eso_c3 push_c3 op_kbc27 c2; do
  LBM_B200_LIB=$PWD/paper_2001_11806_b200/liblbm_b200_sm2.so timeout 300 python bench.py --config $c --steps 20 --warmup 3 --no-probe > gpurun_out/sm2_${c}.json 2> gpurun_out/sm2_${c}.err
done
