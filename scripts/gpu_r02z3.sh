# z-marching AA kernels: tests, then C2 / fp64 TRT AA lines with LBM_ZMARCH=1 vs 0, and KZ / MinBlocks variants.
O=gpurun_out/r02z3; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "zmarch" > $O/tests.log 2>&1; echo "rc=$?" >> $O/tests.log
B="python bench.py --steps 50 --warmup 5 --e2e-reps 0 --no-cpu-baseline --no-probe"
VD=paper_2001_11806_b200/variants
for c in c2 op_trt fig7_trt_aa c2_gen eq_inc_c2; do
  LBM_ZMARCH=0 timeout 300 $B --config $c > $O/${c}_zm0.json 2> $O/${c}_zm0.err
  LBM_ZMARCH=1 timeout 300 $B --config $c > $O/${c}_zm1.json 2> $O/${c}_zm1.err
done
python -c "
from paper_2001_11806_b200 import build
build.build(defines=['LBM_ZM_KZ=8'], out='$VD/kz8.so')
build.build(defines=['LBM_ZM_KZ=2'], out='$VD/kz2.so')
build.build(defines=['LBM_ZM_MINB=3'], out='$VD/zmb3.so')
" > $O/build.log 2>&1
for v in kz8 kz2 zmb3; do
  for c in c2 op_trt; do
    LBM_ZMARCH=1 LBM_B200_LIB=$PWD/$VD/$v.so timeout 300 $B --config $c > $O/${c}_$v.json 2> $O/${c}_$v.err
  done
done
