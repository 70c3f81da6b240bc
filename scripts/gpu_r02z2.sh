# Sweeps on variant builds (built on the box): AA register caps (MinBlocks 4 / 2) for C2's fp32 shear-MRT AA
# kernels, and 7 consumer warps for every fp64 staged kernel.
O=gpurun_out/r02z2; mkdir -p $O
B="python bench.py --steps 50 --warmup 5 --e2e-reps 0 --no-cpu-baseline --no-probe"
VD=paper_2001_11806_b200/variants
python -c "
from paper_2001_11806_b200 import build
build.build(defines=['LBM_MINB_OVERRIDE_AA=4'], out='$VD/aa4.so')
build.build(defines=['LBM_MINB_OVERRIDE_AA=2'], out='$VD/aa2.so')
build.build(defines=['LBM_STAGED_BT224_F64'], out='$VD/bt224.so')
" > $O/build.log 2>&1
for c in c2 eso_c2 fig7_trt_aa; do
  timeout 300 $B --config $c > $O/$c.json 2> $O/$c.err
  LBM_B200_LIB=$PWD/$VD/aa4.so timeout 300 $B --config $c > $O/${c}_aa4.json 2> $O/${c}_aa4.err
  LBM_B200_LIB=$PWD/$VD/aa2.so timeout 300 $B --config $c > $O/${c}_aa2.json 2> $O/${c}_aa2.err
done
for c in op_kbc op_mrt op_smagorinsky op_kbc27 op_gen_mrt; do
  timeout 300 $B --config $c > $O/$c.json 2> $O/$c.err
  LBM_B200_LIB=$PWD/$VD/bt224.so timeout 300 $B --config $c > $O/${c}_bt224.json 2> $O/${c}_bt224.err
done
