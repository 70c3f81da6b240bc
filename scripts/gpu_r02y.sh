# L2::256B prefetch-size hint on the plain kernels' population loads (variant library) vs the default build.
O=gpurun_out/r02y; mkdir -p $O
B="python bench.py --steps 50 --warmup 5 --e2e-reps 0 --no-cpu-baseline --no-probe"
python -c "from paper_2001_11806_b200 import build; build.build(defines=['LBM_L2_PREFETCH=256'], out='paper_2001_11806_b200/variants/liblbm_b200_l2pf.so')" > $O/build.log 2>&1
V=$PWD/paper_2001_11806_b200/variants/liblbm_b200_l2pf.so
for c in c2 c1_f32 c4 c3 fig7_trt_aa c3_aa_links op_cumulant27 c1_f64; do
  timeout 300 $B --config $c > $O/$c.json 2> $O/$c.err
  LBM_B200_LIB=$V timeout 300 $B --config $c > $O/${c}_l2pf.json 2> $O/${c}_l2pf.err
done
