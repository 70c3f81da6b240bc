# C2 two-cells-per-thread kernels: new parity cases, then ncu --set full of both C2 kernels (x2) and the
# one-cell kernels for comparison
O=gpurun_out/r03b; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "c2 or aa_slab" > $O/gpu_tests.log 2>&1; echo rc=$? >> $O/gpu_tests.log
C="python bench.py --config c2 --steps 4 --warmup 3 --e2e-reps 0 --no-cpu-baseline --no-probe"
timeout 300 $C > $O/plain.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_aa -s 6 -c 2 -o $O/prof_c2_x2 $C > $O/ncu_x2.log 2>&1
LBM_AA_X2=0 timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_aa -s 6 -c 2 -o $O/prof_c2_x1 $C > $O/ncu_x1.log 2>&1
for p in x2 x1; do
  ncu -i $O/prof_c2_$p.ncu-rep --page raw --csv > $O/prof_c2_${p}_raw.csv 2>/dev/null
  ncu -i $O/prof_c2_$p.ncu-rep --page details --csv > $O/prof_c2_${p}_details.csv 2>/dev/null
  python scripts/ncu_brief.py $O/prof_c2_$p.ncu-rep > $O/brief_$p.txt 2>&1
  rm -f $O/prof_c2_$p.ncu-rep
done
