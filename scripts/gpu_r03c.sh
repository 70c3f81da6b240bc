# ncu --set full of the C2 odd-step kernels (x2 and one-cell) and of the update-q probe kernels
O=gpurun_out/r03c; mkdir -p $O
C="python bench.py --config c2 --steps 4 --warmup 3 --e2e-reps 0 --no-cpu-baseline --no-probe --graph 0"
timeout 300 $C > $O/plain.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_aa_odd -s 1 -c 1 -o $O/prof_odd_x2 $C > $O/ncu_x2.log 2>&1
LBM_AA_X2=0 timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_aa_odd -s 1 -c 1 -o $O/prof_odd_x1 $C > $O/ncu_x1.log 2>&1
for p in x2 x1; do
  ncu -i $O/prof_odd_$p.ncu-rep --page raw --csv > $O/prof_odd_${p}_raw.csv 2>/dev/null
  ncu -i $O/prof_odd_$p.ncu-rep --page source --csv > $O/prof_odd_${p}_source.csv 2>/dev/null
  python scripts/ncu_brief.py $O/prof_odd_$p.ncu-rep > $O/brief_$p.txt 2>&1
  rm -f $O/prof_odd_$p.ncu-rep
done
