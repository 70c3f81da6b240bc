# ncu --set full of the weakest kernels (next-round targets): KBC D3Q27, cumulant D3Q27 AA, Fig. 8 AA
O=gpurun_out; mkdir -p $O
prof() {  # config kernel-regex skip count
  local C="python bench.py --config $1 --steps 4 --warmup 3 --e2e-reps 0 --no-cpu-baseline --no-probe"
  timeout 300 $C > $O/plain_$1.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$2 -s $3 -c $4 -o $O/prof_$1 $C > $O/ncu_$1.log 2>&1
  echo "prof_$1=$?" >> $O/status_weak.txt
  ncu -i $O/prof_$1.ncu-rep --page raw --csv > $O/prof_$1_raw.csv 2>/dev/null
  ncu -i $O/prof_$1.ncu-rep --page details --csv > $O/prof_$1_details.csv 2>/dev/null
  rm -f $O/prof_$1.ncu-rep
}
prof op_kbc27 k_staged 4 2
prof op_cumulant27 k_staged 4 2
prof fig8_channel_flags k_aa 4 2
cat $O/status_weak.txt
