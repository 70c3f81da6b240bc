# ncu --set full of C2 (shear-only MRT fp32 AA, plain), C3 (in-kernel links pull), Fig. 8 (in-kernel links AA)
O=gpurun_out/r02x; mkdir -p $O
prof() {  # config kernel-regex skip count
  local C="python bench.py --config $1 --steps 4 --warmup 3 --e2e-reps 0 --no-cpu-baseline --no-probe"
  timeout 300 $C > $O/plain_$1.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$2 -s $3 -c $4 -o $O/prof_$1 $C > $O/ncu_$1.log 2>&1
  echo "prof_$1=$?" >> $O/status.txt
  ncu -i $O/prof_$1.ncu-rep --page raw --csv > $O/prof_$1_raw.csv 2>/dev/null
  ncu -i $O/prof_$1.ncu-rep --page details --csv > $O/prof_$1_details.csv 2>/dev/null
  ncu -i $O/prof_$1.ncu-rep --page source --csv > $O/prof_$1_source.csv 2>/dev/null
  rm -f $O/prof_$1.ncu-rep
}
prof c2 "k_aa" 4 2
prof c3 "k_pull|k_links" 4 2
prof fig8_channel_links "k_aa" 4 2
