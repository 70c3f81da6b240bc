#!/bin/bash
# Round-2 evidence on one B200: default bench line (C4), reference arm, per-config lines, the launch list
# of the default command, and ncu --set full captures of the dominant kernel of key configs. Each ncu
# command runs only after the same command exited 0 without ncu.
set -u
O=${OUT:-gpurun_out/r02zz}; mkdir -p $O
timeout 900 python bench.py > $O/bench_default.log 2>&1; echo "default=$?" >> $O/status.txt
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > $O/bench_reference.log 2>&1; echo "reference=$?" >> $O/status.txt
for c in c0 c1_f64 c1_f32 c2 c3 c1_f64_flags c1_f32_flags c3_flags c3_aa c3_aa_links eso_c4 eso_c2 eso_c3 push_c4 push_c3 \
         eq_inc_c4 eq_mm_c4 eq_inc_c2 op_trt op_mrt op_smagorinsky op_kbc op_kbc27 op_cumulant19 op_cumulant27 \
         fig5_srt_pull fig7_trt_aa fig7_trt_aa_q27 fig8_channel_flags fig8_channel_links fig10_small \
         c4_gen c2_gen op_gen_trt op_gen_mrt op_gen_smagorinsky op_gen_srt27 op_trt27 op_kbc_exact op_kbc27_exact \
         fig8_channel_inline c1_f64_inline c3_inline; do
  timeout 300 python bench.py --config $c --steps 50 --warmup 5 --e2e-reps 1 --no-cpu-baseline > $O/bench_$c.log 2>&1
  echo "$c=$?" >> $O/status.txt
done
for hm in 0 1 2; do
  for c in c4 c2; do
    timeout 300 python bench.py --config $c --nccl-self 1 --halo-mode $hm --steps 50 --warmup 5 --e2e-reps 0 --no-cpu-baseline > $O/bench_self_${c}_h$hm.log 2>&1
    echo "self_${c}_h$hm=$?" >> $O/status.txt
  done
done
CMD="python bench.py --steps 5 --warmup 3 --e2e-reps 0 --no-cpu-baseline"
timeout 300 $CMD > $O/plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv --log-file $O/launches_c4.csv $CMD > $O/ncu_launch.log 2>&1
echo "launches=$?" >> $O/status.txt
prof() {  # config kernel-regex skip count
  local C="python bench.py --config $1 --steps 4 --warmup 3 --e2e-reps 0 --no-cpu-baseline --no-probe --graph 0"
  timeout 300 $C > $O/plain_$1.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$2 -s $3 -c $4 -o $O/prof_$1 $C > $O/ncu_$1.log 2>&1
  echo "prof_$1=$?" >> $O/status.txt
  ncu -i $O/prof_$1.ncu-rep --page raw --csv > $O/prof_$1_raw.csv 2>/dev/null
  ncu -i $O/prof_$1.ncu-rep --page details --csv > $O/prof_$1_details.csv 2>/dev/null
  rm -f $O/prof_$1.ncu-rep
}
prof c4 k_pull 3 1
prof c2 "k_aa" 4 2
prof c3 "k_pull|k_links" 6 2
prof c1_f32 "k_pull|k_links" 6 2
prof op_cumulant27 "k_aa" 4 2
prof op_kbc27 k_staged 4 2
prof fig8_channel_flags "k_aa" 6 3
prof fig8_channel_links "k_aa" 6 2
prof c3_aa_links "k_aa" 6 2
cat $O/status.txt
