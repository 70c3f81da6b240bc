# Fig. 8 AA-with-walls breakdown: bench lines of the boundary variants, per-launch times (ncu launch
# list) of the walled and periodic AA steps; ncu --set full of the 7-warp D3Q27 KBC staged kernel.
O=gpurun_out/r02t; mkdir -p $O
B="python bench.py --steps 50 --warmup 5 --e2e-reps 0 --no-cpu-baseline --no-probe"
for c in fig7_trt_aa fig8_channel_flags fig8_channel_links fig8_channel_inline; do
  timeout 300 $B --config $c > $O/$c.json 2> $O/$c.err
done
LBM_FACES=1 timeout 300 $B --config fig8_channel_flags > $O/fig8_faces.json 2> $O/fig8_faces.err
LBM_KERNEL_PATH=plain timeout 300 $B --config fig8_channel_flags > $O/fig8_flags_plain.json 2> $O/fig8_flags_plain.err
LBM_KERNEL_PATH=plain timeout 300 $B --config fig8_channel_links > $O/fig8_links_plain.json 2> $O/fig8_links_plain.err
L="python bench.py --steps 4 --warmup 3 --e2e-reps 0 --no-cpu-baseline --no-probe"
for c in fig7_trt_aa fig8_channel_flags fig8_channel_links; do
  timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 60 --csv --log-file $O/launch_$c.csv $L --config $c > $O/ncu_$c.log 2>&1
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_staged -s 4 -c 1 -o $O/prof_op_kbc27 $L --config op_kbc27 > $O/ncu_kbc27.log 2>&1
ncu -i $O/prof_op_kbc27.ncu-rep --page raw --csv > $O/prof_op_kbc27_raw.csv 2>/dev/null
ncu -i $O/prof_op_kbc27.ncu-rep --page details --csv > $O/prof_op_kbc27_details.csv 2>/dev/null
rm -f $O/prof_op_kbc27.ncu-rep
