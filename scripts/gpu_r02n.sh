mkdir -p gpurun_out/r02n
O=gpurun_out/r02n
for hm in 0 1 2; do
  timeout 300 python bench.py --config c4 --nccl-self 1 --halo-mode $hm --steps 30 --warmup 5 --e2e-reps 0 --no-cpu-baseline --no-probe > $O/self_c4_h$hm.json 2> $O/self_c4_h$hm.err
done
timeout 300 python bench.py --config c1_f32 --graph 1 --steps 50 --warmup 5 --e2e-reps 0 --no-cpu-baseline --no-probe > $O/c1_f32_graph.json 2> $O/c1_f32_graph.err
timeout 300 python bench.py --config c1_f32 --steps 50 --warmup 5 --e2e-reps 0 --no-cpu-baseline --no-probe > $O/c1_f32.json 2> $O/c1_f32.err
timeout 300 python bench.py --config c2 --graph 1 --steps 50 --warmup 5 --e2e-reps 0 --no-cpu-baseline --no-probe > $O/c2_graph.json 2> $O/c2_graph.err
