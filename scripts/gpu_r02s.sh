# D3Q27 KBC staged with 7 consumer warps (no spills at 168-register cap) and tree-summed moments in the
# unit-rate cumulant: tests + bench lines.
mkdir -p gpurun_out/r02s
O=gpurun_out/r02s
timeout 1200 python -m pytest tests/test_gpu_parity.py -m gpu -q -k "kbc or cumulant or cum" > $O/tests.log 2>&1; echo "rc=$?" >> $O/tests.log
for c in op_kbc27 op_kbc27_exact op_cumulant27 c3 c3_aa_links op_kbc; do
  timeout 300 python bench.py --config $c --steps 30 --warmup 3 --no-cpu-baseline --e2e-reps 0 > $O/${c}.json 2> $O/${c}.err
done
LBM_KERNEL_PATH=staged timeout 300 python bench.py --config op_kbc27_exact --steps 20 --warmup 3 --no-cpu-baseline --no-probe --e2e-reps 0 > $O/op_kbc27_exact_staged.json 2> $O/op_kbc27_exact_staged.err
