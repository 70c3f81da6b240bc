mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -k "push or cum" > gpurun_out/pp_tests.log 2>&1; echo "rc=$?" >> gpurun_out/pp_tests.log
for c in push_c3 c3_aa eso_c3 op_cumulant27; do
  timeout 300 python bench.py --config $c --steps 20 --warmup 3 --no-probe > gpurun_out/pp_$c.json 2>&1
done
