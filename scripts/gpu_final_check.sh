# After a rebuild: smoke(), the generated-operator GPU tests, and the new bench lines
mkdir -p gpurun_out
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/fc_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/fc_smoke.log
timeout 900 python -m pytest tests -m gpu -q -k "gen_ or generated or abi" > gpurun_out/fc_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/fc_tests.log
for c in op_gen_mrt27 op_gen_mrt; do
  timeout 300 python bench.py --config $c --steps 20 --warmup 3 --no-probe > gpurun_out/fc_${c}.json 2> gpurun_out/fc_${c}.err
done
