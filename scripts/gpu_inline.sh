mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "inline or abi" > gpurun_out/in_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/in_tests.log
for c in fig8_channel_flags fig8_channel_inline fig8_channel_links c1_f64_flags c1_f64_inline c1_f64 c3_flags c3_inline c3; do
  timeout 300 python bench.py --config $c --steps 20 --warmup 3 --no-probe > gpurun_out/in_${c}.json 2> gpurun_out/in_${c}.err
done
