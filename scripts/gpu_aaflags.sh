mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -k "aa or eso" > gpurun_out/af_tests.log 2>&1; echo "rc=$?" >> gpurun_out/af_tests.log
for c in fig8_channel_flags fig7_trt_aa c4 c2; do
  timeout 300 python bench.py --config $c --steps 20 --warmup 3 --no-probe > gpurun_out/af_$c.json 2>&1
done
