# Flat-row launch indexing (full x-rows with idle lanes at the row end, nx = 300 of Fig. 5 / 7 / 8): the
# new bit-identity test, the whole GPU suite (odd-extent cases now run through the flat rows), then the
# paper-shaped configs with and without (LBM_FLAT=0), three alternating repetitions on one box
O=gpurun_out/r03h; mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_runtime.py -m gpu -x -q -k flat > $O/flat_tests.log 2>&1; echo rc=$? >> $O/flat_tests.log
timeout 1500 python -m pytest tests -m gpu -x -q > $O/gpu_tests.log 2>&1; echo rc=$? >> $O/gpu_tests.log
B="python bench.py --steps 200 --warmup 10 --e2e-reps 0 --no-cpu-baseline --no-probe"
for r in 1 2 3; do
  for c in fig7_trt_aa fig8_channel_links fig8_channel_flags fig8_channel_inline fig5_srt_pull fig7_trt_aa_q27; do
    for f in 1 0; do
      LBM_FLAT=$f timeout 300 $B --config $c 2>>$O/err.log | tail -1 | sed "s/^{/{\"flat\": $f, /" >> $O/bench.jsonl
    done
  done
done
