# compute-sanitizer on representative GPU tests: memcheck (out-of-bounds / misaligned global and shared
# accesses), racecheck (shared-memory hazards of the TMA-staged kernels), synccheck.
mkdir -p gpurun_out/r02l
O=gpurun_out/r02l
CS=/usr/local/cuda/bin/compute-sanitizer
K='c0_full or c2_proxy or aa_cumulant_cavity or st_mrt_f32_aa_walls16 or st_kbc_aa_obst or eso_trt_obstacles_odd or lk_trt_f32_obst_aa or push_trt_force_obst_f64'
timeout 1800 $CS --tool memcheck --error-exitcode 99 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "$K" > $O/memcheck.log 2>&1; echo "rc=$?" >> $O/memcheck.log
timeout 1800 $CS --tool racecheck --error-exitcode 99 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "st_mrt_f32_aa_walls16 or st_kbc_aa_obst or st_cumulant_pull_cavity16 or st_eso_mrt_f32_walls16" > $O/racecheck.log 2>&1; echo "rc=$?" >> $O/racecheck.log
timeout 1800 $CS --tool synccheck --error-exitcode 99 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "st_mrt_f32_aa_walls16 or st_kbc_aa_obst" > $O/synccheck.log 2>&1; echo "rc=$?" >> $O/synccheck.log
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -k "face" > $O/faces_tests.log 2>&1; echo "rc=$?" >> $O/faces_tests.log
