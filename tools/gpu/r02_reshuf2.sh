# raw-box A reshuffle warps A/B (TN_RESHUF_WARPS 2 / 4 / 6), interleaved on one box
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_e2e.py -x -q -k "gather or raw or gathered" > gpurun_out/rs2_tests.log 2>&1; tail -1 gpurun_out/rs2_tests.log
TN_RESHUF_WARPS=2 timeout 900 python -m pytest tests/test_gpu_kernels.py -x -q -k "raw" > gpurun_out/rs2_tests2.log 2>&1; tail -1 gpurun_out/rs2_tests2.log
for r in 1 2; do
for v in 2 4 6; do
  TN_RESHUF_WARPS=$v timeout 300 python tools/step_profile.py c3 3 20 3 > gpurun_out/rs2_${v}_$r.log 2>&1
  echo "w=$v r=$r $(tail -1 gpurun_out/rs2_${v}_$r.log | cut -c1-160)"
  grep -E "^ +(4|13|18|25) m" gpurun_out/rs2_${v}_$r.log | awk '{printf "%s:%s ", $1, $11} END {print ""}'
done; done
