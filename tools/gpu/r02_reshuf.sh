# raw-box A reshuffle with 6 warps (was 2): parity tests of the gathered GEMMs, then the C3 step profile twice
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_e2e.py -x -q -k "gather or raw or gathered" > gpurun_out/rs_tests.log 2>&1; tail -2 gpurun_out/rs_tests.log
for r in 1 2; do
  timeout 300 python tools/step_profile.py c3 3 20 3 > gpurun_out/rs_sp_$r.log 2>&1
  tail -1 gpurun_out/rs_sp_$r.log
  grep -E "^ +(4|13|18|25|30) m" gpurun_out/rs_sp_$r.log
done
