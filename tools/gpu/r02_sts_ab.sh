# 32-bit shared stores in the GEMM epilogues: parity tests, then interleaved A/B vs ab_old/ (previous build)
timeout 1200 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_e2e.py -x -q > gpurun_out/sts_tests.log 2>&1; tail -1 gpurun_out/sts_tests.log
for r in 1 2 3; do
  timeout 300 python tools/step_profile.py c3 3 20 3 > gpurun_out/sts_new_$r.log 2>&1
  (cd ab_old && timeout 300 python tools/step_profile.py c3 3 20 3 > ../gpurun_out/sts_old_$r.log 2>&1)
  for v in new old; do
    echo "$v r=$r $(tail -1 gpurun_out/sts_${v}_$r.log | cut -c1-150)"
  done
done
