timeout 1200 python -m pytest tests/test_gpu_e2e.py tests/test_gpu_loopback.py tests/test_gpu_sparse_state.py -m gpu -q -x > gpurun_out/s3f_t.log 2>&1; tail -2 gpurun_out/s3f_t.log
for r in 1 2 3; do for v in level serial; do
if [ $v = serial ]; then export TN_COMMON_SERIAL=1; else unset TN_COMMON_SERIAL; fi
timeout 600 python tools/step_profile.py c3 3 20 3 > gpurun_out/s3f_sp_${v}_$r.log 2>&1
echo "$v rep $r: $(tail -n 1 gpurun_out/s3f_sp_${v}_$r.log)"
done; done
