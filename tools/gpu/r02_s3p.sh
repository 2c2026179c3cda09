timeout 1200 python -m pytest tests/test_gpu_e2e.py tests/test_gpu_loopback.py -m gpu -q -x > gpurun_out/s3p_t.log 2>&1; tail -2 gpurun_out/s3p_t.log
for r in 1 2; do for v in fold nofold; do
if [ $v = nofold ]; then export TN_NO_FOLD=1; else unset TN_NO_FOLD; fi
timeout 600 python tools/step_profile.py c3 3 20 3 > gpurun_out/s3p_sp.log 2>&1
echo "$v rep $r: $(tail -n 1 gpurun_out/s3p_sp.log)"; grep -E " (14|28) m" gpurun_out/s3p_sp.log | cut -c1-90
done; done
