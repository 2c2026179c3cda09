timeout 600 python -m pytest tests/test_gpu_kernels.py -m gpu -q -x -k "gathered" > gpurun_out/s3q_k.log 2>&1; tail -2 gpurun_out/s3q_k.log
for v in 1 0; do TN_TC2_INTER=$v timeout 300 python tools/gather_bench.py 23,7,9,k2m4k5m19 27,4,4,k2m6k2m21 2>&1 | sed "s/^/inter_tc2=$v /"; done
timeout 900 python -m pytest tests/test_gpu_e2e.py -m gpu -q -x > gpurun_out/s3q_e.log 2>&1; tail -2 gpurun_out/s3q_e.log
for r in 1 2; do for v in 1 0; do
TN_TC2_INTER=$v timeout 600 python tools/step_profile.py c3 3 20 3 > gpurun_out/s3q_sp.log 2>&1
echo "inter_tc2=$v rep $r: $(tail -n 1 gpurun_out/s3q_sp.log)"; grep -E " (26) m" gpurun_out/s3q_sp.log | cut -c1-90
done; done
