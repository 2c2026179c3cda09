timeout 600 python -m pytest tests/test_gpu_kernels.py -m gpu -q -x -k "gathered" > gpurun_out/s3n_k.log 2>&1; tail -2 gpurun_out/s3n_k.log
TN_GATHER_DEBUG=1 timeout 300 python tools/gather_bench.py 16,16,5,k5m11k8m2k3m3 20,10,6,k5m6k2m2k3m12 2>&1 | sort -u
timeout 900 python -m pytest tests/test_gpu_e2e.py -m gpu -q -x > gpurun_out/s3n_e.log 2>&1; tail -2 gpurun_out/s3n_e.log
for r in 1 2; do
timeout 600 python tools/step_profile.py c3 3 20 3 > gpurun_out/s3n_sp.log 2>&1
echo "rep $r: $(tail -n 1 gpurun_out/s3n_sp.log)"; grep -E " (2|31) m" gpurun_out/s3n_sp.log | cut -c1-90
done
