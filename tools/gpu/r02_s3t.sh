timeout 600 python -m pytest tests/test_gpu_kernels.py -m gpu -q -x > gpurun_out/s3t_k.log 2>&1; tail -2 gpurun_out/s3t_k.log
for r in 1 2; do
timeout 600 python tools/step_profile.py c3 3 20 3 > gpurun_out/s3t_sp.log 2>&1
echo "rep $r: $(tail -n 1 gpurun_out/s3t_sp.log)"; grep -E " (29|13|10) m" gpurun_out/s3t_sp.log | cut -c1-90
done
