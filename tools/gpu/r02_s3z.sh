timeout 600 python -m pytest tests/test_gpu_kernels.py -m gpu -q -x > gpurun_out/s3z_k.log 2>&1; tail -2 gpurun_out/s3z_k.log
for t in 1 0; do TN_TC2=$t timeout 300 python tools/mubench.py --m 16 --k 16 --n 5 --iters 5 2>&1 | tail -1 | sed "s/^/tc2=$t /"; done
for r in 1 2; do
timeout 600 python tools/step_profile.py c3 3 20 3 > gpurun_out/s3z_sp.log 2>&1
echo "rep $r: $(tail -n 1 gpurun_out/s3z_sp.log)"; grep -E " (31) m" gpurun_out/s3z_sp.log | cut -c1-90
done
