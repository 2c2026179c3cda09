set -x
timeout 900 python -m pytest tests/test_gpu_loopback.py tests/test_gpu_sparse.py tests/test_gpu_sparse_state.py -m gpu -q -x > gpurun_out/tc2c.log 2>&1; tail -3 gpurun_out/tc2c.log
for r in 1 2; do
  TN_TC2=1 timeout 600 python tools/step_profile.py c3 3 > gpurun_out/sp_ab_tc2_$r.log 2>&1
  TN_TC2=0 timeout 600 python tools/step_profile.py c3 3 > gpurun_out/sp_ab_tc1_$r.log 2>&1
  tail -1 gpurun_out/sp_ab_tc2_$r.log gpurun_out/sp_ab_tc1_$r.log
done
timeout 600 ncu --set full --import-source on --clock-control none -k regex:tc2 -c 1 -o gpurun_out/r02_gemm2_k10n10 python tools/mubench.py --m 23 --k 10 --n 10 --iters 1 > gpurun_out/ncu_tc2.log 2>&1
tail -2 gpurun_out/ncu_tc2.log
