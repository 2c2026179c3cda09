set -x
# CTA-pair GEMM: first contact under a short timeout (a wrong barrier protocol hangs)
timeout 240 python -m pytest tests/test_gpu_kernels.py -m gpu -q -x -k "tensor_core_vs_oracle or scaled_gemm" > gpurun_out/tc2a.log 2>&1
echo "rc=$?" >> gpurun_out/tc2a.log
tail -5 gpurun_out/tc2a.log
if grep -q "passed" gpurun_out/tc2a.log && ! grep -q "failed" gpurun_out/tc2a.log; then
  timeout 600 python tools/mubench.py --m 23 --k 6-10 --n 7-10 --iters 5 > gpurun_out/mb_tc2.txt 2>&1
  TN_TC2=0 timeout 600 python tools/mubench.py --m 23 --k 6-10 --n 7-10 --iters 5 > gpurun_out/mb_tc1.txt 2>&1
  timeout 600 python tools/step_profile.py c3 3 > gpurun_out/sp_tc2_c3.log 2>&1
  cat gpurun_out/mb_tc2.txt gpurun_out/mb_tc1.txt
fi
timeout 300 python tools/debug_sparse_shard.py > gpurun_out/dbg_sparse_shard.log 2>&1
tail -30 gpurun_out/dbg_sparse_shard.log
timeout 900 python -m pytest tests/test_gpu_e2e.py -m gpu -q -k "policies or c2_reduced or random_small or fused_permutation or recompute_on_halves" > gpurun_out/tc2b.log 2>&1
tail -5 gpurun_out/tc2b.log
