set -x
timeout 600 python -m pytest tests/test_gpu_kernels.py -m gpu -q -x -k "mn_ or gathered_runs or tensor_core or scaled" > gpurun_out/s2o_k.log 2>&1; tail -15 gpurun_out/s2o_k.log
timeout 900 python -m pytest tests/test_gpu_e2e.py tests/test_gpu_loopback.py -m gpu -q -x > gpurun_out/s2o_e2e.log 2>&1; tail -5 gpurun_out/s2o_e2e.log
for r in 1 2; do for m in 0 1; do
TN_NO_MN_X=$m
if [ $m = 1 ]; then export TN_NO_MN=1; else unset TN_NO_MN; fi
timeout 600 python tools/step_profile.py c3 3 20 3 > gpurun_out/s2o_sp_nomn${m}_$r.log 2>&1
echo "nomn=$m rep $r: $(tail -n 1 gpurun_out/s2o_sp_nomn${m}_$r.log)"
done; done
unset TN_NO_MN
paste <(cut -c1-100 gpurun_out/s2o_sp_nomn0_1.log) <(cut -c40-62 gpurun_out/s2o_sp_nomn1_1.log)
