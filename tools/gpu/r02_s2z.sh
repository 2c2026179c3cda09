timeout 1200 python -m pytest tests/test_gpu_e2e.py tests/test_gpu_loopback.py tests/test_gpu_sparse.py tests/test_gpu_sparse_state.py -m gpu -q -x > gpurun_out/s2z_t.log 2>&1; tail -3 gpurun_out/s2z_t.log
for r in 1 2; do for v in fold nofold; do
if [ $v = nofold ]; then export TN_NO_FOLD=1; else unset TN_NO_FOLD; fi
timeout 600 python tools/step_profile.py c3 3 20 3 > gpurun_out/s2z_sp_${v}_$r.log 2>&1
echo "$v rep $r: $(tail -n 1 gpurun_out/s2z_sp_${v}_$r.log)"; grep " 14 m29" gpurun_out/s2z_sp_${v}_$r.log
done; done
