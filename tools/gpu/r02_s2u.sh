timeout 600 python -m pytest tests/test_gpu_e2e.py -m gpu -q -x -k "mn_major" > gpurun_out/s2u_t.log 2>&1; tail -2 gpurun_out/s2u_t.log
for r in 1 2 3; do for v in rp norp nomn; do
case $v in rp) E="";; norp) E="TN_MN_ROWPERM=0";; nomn) E="TN_MN_MIN_LOG2=99";; esac
env $E timeout 600 python tools/step_profile.py c3 3 20 3 > gpurun_out/s2u_sp_${v}_$r.log 2>&1
echo "$v rep $r: $(tail -n 1 gpurun_out/s2u_sp_${v}_$r.log)"
done; done
