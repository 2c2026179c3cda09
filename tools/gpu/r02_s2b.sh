set -x
for r in 1 2; do
  TN_TC2=1 timeout 600 python tools/step_profile.py c3 3 > gpurun_out/s2b_sp_tc2_$r.log 2>&1
  TN_TC2=0 timeout 600 python tools/step_profile.py c3 3 > gpurun_out/s2b_sp_tc1_$r.log 2>&1
  tail -1 gpurun_out/s2b_sp_tc2_$r.log gpurun_out/s2b_sp_tc1_$r.log
done
