nvidia-smi --query-gpu=clocks.sm,power.draw,clocks_event_reasons.active --format=csv -lms 50 > gpurun_out/s2k_clocks.csv &
CP=$!
TN_REDO_BITS=0 timeout 600 python tools/step_profile.py c3 3 20 4 > gpurun_out/s2k_sp_noredo.log 2>&1
timeout 600 python tools/step_profile.py c3 3 20 4 > gpurun_out/s2k_sp_redo.log 2>&1
kill $CP
paste <(cut -c1-100 gpurun_out/s2k_sp_noredo.log) <(cut -c40-75 gpurun_out/s2k_sp_redo.log)
