nvidia-smi --query-gpu=clocks.sm,power.draw,clocks_event_reasons.active --format=csv -lms 200 > gpurun_out/s2c_clocks.csv &
CP=$!
TN_GATHER_DEBUG=1 timeout 600 python tools/step_profile.py c3 3 20 6 > gpurun_out/s2c_sp.log 2> gpurun_out/s2c_sp.err
kill $CP
sort -u gpurun_out/s2c_sp.err | head -30
