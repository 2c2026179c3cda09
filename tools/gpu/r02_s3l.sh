timeout 600 python tools/step_profile.py c3 3 20 3 > gpurun_out/s3l_sp.log 2>&1; cat gpurun_out/s3l_sp.log
