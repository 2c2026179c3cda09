TN_GATHER_DEBUG=1 timeout 120 python -m pytest tests/test_gpu_kernels.py -m gpu -q -x -k "gathered_runs" > gpurun_out/s4b_k.log 2>&1; tail -3 gpurun_out/s4b_k.log; grep -c gather gpurun_out/s4b_k.log
