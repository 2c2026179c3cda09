set -x
python -m pytest tests/test_gpu_sparse_state.py tests/test_gpu_kernels.py -m gpu -q --timeout 600 -k "sparse or padded or batched" -rA > gpurun_out/t6.log 2>&1
timeout 900 python tools/debug_parity.py c3 20,22 > gpurun_out/dbg2_c3.log 2>&1
timeout 600 python tools/debug_parity.py c3_sweep 22 > gpurun_out/dbg2_c3sweep.log 2>&1
TN_REDO_BITS=0 timeout 900 python tools/bisect_steps.py c3 20 0 > gpurun_out/bisect_c3_noredo.log 2>&1
tail -3 gpurun_out/t6.log
