set -x
python -m pytest tests/test_gpu_kernels.py tests/test_gpu_sparse_state.py -m gpu -q --timeout 600 -k "batched or padded or sparse" -rA > gpurun_out/t5.log 2>&1
timeout 900 python tools/debug_parity.py c3 20,22 > gpurun_out/dbg_c3.log 2>&1
timeout 600 python tools/debug_parity.py c3_sweep 22 > gpurun_out/dbg_c3sweep.log 2>&1
tail -3 gpurun_out/t5.log
