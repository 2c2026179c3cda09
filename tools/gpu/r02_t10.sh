set -x
python -m pytest tests/test_gpu_loopback.py tests/test_gpu_sparse_state.py tests/test_gpu_kernels.py -m gpu -q --timeout 900 -rf -k "loopback or c3_sub26 or sparse or pad_b" > gpurun_out/t10.log 2>&1
tail -15 gpurun_out/t10.log
