set -x
python -m pytest tests/test_gpu_loopback.py tests/test_gpu_postselect.py tests/test_gpu_multi.py -m gpu -q --timeout 900 -rf > gpurun_out/t11.log 2>&1
tail -15 gpurun_out/t11.log
