set -x
timeout 900 python -m pytest tests/test_gpu_loopback.py -m gpu -q -x -s -k "fused_swap or fp16_vs_one or c3_sub26" > gpurun_out/s2g.log 2>&1; grep -E "world=|passed|failed|Error|error" gpurun_out/s2g.log | head -30
