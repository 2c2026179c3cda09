NG=$(nvidia-smi -L | wc -l)
timeout 900 python -m pytest tests/test_gpu_loopback.py -m gpu -q -x -s -k "fused_swap or fp16_vs_one" > gpurun_out/s2y_lb.log 2>&1; grep -E "world=|passed|failed|rror" gpurun_out/s2y_lb.log | tail -6
timeout 900 python -m pytest tests/test_gpu_multi.py -m gpu -q -x > gpurun_out/s2y_multi_$NG.log 2>&1; tail -2 gpurun_out/s2y_multi_$NG.log
for v in peer nccl; do
if [ $v = nccl ]; then export TN_SWAP_NCCL=1; else unset TN_SWAP_NCCL; fi
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $NG --master-addr 127.0.0.1 --master-port 29581 bench.py --gpus $NG --steps 8 --warmup 3 --no-cpu > gpurun_out/s2y_$v$NG.json 2>/dev/null
python - gpurun_out/s2y_$v$NG.json $v <<'PY'
import json, sys
d = json.loads([l for l in open(sys.argv[1]) if l.startswith("{")][0])
print(sys.argv[2], round(d["ms_per_step"], 1), round(d["value"]), d["clocks"]["sm_mhz"], d["config"]["epilogue_swaps"], d["breakdown_ms"])
PY
done
