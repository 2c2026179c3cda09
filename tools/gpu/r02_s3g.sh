NG=$(nvidia-smi -L | wc -l)
timeout 900 python -m pytest tests/test_gpu_multi.py -m gpu -q -x -s > gpurun_out/s3g_multi_$NG.log 2>&1; grep -E "passed|failed|rror" gpurun_out/s3g_multi_$NG.log | tail -3
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $NG --master-addr 127.0.0.1 --master-port 29601 bench.py --gpus $NG --steps 8 --warmup 3 > gpurun_out/s3g_bench_n$NG.json 2> gpurun_out/s3g_bench_n$NG.err
python - gpurun_out/s3g_bench_n$NG.json <<'PY'
import json, sys
d = json.loads([l for l in open(sys.argv[1]) if l.startswith("{")][0])
print(round(d["ms_per_step"], 1), round(d["value"]), d["clocks"]["sm_mhz"], d["config"]["epilogue_swaps"], d["breakdown_ms"], d["e2e"]["ms_per_step"])
PY
