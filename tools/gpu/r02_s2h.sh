set -x
NG=$(nvidia-smi -L | wc -l)
timeout 900 python -m pytest tests/test_gpu_multi.py -m gpu -q -x -s > gpurun_out/s2h_multi_$NG.log 2>&1; grep -E "world|passed|failed|rror" gpurun_out/s2h_multi_$NG.log | tail -5
for f in 0 1; do
TN_NO_FUSED_SWAP=$f timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $NG --master-addr 127.0.0.1 --master-port 2951$f bench.py --gpus $NG --steps 5 --warmup 3 > gpurun_out/s2h_bench_n${NG}_nofused$f.json 2> gpurun_out/s2h_bench_n${NG}_nofused$f.err
python - <<PY
import json
d=json.loads([l for l in open("gpurun_out/s2h_bench_n${NG}_nofused$f.json") if l.startswith("{")][0])
print("nofused=$f", d["ms_per_step"], d["value"], d["breakdown_ms"], d["clocks"]["sm_mhz"], d["config"].get("fused_swaps"))
PY
tail -3 gpurun_out/s2h_bench_n${NG}_nofused$f.err
done
