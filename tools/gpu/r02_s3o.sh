NG=$(nvidia-smi -L | wc -l)
for r in 1 2; do for g in 0 1; do
TN_GRAPH_NCCL=$g timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $NG --master-addr 127.0.0.1 --master-port 2962$g bench.py --gpus $NG --steps 8 --warmup 3 --no-cpu > gpurun_out/s3o_g$g.json 2>/dev/null
python - gpurun_out/s3o_g$g.json $g <<'PY'
import json, sys
d = json.loads([l for l in open(sys.argv[1]) if l.startswith("{")][0])
print("graph_nccl", sys.argv[2], round(d["ms_per_step"], 1), round(d["value"]), d["clocks"]["sm_mhz"], d["breakdown_ms"])
PY
done; done
