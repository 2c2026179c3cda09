NG=$(nvidia-smi -L | wc -l)
for r in 1 2 3; do for v in 1 0; do
if [ $NG = 1 ]; then
TN_TR_SEARCH=$v timeout 900 python bench.py --steps 6 --warmup 3 --no-cpu > gpurun_out/s3x_$v.json 2>/dev/null
else
TN_TR_SEARCH=$v timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $NG --master-addr 127.0.0.1 --master-port 2967$v bench.py --gpus $NG --steps 6 --warmup 3 --no-cpu > gpurun_out/s3x_$v.json 2>/dev/null
fi
python - gpurun_out/s3x_$v.json $v <<'PY'
import json, sys
d = json.loads([l for l in open(sys.argv[1]) if l.startswith("{")][0])
print("tr_search", sys.argv[2], round(d["ms_per_step"], 1), d["clocks"]["sm_mhz"], round(d["energy"]["joules_per_step"], 1), d["config"]["permutes"], d["breakdown_ms"])
PY
done; done
