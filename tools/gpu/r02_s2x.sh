NG=$(nvidia-smi -L | wc -l)
for r in 1 2; do for v in new old; do
if [ $v = old ]; then export TN_ROWS_TRANSPOSE=1; else unset TN_ROWS_TRANSPOSE; fi
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $NG --master-addr 127.0.0.1 --master-port 2957$r bench.py --gpus $NG --steps 8 --warmup 3 --no-cpu > gpurun_out/s2x_$v$r.json 2>/dev/null
python - gpurun_out/s2x_$v$r.json $v <<'PY'
import json, sys
d = json.loads([l for l in open(sys.argv[1]) if l.startswith("{")][0])
print(sys.argv[2], round(d["ms_per_step"], 1), round(d["value"]), d["clocks"]["sm_mhz"], d["config"]["permutes"], d["breakdown_ms"])
PY
done; done
