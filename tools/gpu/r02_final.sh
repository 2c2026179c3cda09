NG=$(nvidia-smi -L | wc -l)
nvidia-smi --query-gpu=name,clocks.max.sm,power.limit --format=csv,noheader | head -1
if [ $NG = 1 ]; then
  timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/final_n1_a.json 2> gpurun_out/final_n1_a.err
  timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu > gpurun_out/final_n1_b.json 2> gpurun_out/final_n1_b.err
  timeout 600 python tools/step_profile.py c3 3 20 3 > gpurun_out/final_sp_n1.log 2>&1
else
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $NG --master-addr 127.0.0.1 --master-port 29651 bench.py --gpus $NG --steps 8 --warmup 3 > gpurun_out/final_n${NG}_a.json 2> gpurun_out/final_n${NG}_a.err
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $NG --master-addr 127.0.0.1 --master-port 29652 bench.py --gpus $NG --steps 8 --warmup 3 > gpurun_out/final_n${NG}_b.json 2> gpurun_out/final_n${NG}_b.err
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $NG --master-addr 127.0.0.1 --master-port 29653 tools/step_profile_mgpu.py c3 3 > gpurun_out/final_sp_n$NG.log 2>/dev/null
fi
for f in gpurun_out/final_n${NG}_*.json; do python - "$f" <<'PY'
import json, sys
d = json.loads([l for l in open(sys.argv[1]) if l.startswith("{")][0])
r = d["roofline"]
print(sys.argv[1], round(d["ms_per_step"], 1), round(d["value"]), d["clocks"]["sm_mhz"], r["kernel"], round(r["frac"], 3), d["config"].get("epilogue_swaps"), d["breakdown_ms"], round(d["e2e"]["ms_per_step"], 1))
PY
done
