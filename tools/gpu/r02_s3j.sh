timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu > gpurun_out/s3j_bench.json 2> gpurun_out/s3j_bench.err
python - <<'PY'
import json
d = json.loads([l for l in open("gpurun_out/s3j_bench.json") if l.startswith("{")][0])
print(round(d["ms_per_step"], 1), round(d["value"]), d["clocks"]["sm_mhz"])
print(json.dumps(d["roofline"], indent=0)[:1500])
PY
tail -3 gpurun_out/s3j_bench.err
