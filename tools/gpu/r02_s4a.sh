for r in 1 2; do
timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu > gpurun_out/s4a_bench_$r.json 2>/dev/null
python - gpurun_out/s4a_bench_$r.json <<'PY'
import json, sys
d = json.loads([l for l in open(sys.argv[1]) if l.startswith("{")][0]); r = d["roofline"]
print(sys.argv[1], round(d["ms_per_step"], 1), round(d["value"]), d["clocks"]["sm_mhz"], r["kernel"], round(r["frac"], 3), round(d["energy"]["joules_per_step"], 1), d["breakdown_ms"])
PY
done
