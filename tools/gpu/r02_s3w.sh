timeout 1500 python -m pytest tests -m gpu -q --timeout 900 -x > gpurun_out/s3w_tests.log 2>&1; tail -2 gpurun_out/s3w_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s3w_smoke.log 2>&1; tail -3 gpurun_out/s3w_smoke.log
for r in 1 2; do
timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu > gpurun_out/s3w_bench_$r.json 2>/dev/null
python - gpurun_out/s3w_bench_$r.json <<'PY'
import json, sys
d = json.loads([l for l in open(sys.argv[1]) if l.startswith("{")][0]); r = d["roofline"]
print(round(d["ms_per_step"], 1), round(d["value"]), d["clocks"]["sm_mhz"], r["kernel"], round(r["frac"], 3), d["breakdown_ms"], round(d["energy"]["joules_per_step"], 1))
PY
done
