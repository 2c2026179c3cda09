timeout 1500 python -m pytest tests -m gpu -q --timeout 900 -rfs > gpurun_out/s4e_tests.log 2>&1
tail -2 gpurun_out/s4e_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s4e_smoke.log 2>&1; tail -3 gpurun_out/s4e_smoke.log
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/s4e_bench.json 2> gpurun_out/s4e_bench.err
timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu > gpurun_out/s4e_bench_b.json 2> gpurun_out/s4e_bench_b.err
for f in gpurun_out/s4e_bench.json gpurun_out/s4e_bench_b.json; do python - $f <<'PY'
import json, sys
d = json.loads([l for l in open(sys.argv[1]) if l.startswith("{")][0]); r = d["roofline"]
print(sys.argv[1], round(d["ms_per_step"], 1), round(d["value"]), d["clocks"]["sm_mhz"], r["kernel"], round(r["frac"], 3), round(d["energy"]["joules_per_step"], 1), d.get("parity", {}).get("rel_l2_vs_oracle"))
PY
done
