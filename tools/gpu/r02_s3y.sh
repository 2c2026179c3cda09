set -x
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 -rfs > gpurun_out/s3y_tests.log 2>&1
tail -3 gpurun_out/s3y_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s3y_smoke.log 2>&1; tail -3 gpurun_out/s3y_smoke.log
timeout 1800 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/r02c_launches_c3.csv python bench.py --steps 1 --warmup 1 --no-cpu > gpurun_out/s3y_ncu_launch.log 2>&1; tail -1 gpurun_out/s3y_ncu_launch.log
gzip -kf gpurun_out/r02c_launches_c3.csv
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/s3y_bench.json 2> gpurun_out/s3y_bench.err
python - <<'PY'
import json
d = json.loads([l for l in open("gpurun_out/s3y_bench.json") if l.startswith("{")][0]); r = d["roofline"]
print(round(d["ms_per_step"], 1), round(d["value"]), d["clocks"]["sm_mhz"], r["kernel"], round(r["frac"], 3), r.get("traffic"), d.get("parity"))
PY
