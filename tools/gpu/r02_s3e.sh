timeout 900 python bench.py --plan c5 --steps 3 --warmup 3 --no-cpu > gpurun_out/s3e_c5.json 2> gpurun_out/s3e_c5.err; tail -c 1500 gpurun_out/s3e_c5.json
timeout 900 python bench.py --plan c3_sweep --steps 5 --warmup 3 --no-cpu > gpurun_out/s3e_sweep.json 2> gpurun_out/s3e_sweep.err
python - <<'PY'
import json
for f in ("s3e_c5", "s3e_sweep"):
    try:
        d = json.loads([l for l in open(f"gpurun_out/{f}.json") if l.startswith("{")][0])
        print(f, round(d["ms_per_step"], 1), round(d["value"], 1), d["unit"], d["clocks"]["sm_mhz"], d.get("parity"), d["roofline"]["frac"], d["roofline"]["bound"])
    except Exception as e:
        print(f, "err", e, open(f"gpurun_out/{f}.err").read()[-500:])
PY
