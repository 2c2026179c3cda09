set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 -rfs > gpurun_out/s2a_tests.log 2>&1
tail -12 gpurun_out/s2a_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s2a_smoke.log 2>&1; tail -4 gpurun_out/s2a_smoke.log
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/s2a_bench.json 2> gpurun_out/s2a_bench.err; tail -c 3000 gpurun_out/s2a_bench.json
for t in 0 1; do
  TN_TC2=$t timeout 900 python bench.py --steps 8 --warmup 3 --no-cpu > gpurun_out/s2a_bench_tc2_$t.json 2> gpurun_out/s2a_bench_tc2_$t.err
done
python - <<'PY'
import json
for t in (1,0):
    try:
        d=json.loads([l for l in open(f"gpurun_out/s2a_bench_tc2_{t}.json") if l.startswith("{")][0])
        print("tc2" if t else "tc1", round(d["ms_per_step"],2), "MHz", d["clocks"]["sm_mhz"], d.get("breakdown_ms"))
    except Exception as e:
        print(t, "err", e)
PY
for t in 0 1; do TN_TC2=$t timeout 600 python tools/mubench.py --m 23 --k 6-10 --n 6-10 --iters 5 > gpurun_out/s2a_mb_tc2_$t.txt 2>&1; done
tail -30 gpurun_out/s2a_mb_tc2_0.txt gpurun_out/s2a_mb_tc2_1.txt
