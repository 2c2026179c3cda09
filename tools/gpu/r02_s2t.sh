for r in 1 2 3; do for m in 28 99; do
TN_MN_MIN_LOG2=$m timeout 600 python bench.py --steps 6 --warmup 3 --no-cpu > gpurun_out/s2t_b_$m_$r.json 2>/dev/null
python - <<PY
import json
d=json.loads([l for l in open("gpurun_out/s2t_b_$m_$r.json") if l.startswith("{")][0])
print("mn_min=$m rep $r", round(d["ms_per_step"],1), "J", round(d["energy"]["joules_per_step"],1), "MHz", d["clocks"]["sm_mhz"], d["breakdown_ms"])
PY
done; done
