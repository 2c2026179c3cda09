for v in 18 0; do
  TN_REDO_BITS=$v timeout 300 python tools/step_profile.py c3 3 20 3 > gpurun_out/redo_$v.log 2>&1
  echo "redo=$v $(tail -1 gpurun_out/redo_$v.log | cut -c1-170)"
done
python - <<'PY'
import re
def load(f):
    d={}
    for l in open(f):
        m=re.match(r"\s*(\d+) m.*gemm\s+([\d.]+) ms",l)
        if m: d[int(m.group(1))]=float(m.group(2))
    return d
a=load("gpurun_out/redo_18.log"); b=load("gpurun_out/redo_0.log")
for i in sorted(a):
    if abs(a[i]-b[i])>0.3: print(i, a[i], b[i])
PY
