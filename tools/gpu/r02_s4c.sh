for v in 1 0; do TN_TC2_RAW=$v timeout 300 python tools/gather_bench.py 24,8,7,k4m8k4m16 23,9,7,k3m1k6m22 23,9,7,k4m3k5m20 26,6,6,k3m1k3m25 2>&1 | sed "s/^/tc2raw=$v /"; done
python - <<'PY'
import sys, torch, numpy as np
sys.path.insert(0, ".")
from paper_2407_00769_b200 import tn
# exact-integer check of the raw pair path on a step-4-like layout
rng = np.random.default_rng(1)
mlog, klog, N = 14, 8, 128
runs = "k4m8k4m6"
PY
timeout 900 python -m pytest tests/test_gpu_e2e.py -m gpu -q -x > gpurun_out/s4c_e.log 2>&1; tail -2 gpurun_out/s4c_e.log
for r in 1 2; do for v in 1 0; do
TN_TC2_RAW=$v timeout 600 python tools/step_profile.py c3 3 20 3 > gpurun_out/s4c_sp.log 2>&1
echo "tc2raw=$v rep $r: $(tail -n 1 gpurun_out/s4c_sp.log)"; grep -E " (4|13|18|25) m" gpurun_out/s4c_sp.log | cut -c1-90
done; done
