cat > /tmp/one.py <<'PY'
import json, sys, torch
sys.path.insert(0, ".")
from paper_2407_00769_b200 import tn
p = tn.Plan(json.load(open("plans/c3.json")), tn.make_config())
tn.set_graph(p, 0) if hasattr(tn, "set_graph") else None
b = tn.Buffers(p); tn.tn_plan_upload(p, b); tn.tn_stem_contract(p, b, 0); torch.cuda.synchronize()
PY
TN_NO_GRAPH=1 timeout 900 ncu --set full --clock-control none -k regex:permute_pipe -c 8 -o gpurun_out/s3u_perm python /tmp/one.py > gpurun_out/s3u.log 2>&1; tail -2 gpurun_out/s3u.log
