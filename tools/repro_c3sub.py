"""Dev tool: repeat the C3 sub-sliced contraction and compare with the oracle each time."""
import json
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2407_00769_b200 import tn  # noqa: E402
from workload import make_plans as MP  # noqa: E402
from oracle import contract, metrics  # noqa: E402
from oracle.plan import load  # noqa: E402

sub = MP.sub_slice(json.load(open("plans/c3.json")), int(sys.argv[1]) if len(sys.argv) > 1 else 22)
sm = int(sys.argv[2]) if len(sys.argv) > 2 else 14
ref = contract.contract(load(sub), 0)
for pol in (0, 1, 2):
    for rep in range(3):
        p = tn.Plan(sub, tn.make_config(stem_min_log2=sm, layout_policy=pol))
        b = tn.Buffers(p)
        a = tn.contract(p, b, 0)
        r = p.report()
        print("policy", pol, "rep", rep, "rel", metrics.rel_l2(a, ref), "nan", bool(np.isnan(a).any()),
              "tc", sum(s["tc"] for s in r["steps"]), "steps", len(r["steps"]), flush=True)
