"""Dev tool: the GPU path vs the oracle on sub-sliced plans, per layout policy / dtype / fusion knob."""
import json
import sys

import numpy as np

sys.path.insert(0, ".")
from paper_2407_00769_b200 import tn  # noqa: E402
from workload import make_plans as MP  # noqa: E402
from oracle import contract, metrics  # noqa: E402
from oracle.plan import load  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c3"
for tgt in [int(x) for x in (sys.argv[2] if len(sys.argv) > 2 else "20,22,24").split(",")]:
    sub = MP.sub_slice(json.load(open(f"plans/{name}.json")), tgt)
    ref = contract.contract(load(sub), 0)
    for dtype in (0, 1):
        for pol in (0, 1, 2):
            for ng in (0, 1):
                try:
                    p = tn.Plan(sub, tn.make_config(dtype=dtype, stem_min_log2=min(20, tgt - 4), layout_policy=pol,
                                                    no_gather=ng))
                    a = tn.contract(p, tn.Buffers(p), 0)
                    print(f"{name} 2^{tgt} dtype {dtype} policy {pol} no_gather {ng}: rel {metrics.rel_l2(a, ref):.3e} "
                          f"steps {p.info()['n_stem_steps']} perms {p.info()['n_permutes']}", flush=True)
                except Exception as e:
                    print(f"{name} 2^{tgt} dtype {dtype} policy {pol} no_gather {ng}: ERROR {e}", flush=True)
