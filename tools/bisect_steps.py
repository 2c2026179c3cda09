"""Dev tool: localise a GPU/oracle divergence to a stem step.  For stem node T (after step i) the
sub-network under T is written as its own plan (slice 0 applied to the leaves, T's labels open, the
stem path mapped), contracted on the GPU and by the oracle, and compared.

  python tools/bisect_steps.py PLAN SUBSLICE_LOG2 [dtype] [steps...]
"""
import json
import sys

import numpy as np

sys.path.insert(0, ".")
from paper_2407_00769_b200 import tn  # noqa: E402
from workload import make_plans as MP  # noqa: E402
from oracle import contract, metrics  # noqa: E402
from oracle.plan import load  # noqa: E402


def presliced(plan):
    """Leaves with every sliced label fixed to 0 (slice 0), sliced list emptied."""
    out = dict(plan)
    sl = set(plan["sliced"])
    tens = []
    for t in plan["tensors"]:
        labels = t["labels"]
        d = np.asarray(t["data"], dtype=np.float64)
        z = (d[0::2] + 1j * d[1::2]).reshape((2,) * len(labels)) if labels else (d[0::2] + 1j * d[1::2])
        idx = tuple(0 if l in sl else slice(None) for l in labels)
        z = z[idx] if labels else z
        keep = [l for l in labels if l not in sl]
        flat = np.asarray(z).reshape(-1)
        tens.append({"labels": keep, "data": [v for c in flat for v in (float(c.real), float(c.imag))]})
    out["tensors"] = tens
    out["sliced"] = []
    return out


def subtree_plan(plan, node):
    nl = len(plan["tensors"])
    pairs = plan["tree"]
    members = set()

    def walk(k):
        members.add(k)
        if k >= nl:
            u, v = pairs[k - nl]
            walk(u)
            walk(v)
    walk(node)
    leaves = sorted(k for k in members if k < nl)
    internal = sorted(k for k in members if k >= nl)
    newid = {k: i for i, k in enumerate(leaves)}
    for j, k in enumerate(internal):
        newid[k] = len(leaves) + j
    out = {"version": 1, "tensors": [plan["tensors"][k] for k in leaves],
           "tree": [[newid[pairs[k - nl][0]], newid[pairs[k - nl][1]]] for k in internal], "sliced": []}
    cnt = {}
    for k in leaves:
        for l in plan["tensors"][k]["labels"]:
            cnt[l] = cnt.get(l, 0) + 1
    out["open"] = sorted(l for l, c in cnt.items() if c == 1)
    out["stem"] = [newid[k] for k in plan["stem"] if k in members]
    return out


def main():
    name, tgt = sys.argv[1], int(sys.argv[2])
    dtype = int(sys.argv[3]) if len(sys.argv) > 3 else 0
    sub = presliced(MP.sub_slice(json.load(open(f"plans/{name}.json")), tgt))
    p = tn.Plan(sub, tn.make_config(dtype=dtype, stem_min_log2=min(20, tgt - 4)))
    rep = p.report()
    steps = [int(x) for x in sys.argv[4:]] or list(range(len(rep["steps"])))
    for i in steps:
        node = rep["steps"][i]["node"]
        sp = subtree_plan(sub, node)
        if len(sp["open"]) > 24:
            print(f"step {i}: node {node} has {len(sp['open'])} open legs, skipped", flush=True)
            continue
        ref = contract.contract(load(sp), 0)
        q = tn.Plan(sp, tn.make_config(dtype=dtype, stem_min_log2=min(20, tgt - 4)))
        got = tn.contract(q, tn.Buffers(q), 0)
        r = q.report()
        last = r["steps"][-1] if r["steps"] else {}
        print(f"step {i}: node {node} open {len(sp['open'])} gpu steps {len(r['steps'])} "
              f"last m{last.get('m')} k{last.get('k')} n{last.get('n')} perm {last.get('perm')} ga {last.get('ga')} "
              f"tc {last.get('tc')}: rel {metrics.rel_l2(got, ref):.3e} |ref| {np.linalg.norm(ref):.3e} "
              f"|gpu| {np.linalg.norm(got):.3e}", flush=True)


if __name__ == "__main__":
    main()
