"""Write plan JSON files for the BASELINE.json configs (seeded, synthetic).

Plan JSON (the input of ``tn_plan_load``, include/tn.h):
  {"version": 1,
   "tensors": [{"labels": [int...], "data": [re0, im0, re1, im1, ...]}, ...],  # row-major, dims 2
   "open": [labels...],        # output legs, in output order (slowest first)
   "tree": [[u, v], ...],      # SSA pairs; ids < n_tensors are leaves
   "sliced": [labels...],      # bit j of a slice id fixes sliced[j] (C-A20)
   "stem": [node ids...],      # leaf->root stem path (C-A18)
   "circuit": {...}, "bits": [...], "open_qubits": [...], "meta": {...}}   # ignored by the library

Usage:  python -m workload.make_plans [c1 c2 c3 ...]
"""
from __future__ import annotations

import json
import os
import sys
import time

from . import circuit as C
from . import network as NW
from . import planner as PL

HERE = os.path.dirname(os.path.abspath(__file__))
PLAN_DIR = os.path.join(os.path.dirname(HERE), "plans")

# name -> (rows, cols, drop_corner, cycles, n_open, max_log2, trials)
CONFIGS = {
    # C1: 12-qubit depth-8, all legs open (full state), unsliced (BJ configs[0])
    "c1": dict(rows=3, cols=4, drop=False, cycles=8, n_open=12, max_log2=None, trials=8),
    # C2: 30-qubit 14-cycle, stem <= 2^28, 10 open legs (BJ configs[1])
    "c2": dict(rows=5, cols=6, drop=False, cycles=14, n_open=10, max_log2=30, trials=0),
    # C3: 53-qubit (6x9 minus a corner) 20-cycle, 6 open legs (BJ configs[2]).  Branch grouping over
    # up to 24 consecutive stem branches (MB-scale non-stem tensors), then as few sliced edges
    # as keep the largest stem at 2^32 ("~2^32 complex-half in double buffers")
    # fSim angles jittered per coupler (reading C-A2, revised): at theta = pi/2 exactly fSim is a phased
    # SWAP whose zero pattern makes most slices of a heavily sliced 53-qubit network structurally zero
    "c3": dict(rows=6, cols=9, drop=True, cycles=20, n_open=6, max_log2=35, trials=0, max_group=24, stem_log2=32,
               jitter=0.2),
    # round-1 C3 plan (kept as the memory-bound variant): 12-branch groups, 188 sliced edges, stem 2^33
    "c3_sweep": dict(rows=6, cols=9, drop=True, cycles=20, n_open=6, max_log2=35, trials=0, jitter=0.2),
    # C5 (BJ configs[4]): the C3 circuit with 22 output legs open: the 12 that enter the stem last are
    # the sparse-state legs (a correlated subspace = one value of them, "sparse state occurs in
    # the final stage"), the other 10 the members of each subspace (q_open = 10)
    "c5": dict(rows=6, cols=9, drop=True, cycles=20, n_open=22, max_log2=35, trials=0, max_group=24, stem_log2=32,
               jitter=0.2, sparse=12),
}


def choose_sparse_legs(plan, n_sparse):
    """The n_sparse open legs whose first appearance along the stem (in a stem branch) is latest;
    legs already in the first stem tensors are never chosen (they would have to be batch modes of
    the whole stem)."""
    masks = []
    for t in plan["tensors"]:
        m = 0
        for l in t["labels"]:
            m |= 1 << l
        masks.append(m)
    tree = PL.Tree(masks, [tuple(p) for p in plan["tree"]])
    stem = plan["stem"]
    first = {}
    for s, (a, b) in enumerate(zip(stem[:-1], stem[1:])):
        u, v = tree.children[b]
        br = v if u == a else u
        for l in PL.bits_of(tree.masks[br]):
            first.setdefault(l, s + 1)
    cand = [l for l in plan["open"] if l in first]
    cand.sort(key=lambda l: -first[l])
    if len(cand) < n_sparse:
        raise RuntimeError("not enough late-entering open legs for the sparse state")
    return sorted(cand[:n_sparse], key=plan["open"].index)


def open_qubit_choice(n, n_open):
    """Open the last n_open qubits (a contiguous block at the grid edge)."""
    return list(range(n - n_open, n))


def sweep_orders(circ, net):
    """Leaf orders that sweep the grid column by column (and row by row), time-forward inside a
    column: the stem then carries the bonds across one cut of the 2-D grid."""
    sites = circ["sites"]
    info = []
    for ls, _ in net.tensors:
        qs = [net.label_pos[l][0] for l in ls]
        ts = [net.label_pos[l][1] for l in ls]
        rows = [sites[q][0] for q in qs]
        cols = [sites[q][1] for q in qs]
        if not ls:  # scalar factor (a qubit without two-qubit gates, fully closed)
            rows, cols, ts = [0], [0], [0]
        info.append((rows, cols, sum(ts) / len(ts)))
    idx = range(len(info))
    orders = []
    orders.append(sorted(idx, key=lambda i: (max(info[i][1]), info[i][2], min(info[i][0]))))
    orders.append(sorted(idx, key=lambda i: (max(info[i][1]), min(info[i][0]), info[i][2])))
    orders.append(sorted(idx, key=lambda i: (max(info[i][0]), info[i][2], min(info[i][1]))))
    orders.append(sorted(idx, key=lambda i: (min(info[i][1]), info[i][2], min(info[i][0]))))
    return orders


def build_plan(rows, cols, drop, cycles, n_open, max_log2, trials, seed=0, group=True,
               max_branch_log2=20, max_group=12, stem_log2=None, jitter=0.0):
    circ = C.make_circuit(rows, cols, cycles, seed=seed, drop_corner=drop, jitter=jitter)
    n = circ["n_qubits"]
    bits = C.random_bits(n, seed + 1000)
    oq = open_qubit_choice(n, n_open)
    net = NW.simplify(NW.build_network(circ, bits=bits, open_qubits=oq))
    leaf_masks = []
    for ls, _ in net.tensors:
        m = 0
        for l in ls:
            m |= 1 << l
        leaf_masks.append(m)
    open_mask = 0
    for l in net.open:
        open_mask |= 1 << l
    if max_log2 is None:
        max_log2 = 10 ** 6
    res = PL.plan_network(leaf_masks, open_mask, max_log2, trials=trials, seed=seed, group=group,
                          max_branch_log2=max_branch_log2, sweeps=sweep_orders(circ, net), max_group=max_group,
                          stem_log2=stem_log2)
    tree, sliced, stem = res["tree"], res["sliced"], res["stem"]
    tensors = []
    for ls, d in net.tensors:
        flat = d.reshape(-1)
        data = []
        for z in flat:
            data.append(float(z.real))
            data.append(float(z.imag))
        tensors.append({"labels": list(ls), "data": data})
    geo = PL.stem_report(tree, sliced, stem)
    meta = {
        "n_qubits": n, "cycles": cycles, "seed": seed,
        "n_tensors": len(tensors), "n_sliced": PL.popcount(sliced),
        "slice_cost_cmacs": tree.total_cost(sliced),
        "max_log2": tree.max_log2(sliced),
        "stem_steps_mkn_log2": geo,
        "est_time_s": res["est_time"],
    }
    return {
        "version": 1,
        "tensors": tensors,
        "open": list(net.open),
        "tree": [list(p) for p in tree.pairs],
        "sliced": PL.bits_of(sliced),
        "stem": stem,
        "circuit": circ,
        "bits": bits,
        "open_qubits": oq,
        "meta": meta,
    }


def write_plan(name, plan):
    os.makedirs(PLAN_DIR, exist_ok=True)
    path = os.path.join(PLAN_DIR, f"{name}.json")
    with open(path, "w") as f:
        json.dump(plan, f, separators=(",", ":"))
    return path


def main(argv):
    names = argv or list(CONFIGS)
    for name in names:
        cfg = CONFIGS[name]
        t0 = time.time()
        plan = build_plan(cfg["rows"], cfg["cols"], cfg["drop"], cfg["cycles"], cfg["n_open"],
                          cfg["max_log2"], cfg["trials"], max_group=cfg.get("max_group", 12),
                          stem_log2=cfg.get("stem_log2"), jitter=cfg.get("jitter", 0.0))
        if cfg.get("sparse"):
            plan["sparse_legs"] = choose_sparse_legs(plan, cfg["sparse"])
        p = write_plan(name, plan)
        m = plan["meta"]
        print(f"{name}: {p} tensors={m['n_tensors']} sliced={m['n_sliced']} "
              f"max_log2={m['max_log2']} slice_cmacs={m['slice_cost_cmacs']:.3e} "
              f"stem_steps={len(m['stem_steps_mkn_log2'])} est={m['est_time_s']} "
              f"({time.time() - t0:.1f}s)")


if __name__ == "__main__":
    main(sys.argv[1:])


def sub_slice(plan, target_log2):
    """Reduced-scale protocol: slice extra closed labels of an existing plan
    (same tree, same leaves) until every intermediate has <= 2^target_log2 elements.  The result
    is another valid plan; its slices are sub-slices of the original."""
    import copy
    leaf_masks = []
    for t in plan["tensors"]:
        m = 0
        for l in t["labels"]:
            m |= 1 << l
        leaf_masks.append(m)
    tree = PL.Tree(leaf_masks, [tuple(p) for p in plan["tree"]])
    sliced = 0
    for l in plan["sliced"]:
        sliced |= 1 << l
    open_mask = 0
    for l in plan["open"]:
        open_mask |= 1 << l
    extra = []
    while tree.max_log2(sliced) > target_log2:
        worst = tree.max_log2(sliced)
        score = {}
        for m in tree.masks:
            if PL.popcount(m & ~sliced) >= worst - 2:
                for l in PL.bits_of(m & ~sliced & ~open_mask):
                    score[l] = score.get(l, 0) + (4 if PL.popcount(m & ~sliced) == worst else 1)
        if not score:  # only open legs remain in the widest intermediates
            break
        l = max(sorted(score), key=lambda x: score[x])
        sliced |= 1 << l
        extra.append(l)
    out = copy.deepcopy(plan)
    out["sliced"] = list(plan["sliced"]) + extra
    return out
