"""Oracle contraction of one sliced subtask, complex128.

Definition followed, step by step:
* tensor network of the RQC (§2.2); every mode has dimension 2;
* slicing: each sliced edge e_j is fixed to bit j of the slice id ("breaking edges",
  P:318 independent sub-networks; bit order = reading C-A20);
* pairwise contraction in the plan's SSA order, Eq. 3: C = sum over the shared
  (reduced) indices of A*B, with the pure-GEMM condition delta = (alpha) cap (beta) and the
  output indices by Eq. 4: (alpha) cup (beta) minus delta, in canonical order
  (u-free, v-free).  ``np.tensordot`` is the library primitive for one pair;
* the root is transposed to the plan's ``open`` order.

The slicing identity sum_s a_s = unsliced and agreement with the state vector are pinned
in tests/test_oracle.py.
"""
import numpy as np

from .plan import Plan, load


def slice_leaves(plan: Plan, slice_id: int):
    """Leaves with every sliced label fixed to its bit of ``slice_id`` (mode dropped)."""
    if slice_id < 0 or slice_id >= (1 << min(len(plan.sliced), 64)):
        raise ValueError("slice id out of range")
    val = {l: (slice_id >> j) & 1 for j, l in enumerate(plan.sliced)}
    out = []
    for labels, t in plan.tensors:
        idx = tuple(val[l] if l in val else slice(None) for l in labels)
        out.append(([l for l in labels if l not in val], t[idx] if labels else t))
    return out


def contract_pair(a, b):
    """Eq. 3/4 for one pair: reduce over the shared labels, keep u-free then v-free."""
    la, ta = a
    lb, tb = b
    shared = [l for l in la if l in lb]
    ia = [la.index(l) for l in shared]
    ib = [lb.index(l) for l in shared]
    out = [l for l in la if l not in shared] + [l for l in lb if l not in shared]
    return out, np.tensordot(ta, tb, axes=(ia, ib))


def contract(plan, slice_id: int = 0, record=None, override=None):
    """Partial amplitudes a_s over the open legs (array with shape (2,)*len(open)).

    ``record``: optional dict; if given, record[node_id] = (labels, tensor) for every node id in
    it on entry (used to compare stem intermediates by label, not by layout).
    ``override``: optional dict node_id -> (labels, tensor) replacing that node's value as soon as
    it is formed (the contraction is linear in every node, so overriding a stem node with a
    perturbation e yields the perturbation's image at the root; used to propagate swap errors)."""
    if not isinstance(plan, Plan):
        plan = load(plan)
    nodes = slice_leaves(plan, slice_id)
    count = {}
    for labels, _ in nodes:
        for l in labels:
            count[l] = count.get(l, 0) + 1
    if any(c > 2 for c in count.values()):
        raise ValueError("hyper-edges are not part of the RQC network")
    for u, v in plan.tree:
        nodes.append(contract_pair(nodes[u], nodes[v]))
        if override is not None and len(nodes) - 1 in override:
            lab, t = override[len(nodes) - 1]
            if sorted(lab) != sorted(nodes[-1][0]) or t.shape != nodes[-1][1].shape:
                raise ValueError("override must carry the node's labels and shape")
            nodes[-1] = (list(lab), t)
        if record is not None and len(nodes) - 1 in record:
            record[len(nodes) - 1] = nodes[-1]
    labels, t = nodes[-1]
    if sorted(labels) != sorted(plan.open):
        raise ValueError("root labels do not match the open legs")
    return np.transpose(t, [labels.index(l) for l in plan.open]) if plan.open else t


def contract_all_slices(plan):
    if not isinstance(plan, Plan):
        plan = load(plan)
    acc = None
    for s in range(1 << len(plan.sliced)):
        a = contract(plan, s)
        acc = a if acc is None else acc + a
    return acc


def flops(plan):
    """8 real flops per complex MAC (reading C-A21) of one slice, summed over the tree."""
    if not isinstance(plan, Plan):
        plan = load(plan)
    sl = set(plan.sliced)
    labs = [set(l for l in labels if l not in sl) for labels, _ in plan.tensors]
    total = 0
    for u, v in plan.tree:
        total += 8 * (1 << len(labs[u] | labs[v]))
        labs.append(labs[u] ^ labs[v])
    return total
