"""Circuit -> tensor network (§2.2): "Single-qubit and two-qubit quantum gate
operations can be represented by rank-2 and rank-4 tensors".

Input generator (L0).  Builds the closed/open network of <x|U|0...0> for a circuit from
``workload.circuit`` and applies exact rank simplification (absorbing rank<=2 tensors into a
neighbour) so the leaves are the fused fSim tensors a Sycamore network consists of.

Gate matrices follow P:183-201 with conventions C-A1 (principal roots for sqrt(i), sqrt(-i)) and
C-A4 (gate tensor G[out..., in...]; 2-qubit basis |q_a q_b> with a < b).  The oracle keeps its
OWN gate library (oracle/gates.py) and pins these leaves indirectly through the state-vector
comparison; nothing here is imported by the oracle or the CUDA library.
"""
from __future__ import annotations

import cmath
import math

import numpy as np


def gate_matrix(g):
    k = g["kind"]
    s = 1.0 / math.sqrt(2.0)
    if k == "sqrt_x":
        return s * np.array([[1, -1j], [-1j, 1]], dtype=np.complex128)
    if k == "sqrt_y":
        return s * np.array([[1, -1], [1, 1]], dtype=np.complex128)
    if k == "sqrt_w":
        return s * np.array([[1, -cmath.exp(1j * math.pi / 4)],
                             [cmath.exp(-1j * math.pi / 4), 1]], dtype=np.complex128)
    if k == "fsim":
        th, ph = g["theta"], g["phi"]
        c, sn = math.cos(th), math.sin(th)
        return np.array([[1, 0, 0, 0],
                         [0, c, -1j * sn, 0],
                         [0, -1j * sn, c, 0],
                         [0, 0, 0, cmath.exp(-1j * ph)]], dtype=np.complex128)
    raise ValueError(f"unknown gate kind {k}")


class Network:
    """tensors: list of (labels tuple, ndarray with shape (2,)*rank); open: list of labels."""

    def __init__(self):
        self.tensors = []
        self.open = []
        self.next_label = 0
        self.label_pos = {}  # label -> (qubit, time); used only by the sweep-order planner

    def new_label(self, qubit=None, time=None):
        self.label_pos[self.next_label] = (qubit, time)
        self.next_label += 1
        return self.next_label - 1


def build_network(circ, bits=None, open_qubits=()):
    """Network of <bits|U|0..0> with the qubits in ``open_qubits`` left open (legs in the order
    given).  ``bits`` covers all qubits (entries of open qubits are ignored)."""
    n = circ["n_qubits"]
    net = Network()
    cur = []
    for q in range(n):
        l = net.new_label(q, -1)
        net.tensors.append(((l,), np.array([1.0, 0.0], dtype=np.complex128)))
        cur.append(l)
    for g in circ["gates"]:
        m = gate_matrix(g)
        if len(g["qubits"]) == 1:
            q = g["qubits"][0]
            lo = net.new_label(q, 2 * g["cycle"])
            net.tensors.append(((lo, cur[q]), m.copy()))
            cur[q] = lo
        else:
            a, b = g["qubits"]
            assert a < b
            la, lb = net.new_label(a, 2 * g["cycle"] + 1), net.new_label(b, 2 * g["cycle"] + 1)
            net.tensors.append(((la, lb, cur[a], cur[b]), m.reshape(2, 2, 2, 2).copy()))
            cur[a], cur[b] = la, lb
    open_set = set(open_qubits)
    for q in range(n):
        if q in open_set:
            continue
        x = 0 if bits is None else bits[q]
        v = np.zeros(2, dtype=np.complex128)
        v[x] = 1.0
        net.tensors.append(((cur[q],), v))
    net.open = [cur[q] for q in open_qubits]
    return net


def _contract_pair(ta, tb, open_set):
    la, da = ta
    lb, db = tb
    shared = [l for l in la if l in lb]
    out = [l for l in la if l not in shared] + [l for l in lb if l not in shared]
    letters = {}
    for l in list(la) + list(lb):
        if l not in letters:
            letters[l] = chr(ord("a") + len(letters)) if len(letters) < 26 else chr(ord("A") + len(letters) - 26)
    spec = "".join(letters[l] for l in la) + "," + "".join(letters[l] for l in lb) + "->" + "".join(letters[l] for l in out)
    return tuple(out), np.einsum(spec, da, db)


def simplify(net, max_rank=4):
    """Exact rank simplification: absorb tensors of rank <= 2 into a neighbour (fewest legs first)
    as long as the result keeps rank <= max_rank."""
    tensors = list(net.tensors)
    open_set = set(net.open)
    changed = True
    while changed:
        changed = False
        where = {}
        for i, (ls, _) in enumerate(tensors):
            for l in ls:
                where.setdefault(l, []).append(i)
        order = sorted(range(len(tensors)), key=lambda i: len(tensors[i][0]))
        dead = set()
        new = []
        for i in order:
            if i in dead:
                continue
            ls, _ = tensors[i]
            if len(ls) > 2:
                break
            nbrs = sorted({j for l in ls for j in where[l] if j != i and j not in dead})
            best = None
            for j in nbrs:
                lj = tensors[j][0]
                r = len(set(ls) ^ set(lj))
                if r <= max_rank and (best is None or r < best[0]):
                    best = (r, j)
            if best is None:
                continue
            j = best[1]
            merged = _contract_pair(tensors[j], tensors[i], open_set)
            dead.add(i)
            dead.add(j)
            new.append(merged)
            changed = True
        if changed:
            tensors = [t for k, t in enumerate(tensors) if k not in dead] + new
    # relabel densely for compact plans
    relabel = {}
    out = []
    for ls, d in tensors:
        for l in ls:
            relabel.setdefault(l, len(relabel))
        out.append((tuple(relabel[l] for l in ls), d))
    for l in net.open:
        relabel.setdefault(l, len(relabel))
    res = Network()
    res.tensors = out
    res.open = [relabel[l] for l in net.open]
    res.next_label = len(relabel)
    res.label_pos = {relabel[l]: p for l, p in net.label_pos.items() if l in relabel}
    return res
