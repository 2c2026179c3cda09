"""Seeded Sycamore-style random quantum circuit (RQC) generator.

Input generator only: it emits gate *names*, qubit indices and fSim parameters; it holds none of
the method's arithmetic (no matrices, no contraction).  Both the CUDA path (through the plan
JSON written by ``workload.network``/``workload.planner``) and the oracle consume its output.

Structure follows PAPER.md §2.1: ``m`` full cycles, each "a single-qubit gate is
applied to each qubit. Next, two-qubit gates are applied to pairs of qubits", followed by a half
cycle of single-qubit gates.  Readings the paper leaves open:

* C-A2: fSim(theta, phi) = (pi/2, pi/6) for every pair (Sycamore nominal), optional seeded jitter.
* C-A3: single-qubit gate drawn uniformly from {sqrt_x, sqrt_y, sqrt_w} excluding the gate the
  same qubit received in the previous cycle; two-qubit couplers of a 2-D grid in classes
  A (horizontal, even column), B (horizontal, odd column), C (vertical, even row),
  D (vertical, odd row), applied in the sequence ABCDCDAB.
* C-A4: qubit q = row * cols + col; bitstring integer has qubit 0 as the most significant bit.
"""
from __future__ import annotations

import math
import random

GATES_1Q = ("sqrt_x", "sqrt_y", "sqrt_w")
PATTERN = "ABCDCDAB"


def grid_qubits(rows: int, cols: int, drop_corner: bool = False):
    """Return the list of (row, col) sites; ``drop_corner`` removes the last site (53 = 6x9-1)."""
    sites = [(r, c) for r in range(rows) for c in range(cols)]
    if drop_corner:
        sites = sites[:-1]
    return sites


def couplers(sites, cls: str):
    idx = {s: i for i, s in enumerate(sites)}
    out = []
    for (r, c), q in idx.items():
        if cls == "A" and c % 2 == 0 and (r, c + 1) in idx:
            out.append((q, idx[(r, c + 1)]))
        elif cls == "B" and c % 2 == 1 and (r, c + 1) in idx:
            out.append((q, idx[(r, c + 1)]))
        elif cls == "C" and r % 2 == 0 and (r + 1, c) in idx:
            out.append((q, idx[(r + 1, c)]))
        elif cls == "D" and r % 2 == 1 and (r + 1, c) in idx:
            out.append((q, idx[(r + 1, c)]))
    return sorted(out)


def make_circuit(rows: int, cols: int, cycles: int, seed: int, drop_corner: bool = False,
                 theta: float = math.pi / 2, phi: float = math.pi / 6, jitter: float = 0.0):
    """Seeded RQC description (dict, JSON-serialisable)."""
    rng = random.Random(seed)
    sites = grid_qubits(rows, cols, drop_corner)
    n = len(sites)
    gates = []
    prev = [None] * n

    def layer_1q(cyc):
        for q in range(n):
            choices = [g for g in GATES_1Q if g != prev[q]]
            g = rng.choice(choices)
            prev[q] = g
            gates.append({"kind": g, "qubits": [q], "cycle": cyc})

    for cyc in range(cycles):
        layer_1q(cyc)
        for a, b in couplers(sites, PATTERN[cyc % len(PATTERN)]):
            th = theta + (rng.uniform(-jitter, jitter) if jitter else 0.0)
            ph = phi + (rng.uniform(-jitter, jitter) if jitter else 0.0)
            gates.append({"kind": "fsim", "qubits": [a, b], "cycle": cyc, "theta": th, "phi": ph})
    layer_1q(cycles)  # final half cycle
    return {"n_qubits": n, "rows": rows, "cols": cols, "drop_corner": drop_corner,
            "cycles": cycles, "seed": seed, "sites": sites, "gates": gates}


def random_bits(n: int, seed: int):
    rng = random.Random(seed)
    return [rng.randint(0, 1) for _ in range(n)]
