"""State-vector method (§2.2): brute-force evolution of the full 2^n state.

The independent textbook routine that pins the tensor-network oracle.
Qubit 0 is axis 0 (the most significant bit of a bitstring index, reading C-A4); input |0...0>.
Gate order is the circuit's list order: per cycle all single-qubit gates then the two-qubit gates,
then the final half cycle.
"""
import numpy as np

from . import gates


def simulate(circ):
    n = circ["n_qubits"]
    psi = np.zeros((2,) * n, dtype=np.complex128)
    psi[(0,) * n] = 1.0
    for g in circ["gates"]:
        m = gates.matrix(g)
        qs = g["qubits"]
        if len(qs) == 1:
            q = qs[0]
            psi = np.moveaxis(np.tensordot(m, psi, axes=([1], [q])), 0, q)
        else:
            a, b = qs
            g4 = m.reshape(2, 2, 2, 2)  # (out_a, out_b, in_a, in_b)
            psi = np.moveaxis(np.tensordot(g4, psi, axes=([2, 3], [a, b])), [0, 1], [a, b])
    return psi


def amplitudes(psi, bits, open_qubits):
    """Amplitude block <bits|psi> over the open qubits (in the order given)."""
    n = psi.ndim
    idx = []
    for q in range(n):
        idx.append(slice(None) if q in open_qubits else bits[q])
    block = psi[tuple(idx)]
    # remaining axes are the open qubits in increasing qubit order -> reorder as requested
    inc = sorted(open_qubits)
    perm = [inc.index(q) for q in open_qubits]
    return np.transpose(block, perm) if perm else block
