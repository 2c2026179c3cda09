"""Result metrics.

* rel_l2(result, reference) = ||r - o||_2 / ||o||_2 (BASELINE.json tolerances are stated in it).
* fidelity, PAPER.md Eq. "fidelity", reading C-A15:
  |<b, r>|^2 / (||b||^2 ||r||^2) with the sesquilinear <b, r> = sum conj(b) r.
* linear XEB = 2^n * mean(p) - 1 (reading C-A22; the paper never defines the estimator).
* post-selection: keep the top-k probability members of each correlated subspace; ties go
  to the lexicographically smallest bitstring (C-A23).
"""
import numpy as np


def rel_l2(result, reference):
    r = np.asarray(result, dtype=np.complex128).reshape(-1)
    o = np.asarray(reference, dtype=np.complex128).reshape(-1)
    return float(np.linalg.norm(r - o) / np.linalg.norm(o))


def fidelity(benchmark, result):
    b = np.asarray(benchmark, dtype=np.complex128).reshape(-1)
    r = np.asarray(result, dtype=np.complex128).reshape(-1)
    nb = np.vdot(b, b).real
    nr = np.vdot(r, r).real
    if nb == 0 or nr == 0:
        raise ValueError("fidelity undefined for a zero-norm argument")
    ip = np.vdot(b, r)
    return float(abs(ip) ** 2 / (nb * nr))


def linear_xeb(probs, n_qubits):
    p = np.asarray(probs, dtype=np.float64)
    if p.size == 0:
        raise ValueError("empty sample set")
    return float(2.0 ** n_qubits * p.mean() - 1.0)


def post_select(probs_per_subspace, k=1):
    """probs_per_subspace: array [S, N].  Returns [S, k] member indices (descending probability,
    ties -> smaller index)."""
    p = np.asarray(probs_per_subspace, dtype=np.float64)
    # stable sort on -p keeps the smaller index first among equal probabilities
    order = np.argsort(-p, axis=1, kind="stable")
    return order[:, :k]


def harmonic(n):
    return float(sum(1.0 / k for k in range(1, n + 1)))
