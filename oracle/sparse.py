"""Sparse-state gathered contraction, §3.4.2 / Fig. 5, complex128.

* gather_contract: C[n] = A[Index_A[n]] x B[Index_B[n]] (Fig. 5 bottom, "retrieving tensors
  through indices"); A[a, M, K] and B[b, K, N] -> C[n, M, N].
* build_padded_index: m_r = max repeat count of a value in Index_A; table [m_a, m_r] of Index_B
  values in Index_A order, excess positions = -1.
* padded_contract: C_P = A x B_P with B_P gathered through the table (-1 -> zero block), then
  flatten and extract the valid rows (Fig. 5 top).
"""
import numpy as np


def gather_contract(a, b, index_a, index_b):
    a = np.asarray(a, dtype=np.complex128)
    b = np.asarray(b, dtype=np.complex128)
    return np.stack([a[i] @ b[j] for i, j in zip(index_a, index_b)]) if len(index_a) else \
        np.zeros((0, a.shape[1], b.shape[2]), dtype=np.complex128)


def build_padded_index(index_a, index_b, m_a):
    reps = np.zeros(m_a, dtype=np.int64)
    for i in index_a:
        reps[i] += 1
    m_r = int(reps.max()) if len(index_a) else 0
    table = -np.ones((m_a, m_r), dtype=np.int64)
    fill = np.zeros(m_a, dtype=np.int64)
    for i, j in zip(index_a, index_b):
        table[i, fill[i]] = j
        fill[i] += 1
    return table, m_r


def padded_contract(a, b, index_a, index_b):
    a = np.asarray(a, dtype=np.complex128)
    b = np.asarray(b, dtype=np.complex128)
    m_a = a.shape[0]
    table, m_r = build_padded_index(index_a, index_b, m_a)
    K, N = b.shape[1], b.shape[2]
    bp = np.zeros((m_a, m_r, K, N), dtype=np.complex128)
    for i in range(m_a):
        for r in range(m_r):
            if table[i, r] >= 0:
                bp[i, r] = b[table[i, r]]
    cp = np.einsum("amk,arkn->armn", a, bp)          # C_P = A x B_P
    # extract: the k-th occurrence of value i in Index_A is C_P[i, k]
    occ = np.zeros(m_a, dtype=np.int64)
    out = []
    for i in index_a:
        out.append(cp[i, occ[i]])
        occ[i] += 1
    return np.stack(out) if out else np.zeros((0, a.shape[1], N), dtype=np.complex128)
