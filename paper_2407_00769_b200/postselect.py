"""Multi-subtask post-selection pipeline ("computing ... independent correlated
subspaces, each containing thousands of samples, and subsequently selecting the sample with the
highest probability from each correlated subspace").

Global level of the method: every conducted slice (subtask) contributes its partial amplitudes of
the requested correlated subspaces (the sparse-state batch of one tn_sample_amplitudes call); the
caller sums them over the slices it conducts (reading C-A25: a fraction f of the
2^|sliced| subtasks), post-selects the most probable member of each subspace (top-1, ties to the
smaller member index, C-A23) and scores the selected bitstrings with the linear XEB
2^n <p> - 1 (reading C-A22).  All contraction work runs in libtn's kernels; this module only
accumulates the returned complex128 blocks (the a.9 slice sum, <= 2^20 numbers per subtask).
"""
from __future__ import annotations

import numpy as np

from . import tn


def contract_subspaces(plan_json, prefixes, slices, cfg=None, stem_bytes=None):
    """Sum over `slices` of the partial amplitudes of the subspaces `prefixes` (a sparse-state plan:
    prefixes are values of the plan's sparse legs).  Returns (amplitudes [S, members] complex128,
    plan)."""
    p = tn.Plan(plan_json, cfg or tn.make_config(stem_min_log2=20))
    b = tn.Buffers(p, stem_bytes=stem_bytes)
    tn.tn_plan_upload(p, b)
    acc = None
    for s in slices:
        tn.tn_stem_contract(p, b, int(s))
        amps, _ = tn.tn_sample_sparse(p, b, prefixes, k=0)
        acc = amps.copy() if acc is None else acc + amps
    return acc, p


def post_select(amps):
    """Most probable member of each subspace (ties -> smaller member index, C-A23); returns
    (member index per subspace, its probability)."""
    prob = np.abs(amps) ** 2
    top = np.argmax(prob, axis=1)          # numpy argmax returns the first (smallest) index on ties
    return top, prob[np.arange(len(top)), top]


def linear_xeb(p_selected, n_qubits):
    """Linear XEB of the selected bitstrings (reading C-A22): 2^n * mean(p) - 1."""
    return float(2.0 ** n_qubits * np.mean(p_selected) - 1.0)
