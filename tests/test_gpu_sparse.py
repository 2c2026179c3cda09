"""Sparse-state batch output + post-selection + XEB.

The correlated subspaces are values of the split legs; only the requested chunks of the stem tail
are contracted (Fig. 5's gather on the stem operand).  Amplitudes vs the oracle; device top-1 per
subspace (ties -> smaller index, C-A23) is a valid pick (C-A24); XEB of the picks on exact
probabilities matches the Porter-Thomas closed form H_N - 1 (C-A22)."""
import math

import numpy as np
import pytest

from oracle import contract, metrics, statevector
from oracle.plan import load
from workload import make_plans as MP

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def tn():
    import torch
    from paper_2407_00769_b200 import build as B
    B.build()
    from paper_2407_00769_b200 import tn as T
    assert torch.cuda.is_available()
    return T


def _blocks(ref, open_labels, split_modes):
    """oracle full-state array [open...] -> [prefix (split legs in open order, include/tn.h), members
    (open order)]"""
    split_modes = [l for l in open_labels if l in split_modes]
    rest = [l for l in open_labels if l not in split_modes]
    t = np.transpose(ref, [open_labels.index(l) for l in split_modes + rest])
    return t.reshape(2 ** len(split_modes), -1)


@pytest.mark.parametrize("dtype,tol", [(0, 2e-2), (1, 1e-5)])
def test_sparse_batch_vs_oracle(tn, dtype, tol):
    plan = MP.build_plan(3, 4, False, 8, 12, None, trials=2, seed=0)
    p = tn.Plan(plan, tn.make_config(dtype=dtype, stem_min_log2=6, split_log2=5))
    b = tn.Buffers(p)
    tn.tn_plan_upload(p, b)
    tn.tn_stem_contract(p, b, 0)
    rep = p.report()
    ref = _blocks(contract.contract(load(plan), 0), plan["open"], rep["split_modes"])
    rng = np.random.default_rng(0)
    pre = rng.choice(32, size=11, replace=False)
    amps, top = tn.tn_sample_sparse(p, b, pre, k=1)
    for i, v in enumerate(pre):
        assert metrics.rel_l2(amps[i], ref[v]) <= tol
        pr = np.abs(ref[v]) ** 2
        assert pr[int(top[i, 0])] >= (1 - 2 * tol) * pr.max()     # a valid post-selected pick
    # the dense readout after a sparse batch still returns every chunk
    full = tn.tn_sample_amplitudes(p, b)[0]
    assert metrics.rel_l2(full, contract.contract(load(plan), 0)) <= tol


def test_post_selection_xeb_porter_thomas(tn):
    """Deep 12-qubit circuit, 64 subspaces of 64 members: top-1 XEB on exact probabilities
    = H_64 - 1 within 4 standard errors (reading C-A22)."""
    plan = MP.build_plan(3, 4, False, 14, 12, None, trials=2, seed=11)
    p = tn.Plan(plan, tn.make_config(dtype=0, stem_min_log2=6, split_log2=6))
    b = tn.Buffers(p)
    tn.tn_plan_upload(p, b)
    tn.tn_stem_contract(p, b, 0)
    rep = p.report()
    amps, top = tn.tn_sample_sparse(p, b, np.arange(64), k=1)
    psi = statevector.simulate(plan["circuit"])
    # exact probabilities in the same [prefix, member] arrangement, via the oracle (unsliced = exact;
    # the oracle equals the state vector, tests/test_oracle.py)
    ref = _blocks(contract.contract(load(plan), 0), plan["open"], rep["split_modes"])
    pr = np.abs(ref) ** 2
    chosen = pr[np.arange(64), top[:, 0].astype(np.int64)]
    assert np.all(chosen >= (1 - 4e-2) * pr.max(axis=1))
    xeb = metrics.linear_xeb(chosen, 12)
    N = 64
    se = math.sqrt(sum(1.0 / k ** 2 for k in range(1, N + 1))) / math.sqrt(64)
    assert abs(xeb - (metrics.harmonic(N) - 1.0)) < 4 * se
    assert abs(np.sum(pr) - 1.0) < 1e-12 and psi.size == 4096
