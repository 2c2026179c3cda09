"""Multi-subtask post-selection pipeline on the GPU: the
partial amplitudes of every slice (subtask) of a sliced network, each from one sparse-state call,
summed by the caller (a.9), top-1 per correlated subspace, linear XEB of the picks.

Pins: the slice sum equals the oracle's unsliced amplitudes (slicing identity) within the
fp16 bound; with all slices conducted (f = 1) the picks are exact top-1 samples of a Porter-Thomas
distribution, whose linear XEB is H_N - 1 (reading C-A22) within 4 standard errors."""
import math

import numpy as np
import pytest

from oracle import contract, metrics
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


def test_all_slices_post_selection_xeb(tn):
    from paper_2407_00769_b200 import postselect
    plan = MP.build_plan(3, 4, False, 14, 12, None, trials=2, seed=11)
    sub = MP.sub_slice(plan, plan["meta"]["max_log2"] - 2)
    n_sl = len(sub["sliced"])
    assert 1 <= n_sl <= 12
    # the 6 open legs entering the stem last are the sparse legs: 64 subspaces x 64 members
    p0 = tn.Plan(sub, tn.make_config(stem_min_log2=6))
    rep = p0.report()
    first = {}
    for i, st in enumerate(rep["steps"]):
        for l in st["in"] + st["out"]:
            first.setdefault(l, i)
    cand = sorted([l for l in sub["open"] if l not in rep["entry_layout"]], key=lambda l: -first.get(l, 10 ** 9))
    sub["sparse_legs"] = sorted(cand[:6], key=sub["open"].index)
    rest = [l for l in sub["open"] if l not in sub["sparse_legs"]]
    exact = contract.contract(load(plan), 0)            # unsliced = exact amplitudes
    ref = np.transpose(exact, [sub["open"].index(l) for l in sub["sparse_legs"] + rest]).reshape(64, 64)
    amps, _ = postselect.contract_subspaces(sub, np.arange(64, dtype=np.uint64), range(2 ** n_sl),
                                            tn.make_config(stem_min_log2=6))
    assert metrics.rel_l2(amps, ref) <= 2e-2
    top, _ = postselect.post_select(amps)
    pr = np.abs(ref) ** 2
    chosen = pr[np.arange(64), top]
    assert np.all(chosen >= (1 - 4e-2) * pr.max(axis=1))        # valid picks (C-A24)
    xeb = postselect.linear_xeb(chosen, 12)
    se = math.sqrt(sum(1.0 / k ** 2 for k in range(1, 65))) / math.sqrt(64)
    assert abs(xeb - (metrics.harmonic(64) - 1.0)) < 4 * se
