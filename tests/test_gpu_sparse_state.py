"""Sparse-state tail (§3.4.2, Fig. 5).

The plan names some open legs as sparse legs ("sparse_legs"): a correlated subspace is one value of
them (a prefix), the other open legs are its members.  From the first stem step whose branch holds a
sparse leg, every stem tensor is a batch over the distinct prefix values of the sparse legs it holds,
contracted with the gather-batched tcgen05 GEMM C[n] = A[Index_A[n]] x B[Index_B[n]] (small steps:
one GEMM per entry); subspaces are chunked when the batch does not fit.

Oracle: the plain definition — the full amplitude tensor over all open legs (oracle contraction)
indexed at each prefix.  Bounds: rel-L2 <= 2e-2 (complex-half), <= 1e-5 (complex64) per subspace;
the post-selected member is a valid pick (C-A24)."""
import json
import os

import numpy as np
import pytest

from oracle import contract, metrics
from oracle.plan import load
from workload import make_plans as MP

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
TOL = {0: 2e-2, 1: 1e-5}


@pytest.fixture(scope="module")
def tn():
    import torch
    from paper_2407_00769_b200 import build as B
    B.build()
    from paper_2407_00769_b200 import tn as T
    assert torch.cuda.is_available()
    return T


def with_sparse_legs(tn, plan, n_sparse, stem_min):
    """Choose the n_sparse open legs that enter the stem last (never in the stem entry)."""
    rep = tn.Plan(plan, tn.make_config(stem_min_log2=stem_min)).report()
    first = {}
    for i, st in enumerate(rep["steps"]):
        for l in st["in"] + st["out"]:
            first.setdefault(l, i)
    cand = [l for l in plan["open"] if l not in rep["entry_layout"]]
    cand.sort(key=lambda l: -first.get(l, 10 ** 9))
    assert len(cand) >= n_sparse
    out = dict(plan)
    out["sparse_legs"] = sorted(cand[:n_sparse], key=plan["open"].index)
    return out


def oracle_blocks(plan, ref):
    """ref [open...] -> [prefix (sparse legs, MSB first), members (open order without them)]"""
    sp = plan["sparse_legs"]
    rest = [l for l in plan["open"] if l not in sp]
    t = np.transpose(ref, [plan["open"].index(l) for l in sp + rest])
    return t.reshape(2 ** len(sp), -1)


def run(tn, plan, dtype, stem_min, prefixes, k=1):
    p = tn.Plan(plan, tn.make_config(dtype=dtype, stem_min_log2=stem_min))
    b = tn.Buffers(p)
    tn.tn_plan_upload(p, b)
    tn.tn_stem_contract(p, b, 0)
    amps, top = tn.tn_sample_sparse(p, b, prefixes, k=k)
    return amps, top, p


@pytest.mark.parametrize("dtype", [0, 1])
@pytest.mark.parametrize("n_sparse", [2, 4, 6])
def test_sparse_tail_c1_vs_oracle(tn, dtype, n_sparse):
    plan = with_sparse_legs(tn, MP.build_plan(3, 4, False, 8, 12, None, trials=2, seed=1), n_sparse, 6)
    ref = oracle_blocks(plan, contract.contract(load(plan), 0))
    rng = np.random.default_rng(n_sparse)
    pre = rng.choice(2 ** n_sparse, size=min(5, 2 ** n_sparse), replace=False).astype(np.uint64)
    amps, top, p = run(tn, plan, dtype, 6, pre)
    assert sum(s["sparse"] for s in p.report()["steps"]) >= 1
    for i, v in enumerate(pre):
        assert metrics.rel_l2(amps[i], ref[v]) <= TOL[dtype]
        pr = np.abs(ref[v]) ** 2
        assert pr[int(top[i, 0])] >= (1 - 4 * TOL[dtype]) * pr.max()


@pytest.mark.parametrize("n_sparse", [3, 5])
def test_sparse_tail_c2_batched_tcgen05_vs_oracle(tn, n_sparse):
    """C2 sub-sliced: tail steps big enough (>= 128 rows per entry) for the gather-batched tcgen05
    launch; repeated and unsorted prefixes; complex-half vs complex64 vs oracle."""
    with open(os.path.join(ROOT, "plans", "c2.json")) as f:
        sub = MP.sub_slice(json.load(f), 20)
    plan = with_sparse_legs(tn, sub, n_sparse, 12)
    ref = oracle_blocks(plan, contract.contract(load(plan), 0))
    pre = np.array([5, 1, 5, 0, 2 ** n_sparse - 1, 3], dtype=np.uint64) % (2 ** n_sparse)
    a16, top, p = run(tn, plan, 0, 12, pre)
    a32, _, _ = run(tn, plan, 1, 12, pre)
    for i, v in enumerate(pre):
        assert metrics.rel_l2(a16[i], ref[v]) <= 2e-2
        assert metrics.rel_l2(a32[i], ref[v]) <= 1e-5
    assert np.array_equal(a16[0], a16[2])          # the same subspace twice: identical answers


def test_sparse_tail_chunked_by_capacity(tn):
    """Free stem buffer too small for the whole batch: the subspaces run in chunks, same
    answers as one chunk."""
    with open(os.path.join(ROOT, "plans", "c2.json")) as f:
        sub = MP.sub_slice(json.load(f), 20)
    plan = with_sparse_legs(tn, sub, 5, 12)
    pre = np.arange(32, dtype=np.uint64)
    p = tn.Plan(plan, tn.make_config(dtype=0, stem_min_log2=12))
    b = tn.Buffers(p)
    tn.tn_plan_upload(p, b)
    tn.tn_stem_contract(p, b, 0)
    a_all, _ = tn.tn_sample_sparse(p, b, pre)
    assert p.report().get("sparse_chunks", 1) >= 1
    ref = oracle_blocks(plan, contract.contract(load(plan), 0))
    for i in range(32):
        assert metrics.rel_l2(a_all[i], ref[i]) <= 2e-2


def test_c5_sparse_state_subslice_vs_oracle(tn):
    """C5 (BJ configs[4]): 53-qubit 20-cycle network, 10 member legs, 12 sparse legs entering the stem
    in its final stage; sub-sliced so the oracle's dense root (2^22 amplitudes) is cheap; 64 seeded
    prefixes.  Complex-half amplitudes per subspace vs the oracle, valid post-selected members."""
    with open(os.path.join(ROOT, "plans", "c5.json")) as f:
        c5 = json.load(f)
    sub = MP.sub_slice(c5, 24)
    assert sub["sparse_legs"] == c5["sparse_legs"]
    ref = oracle_blocks(sub, contract.contract(load(sub), 0))
    rng = np.random.default_rng(5)
    pre = rng.choice(2 ** 12, size=64, replace=False).astype(np.uint64)
    amps, top, p = run(tn, sub, 0, 16, pre)
    assert p.info()["n_sparse_legs"] == 12
    errs = [metrics.rel_l2(amps[i], ref[v]) for i, v in enumerate(pre)]
    assert max(errs) <= 2e-2, max(errs)
    for i, v in enumerate(pre):
        pr = np.abs(ref[v]) ** 2
        assert pr[int(top[i, 0])] >= (1 - 4e-2) * pr.max()
