"""End-to-end parity through the C-ABI on a B200: the full stem path (common phase, Eq. 6
padding, permutations, tcgen05/SIMT GEMMs, power-of-two scaling) vs the complex128 oracle on
the same plan and slice.  Tolerances (BASELINE.json north_star): rel-L2 <= 1e-5 (complex64 path),
<= 2e-2 (complex-half path)."""
import json
import os

import numpy as np
import pytest

from oracle import contract, metrics
from oracle.plan import load
from workload import make_plans as MP

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
TOL = {0: 2e-2, 1: 1e-5}   # TN_CHALF, TN_CFLOAT


@pytest.fixture(scope="module")
def tn():
    import torch
    from paper_2407_00769_b200 import build as B
    B.build()
    from paper_2407_00769_b200 import tn as T
    assert torch.cuda.is_available()
    return T


def _plan(name):
    with open(os.path.join(ROOT, "plans", f"{name}.json")) as f:
        return json.load(f)


def run_gpu(tn, plan, dtype, slice_id=0, stem_min_log2=6, policy=0):
    p = tn.Plan(plan, tn.make_config(dtype=dtype, stem_min_log2=stem_min_log2, layout_policy=policy))
    bufs = tn.Buffers(p)
    amps = tn.contract(p, bufs, slice_id)
    return amps, p


@pytest.mark.parametrize("policy", [0, 1, 2, 3])
@pytest.mark.parametrize("dtype", [0, 1])
@pytest.mark.parametrize("stem_min", [6, 8, 10])
def test_c1_full_state_vs_oracle(tn, dtype, stem_min, policy):
    """public layout policies (tn.h): 0 = identity outputs + fused/standalone permutations, 1 = hybrid,
    2 = scatter-epilogue layouts (no permutation passes)."""
    plan = _plan("c1")
    ref = contract.contract(load(plan), 0)
    got, p = run_gpu(tn, plan, dtype, 0, stem_min, policy)
    assert p.info()["n_stem_steps"] >= 1
    assert metrics.rel_l2(got, ref) <= TOL[dtype]
    assert abs(np.sum(np.abs(got) ** 2) - 1.0) <= (2 * TOL[dtype])


@pytest.mark.parametrize("seed", range(6))
@pytest.mark.parametrize("dtype", [0, 1])
@pytest.mark.parametrize("policy", [0, 1, 2, 3])
def test_random_small_circuits_sliced(tn, seed, dtype, policy):
    """Seeded small circuits with extra sliced edges: every slice vs the oracle slice, and the
    GPU sum over slices vs the unsliced oracle (slicing identity)."""
    rng = np.random.default_rng(seed)
    rows, cols = [(3, 4), (3, 3), (2, 5)][seed % 3]
    plan = MP.build_plan(rows, cols, False, int(rng.integers(4, 9)), int(rng.integers(2, 7)), None, trials=2,
                         seed=seed)
    sub = MP.sub_slice(plan, max(4, plan["meta"]["max_log2"] - 2))
    full = contract.contract(load(plan), 0)
    tot = 0
    for s in range(1 << len(sub["sliced"])):
        ref = contract.contract(load(sub), s)
        got, _ = run_gpu(tn, sub, dtype, s, stem_min_log2=3, policy=policy)
        if np.linalg.norm(ref) > 1e-12:
            assert metrics.rel_l2(got, ref) <= TOL[dtype]
        tot = tot + got
    assert metrics.rel_l2(tot, full) <= TOL[dtype]


@pytest.mark.parametrize("dtype", [0, 1])
@pytest.mark.parametrize("policy", [0, 1, 2, 3])
def test_c2_reduced_vs_oracle(tn, dtype, policy):
    """C2 (30 qubits, 14 cycles) with extra sub-slicing so the oracle finishes in seconds
    (SURVEY §8(c) c.6): same tree, same kernels, stems up to 2^22."""
    sub = MP.sub_slice(_plan("c2"), 22)
    for s in (0, (1 << len(sub["sliced"])) - 1):
        ref = contract.contract(load(sub), s)
        got, p = run_gpu(tn, sub, dtype, s, stem_min_log2=12, policy=policy)
        assert p.info()["n_stem_steps"] >= 3
        assert metrics.rel_l2(got, ref) <= TOL[dtype]


def test_c2_full_fp32_vs_fp16(tn):
    """Full-size C2 slice: the complex-half path vs the complex64 path (same plan, same slice)."""
    plan = _plan("c2")
    a32, _ = run_gpu(tn, plan, 1, 0, stem_min_log2=16)
    a16, _ = run_gpu(tn, plan, 0, 0, stem_min_log2=16)
    assert metrics.rel_l2(a16, a32) <= 2e-2


def test_slice_id_out_of_range(tn):
    plan = _plan("c2")
    p = tn.Plan(plan, tn.make_config(stem_min_log2=16))
    bufs = tn.Buffers(p)
    tn.tn_plan_upload(p, bufs)
    with pytest.raises(tn.TnError) as e:
        tn.tn_stem_contract(p, bufs, 1 << len(plan["sliced"]))
    assert e.value.code == -1


@pytest.mark.parametrize("policy", [0, 2])
@pytest.mark.parametrize("split", [1, 2, 3])
@pytest.mark.parametrize("dtype", [0, 1])
def test_split_tail_vs_oracle(tn, split, policy, dtype):
    """Split-type tail: the last stem steps run on 2^j chunks inside the
    stem buffers.  Same amplitudes as the oracle; the complex64 path is bit-identical to the
    unsplit run (chunking does not change any per-element sum)."""
    sub = MP.sub_slice(_plan("c2"), 20)
    ref = contract.contract(load(sub), 0)
    p = tn.Plan(sub, tn.make_config(dtype=dtype, stem_min_log2=12, split_log2=split, layout_policy=policy))
    assert p.info()["split_chunks"] == 2 ** split
    rep = p.report()
    assert sum(s["split"] for s in rep["steps"]) >= 1
    got = tn.contract(p, tn.Buffers(p), 0)
    assert metrics.rel_l2(got, ref) <= TOL[dtype]
    if dtype == 1:
        p0 = tn.Plan(sub, tn.make_config(dtype=dtype, stem_min_log2=12, layout_policy=policy))
        assert np.array_equal(tn.contract(p0, tn.Buffers(p0), 0), got)


@pytest.mark.parametrize("dtype", [0, 1])
def test_graph_replay_across_slices(tn, dtype):
    """One plan, one buffer set, every slice in turn: the CUDA-graph replay (slice id read on the
    device) matches the oracle per slice and is bit-identical to eager launches; toggling timing
    re-captures and still matches."""
    sub = MP.sub_slice(_plan("c2"), 18)
    p = tn.Plan(sub, tn.make_config(dtype=dtype, stem_min_log2=10))
    bufs = tn.Buffers(p)
    n = 1 << len(sub["sliced"])
    picks = sorted({0, 1, n // 2, n - 1, 5 % n})
    graph = {}
    for k, s in enumerate(picks + picks[::-1]):
        p.set_timing(k % 3 == 1)
        graph[s] = tn.contract(p, bufs, s)
        assert metrics.rel_l2(graph[s], contract.contract(load(sub), s)) <= TOL[dtype]
    p.set_timing(False)
    p.set_graph(False)
    for s in picks:
        assert np.array_equal(tn.contract(p, bufs, s), graph[s])
    # timing events recorded by the graph replay feed the report
    p.set_graph(True)
    p.set_timing(True)
    tn.tn_stem_contract(p, bufs, picks[-1])
    ms = p.report()["ms"]
    assert len(ms) == 2 + 2 * p.info()["n_stem_steps"] and all(m >= 0 for m in ms) and sum(ms) > 0


@pytest.mark.parametrize("dtype", [0])
def test_fused_permutation_matches_permute_pass(tn, dtype):
    """Gathered-A GEMMs (permutation fused into the load) vs explicit permutation passes on the
    same plan: same operands, same K order, same accumulation -> bit-identical amplitudes; and the
    oracle within tolerance.  (Layout policy 0: under policy 3 the output layouts, and so the K
    orders, depend on which steps can gather.)"""
    sub = MP.sub_slice(_plan("c2"), 22)
    out = {}
    for ng in (0, 1):
        p = tn.Plan(sub, tn.make_config(dtype=dtype, stem_min_log2=12, no_gather=ng, layout_policy=0))
        rep = p.report()
        out[ng] = (tn.contract(p, tn.Buffers(p), 0), sum(s["ga"] for s in rep["steps"]), p.info()["n_permutes"])
    assert out[0][1] >= 1 and out[1][1] == 0 and out[0][2] < out[1][2]
    assert np.array_equal(out[0][0], out[1][0])
    assert metrics.rel_l2(out[0][0], contract.contract(load(sub), 0)) <= TOL[dtype]


def _free():
    import gc
    import torch
    gc.collect()
    torch.cuda.empty_cache()


def test_c3_split_auto_capacity(tn):
    """SURVEY a.7 protocol at full C3 size: buffers sized below the unsplit stem force the automatic
    chunk count (split_log2 = -1, C-A19) to c >= 2; same amplitudes as the unsplit run (chunk
    scales are powers of two, so only fp16 subnormals could differ)."""
    c3 = _plan("c3_sweep")  # the round-1 C3 plan: its largest stem is in the tail
    p0 = tn.Plan(c3, tn.make_config(stem_min_log2=20))
    one = tn.contract(p0, tn.Buffers(p0), 0)
    need0 = p0.info()["stem_bytes"]
    del p0
    _free()
    cap = tn.Plan(c3, tn.make_config(stem_min_log2=20, split_log2=3)).info()["stem_bytes"]
    assert cap < need0
    p = tn.Plan(c3, tn.make_config(stem_min_log2=20, split_log2=-1, stem_capacity_bytes=cap))
    assert p.info()["split_chunks"] >= 2 and p.info()["stem_bytes"] <= cap
    got = tn.contract(p, tn.Buffers(p, stem_bytes=cap), 0)
    del p
    _free()
    # the split legs sort outermost, which changes M/K orders and thus fp32 summation order: the
    # two complex-half runs agree to fp16 accuracy (measured 1.1e-4), not bit for bit
    assert metrics.rel_l2(got, one) <= 1e-2


def test_c2_split_auto_capacity(tn):
    """Full-size C2 (stem 2^28): capacity below the unsplit and the 4-chunk need forces the automatic
    chunk count to 8; complex-half and complex64 split runs vs the unsplit complex64 run."""
    c2 = _plan("c2")
    need = [tn.Plan(c2, tn.make_config(stem_min_log2=16, split_log2=j)).info()["stem_bytes"] for j in range(4)]
    assert need[3] < need[2] < need[0]
    ref, _ = run_gpu(tn, c2, 1, 0, stem_min_log2=16)
    _free()
    for dtype, tol in ((1, 1e-5), (0, 2e-2)):
        cap = tn.Plan(c2, tn.make_config(dtype=dtype, stem_min_log2=16, split_log2=3)).info()["stem_bytes"]
        p = tn.Plan(c2, tn.make_config(dtype=dtype, stem_min_log2=16, split_log2=-1, stem_capacity_bytes=cap))
        assert p.info()["split_chunks"] == 8
        got = tn.contract(p, tn.Buffers(p, stem_bytes=cap), 0)
        del p
        _free()
        assert metrics.rel_l2(got, ref) <= tol


def test_c3_full_equals_sum_of_gpu_subslices(tn):
    """SURVEY c.6 step 2 at full size: the full C3 subtask (stem 2^32) = the sum of its GPU
    sub-slices over 2 extra sliced edges (slicing identity P:318), within the fp16 bound."""
    c3 = _plan("c3")
    p = tn.Plan(c3, tn.make_config(stem_min_log2=20))
    full = tn.contract(p, tn.Buffers(p), 0)
    assert p.info()["max_stem_log2"] >= 32
    del p
    _free()
    sub = MP.sub_slice(c3, 31)
    extra = sub["sliced"][len(c3["sliced"]):]
    assert len(extra) >= 2
    sub["sliced"] = extra + c3["sliced"]  # extra edges first: slice e sets them, the rest stay 0
    p = tn.Plan(sub, tn.make_config(stem_min_log2=20))
    b = tn.Buffers(p)
    tot = 0
    for e in range(1 << len(extra)):
        tot = tot + tn.contract(p, b, e)
    del p, b
    _free()
    assert metrics.rel_l2(tot, full) <= 2e-2


def test_c3_subslice_fp16_vs_complex64(tn):
    """SURVEY c.6 step 3: C3 sub-sliced by one edge (stem 2^32): complex-half vs the complex64 path."""
    sub = MP.sub_slice(_plan("c3"), 32)
    a32, p = run_gpu(tn, sub, 1, 0, stem_min_log2=20)
    assert p.info()["max_stem_log2"] >= 31
    del p
    _free()
    a16, p = run_gpu(tn, sub, 0, 0, stem_min_log2=20)
    del p
    _free()
    assert metrics.rel_l2(a16, a32) <= 2e-2


def test_recompute_on_halves_full_c3(tn):
    """Recomputation on halves at full size (round-1 C3 plan, stem 2^33): the two halves, each run
    through the rest of the path inside the stem buffers and concatenated, give the same amplitudes
    as the unhalved run with half the stem-buffer bytes."""
    c3 = _plan("c3_sweep")
    p0 = tn.Plan(c3, tn.make_config(stem_min_log2=20))
    one = tn.contract(p0, tn.Buffers(p0), 0)
    need0 = p0.info()["stem_bytes"]
    del p0
    _free()
    p = tn.Plan(c3, tn.make_config(stem_min_log2=20, recompute=1))
    assert p.info()["stem_bytes"] <= 0.52 * need0
    got = tn.contract(p, tn.Buffers(p), 0)
    del p
    _free()
    assert metrics.rel_l2(got, one) <= 1e-2


@pytest.mark.parametrize("dtype", [0, 1])
def test_recompute_on_halves_vs_oracle(tn, dtype):
    """C2 sub-slice: recomputed halves vs the oracle, and complex64 bit-identical to no recompute
    (layout policy 0 for that: policy 3 picks transposed outputs only before the tail, which
    recomputation moves, so the two plans' K orders differ)."""
    sub = MP.sub_slice(_plan("c2"), 22)
    ref = contract.contract(load(sub), 0)
    p = tn.Plan(sub, tn.make_config(dtype=dtype, stem_min_log2=12, recompute=1))
    assert p.info()["split_chunks"] == 2
    got = tn.contract(p, tn.Buffers(p), 0)
    assert metrics.rel_l2(got, ref) <= TOL[dtype]
    if dtype == 1:
        p = tn.Plan(sub, tn.make_config(dtype=1, stem_min_log2=12, recompute=1, layout_policy=0))
        got = tn.contract(p, tn.Buffers(p), 0)
        p0 = tn.Plan(sub, tn.make_config(dtype=1, stem_min_log2=12, layout_policy=0))
        assert np.array_equal(tn.contract(p0, tn.Buffers(p0), 0), got)


@pytest.mark.parametrize("policy", [0, 3])
def test_c3_subslice_policies_vs_oracle(tn, policy):
    """The headline plan sub-sliced to 2^22: identity outputs (policy 0) and transposed C[n][m] stores
    where they put the next step's contracted modes innermost (policy 3) vs the oracle."""
    sub = MP.sub_slice(_plan("c3"), 22)
    ref = contract.contract(load(sub), 0)
    got, p = run_gpu(tn, sub, 0, 0, stem_min_log2=16, policy=policy)
    assert metrics.rel_l2(got, ref) <= 2e-2


def test_mn_major_steps_vs_oracle(tn):
    """Steps stored [kept | contracted | >= 7 kept] run on the MN-major operand (no permutation pass,
    k_gemm_tc2.cu): C3 sub-sliced to 2^25 with the fold enabled down to 2^18-element steps, one GPU
    and 4 loopback ranks, against the oracle (fp16 bound); also with the row-permuted output
    (TN_MN_ROWPERM=1), with the split block (TN_MN_SPLIT=1: [.. | k_hi | m_mid | k_lo | m_lo]
    stored steps on a 5-d A map instead of a pass) and with the fold off."""
    import subprocess
    import sys
    import tempfile
    sub = MP.sub_slice(_plan("c3"), 25)
    ref = contract.contract(load(sub), 0)
    got = {}
    for mode, env in (("mn", {"TN_MN_MIN_LOG2": "18"}), ("mn_rowperm", {"TN_MN_MIN_LOG2": "18", "TN_MN_ROWPERM": "1"}),
                      ("mn_split", {"TN_MN_MIN_LOG2": "18", "TN_MN_SPLIT": "1"}), ("pass", {"TN_NO_MN": "1"})):
        with tempfile.NamedTemporaryFile(suffix=".npz", delete=False) as f:
            path = f.name
        r = subprocess.run([sys.executable, os.path.join(ROOT, "tests", "mn_worker.py"), path],
                           env=dict(os.environ, **env), capture_output=True, text=True, timeout=600)
        assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
        got[mode] = np.load(path)
    assert len(got["mn"]["mn_one"]) >= 1 and len(got["mn"]["mn_four"]) >= 1
    assert len(got["mn_rowperm"]["mn_one"]) >= 1
    assert len(got["pass"]["mn_one"]) == 0
    assert len(got["mn_split"]["split_one"]) >= 1 and len(got["mn"]["split_one"]) == 0
    for mode in got:
        for key in ("one", "four"):
            assert metrics.rel_l2(got[mode][key], ref) <= 2e-2, (mode, key)

