"""Pins of the CPU oracle against what the paper and the mathematics fix (no GPU).

Every oracle function is checked against something other than itself: closed forms, the paper's
worked example (tests/golden/), an independent textbook routine (state vector), brute force, or
invariants (slicing identity, tree independence)."""
import json
import math
import os

import numpy as np
import pytest

from oracle import codec, contract, embed, gates, metrics, sparse, statevector
from oracle.plan import load
from workload import circuit as C
from workload import make_plans as MP

GOLD = os.path.join(os.path.dirname(__file__), "golden")


# ---------------------------------------------------------------- gates
def test_gates_unitary_and_closed_forms():
    for m in (gates.sqrt_x(), gates.sqrt_y(), gates.sqrt_w(), gates.fsim(np.pi / 2, np.pi / 6),
              gates.fsim(0.3, 1.1)):
        assert np.allclose(m @ m.conj().T, np.eye(m.shape[0]), atol=1e-15)
    assert np.allclose(gates.fsim(0, 0), np.eye(4), atol=0)
    exp = np.array([[1, 0, 0, 0], [0, 0, -1j, 0], [0, -1j, 0, 0], [0, 0, 0, 1]])
    assert np.allclose(gates.fsim(np.pi / 2, 0), exp, atol=1e-16)
    # sqrt(X)|0> = (1, -i)/sqrt2
    assert np.allclose(gates.sqrt_x() @ [1, 0], np.array([1, -1j]) / np.sqrt(2), atol=1e-16)
    # sqrt(X)^2 = X up to global phase: X = [[0,1],[1,0]]; sqrtX^2 = -i X
    assert np.allclose(gates.sqrt_x() @ gates.sqrt_x(), -1j * np.array([[0, 1], [1, 0]]), atol=1e-15)
    assert np.allclose(gates.sqrt_y() @ gates.sqrt_y(), np.array([[0, -1], [1, 0]]), atol=1e-15)
    # fSim is symmetric under swapping the two qubits
    swap = np.eye(4)[[0, 2, 1, 3]]
    f = gates.fsim(0.7, 0.4)
    assert np.allclose(swap @ f @ swap, f, atol=0)


# ---------------------------------------------------------------- state vector
def test_statevector_norm_and_trivial_cases():
    empty = {"n_qubits": 3, "gates": []}
    psi = statevector.simulate(empty)
    assert psi[0, 0, 0] == 1 and abs(np.linalg.norm(psi) - 1) == 0
    one = {"n_qubits": 1, "gates": [{"kind": "sqrt_x", "qubits": [0], "cycle": 0}]}
    assert np.allclose(statevector.simulate(one), np.array([1, -1j]) / np.sqrt(2), atol=1e-16)
    circ = C.make_circuit(3, 4, 8, seed=3)
    psi = statevector.simulate(circ)
    assert abs(np.linalg.norm(psi) - 1.0) < 1e-12
    # fSim(pi/2, 0) on |01> (a=0 -> 0, b=1 -> 1): maps |01> -> -i|10>
    c2 = {"n_qubits": 2, "gates": [{"kind": "sqrt_y", "qubits": [1], "cycle": 0},
                                   {"kind": "sqrt_y", "qubits": [1], "cycle": 0},
                                   {"kind": "fsim", "qubits": [0, 1], "theta": np.pi / 2, "phi": 0.0, "cycle": 0}]}
    p = statevector.simulate(c2)   # sqrtY^2 |0> = |1> on qubit 1 -> |01> -> -i |10>
    assert np.allclose(p, np.array([[0, 0], [-1j, 0]]), atol=1e-15)


def _small_plan(rows, cols, cycles, seed, n_open, max_log2=None):
    return MP.build_plan(rows, cols, False, cycles, n_open, max_log2, trials=4, seed=seed)


# ---------------------------------------------------------------- oracle vs state vector
@pytest.mark.parametrize("seed", range(50))
def test_oracle_matches_statevector_c1_class(seed):
    """50 seeded C1-class circuits (n <= 12, m <= 8); |da| <= 1e-12."""
    rng = np.random.default_rng(seed)
    rows, cols = [(3, 4), (2, 4), (3, 3), (2, 5), (2, 6)][seed % 5]
    cycles = int(rng.integers(1, 9))
    n_open = int(rng.integers(0, rows * cols + 1))
    plan = _small_plan(rows, cols, cycles, seed, n_open)
    amps = contract.contract(load(plan), 0)
    psi = statevector.simulate(plan["circuit"])
    ref = statevector.amplitudes(psi, plan["bits"], plan["open_qubits"])
    assert amps.shape == ref.shape
    assert np.max(np.abs(amps - ref)) <= 1e-12


def test_full_state_norm_c1():
    plan = _small_plan(3, 4, 8, 0, 12)
    amps = contract.contract(load(plan), 0)
    assert abs(np.sum(np.abs(amps) ** 2) - 1.0) < 1e-12


def test_slicing_identity_and_order_independence():
    plan = _small_plan(3, 4, 6, 7, 4)
    p = load(plan)
    full = contract.contract(p, 0)
    # slice k = 1..4 extra closed labels: sum over slices equals the unsliced result
    closed = sorted({l for ls, _ in p.tensors for l in ls} - set(p.open))
    rng = np.random.default_rng(1)
    for k in range(1, 5):
        d = dict(plan)
        d["sliced"] = [int(x) for x in rng.choice(closed, size=k, replace=False)]
        tot = contract.contract_all_slices(load(d))
        assert np.linalg.norm(tot - full) <= 1e-12 * np.linalg.norm(full)
    # a different tree (another planner seed) gives the same amplitudes
    plan2 = MP.build_plan(3, 4, False, 6, 4, None, trials=1, seed=7, group=False)
    assert plan2["tree"] != plan["tree"]
    other = contract.contract(load(plan2), 0)
    assert np.linalg.norm(other - full) <= 1e-12 * np.linalg.norm(full)


def test_slice_id_range():
    plan = _small_plan(2, 3, 3, 0, 2)
    plan["sliced"] = [plan["tree"][0][0] * 0 + sorted({l for t in plan["tensors"] for l in t["labels"]} - set(plan["open"]))[0]]
    with pytest.raises(ValueError):
        contract.contract(load(plan), 2)


# ---------------------------------------------------------------- Eq. 6
def test_eq6_worked_example_golden():
    g = json.load(open(os.path.join(GOLD, "eq6_worked_example.json")))
    a = np.array(g["A_complex"], dtype=float)
    a_c = a[:, 0] + 1j * a[:, 1]               # A = [(1+2i), (3+4i)] along a1
    b_c = np.array([g["B_complex"][0] + 1j * g["B_complex"][1]])  # b1 has dim 1
    assert np.array_equal(embed.real_view(a_c), np.array(g["A_real"], dtype=float))
    bp = embed.pad_b(b_c)                       # [c0, b1, a2]
    assert np.array_equal(bp, np.array(g["B_padded_c_b_a"], dtype=float))
    c_real = np.einsum("ij,kmj->imk", embed.real_view(a_c), bp)   # a1a2,c0b1a2->a1b1c0
    assert np.array_equal(c_real, np.array(g["C_real_expected"], dtype=float))
    exp_c = np.array([complex(*z) for z in g["C_complex_expected"]])
    assert np.array_equal(np.outer(a_c, b_c)[:, 0], exp_c)


def test_eq6_gemm_form_random():
    rng = np.random.default_rng(0)
    for m, k, n in [(7, 4, 3), (16, 8, 8), (3, 1, 5)]:
        a = rng.standard_normal((m, k)) + 1j * rng.standard_normal((m, k))
        b = rng.standard_normal((k, n)) + 1j * rng.standard_normal((k, n))
        cr = embed.cgemm_real(embed.real_view(a).reshape(m, 2 * k), embed.pad_b(b))
        c = cr.reshape(m, n, 2)
        ref = a @ b
        assert np.max(np.abs(c[..., 0] + 1j * c[..., 1] - ref)) < 1e-13
        # integer-valued data: exact
        ai = rng.integers(-5, 5, (m, k)) + 1j * rng.integers(-5, 5, (m, k))
        bi = rng.integers(-5, 5, (k, n)) + 1j * rng.integers(-5, 5, (k, n))
        ci = embed.cgemm_real(embed.real_view(ai).reshape(m, 2 * k), embed.pad_b(bi)).reshape(m, n, 2)
        assert np.array_equal(ci[..., 0] + 1j * ci[..., 1], ai @ bi)


# ---------------------------------------------------------------- codec (Eq. 1, Table 1)
def test_codec_examples_golden():
    g = json.load(open(os.path.join(GOLD, "codec_examples.json")))
    for key in ("int4_identity", "int8_exp02_pm1"):
        e = g[key]
        codes, s, z = codec.quantize(np.array(e["x"], np.float32), np.float32(e["qmin"]),
                                     np.float32(e["qmax"]), e["exp"])
        assert codes.tolist() == e["codes"]
        assert float(s[0]) == e["scale"] and float(z[0]) == e["zero"]
    cr = g["cr_percent_n65536"]
    n = 65536
    assert abs(100 * codec.compression_rate(n, 16, 1) - cr["half"]) < 1e-9
    assert abs(100 * codec.compression_rate(n, 8, 1) - cr["int8_entire"]) < 1e-9
    assert abs(100 * codec.compression_rate(n, 4, n // 128) - cr["int4_g128"]) < 1e-12


def test_codec_closed_form_endpoints_and_invariants():
    rng = np.random.default_rng(0)
    x = rng.standard_normal(1024).astype(np.float32)
    qmin, qmax = np.float32(-128), np.float32(127)
    codes, s, z = codec.quantize(x, qmin, qmax, 1.0, group=128)
    assert codes.min() >= -128 and codes.max() <= 127
    for gi in range(8):
        seg = x[gi * 128:(gi + 1) * 128]
        # Eq. 1 maps the group max to q_max and the min to q_min (up to fp32 rounding)
        assert codes[gi * 128 + int(np.argmax(seg))] == 127
        assert codes[gi * 128 + int(np.argmin(seg))] == -128
        assert abs(float(s[gi]) * (seg.max() - seg.min()) - 255.0) < 1e-3
    y = codec.dequantize(codes, s, z, 1.0, group=128)
    step = 1.0 / s.repeat(128)
    assert np.all(np.abs(y - x) <= 0.5 * step * (1 + 1e-5) + 1e-7)
    # idempotence: quantize(dequantize(q)) == q
    codes2, _, _ = codec.quantize(y, qmin, qmax, 1.0, group=128)
    assert np.array_equal(codes2, codes)
    # constant block exact (C-A11)
    c = np.full(128, 0.37, np.float32)
    cc, cs, cz = codec.quantize(c, qmin, qmax, 1.0, group=128)
    assert np.all(cc == -128) and np.array_equal(codec.dequantize(cc, cs, cz, 1.0, 128), c)
    # int4 packing round trip (C-A14)
    q4, _, _ = codec.quantize(x[:256], np.float32(0), np.float32(15), 1.0, group=128)
    assert np.array_equal(codec.unpack_int4(codec.pack_int4(q4)), q4.astype(np.uint8))
    assert codec.pack_int4(np.array([1, 2]))[0] == 0x21


# ---------------------------------------------------------------- metrics
def test_metrics_closed_forms():
    assert metrics.fidelity([1, 0], [1, 1]) == pytest.approx(0.5, abs=1e-15)
    rng = np.random.default_rng(0)
    t = rng.standard_normal(16) + 1j * rng.standard_normal(16)
    assert metrics.fidelity(t, t) == pytest.approx(1.0, abs=1e-14)
    assert metrics.fidelity(t, np.exp(0.7j) * 3.0 * t) == pytest.approx(1.0, abs=1e-14)
    # orthogonal error e with |e| = eps |t|  ->  fidelity = 1/(1+eps^2) (C-A15)
    e = rng.standard_normal(16) + 1j * rng.standard_normal(16)
    e -= np.vdot(t, e) / np.vdot(t, t) * t
    e *= 0.1 * np.linalg.norm(t) / np.linalg.norm(e)
    assert metrics.fidelity(t, t + e) == pytest.approx(1 / 1.01, rel=1e-12)
    assert metrics.rel_l2(t + e, t) == pytest.approx(0.1, rel=1e-12)
    n = 10
    assert metrics.linear_xeb(np.full(5, 2.0 ** -n), n) == 0.0
    assert metrics.linear_xeb(np.full(5, 2 * 2.0 ** -n), n) == 1.0
    sel = metrics.post_select(np.array([[0.1, 0.4, 0.25], [0.2, 0.2, 0.1]]), k=1)
    assert sel[:, 0].tolist() == [1, 0]


def test_xeb_porter_thomas_top1():
    """Exact probabilities of a deep 12-qubit circuit: top-1-of-N post-selected XEB = H_N - 1
    (C-A22) within 4 standard errors."""
    circ = C.make_circuit(3, 4, 14, seed=11)
    p = np.abs(statevector.simulate(circ).reshape(-1)) ** 2
    n_open = 6
    subsp = p.reshape(2 ** (12 - n_open), 2 ** n_open)      # last 6 qubits open
    sel = metrics.post_select(subsp, k=1)[:, 0]
    chosen = subsp[np.arange(subsp.shape[0]), sel]
    xeb = metrics.linear_xeb(chosen, 12)
    N = 2 ** n_open
    expect = metrics.harmonic(N) - 1.0
    se = math.sqrt(sum(1.0 / k ** 2 for k in range(1, N + 1))) / math.sqrt(subsp.shape[0])
    assert abs(xeb - expect) < 4 * se
    # the plain (unselected) XEB of the exact distribution is ~1 (PT second moment)
    assert abs(2 ** 12 * np.sum(p ** 2) - 2.0) < 0.2


# ---------------------------------------------------------------- sparse state
def test_sparse_padded_index_and_equivalence():
    table, m_r = sparse.build_padded_index([0, 0, 1, 1, 1, 3, 4], [0, 1, 2, 0, 1, 2, 0], 5)
    assert m_r == 3                                   # "m_r is 3 since 1 had appeared 3 times"
    assert table[2].tolist() == [-1, -1, -1]
    rng = np.random.default_rng(0)
    a = rng.standard_normal((5, 3, 4)) + 1j * rng.standard_normal((5, 3, 4))
    b = rng.standard_normal((3, 4, 2)) + 1j * rng.standard_normal((3, 4, 2))
    ia, ib = [0, 0, 1, 1, 1, 3, 4], [0, 1, 2, 0, 1, 2, 0]
    g = sparse.gather_contract(a, b, ia, ib)
    for n, (i, j) in enumerate(zip(ia, ib)):       # brute force per pair
        assert np.allclose(g[n], np.einsum("mk,kn->mn", a[i], b[j]), atol=1e-14)
    assert np.allclose(sparse.padded_contract(a, b, ia, ib), g, atol=1e-14)


def test_flops_convention():
    # chain "ij,jk->ik" with dims 2 -> 8 * 2^3 = 64 flops
    plan = {"tensors": [{"labels": [0, 1], "data": [0.0] * 8}, {"labels": [1, 2], "data": [0.0] * 8}],
            "open": [0, 2], "tree": [[0, 1]], "sliced": []}
    assert contract.flops(plan) == 64


def test_override_is_linear_and_consistent():
    """contract(override=...) (used to propagate swap errors): overriding a node with its own value
    changes nothing; overriding with zeros gives zero; the root is linear in the overridden node."""
    from oracle.plan import load as _load
    plan = MP.build_plan(3, 3, False, 5, 3, None, trials=2, seed=3)
    P = _load(plan)
    nl = len(P.tensors)
    node = nl + len(P.tree) // 2
    rec = {node: None}
    ref = contract.contract(P, 0, record=rec)
    lab, t = rec[node]
    assert np.array_equal(contract.contract(P, 0, override={node: (lab, t)}), ref)
    assert np.all(contract.contract(P, 0, override={node: (lab, np.zeros_like(t))}) == 0)
    rng = np.random.default_rng(0)
    a = rng.standard_normal(t.shape) + 1j * rng.standard_normal(t.shape)
    b = rng.standard_normal(t.shape) + 1j * rng.standard_normal(t.shape)
    la = contract.contract(P, 0, override={node: (lab, a)})
    lb = contract.contract(P, 0, override={node: (lab, b)})
    lab_ = contract.contract(P, 0, override={node: (lab, 2 * a - 3j * b)})
    assert np.allclose(lab_, 2 * la - 3j * lb, rtol=1e-12, atol=1e-14 * np.abs(lab_).max())


def test_codec_exp02_dequantize_worked_example():
    """Eq. 1 with exp = 0.2 (Table 1 int8 preset; reading C-A10) on x = [-1, 0, 1, 1/32]:
    x' = sign(x)|x|^0.2 = [-1, 0, 1, 1/2]; scale = 255/2 = 127.5, zero = (-128*1 - 127*(-1))/2 = -0.5;
    codes = rint(x'*127.5 - 0.5) = [-128, -0 -> 0 (half to even), 127, rint(63.25) = 63];
    dequantised y' = (code + 0.5)/127.5 = [-1, 1/255, 1, 63.5/127.5], y = sign(y')|y'|^5.
    (Worked by hand; pins the exp != 1 branch of dequantize, which the golden codes do not reach.)"""
    x = np.array([-1.0, 0.0, 1.0, 1.0 / 32.0], dtype=np.float32)
    c, s, z = codec.quantize(x, np.float32(-128), np.float32(127), exp=0.2, group=None)
    assert list(c) == [-128.0, 0.0, 127.0, 63.0]
    assert s[0] == np.float32(127.5) and z[0] == np.float32(-0.5)
    y = codec.dequantize(c, s, z, exp=0.2, group=None)
    want = [-1.0, (1.0 / 255.0) ** 5, 1.0, (63.5 / 127.5) ** 5]
    assert np.allclose(y, want, rtol=1e-6, atol=0)
    # the inverse transform is exact on codes that hit x' exactly: x' = +-1 round-trips to +-1
    assert y[0] == -1.0 and y[2] == 1.0
