"""C-ABI library checks that need no GPU: it builds/loads, exports every symbol include/tn.h
declares, and the host-side plan parsing/validation/lowering behaves."""
import copy
import json
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="session")
def tnmod():
    from paper_2407_00769_b200 import build as B
    B.build()
    from paper_2407_00769_b200 import tn
    return tn


def header_symbols():
    src = open(os.path.join(ROOT, "include", "tn.h")).read()
    return sorted(set(re.findall(r"TN_API[^;(]*?\b(tn_\w+)\s*\(", src)))


def test_exports_every_header_symbol(tnmod):
    L = tnmod.lib()
    syms = header_symbols()
    assert len(syms) >= 18
    for s in syms:
        assert hasattr(L, s), f"libtn.so does not export {s}"
    assert L.tn_version() == 1


@pytest.fixture(scope="session")
def c1_plan():
    with open(os.path.join(ROOT, "plans", "c1.json")) as f:
        return json.load(f)


def _load(tnmod, plan, **cfg):
    return tnmod.Plan(plan, tnmod.make_config(**cfg))


def test_plan_load_info_and_lowering_invariants(tnmod, c1_plan):
    p = _load(tnmod, c1_plan, stem_min_log2=6)
    info = p.info()
    assert info["n_open"] == 12 and info["n_slices_log2"] == 0
    assert info["n_stem_steps"] >= 1 and info["ws_bytes"] > 0
    rep = p.report()
    prev = None
    for st in rep["steps"]:
        lay = st["in"]
        if prev is not None:
            assert lay == prev
        R = st["R"]
        assert len(R) == st["k"]
        out = st["out"]
        assert len(out) == st["m"] + st["n"]
        if st["ga"]:
            # permutation fused into the GEMM load: 16-byte pieces (the two innermost stored modes are
            # contracted) or 4-byte pieces whose lanes read 32 contiguous complex (the 5 innermost
            # stored modes are tile bits: the 7 innermost kept or the innermost contracted modes)
            kept = [l for l in lay if l not in R]
            tile = set(kept[-7:]) | set(R[-min(5, len(R)):])
            assert not st["perm"] and st["tc"] and st["m"] >= 7 and st["k"] >= 3
            assert set(lay[-2:]) <= set(R) or set(lay[-5:]) <= tile
        elif not st["perm"]:
            assert lay[len(lay) - len(R):] == R           # R innermost: GEMM reads A as stored
        assert (set(lay) - set(R)) <= set(out)              # Eq. 4: kept modes remain
        assert not (set(out) & set(R))                       # contracted modes are gone
        prev = out
    assert sorted(rep["final_layout"]) == sorted(c1_plan["open"])


@pytest.mark.parametrize("name", ["c1", "c2", "c3"])
def test_scatter_layout_policy_needs_no_permutation(tnmod, name):
    """Layout policy 2: each GEMM writes the next step's contracted modes innermost, so every stem
    operand is read as stored and the result lands in output order."""
    with open(os.path.join(ROOT, "plans", f"{name}.json")) as f:
        plan = json.load(f)
    p = _load(tnmod, plan, stem_min_log2=6 if name == "c1" else 16, layout_policy=2)
    rep = p.report()
    assert p.info()["n_permutes"] == 0 and rep["final_perm"] == 0
    for a, b in zip(rep["steps"], rep["steps"][1:]):
        assert b["in"][len(b["in"]) - len(b["R"]):] == b["R"]
    assert rep["final_layout"] == plan["open"]


def test_flops_match_oracle_definition(tnmod, c1_plan):
    from oracle import contract
    p = _load(tnmod, c1_plan, stem_min_log2=6)
    assert p.info()["total_flops"] == contract.flops(c1_plan)


def test_plan_errors(tnmod, c1_plan):
    with pytest.raises(tnmod.TnError) as e:
        tnmod.Plan('{"tensors": [', tnmod.make_config())
    assert e.value.code == -2
    bad = copy.deepcopy(c1_plan)
    bad["tensors"][0]["data"] = bad["tensors"][0]["data"][:-2]
    with pytest.raises(tnmod.TnError) as e:
        tnmod.Plan(bad, tnmod.make_config())
    assert e.value.code == -1
    hyper = copy.deepcopy(c1_plan)
    l0 = hyper["tensors"][0]["labels"][0]
    t = hyper["tensors"][1]
    t["labels"] = t["labels"] + [l0]
    t["data"] = t["data"] + t["data"]
    with pytest.raises(tnmod.TnError) as e:
        tnmod.Plan(hyper, tnmod.make_config())
    assert e.value.code == -1
    sl_open = copy.deepcopy(c1_plan)
    sl_open["sliced"] = [sl_open["open"][0]]
    with pytest.raises(tnmod.TnError) as e:
        tnmod.Plan(sl_open, tnmod.make_config())
    assert e.value.code == -1
    with pytest.raises(tnmod.TnError) as e:
        _load(tnmod, c1_plan, stem_min_log2=6, stem_capacity_bytes=64)
    assert e.value.code == -3
    tree = copy.deepcopy(c1_plan)
    tree["tree"] = tree["tree"][:-1]
    with pytest.raises(tnmod.TnError) as e:
        tnmod.Plan(tree, tnmod.make_config())
    assert e.value.code == -1


def test_header_documents_citations():
    src = open(os.path.join(ROOT, "include", "tn.h")).read()
    for cite in ("P:496-514", "P:18-22", "P:230", "Eq. 1"):
        assert cite in src


@pytest.mark.parametrize("j", [1, 2, 3])
def test_split_tail_lowering(tnmod, j):
    """Split modes are open legs, stay the outermost block through the tail, and are never
    contracted there (chunks of the stem contract with chunked non-stem inputs)."""
    with open(os.path.join(ROOT, "plans", "c3.json")) as f:
        plan = json.load(f)
    for policy in (0, 2):
        p = _load(tnmod, plan, stem_min_log2=20, split_log2=j, layout_policy=policy)
        rep = p.report()
        assert p.info()["split_chunks"] == 2 ** j
        tail = [s for s in rep["steps"] if s["split"]]
        assert tail and tail[-1] is rep["steps"][-1]
        first = tail[0]["out"][:j]
        assert set(first) <= set(plan["open"])
        for s in tail:
            assert s["out"][:j] == first and not (set(s["R"]) & set(first))


@pytest.mark.parametrize("name", ["c2", "c3"])
def test_fused_permutation_lowering(tnmod, name):
    """Gathered-A steps (the permutation folded into the GEMM load): only tensor-core steps with
    M >= 128 and either the two innermost stored modes contracted (16-byte pieces) or the 5 innermost
    stored modes tile bits (4-byte pieces, coalesced); their kept modes stay in stored order;
    the output layout is kept ++ new exactly as after a permutation pass; fusing only removes
    passes (same GEMM geometry and flops)."""
    with open(os.path.join(ROOT, "plans", f"{name}.json")) as f:
        plan = json.load(f)
    fused = _load(tnmod, plan, stem_min_log2=16)
    plain = _load(tnmod, plan, stem_min_log2=16, no_gather=1)
    rf, rp = fused.report(), plain.report()
    assert sum(s["ga"] for s in rf["steps"]) >= 1 and sum(s["ga"] for s in rp["steps"]) == 0
    assert fused.info()["n_permutes"] < plain.info()["n_permutes"]
    assert fused.info()["perm_bytes"] < plain.info()["perm_bytes"]
    assert fused.info()["stem_flops"] == plain.info()["stem_flops"]
    for s in rf["steps"]:
        if not s["ga"]:
            continue
        lay, R = s["in"], set(s["R"])
        assert s["tc"] and not s["perm"] and s["m"] >= 7 and s["k"] >= 3
        kept = [l for l in lay if l not in R]
        Rl = [l for l in lay if l in R]
        tile = set(kept[-7:]) | set(Rl[-min(5, len(Rl)):])
        assert (lay[-1] in R and lay[-2] in R) or set(lay[-5:]) <= tile   # 16-byte or 4-byte pieces
        new = [l for l in s["out"] if l not in kept]
        # kept modes in stored order, then the new modes (or, layout policy 3, the transposed C[n][m])
        assert s["out"] == kept + new or s["out"] == new + kept


@pytest.mark.parametrize("world,g", [(8, 128), (4, 32), (2, 16)])
def test_fused_swap_codec_lowering(tnmod, world, g):
    """Sender permutation folded into the swap codec (north_star (5)): a swap is marked fuse_quant
    exactly when it is quantised, needs a sender permutation, and that permutation keeps the
    innermost log2(g/2) local modes in place (so every codec group is contiguous in the unpermuted
    stem).  The pre-swap local layout is the previous step's output layout.  no_fuse_swap_quant=1
    clears every mark and changes nothing else in the lowering."""
    from workload import make_plans as MP
    with open(os.path.join(ROOT, "plans", "c3.json")) as f:
        plan = MP.sub_slice(json.load(f), 22)
    b = (g // 2).bit_length() - 1
    kw = dict(stem_min_log2=14, virtual_world=world, quant_from_pct=0, comm_group=g)
    rf = tnmod.Plan(plan, tnmod.make_config(**kw)).report()["steps"]
    ru = tnmod.Plan(plan, tnmod.make_config(no_fuse_swap_quant=1, **kw)).report()["steps"]
    n_fused = 0
    for i, s in enumerate(rf):
        if not s["swap"] or i == 0:
            assert not s["fuse_quant"]
            continue
        snd = s["send_layout"]
        pre = [l for l in rf[i - 1]["out"] if l in snd]          # local modes, stored order
        assert sorted(pre) == sorted(snd)
        want = bool(s["quant"]) and pre != snd and pre[len(pre) - b:] == snd[len(snd) - b:]
        assert bool(s["fuse_quant"]) == want, (i, s["quant"], pre[-b:], snd[-b:])
        n_fused += want
    assert n_fused >= 1
    assert all(not s["fuse_quant"] for s in ru)
    strip = lambda st: [{k: v for k, v in s.items() if k != "fuse_quant"} for s in st]  # noqa: E731
    assert strip(rf) == strip(ru)


def test_split_auto_chunk_count(tnmod):
    """split_log2 = -1 (reading C-A19): the smallest power-of-two chunk count whose lowering
    fits stem_capacity_bytes; no capacity -> no split; nothing fits -> TN_E_CAPACITY."""
    with open(os.path.join(ROOT, "plans", "c3_sweep.json")) as f:
        c3 = json.load(f)
    need = {}
    for j in range(4):
        need[j] = _load(tnmod, c3, stem_min_log2=20, split_log2=j).info()["stem_bytes"]
    assert need[0] > need[3]
    assert _load(tnmod, c3, stem_min_log2=20, split_log2=-1).info()["split_chunks"] == 1
    for cap in (need[0], need[0] - 1, need[3]):
        p = _load(tnmod, c3, stem_min_log2=20, split_log2=-1, stem_capacity_bytes=cap)
        c = p.info()["split_chunks"]
        j = c.bit_length() - 1
        assert need[j] <= cap and all(need[i] > cap for i in range(j))
    with pytest.raises(tnmod.TnError) as e:
        _load(tnmod, c3, stem_min_log2=20, split_log2=-1, stem_capacity_bytes=1 << 30)
    assert e.value.code == -4


@pytest.mark.parametrize("world", [2, 4, 8])
def test_split_tail_with_sharded_stem_lowering(tnmod, world):
    """Split tail on a sharded stem: split legs are never shard or swap-in modes, and the tail starts
    after the last mode swap (host lowering for `world` virtual ranks)."""
    from workload import make_plans as MP
    with open(os.path.join(ROOT, "plans", "c2.json")) as f:
        sub = MP.sub_slice(json.load(f), 20)
    for j in (1, 2, 3):
        p = _load(tnmod, sub, stem_min_log2=12, split_log2=j, virtual_world=world)
        rep = p.report()
        assert p.info()["split_chunks"] == 2 ** j
        sm = set(rep["split_modes"])
        assert not sm & set(rep["shard0"])
        tail = [s for s in rep["steps"] if s["split"]]
        assert tail and all(not s["swap"] for s in tail)
        for s in rep["steps"]:
            if s["swap"]:
                assert not sm & set(s["swap_in"])
            if s["split"]:
                assert set(s["in"][:j]) == sm or s is tail[0]


def test_codec_group_validation(tnmod, c1_plan):
    """ADVICE (round 1): the group codecs stage codes + scales + zeros in one stem buffer, which only
    fits for groups of >= 16 reals; other groups are refused at load time."""
    for g in (8, 24, 0x7fff):
        with pytest.raises(tnmod.TnError) as e:
            _load(tnmod, c1_plan, stem_min_log2=6, comm_codec=tnmod.TN_COMM_INT8, comm_group=g)
        assert e.value.code == -1
    _load(tnmod, c1_plan, stem_min_log2=6, comm_codec=tnmod.TN_COMM_INT8, comm_group=16)
    _load(tnmod, c1_plan, stem_min_log2=6, comm_codec=tnmod.TN_COMM_INT8_TENSOR, comm_group=8)
    with pytest.raises(tnmod.TnError):
        _load(tnmod, c1_plan, stem_min_log2=6, comm_codec=7)


@pytest.mark.parametrize("world", [1, 2, 4, 8])
def test_recompute_on_halves_halves_peak(tnmod, world):
    """Recomputation on halves: the stem is halved along an open leg
    right before the step that produces its largest tensor; per-buffer stem bytes halve (+ the
    tail input), no mode swap falls into the recomputed region, two chunks."""
    with open(os.path.join(ROOT, "plans", "c3_sweep.json")) as f:
        plan = json.load(f)
    base = _load(tnmod, plan, stem_min_log2=20, virtual_world=world).info()["stem_bytes"]
    p = _load(tnmod, plan, stem_min_log2=20, virtual_world=world, recompute=1)
    rep = p.report()
    assert p.info()["split_chunks"] == 2 and rep["recompute_from"] >= 0
    assert rep["split_from"] >= rep["recompute_from"]
    sizes = [s["m"] + s["n"] for s in rep["steps"]]
    assert p.info()["stem_bytes"] <= 0.52 * base
    assert all(not s["swap"] for s in rep["steps"] if s["split"])
    with pytest.raises(tnmod.TnError):
        _load(tnmod, plan, stem_min_log2=20, recompute=1, split_log2=2)
    assert max(sizes) + (world.bit_length() - 1) >= 32    # the recomputed region holds the 2^33 tensor


def _runs(step):
    """Stored order of a step's input, innermost first, as 'k'/'m' per mode."""
    R = set(step["R"])
    return ["k" if x in R else "m" for x in reversed(step["in"])]


@pytest.mark.parametrize("world", [1, 4])
def test_mn_major_lowering(tnmod, world):
    """Steps folded into the MN-major operand (plan.cpp, StemStep::mn): stored order
    [kept | contracted | >= 7 kept] (or the contracted block split by one kept run), K >= 64, N >= 64, >= 2^28 elements; the permutation stays as the
    fallback (perm = 1) but is not counted in n_permutes / perm_bytes."""
    with open(os.path.join(ROOT, "plans", "c3.json")) as f:
        plan = json.load(f)
    p = _load(tnmod, plan, virtual_world=world)
    rep, info = p.report(), p.info()
    mn = [s for s in rep["steps"] if s["mn"]]
    assert len(mn) >= 1
    for s in mn:
        runs = _runs(s)
        ma = s["mn"]
        kl, mm = s["mn_split"]
        if kl == 0:
            assert mm == 0
            assert ma >= 7 and runs[:ma] == ["m"] * ma and runs[ma:ma + s["k"]] == ["k"] * s["k"]
            assert set(runs[ma + s["k"]:]) <= {"m"}
        else:
            # split block [.. | k_hi | m_mid | k_lo | m_lo]: one kept run inside the contracted modes
            assert ma >= 7 and mm >= 1 and 1 <= kl < s["k"]
            assert runs[:ma] == ["m"] * ma and runs[ma:ma + kl] == ["k"] * kl
            assert runs[ma + kl:ma + kl + mm] == ["m"] * mm
            assert runs[ma + kl + mm:ma + mm + s["k"]] == ["k"] * (s["k"] - kl)
            assert set(runs[ma + mm + s["k"]:]) <= {"m"}
        assert s["k"] >= 6 and s["n"] >= 6 and len(s["in"]) >= 28 and s["perm"] == 1 and s["ga"] == 0
    # (+1: the final permutation into output order, one GPU)
    assert info["n_permutes"] - sum(1 for s in rep["steps"] if s["perm"] and not s["mn"]) in (0, 1)


@pytest.mark.parametrize("name", ["c2", "c3"])
def test_row_folding_lowering(tnmod, name):
    """Row folding (StemStep::fold): only plain A (as stored or after a pass; no gather), row-major outputs with rows of
    2K fp16 < 128 B, f = 128 B / row bytes, at least 2^8 folded rows; such steps run on tcgen05."""
    with open(os.path.join(ROOT, "plans", f"{name}.json")) as f:
        plan = json.load(f)
    for world in (1, 4):
        rep = _load(tnmod, plan, virtual_world=world).report()
        for s in rep["steps"]:
            if s["fold"] > 1:
                assert s["ga"] == 0 and s["mn"] == 0 and s["k"] <= 4 and s["tc"] == 1
                # row-major output, or transposed for f = 2 and N = 16 (one C^T box per folded tile)
                assert s["out_kind"] == 0 or (s["out_kind"] == 1 and s["fold"] == 2 and s["n"] == 4)
                assert s["fold"] * (4 << s["k"]) == 128 and s["m"] - (s["fold"].bit_length() - 1) >= 8


def test_no_transposed_output_for_row_streaming_steps(tnmod):
    """Layout policy 3 never gives a SIMT row-streaming step (K <= 16, N <= 32, K N <= 128) a
    transposed output: its stores would be 4-byte scatters."""
    with open(os.path.join(ROOT, "plans", "c3.json")) as f:
        plan = json.load(f)
    for world in (1, 2, 4, 8):
        rep = _load(tnmod, plan, virtual_world=world).report()
        for s in rep["steps"]:
            if s["k"] <= 4 and s["n"] <= 5 and s["k"] + s["n"] <= 7:
                assert s["out_kind"] != 1


@pytest.mark.parametrize("world,routable", [(4, 5), (8, 10)])
def test_swaps_routable_by_the_epilogue(tnmod, world, routable):
    """The C3 swap schedule at 4 / 8 ranks: every swapped-in mode is a bit of the previous tcgen05
    step's output that a store box keeps constant (m bit >= 7 or n bit >= 5 of its M / N index), so
    every swap can be done by that GEMM's epilogue (runtime.cu fused_swap_target)."""
    with open(os.path.join(ROOT, "plans", "c3.json")) as f:
        plan = json.load(f)
    rep = _load(tnmod, plan, virtual_world=world).report()
    ok = 0
    for i, s in enumerate(rep["steps"]):
        if not s["swap"]:
            continue
        pv = rep["steps"][i - 1]
        pos = [len(pv["out"]) - 1 - pv["out"].index(x) for x in s["swap_in"]]
        if pv["out_kind"] == 0:
            good = all(q >= pv["n"] + 7 or 5 <= q < pv["n"] for q in pos)
        elif pv["out_kind"] == 1:
            good = all(7 <= q < pv["m"] or q >= pv["m"] + 5 for q in pos)
        else:
            good = False
        ok += bool(good and pv["tc"] and pv["fold"] == 1)
    assert rep["n_swaps"] == routable and ok == routable
