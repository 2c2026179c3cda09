"""Host-side check of the sharded-stem schedule without GPUs: the library lowers
the plan for G virtual ranks (tn_config.reserved[0]); this test replays that schedule on G
in-memory numpy shards — entry split on the shard modes, Alg. 1 mode swaps (chunk v of the
swapped-in modes goes to the member whose swapped-out bits are v, stored at the sender's slot),
local contractions with the oracle's branch tensors, final gather — and requires the result to equal
the oracle's unsharded contraction.  Validates the swap bookkeeping the NCCL path executes."""
import json
import os

import numpy as np
import pytest

from oracle import contract
from oracle.plan import load
from workload import make_plans as MP

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def tnmod():
    from paper_2407_00769_b200 import build as B
    B.build()
    from paper_2407_00769_b200 import tn
    return tn


def _to_layout(labels, t, layout):
    return np.transpose(t, [labels.index(l) for l in layout])


def emulate(tnmod, plan, world, stem_min):
    p = tnmod.Plan(plan, tnmod.make_config(stem_min_log2=stem_min, virtual_world=world))
    rep = p.report()
    record = {rep["stem_entry"]: None}
    for st in rep["steps"]:
        record[st["branch"]] = None
    P = load(plan)
    ref = contract.contract(P, 0, record=record)
    nl = len(P.tensors)
    sl = contract.slice_leaves(P, 0)
    for st in rep["steps"]:
        if st["branch"] < nl:
            record[st["branch"]] = sl[st["branch"]]
    S = len(rep["shard0"])
    assert (1 << S) == world
    el, et = record[rep["stem_entry"]]
    full = _to_layout(el, et, rep["entry_layout"])
    shards = [full[tuple((r >> (S - 1 - j)) & 1 for j in range(S))] for r in range(world)]
    layout = rep["entry_layout"][S:]
    shard = list(rep["shard0"])
    for st in rep["steps"]:
        if st.get("swap"):
            assert st["shard_before"] == shard
            pos, sin = st["swap_out_pos"], st["swap_in"]
            sx = len(pos)
            snd = st["send_layout"]
            send = [_to_layout(layout, x, snd) for x in shards]

            def member(r):
                m = 0
                for q in pos:
                    m = (m << 1) | ((r >> (S - 1 - q)) & 1)
                return m

            def peer(r, v):
                for t, q in enumerate(pos):
                    bit = (v >> (sx - 1 - t)) & 1
                    r = (r & ~(1 << (S - 1 - q))) | (bit << (S - 1 - q))
                return r

            new = []
            for r in range(world):
                parts = []
                for v in range(1 << sx):
                    src = peer(r, v)                     # member v of my group
                    chunk = send[src].reshape((1 << sx,) + send[src].shape[sx:])[member(r)]
                    parts.append(chunk)
                new.append(np.stack(parts).reshape((2,) * sx + parts[0].shape))
            shards = new
            layout = [shard[q] for q in pos] + snd[sx:]
            for t, q in enumerate(pos):
                shard[q] = sin[t]
            assert shard == st["shard_after"]
        assert layout == st["in"] or st["perm"]
        bl, bt = record[st["branch"]]
        out = st["out"]
        letters = {l: chr(97 + i) if i < 26 else chr(65 + i - 26) for i, l in enumerate(sorted(set(layout) | set(bl)))}
        spec = "".join(letters[l] for l in layout) + "," + "".join(letters[l] for l in bl) + "->" + \
            "".join(letters[l] for l in out)
        shards = [np.einsum(spec, x, bt) for x in shards]
        layout = out
    assert shard == rep["final_shard"] and layout == rep["final_layout"]
    gathered = np.stack(shards).reshape((2,) * S + shards[0].shape)
    got = _to_layout(shard + layout, gathered, plan["open"])
    return got, ref, rep


@pytest.mark.parametrize("world", [2, 4, 8])
def test_sharded_schedule_reproduces_oracle(tnmod, world):
    plan = MP.sub_slice(json.load(open(os.path.join(ROOT, "plans", "c2.json"))), 18)
    got, ref, rep = emulate(tnmod, plan, world, 10)
    assert np.linalg.norm(got - ref) <= 1e-12 * np.linalg.norm(ref)
    if world >= 4:
        assert rep["n_swaps"] >= 1


def test_c3_schedule_swaps_only_contracted_shard_modes(tnmod):
    plan = json.load(open(os.path.join(ROOT, "plans", "c3.json")))
    for world in (2, 4, 8):
        p = tnmod.Plan(plan, tnmod.make_config(stem_min_log2=20, virtual_world=world))
        rep = p.report()
        shard = rep["shard0"]
        for st in rep["steps"]:
            R = set(st["R"])
            if st.get("swap"):
                outs = {st["shard_before"][q] for q in st["swap_out_pos"]}
                assert outs == R & set(st["shard_before"])      # only the contracted shard modes move
                assert not (set(st["swap_in"]) & R)              # swapped-in modes survive this step
                shard = st["shard_after"]
            assert not (R & set(shard))                          # the GEMM never contracts a shard mode
        assert p.info()["stem_bytes"] * world == tnmod.Plan(plan, tnmod.make_config(stem_min_log2=20)).info()["stem_bytes"]
