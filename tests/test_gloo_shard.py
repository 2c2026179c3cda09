"""World-size-2/4 multi-PROCESS check of the sharded-stem schedule on CPU (gloo): each process is one
rank, lowers the plan for its rank through the C-ABI library (host-only lowering, virtual_world),
holds only its 1/G shard of the stem, performs every Alg. 1 mode swap as real
point-to-point messages (chunk v of the send layout goes to the group member whose swapped-out
bits are v, and lands at the sender's member slot), contracts its shard locally, and finally
all-gathers the shards in rank order.  Rank 0 requires the oracle's unsharded amplitudes.
This exercises the rank arithmetic and message matching of the N>1 path with real processes;
the device byte movers are covered by tests/test_gpu_loopback.py and tests/test_gpu_multi.py."""
import json
import os
import socket
import tempfile

import numpy as np
import pytest
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, out_path):
    import sys
    sys.path.insert(0, ROOT)
    import torch
    import torch.distributed as dist
    from oracle import contract
    from oracle.plan import load
    from paper_2407_00769_b200 import tn
    from workload import make_plans as MP
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    plan = MP.sub_slice(json.load(open(os.path.join(ROOT, "plans", "c2.json"))), 18)
    rep = tn.Plan(plan, tn.make_config(stem_min_log2=10, virtual_world=world)).report()
    P = load(plan)
    record = {rep["stem_entry"]: None}
    for st in rep["steps"]:
        record[st["branch"]] = None
    ref = contract.contract(P, 0, record=record)
    sl = contract.slice_leaves(P, 0)
    for st in rep["steps"]:
        if st["branch"] < len(P.tensors):
            record[st["branch"]] = sl[st["branch"]]
    S = len(rep["shard0"])
    el, et = record[rep["stem_entry"]]
    full = np.transpose(et, [el.index(l) for l in rep["entry_layout"]])
    x = full[tuple((rank >> (S - 1 - j)) & 1 for j in range(S))]   # only my shard is kept
    layout = rep["entry_layout"][S:]
    shard = list(rep["shard0"])
    n_msgs = 0
    for st in rep["steps"]:
        if st.get("swap"):
            pos, snd = st["swap_out_pos"], st["send_layout"]
            sx = len(pos)
            send = np.ascontiguousarray(np.transpose(x, [layout.index(l) for l in snd]))
            chunks = send.reshape((1 << sx, -1))
            me = 0
            for q in pos:
                me = (me << 1) | ((rank >> (S - 1 - q)) & 1)

            def peer(v):
                r = rank
                for t, q in enumerate(pos):
                    bit = (v >> (sx - 1 - t)) & 1
                    r = (r & ~(1 << (S - 1 - q))) | (bit << (S - 1 - q))
                return r
            recv = np.empty_like(chunks)
            recv[me] = chunks[me]
            reqs = []
            bufs = {}
            for v in range(1 << sx):
                if v == me:
                    continue
                sb = torch.from_numpy(np.ascontiguousarray(chunks[v]).view(np.float64).copy())
                rb = torch.empty_like(sb)
                bufs[v] = rb
                reqs.append(dist.isend(sb, peer(v)))
                reqs.append(dist.irecv(rb, peer(v)))
                n_msgs += 1
            for q in reqs:
                q.wait()
            for v, rb in bufs.items():
                recv[v] = rb.numpy().view(np.complex128)
            x = recv.reshape((2,) * sx + send.shape[sx:])
            layout = [shard[q] for q in pos] + snd[sx:]
            for t, q in enumerate(pos):
                shard[q] = st["swap_in"][t]
            assert shard == st["shard_after"]
        bl, bt = record[st["branch"]]
        out = st["out"]
        letters = {l: chr(97 + i) if i < 26 else chr(65 + i - 26) for i, l in enumerate(sorted(set(layout) | set(bl)))}
        spec = "".join(letters[l] for l in layout) + "," + "".join(letters[l] for l in bl) + "->" + \
            "".join(letters[l] for l in out)
        x = np.einsum(spec, x, bt)
        layout = out
    assert shard == rep["final_shard"] and layout == rep["final_layout"]
    flat = torch.from_numpy(np.ascontiguousarray(x).reshape(-1).view(np.float64).copy())
    parts = [torch.empty_like(flat) for _ in range(world)]
    dist.all_gather(parts, flat)
    if rank == 0:
        g = np.stack([p.numpy().view(np.complex128).reshape(x.shape) for p in parts])
        g = g.reshape((2,) * S + x.shape)
        got = np.transpose(g, [(shard + layout).index(l) for l in plan["open"]])
        with open(out_path, "w") as f:
            json.dump({"err": float(np.linalg.norm(got - ref) / np.linalg.norm(ref)), "swaps": rep["n_swaps"],
                       "msgs": n_msgs}, f)
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4])
def test_gloo_sharded_schedule_matches_oracle(world):
    from paper_2407_00769_b200 import build as B
    B.build()
    with tempfile.NamedTemporaryFile(suffix=".json", delete=False) as f:
        out = f.name
    mp.start_processes(_worker, args=(world, _free_port(), out), nprocs=world, join=True, start_method="spawn")
    v = json.load(open(out))
    os.unlink(out)
    assert v["err"] <= 1e-12
    assert v["swaps"] >= 1
