"""Dev tool: repeated sharded runs in one process, each checked against the oracle."""
import json
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, ".")
from paper_2407_00769_b200 import tn  # noqa: E402
from workload import make_plans as MP  # noqa: E402
from oracle import contract, metrics  # noqa: E402
from oracle.plan import load  # noqa: E402

rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
local = int(os.environ.get("LOCAL_RANK", rank))
torch.cuda.set_device(local)
dist.init_process_group("nccl", device_id=torch.device("cuda", local))
sub = MP.sub_slice(json.load(open("plans/c3.json")), 22)
ref = contract.contract(load(sub), 0) if rank == 0 else None
comm = tn.Comm(rank, world, local)
keep = []
for it in range(4):
    for use_comm in (True, False):
        if not use_comm and rank != 0:
            continue
        p = tn.Plan(sub, tn.make_config(stem_min_log2=14, comm_codec=tn.TN_COMM_FP16), comm=comm if use_comm else None)
        b = tn.Buffers(p)
        a = tn.contract(p, b, 0)
        if rank == 0:
            print(it, "comm" if use_comm else "single", "rel", metrics.rel_l2(a, ref), "norm", float(np.linalg.norm(a)),
                  flush=True)
        if it % 2:
            keep.append((p, b))
dist.barrier()
dist.destroy_process_group()
