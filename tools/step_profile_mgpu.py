"""Dev tool: per-stem-step timing of one SHARDED subtask (CUDA events inside libtn, rank 0 shown;
max over ranks per step printed beside it).  Launch with torchrun:

  python -m torch.distributed.run --nproc-per-node N tools/step_profile_mgpu.py [plan] [repeats]"""
import json
import os
import statistics
import sys

import torch
import torch.distributed as dist

sys.path.insert(0, ".")
from paper_2407_00769_b200 import tn  # noqa: E402


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "c3"
    reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    comm = tn.Comm(rank, world, local)
    plan = json.load(open(f"plans/{name}.json"))
    p = tn.Plan(plan, tn.make_config(stem_min_log2=20, comm_codec=tn.TN_COMM_INT8), comm=comm)
    b = tn.Buffers(p)
    tn.tn_plan_upload(p, b)
    for _ in range(2):
        tn.tn_stem_contract(p, b, 0)
    torch.cuda.synchronize()
    p.set_timing(True)
    runs = []
    for _ in range(reps):
        dist.barrier()
        tn.tn_stem_contract(p, b, 0)
        torch.cuda.synchronize()
        runs.append(p.report())
    ms = torch.tensor([[statistics.median(x["ms"][j] for x in runs) for j in range(len(runs[0]["ms"]))]],
                      device="cuda")
    mx = ms.clone()
    dist.all_reduce(mx, op=dist.ReduceOp.MAX)
    if rank == 0:
        r = runs[0]
        m0, mm = ms[0].tolist(), mx[0].tolist()
        print(f"world {world}: swaps {r['n_swaps']} in-epilogue {r['n_fused_swaps']}; common {m0[0]:.2f} ms")
        for i, s in enumerate(r["steps"]):
            tag = ("swap" + ("q" if s["quant"] else "") if s["swap"] else "") + (" perm" if s["perm"] else "")
            nxt = r["steps"][i + 1] if i + 1 < len(r["steps"]) else None
            if nxt is not None and nxt["swap"]:
                tag += " ->swap"
            print(f"{i:3d} m{s['m']:2d} k{s['k']:2d} n{s['n']:2d} {'tc' if s['tc'] else 'simt'} ga{s['ga']} "
                  f"pre {m0[1 + 2 * i]:7.3f} ({mm[1 + 2 * i]:7.3f}) gemm {m0[2 + 2 * i]:7.3f} ({mm[2 + 2 * i]:7.3f}) {tag}")
        print("sum", round(sum(m0), 2), "max-over-ranks sum", round(sum(mm), 2))
    dist.barrier()
    del p, b
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
