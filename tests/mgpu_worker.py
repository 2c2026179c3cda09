"""Multi-GPU worker (launched by tests/test_gpu_multi.py through torch.distributed.run).

Each rank holds 1/G of the stem (sharded on its log2 G outermost modes); contracted
shard modes are swapped by NCCL send/recv with int8 group quantisation or fp16 (Alg. 1,
P:352-363).  Rank 0 compares the gathered amplitudes with the oracle (same plan, same slice) and
with the single-GPU run, and writes a JSON verdict."""
import json
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

from paper_2407_00769_b200 import tn  # noqa: E402
from swap_error import predicted_swap_error  # noqa: E402


def main():
    out_path = sys.argv[1]
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    from workload import make_plans as MP
    from oracle import contract, metrics
    from oracle.plan import load
    with open(os.path.join(ROOT, "plans", "c3.json")) as f:
        full = json.load(f)
    sub = MP.sub_slice(full, 22)   # C3 (53 qubits, 20 cycles) sub-sliced so the oracle is quick
    one_first = None
    if rank == 0:  # single-GPU reference run before any communicator exists
        p0 = tn.Plan(sub, tn.make_config(stem_min_log2=14))
        one_first = tn.contract(p0, tn.Buffers(p0), 0)
        del p0
    comm = tn.Comm(rank, world, local)
    results = {}
    # int8: every swap quantised on C2 (quant_from_pct=0); default late-stage policy on C3
    with open(os.path.join(ROOT, "plans", "c2.json")) as f:
        c2 = MP.sub_slice(json.load(f), 20)
    for codec, name, plan, pct, sm in ((tn.TN_COMM_FP16, "fp16", sub, -1, 14),
                                       (tn.TN_COMM_FP16, "fp16_nofused", sub, -1, 14),
                                       (tn.TN_COMM_INT8, "int8", sub, -1, 14),
                                       (tn.TN_COMM_INT8, "int8_all_c2", c2, 0, 12),
                                       (tn.TN_COMM_INT8, "int8_all_c3", sub, 0, 14),
                                       (tn.TN_COMM_INT8, "int8_all_c3_unfused", sub, 0, 14),
                                       (tn.TN_COMM_INT4, "int4", sub, -1, 14),
                                       (tn.TN_COMM_INT4, "int4_all", sub, 0, 14),
                                       (tn.TN_COMM_INT8_TENSOR, "int8_tensor_all", sub, 0, 14)):
        p = tn.Plan(plan, tn.make_config(stem_min_log2=sm, comm_codec=codec, quant_from_pct=pct,
                                         no_fuse_swap_quant=int(name.endswith("_unfused")),
                                         no_fused_swap=int(name.endswith("_nofused"))), comm=comm)
        b = tn.Buffers(p)
        amps = tn.contract(p, b, 0)
        torch.cuda.synchronize()
        print(f"rank {rank} {name}: norm {float(np.linalg.norm(amps))}", flush=True)
        results[name] = (amps, p.report())
    if rank == 0:
        ref = contract.contract(load(sub), 0)
        p1 = tn.Plan(sub, tn.make_config(stem_min_log2=14))
        one = tn.contract(p1, tn.Buffers(p1), 0)
        print(f"rank {rank} single-after: norm {float(np.linalg.norm(one))} first {float(np.linalg.norm(one_first))}", flush=True)
        ref2 = contract.contract(load(c2), 0)
        verdict = {"world": world, "rel_1gpu_first_vs_after": metrics.rel_l2(one, one_first),
                   "rel_fp16_vs_1gpu_first": metrics.rel_l2(results["fp16"][0], one_first),
                   "rel_int8_all_c2_oracle": metrics.rel_l2(results["int8_all_c2"][0], ref2),
                   "int8_swaps_c2": sum(1 for s in results["int8_all_c2"][1]["steps"] if s.get("quant")),
                   "fused_swaps_c3": sum(1 for s in results["int8_all_c3"][1]["steps"] if s.get("fuse_quant")),
                   "fused_swaps_c3_unfused_run": sum(1 for s in results["int8_all_c3_unfused"][1]["steps"]
                                                     if s.get("fuse_quant")),
                   "rel_int8_all_c3_oracle": metrics.rel_l2(results["int8_all_c3"][0], ref),
                   "rel_int8_c3_fused_vs_unfused": metrics.rel_l2(results["int8_all_c3"][0],
                                                                  results["int8_all_c3_unfused"][0]),
                   "int8_swaps_c3": sum(1 for s in results["int8"][1]["steps"] if s.get("quant")),
                   "rel_fp16_oracle": metrics.rel_l2(results["fp16"][0], ref),
                   "rel_int8_oracle": metrics.rel_l2(results["int8"][0], ref),
                   "rel_int4_oracle": metrics.rel_l2(results["int4"][0], ref),
                   "int4_swaps_c3": sum(1 for s in results["int4"][1]["steps"] if s.get("quant")),
                   "rel_int4_all_oracle": metrics.rel_l2(results["int4_all"][0], ref),
                   "rel_int8_tensor_all_oracle": metrics.rel_l2(results["int8_tensor_all"][0], ref),
                   "fp16_oracle": metrics.rel_l2(results["fp16"][0], ref),
                   "pred_int8_all": predicted_swap_error(sub, results["int8_all_c3"][1], ref, "int8_g128"),
                   "pred_int8": predicted_swap_error(sub, results["int8"][1], ref, "int8_g128"),
                   "pred_int4_all": predicted_swap_error(sub, results["int4_all"][1], ref, "int4"),
                   "pred_int8_tensor_all": predicted_swap_error(sub, results["int8_tensor_all"][1], ref, "int8"),
                   "rel_fp16_vs_1gpu": metrics.rel_l2(results["fp16"][0], one),
                   "fp16_epilogue_swaps": results["fp16"][1]["n_fused_swaps"],
                   "fp16_nofused_epilogue_swaps": results["fp16_nofused"][1]["n_fused_swaps"],
                   "fp16_fused_equal_transport": bool(np.array_equal(results["fp16"][0], results["fp16_nofused"][0])),
                   "fp16_peer_pass_swaps": results["fp16"][1]["n_peer_swaps"],
                   "rel_1gpu_oracle": metrics.rel_l2(one, ref),
                   "swaps": sum(1 for s in results["int8"][1]["steps"] if s.get("swap")),
                   "steps": len(results["int8"][1]["steps"])}
        with open(out_path, "w") as f:
            json.dump(verdict, f)
        print(json.dumps(verdict))
    dist.barrier()
    del results
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
