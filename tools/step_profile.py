"""Dev tool: per-stem-step timing table of one subtask (CUDA events inside libtn)."""
import json
import sys

import torch

sys.path.insert(0, ".")
from paper_2407_00769_b200 import tn  # noqa: E402


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "c3"
    pol = int(sys.argv[2]) if len(sys.argv) > 2 else 0
    plan = json.load(open(f"plans/{name}.json"))
    sm = int(sys.argv[3]) if len(sys.argv) > 3 else 20
    p = tn.Plan(plan, tn.make_config(stem_min_log2=sm, layout_policy=pol))
    print(p.info()["n_permutes"], "permutes")
    b = tn.Buffers(p)
    tn.tn_plan_upload(p, b)
    for _ in range(2):
        tn.tn_stem_contract(p, b, 0)
    p.set_timing(True)
    tn.tn_stem_contract(p, b, 0)
    torch.cuda.synchronize()
    r = p.report()
    ms = r["ms"]
    print(f"policy {pol} common {ms[0]:.2f} ms")
    tot = {}
    for i, s in enumerate(r["steps"]):
        M, K, N = 2 ** s["m"], 2 ** s["k"], 2 ** s["n"]
        by = 4 * (M * K + M * N)
        pm, gm = ms[1 + 2 * i], ms[2 + 2 * i]
        key = ("tc" if s["tc"] else "simt")
        tot[key] = tot.get(key, 0) + gm
        print(f"{i:3d} m{s['m']:2d} k{s['k']:2d} n{s['n']:2d} {key:4s} perm {pm:7.3f} gemm {gm:7.3f} ms "
              f"{by / gm / 1e6 if gm > 0 else 0:7.0f} GB/s  in {4*M*K/2**30:.2f} GiB out {4*M*N/2**30:.2f} GiB")
    perm_tot = sum(ms[1 + 2 * i] for i in range(len(r["steps"])))
    print("totals", {k: round(v, 2) for k, v in tot.items()}, "perm", round(perm_tot, 2), "final", round(ms[-1], 3),
          "common", round(ms[0], 2), "sum", round(sum(ms), 2))


if __name__ == "__main__":
    main()
