"""Dev tool: per-stem-step timing table of one subtask (CUDA events inside libtn).

  python tools/step_profile.py [plan] [policy] [stem_min_log2] [repeats]

With repeats > 1 every step shows the min and the max over the repeated subtasks (the box runs
under a 1 kW power cap, so single replays vary with the SM clock)."""
import json
import statistics
import sys

import torch

sys.path.insert(0, ".")
from paper_2407_00769_b200 import tn  # noqa: E402


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "c3"
    pol = int(sys.argv[2]) if len(sys.argv) > 2 else 3
    plan = json.load(open(f"plans/{name}.json"))
    sm = int(sys.argv[3]) if len(sys.argv) > 3 else 20
    reps = int(sys.argv[4]) if len(sys.argv) > 4 else 1
    p = tn.Plan(plan, tn.make_config(stem_min_log2=sm, layout_policy=pol))
    print(p.info()["n_permutes"], "permutes")
    b = tn.Buffers(p)
    tn.tn_plan_upload(p, b)
    for _ in range(2):
        tn.tn_stem_contract(p, b, 0)
    p.set_timing(True)
    runs = []
    for _ in range(reps):
        tn.tn_stem_contract(p, b, 0)
        torch.cuda.synchronize()
        runs.append(p.report())
    r = runs[0]
    print(f"policy {pol} common {statistics.median(x['ms'][0] for x in runs):.2f} ms (median of {reps})")
    tot = {}
    for i, s in enumerate(r["steps"]):
        M, K, N = 2 ** s["m"], 2 ** s["k"], 2 ** s["n"]
        by = 4 * (M * K + M * N)
        fl = 8 * M * K * N
        pms = [x["ms"][1 + 2 * i] for x in runs]
        gms = [x["ms"][2 + 2 * i] for x in runs]
        pm, gm = statistics.median(pms), statistics.median(gms)
        key = s.get("kern") or ("tc" if s["tc"] else "simt")
        tot[key] = tot.get(key, 0) + gm
        print(f"{i:3d} m{s['m']:2d} k{s['k']:2d} n{s['n']:2d} {key:6s} ga{s['ga']} perm {pm:7.3f} gemm {gm:7.3f} ms "
              f"[{min(gms):7.3f} {max(gms):7.3f}] {by / gm / 1e6 if gm > 0 else 0:5.0f} GB/s "
              f"{fl / gm / 1e9 if gm > 0 else 0:6.0f} TF/s  in {4*M*K/2**30:.2f} GiB out {4*M*N/2**30:.2f} GiB")
    perm_tot = sum(statistics.median(x["ms"][1 + 2 * i] for x in runs) for i in range(len(r["steps"])))
    sums = [sum(x["ms"]) for x in runs]
    print("totals", {k: round(v, 2) for k, v in tot.items()}, "perm", round(perm_tot, 2),
          "common", round(statistics.median(x["ms"][0] for x in runs), 2),
          "sum median", round(statistics.median(sums), 2), "min", round(min(sums), 2), "max", round(max(sums), 2))


if __name__ == "__main__":
    main()
