"""Summarise an ncu launch list (--metrics gpu__time_duration.sum,dram__bytes_read.sum,
dram__bytes_write.sum --csv) of bench.py into per-kernel-family totals per subtask.

usage: python tools/ncu_summary.py LAUNCHES.csv RUNS [OUT.json]
RUNS = how many tn_stem_contract calls the profiled command made (bench.py --steps K --warmup W:
W + K + 3 end-to-end calls).  ncu serialises launches and runs them cold: use the SHARE of each
family, not the absolute times (profiles/README)."""
import collections
import csv
import io
import json
import sys


def family(name):
    if "gemm_chalf_tc2" in name:
        return "gemm_tc2"  # the CTA-pair kernel (plain, N-d box and MN-major forms)
    if "gemm_chalf_tc" in name:
        return "gemm_tc"
    if "gemm_chalf_rows" in name or "gemm_chalf_simt" in name:
        return "gemm_simt"
    if "gemm_c64" in name:
        return "gemm_c64"
    if "permute" in name:
        return "permute"
    if "contract_c64" in name:
        return "common"
    return "prep/other"


def main():
    path, runs = sys.argv[1], int(sys.argv[2])
    lines = [ln for ln in open(path) if ln.startswith('"')]
    rd = csv.DictReader(io.StringIO("".join(lines)))
    per = collections.defaultdict(dict)
    for row in rd:
        per[int(row["ID"])]["name"] = row["Kernel Name"]
        v = float(row["Metric Value"].replace(",", ""))
        unit = row["Metric Unit"]
        if row["Metric Name"] == "gpu__time_duration.sum":
            v *= {"ns": 1e-6, "nsecond": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0}.get(unit, 1e-6)
        else:
            v *= {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)
        per[int(row["ID"])][row["Metric Name"]] = v
    fam = collections.defaultdict(lambda: {"launches": 0, "ms": 0.0, "dram_read": 0.0, "dram_write": 0.0})
    for k in per.values():
        f = fam[family(k["name"])]
        f["launches"] += 1
        f["ms"] += k.get("gpu__time_duration.sum", 0.0)
        f["dram_read"] += k.get("dram__bytes_read.sum", 0.0)
        f["dram_write"] += k.get("dram__bytes_write.sum", 0.0)
    tot_ms = sum(f["ms"] for f in fam.values())
    out = {"source": path, "runs": runs, "launches_total": len(per), "per_subtask": {}}
    for name, f in sorted(fam.items(), key=lambda x: -x[1]["ms"]):
        out["per_subtask"][name] = {"launches": f["launches"] / runs, "ms_cold_serialised": f["ms"] / runs,
                                    "share": f["ms"] / tot_ms, "dram_bytes": (f["dram_read"] + f["dram_write"]) / runs}
    print(json.dumps(out, indent=1))
    if len(sys.argv) > 3:
        with open(sys.argv[3], "w") as fh:
            json.dump(out, fh, indent=1)


if __name__ == "__main__":
    main()
