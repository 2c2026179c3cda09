"""Dev tool: per-step table of gathered-A steps from a step_profile.py output file."""
import json
import re
import sys

sys.path.insert(0, ".")
from paper_2407_00769_b200 import tn  # noqa: E402

plan = json.load(open("plans/c3.json"))
p = tn.Plan(plan, tn.make_config(stem_min_log2=20))
ga = [s["ga"] for s in p.report()["steps"]]
tot = 0.0
for line in open(sys.argv[1]):
    m = re.match(r"\s*(\d+) m\s*(\d+) k\s*(\d+) n\s*(\d+) (\w+)\s+perm\s+([\d.]+) gemm\s+([\d.]+) ms", line)
    if m and ga[int(m.group(1))]:
        print(line.rstrip())
        tot += float(m.group(7))
print("gathered-A GEMM total ms", round(tot, 2))
