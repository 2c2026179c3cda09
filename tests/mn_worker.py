"""Subprocess helper of tests/test_gpu_e2e.py::test_mn_major_steps_vs_oracle: contracts the C3 plan
sub-sliced to 2^25 with the MN-major operand enabled down to 2^18-element steps (TN_MN_MIN_LOG2 is
read once per process, hence the subprocess), on one GPU and on 4 loopback ranks, and saves the
amplitudes and the MN steps of each lowering (and the split-block ones of the one-GPU lowering)."""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    out = sys.argv[1]
    from paper_2407_00769_b200 import tn
    from workload import make_plans as MP
    with open(os.path.join(ROOT, "plans", "c3.json")) as f:
        sub = MP.sub_slice(json.load(f), 25)
    kw = dict(stem_min_log2=16, comm_codec=tn.TN_COMM_FP16)
    p = tn.Plan(sub, tn.make_config(**kw))
    one = tn.contract(p, tn.Buffers(p), 0)
    mn_one = [s["mn"] for s in p.report()["steps"] if s["mn"]]
    split_one = [s["mn_split"][0] for s in p.report()["steps"] if s["mn"] and s["mn_split"][0]]
    group = tn.LoopbackComm(4)

    def rank_fn(r):
        q = tn.Plan(sub, tn.make_config(**kw), comm=group.ranks[r])
        return tn.contract(q, tn.Buffers(q), 0), [s["mn"] for s in q.report()["steps"] if s["mn"]]

    res = tn.run_ranks(4, rank_fn)
    np.savez(out, one=one, four=res[0][0], mn_one=np.array(mn_one), mn_four=np.array(res[0][1]),
             split_one=np.array(split_one))


if __name__ == "__main__":
    main()
