"""Dev tool: sharded (loopback, 2 ranks) vs one-GPU sparse-state batch and dense readout on the C2
sub-slice, per layout policy: relative errors, whether the blocks match up to a member permutation,
and the layouts involved."""
import sys

import numpy as np

sys.path.insert(0, ".")
sys.path.insert(0, "tests")
from paper_2407_00769_b200 import tn  # noqa: E402
import test_gpu_loopback as T  # noqa: E402


def rel(a, b):
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def main():
    plan = T.MP.sub_slice(T._plan("c2"), 20)
    pre = np.array([3, 0, 7, 5], dtype=np.uint64)
    for pol in (0, 3):
        kw = dict(dtype=0, stem_min_log2=12, split_log2=3, comm_codec=tn.TN_COMM_FP16, layout_policy=pol)
        p1 = tn.Plan(plan, tn.make_config(**kw))
        b1 = tn.Buffers(p1)
        tn.tn_plan_upload(p1, b1)
        tn.tn_stem_contract(p1, b1, 0)
        a1, t1 = tn.tn_sample_sparse(p1, b1, pre, k=1)
        d1 = tn.contract(p1, b1, 0)
        r1 = p1.report()
        out = T.run_loopback(tn, plan, 2, kw, sparse=pre)
        a2, t2 = out[0][0]
        r2 = out[0][1]
        outd = T.run_loopback(tn, plan, 2, kw)
        d2 = outd[0][0]
        print(f"policy {pol}: sparse rel {rel(a2, a1):.3e} dense rel {rel(d2, d1):.3e} tops {list(t1)} {list(t2)}")
        for i in range(len(pre)):
            s1 = np.sort(np.abs(a1[i]).ravel())
            s2 = np.sort(np.abs(a2[i]).ravel())
            print(f"  block {i}: rel {rel(a2[i], a1[i]):.3e} sorted-abs rel {rel(s2, s1):.3e}")
        # dense blocks vs the sparse blocks (one GPU and sharded)
        for key in ("split_modes", "final_layout", "final_shard", "split_from", "shard0"):
            print(f"  {key}: 1gpu {r1.get(key)} 2rk {r2.get(key)}")
        print("  steps 2rk:", [(s["m"], s["k"], s["n"], s["swap"], s["split"]) for s in r2["steps"]][-8:])
        print("  steps 1gpu:", [(s["m"], s["k"], s["n"], s["swap"], s["split"]) for s in r1["steps"]][-8:])


if __name__ == "__main__":
    main()
