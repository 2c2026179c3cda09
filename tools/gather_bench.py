"""Dev tool: time the gathered-A tcgen05 GEMM for a run pattern of the source layout.

usage: python tools/gather_bench.py mlog klog nlog RUNS  (RUNS like k2m8k5m15: innermost first)"""
import re
import sys

import torch

sys.path.insert(0, ".")
from paper_2407_00769_b200 import tn  # noqa: E402


def run(mlog, klog, nlog, runs, iters=5):
    kpos, mpos, b = [], [], 0
    for kind, cnt in re.findall(r"([km])(\d+)", runs):
        for _ in range(int(cnt)):
            (kpos if kind == "k" else mpos).append(b)
            b += 1
    assert len(kpos) == klog and len(mpos) == mlog, (len(kpos), len(mpos))
    ms, ks = [1 << p for p in mpos], [1 << p for p in kpos]
    M, K, N = 1 << mlog, 1 << klog, 1 << nlog
    X = torch.randn(M * K * 2, device="cuda", dtype=torch.float16)
    BP = torch.randn(max(2 * N, 16) * 2 * K, device="cuda", dtype=torch.float16) * 0.01
    C = torch.empty(M * N * 2, device="cuda", dtype=torch.float16)
    tn.tn_gemm_chalf_gather(C, X, BP, mlog, klog, N, ms, ks)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(iters):
        tn.tn_gemm_chalf_gather(C, X, BP, mlog, klog, N, ms, ks)
    e1.record()
    torch.cuda.synchronize()
    ms_ = e0.elapsed_time(e1) / iters
    by = 4 * (M * K + M * N)
    print(f"m{mlog} k{klog} n{nlog} {runs}: {ms_:.3f} ms  {by / ms_ / 1e6:.0f} GB/s", flush=True)


if __name__ == "__main__":
    for spec in sys.argv[1:]:
        a = spec.split(",")
        run(int(a[0]), int(a[1]), int(a[2]), a[3])
