"""Dev tool: time the tcgen05 complex-half GEMM (identity output) for one shape via the C-ABI."""
import sys

import torch

sys.path.insert(0, ".")
from paper_2407_00769_b200 import tn  # noqa: E402


def run(mlog, klog, nlog, iters=5):
    M, K, N = 1 << mlog, 1 << klog, 1 << nlog
    A = torch.randn(M * K * 2, device="cuda", dtype=torch.float16)
    BP = torch.randn(4 * K * N, device="cuda", dtype=torch.float16) * 0.01
    C = torch.empty(M * N * 2, device="cuda", dtype=torch.float16)
    tn.tn_gemm_chalf(C, A, BP, M, K, N)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(iters):
        tn.tn_gemm_chalf(C, A, BP, M, K, N)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / iters
    by = 4 * (M * K + M * N)
    fl = 8 * M * K * N
    print(f"m{mlog} k{klog} n{nlog}: {ms:.3f} ms  {by / ms / 1e6:.0f} GB/s  {fl / ms / 1e9:.1f} TFLOP/s", flush=True)


if __name__ == "__main__":
    shapes = [tuple(int(x) for x in s.split(",")) for s in sys.argv[1:]] or [(23, 5, 8), (22, 6, 10), (23, 8, 6),
                                                                           (24, 6, 6), (20, 10, 10), (18, 12, 12)]
    for s in shapes:
        run(*s)
