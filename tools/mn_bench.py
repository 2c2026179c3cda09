"""Dev tool: the MN-major A GEMM (tn_gemm_chalf_mn, permutation folded into the operand) against the
permutation pass + plain GEMM (tn_permute + tn_gemm_chalf) on the same stem-shaped step.

  python tools/mn_bench.py mlog klog nlog ma [iters]"""
import sys

import torch

sys.path.insert(0, ".")
from paper_2407_00769_b200 import tn  # noqa: E402


def timed(fn, iters):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(iters):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / iters


def main():
    mlog, klog, nlog, ma = (int(x) for x in sys.argv[1:5])
    iters = int(sys.argv[5]) if len(sys.argv) > 5 else 5
    M, K, N = 1 << mlog, 1 << klog, 1 << nlog
    g = torch.Generator(device="cuda").manual_seed(0)
    X = torch.randn(2 * M * K, device="cuda", dtype=torch.float16, generator=g)
    Y = torch.empty_like(X)
    B = (torch.randn(2 * K * N, device="cuda", generator=g) / K ** 0.5).float()
    BPM = torch.empty(2 * N * K, dtype=torch.float16, device="cuda")
    BP = torch.empty(4 * N * K, dtype=torch.float16, device="cuda")
    scratch = torch.zeros(4, dtype=torch.int32, device="cuda")
    tn.tn_pad_b_mn(BPM, B, K, N, None, None, scratch)
    tn.tn_pad_b(BP, B, K, N, None, None, scratch)
    C = torch.empty(2 * M * N, dtype=torch.float16, device="cuda")
    # stored [M >> ma][K][2^ma] -> permuted [M][K]: axes (outermost first) hi, k, lo -> hi, lo, k
    nb = mlog + klog
    axes = list(range(mlog - ma)) + list(range(mlog - ma + klog, nb)) + list(range(mlog - ma, mlog - ma + klog))
    t_mn = timed(lambda: tn.tn_gemm_chalf_mn(C, X, BPM, M, K, N, ma), iters)
    t_p = timed(lambda: tn.tn_permute_bytes(Y, X, 4, axes), iters)
    t_g = timed(lambda: tn.tn_gemm_chalf(C, Y, BP, M, K, N), iters)
    fl = 8.0 * M * K * N
    print(f"m{mlog} k{klog} n{nlog} ma{ma}: mn {t_mn:.3f} ms ({fl / t_mn / 1e9:.0f} TF/s) | perm {t_p:.3f} + "
          f"gemm {t_g:.3f} = {t_p + t_g:.3f} ms ({fl / t_g / 1e9:.0f} TF/s gemm)", flush=True)


if __name__ == "__main__":
    main()
