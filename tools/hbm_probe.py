"""Dev tool: HBM read-only / write-only / copy bandwidth on this GPU (torch kernels, CUDA events)."""
import torch

n = 1 << 31  # 8 GiB of fp32
a = torch.empty(n, dtype=torch.float32, device="cuda")
b = torch.empty(n, dtype=torch.float32, device="cuda")
a.fill_(1.0)


def t(fn, iters=5):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(iters):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / iters


ms = t(lambda: b.copy_(a))
print(f"copy  : {2 * 4 * n / ms / 1e6:.0f} GB/s (read+write)")
ms = t(lambda: b.fill_(2.0))
print(f"write : {4 * n / ms / 1e6:.0f} GB/s (fill)")
ms = t(lambda: torch.cuda.memset_async if False else b.zero_())
print(f"write : {4 * n / ms / 1e6:.0f} GB/s (zero_)")
ms = t(lambda: a.sum())
print(f"read  : {4 * n / ms / 1e6:.0f} GB/s (sum)")
c = a[: n // 8]
d = torch.empty(n, dtype=torch.float32, device="cuda")
ms = t(lambda: d.view(8, -1).copy_(c.expand(8, -1)))
print(f"1:8 read:write : {(4 * n / 8 + 4 * n) / ms / 1e6:.0f} GB/s (broadcast copy)")
