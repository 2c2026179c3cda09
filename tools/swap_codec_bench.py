"""Dev tool: sender side of a quantised mode swap on a stem-sized complex-half tensor — fused
permute + int8 codec (tn_permute_quant_f16) vs permutation pass + codec — CUDA events, GB/s of
algorithmic bytes (read 4 B per complex element; write 2 codes + 8 B of scale/zero per g reals)."""
import sys

import torch

sys.path.insert(0, ".")
from paper_2407_00769_b200 import tn  # noqa: E402


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 28
    g = 128
    b = 6  # log2(g/2)
    gen = torch.Generator(device="cuda").manual_seed(0)
    x = torch.randn(2 << n, device="cuda", generator=gen).half()
    y = torch.empty_like(x)
    codes = torch.empty(2 << n, dtype=torch.int8, device="cuda")
    sc = torch.empty((2 << n) // g, dtype=torch.float32, device="cuda")
    ze = torch.empty_like(sc)
    # a swap-like permutation: two inner-ish modes move outermost, the innermost b stay
    outer = list(range(n - b))
    perm = [outer[-1], outer[-2]] + outer[:-2] + list(range(n - b, n))
    alg = (4 << n) + (2 << n) + 8 * ((2 << n) // g)
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]

    def run(fn, reps=10):
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        ev[0].record()
        for _ in range(reps):
            fn()
        ev[1].record()
        torch.cuda.synchronize()
        return ev[0].elapsed_time(ev[1]) / reps

    def fused():
        tn.tn_permute_quant_f16(codes, sc, ze, x, perm, g)

    def separate():
        tn.tn_permute(y.view(torch.complex32), x.view(torch.complex32), perm)
        tn.tn_quant_int8_f16(codes, sc, ze, y, g)

    def deq():
        tn.tn_dequant_int8_f16(y, codes, sc, ze, g)

    tf, ts, td = run(fused), run(separate), run(deq)
    dalg = (2 << n) + 8 * ((2 << n) // g) + (4 << n)
    print(f"dequant int8 -> complex-half: {td:.3f} ms ({dalg / td / 1e6:.0f} GB/s algorithmic)")
    print(f"n={n} ({(4 << n) / 2**30:.1f} GiB stem): fused {tf:.3f} ms ({alg / tf / 1e6:.0f} GB/s algorithmic), "
          f"permute+quant {ts:.3f} ms, speed-up {ts / tf:.2f}x")


if __name__ == "__main__":
    main()
