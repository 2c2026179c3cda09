"""SURVEY §8(d) μ-bench: the tcgen05 complex-half stem GEMM (Eq. 6 as one real fp16 GEMM,
P:496-514) on synthetic stem-shaped steps, M = 2^23 (default) rows, (log2 K, log2 N) over a grid
(default {4..10}^2), identity output layout, through the C-ABI kernel entry (tn_gemm_chalf).

Per shape: CUDA-event time (median of `iters` after warm-up), effective TFLOP/s (8 flops per complex
MAC, C-A21) against the measured bf16 burst peak (MEASURED_PEAKS.json, same rate as fp16 dense) and
the 2.25 PF spec, algorithmic HBM GB/s (4 B per complex element of A and C + B_P) against the
measured copy bandwidth, and the roofline bound max(F/P_burst, B/BW).  Inputs: A ~ N(0, 1/2) per
component, B_P ~ N(0, 1/(2K)) so |C| stays O(1) (the library's scale is not used: exp slots NULL).

  python tools/mubench.py [--m 23] [--k 4-10] [--n 4-10] [--iters 5] [--out file]
"""
import argparse
import json
import os
import statistics
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2407_00769_b200 import tn  # noqa: E402


def rng_arg(s):
    a, b = s.split("-") if "-" in s else (s, s)
    return list(range(int(a), int(b) + 1))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--m", type=int, default=23)
    ap.add_argument("--k", type=rng_arg, default=list(range(4, 11)))
    ap.add_argument("--n", type=rng_arg, default=list(range(4, 11)))
    ap.add_argument("--iters", type=int, default=5)
    ap.add_argument("--out", default=None)
    args = ap.parse_args()
    try:
        pk = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
        bw, tc = float(pk["hbm_gbs"]), float(pk["bf16_tflops"])
        src = "measured"
    except Exception:
        bw, tc, src = 6650.0, 1590.0, "fallback"
    torch.cuda.set_device(0)
    tn.set_device()
    M = 1 << args.m
    kmax, nmax = 1 << max(args.k), 1 << max(args.n)
    g = torch.Generator(device="cuda").manual_seed(0)
    A = torch.randn(M * kmax * 2, device="cuda", dtype=torch.float16, generator=g).mul_(0.7071)
    C = torch.empty(M * nmax * 2, device="cuda", dtype=torch.float16)
    rows = []
    lines = [f"# tcgen05 complex-half GEMM, M = 2^{args.m}, peaks ({src}): {tc:.0f} TF/s burst bf16/fp16, "
             f"{bw:.0f} GB/s copy; spec 2250 TF/s",
             "# log2K log2N     ms   TFLOP/s  %burst  %spec    GB/s  %hbm  bound  roof_frac"]
    for kl in args.k:
        for nl in args.n:
            K, N = 1 << kl, 1 << nl
            bp = (torch.randn(max(2 * N, 16) * 2 * K, device="cuda", dtype=torch.float32, generator=g)
                  * (0.5 / K ** 0.5)).half()
            if N < 8:
                bp.view(max(2 * N, 16), 2 * K)[2 * N:] = 0
            for _ in range(2):
                tn.tn_gemm_chalf(C, A, bp, M, K, N)
            torch.cuda.synchronize()
            ts = []
            for _ in range(args.iters):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                tn.tn_gemm_chalf(C, A, bp, M, K, N)
                e1.record()
                torch.cuda.synchronize()
                ts.append(e0.elapsed_time(e1))
            ms = statistics.median(ts)
            fl = 8.0 * M * K * N
            by = 4.0 * (M * K + M * N) + 8.0 * K * N
            tf = fl / ms / 1e9
            gbs = by / ms / 1e6
            t_roof = max(fl / (tc * 1e12), by / (bw * 1e9)) * 1e3
            bound = "tensor" if fl / (tc * 1e12) >= by / (bw * 1e9) else "hbm"
            r = dict(klog=kl, nlog=nl, ms=ms, tflops=tf, frac_burst=tf / tc, frac_spec=tf / 2250.0, gbs=gbs,
                     frac_hbm=gbs / bw, bound=bound, roof_frac=t_roof / ms)
            rows.append(r)
            lines.append(f"  {kl:5d} {nl:5d} {ms:8.3f} {tf:9.1f} {100 * tf / tc:6.1f} {100 * tf / 2250:6.1f} "
                         f"{gbs:7.0f} {100 * gbs / bw:5.1f} {bound:>6s} {r['roof_frac']:9.3f}")
            print(lines[-1], flush=True)
    text = "\n".join(lines)
    print(text)
    if args.out:
        with open(args.out, "w") as f:
            f.write(text + "\n")
        with open(os.path.splitext(args.out)[0] + ".json", "w") as f:
            json.dump({"m_log2": args.m, "peaks": {"tc_burst": tc, "hbm": bw, "source": src}, "rows": rows}, f, indent=1)


if __name__ == "__main__":
    main()
