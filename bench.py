#!/usr/bin/env python
"""Benchmark: stem-path contraction of one sliced subtask of the C3 workload (53-qubit, 20-cycle
Sycamore-style RQC network, largest stem 2^33 complex-half) on B200 — BASELINE.json metric
"stem-contraction effective TFLOPS/GPU and subtask time-to-solution".

A step = one subtask: tn_stem_contract (common phase + Eq. 6 padding + all stem steps) +
tn_split_contract, inputs (leaves) resident in HBM.  value = effective TFLOPS of the job (8 flops
per complex MAC of the stem GEMMs, reading C-A21) / max-over-ranks device time.
Multi-GPU (C4): ONE subtask sharded across the N GPUs on its log2 N outermost modes, with
int8-quantised (late-stage) or fp16 NCCL mode swaps (Alg. 1) — strong scaling.
--replicas runs independent slices per GPU instead (weak scaling, no collective).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference] [--plan c3]
"""
import os

_CORES = len(os.sched_getaffinity(0))
for _v in ("OPENBLAS_NUM_THREADS", "OMP_NUM_THREADS", "MKL_NUM_THREADS"):
    os.environ.setdefault(_v, str(_CORES))

import argparse  # noqa: E402
import json  # noqa: E402
import statistics  # noqa: E402
import subprocess  # noqa: E402
import sys  # noqa: E402
import tempfile  # noqa: E402
import time  # noqa: E402

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "stem-contraction effective TFLOPS/GPU and subtask time-to-solution at 1/2/4/8 B200"
WORKLOADS = {
    "c3": "C3: 53-qubit (6x9 grid minus a corner) 20-cycle Sycamore-style RQC network, one sliced subtask "
          "(158 sliced edges, branch-grouped stem: MB-scale non-stem tensors), 6 open legs, largest stem 2^32 "
          "complex-half, stem buffers 2 x 16 GiB",
    "c3_sweep": "C3 (round-1 plan, memory-bound variant): same network, 188 sliced edges, 12-branch groups, "
                "largest stem 2^33 complex-half, stem buffers 2 x 32 GiB",
    "c2": "C2: 30-qubit (5x6) 14-cycle RQC, one sliced subtask, 10 open legs",
    "c5": "C5: the C3 network with 22 output legs open: sparse-state batch of 1024 seeded correlated subspaces "
          "(values of the 12 legs entering the stem last) x 1024 members, top-1 post-selection per subspace",
}


# layout policy per plan (tn.h tn_config.layout_policy): 3 = identity outputs, transposed C[n][m] TMA
# stores where they put the next step's contracted modes innermost, permutations fused into the next
# GEMM's load or passes otherwise (C3: 280 ms vs 325 ms for policy 0 and 2.5x that for policy 2)
DEFAULT_POLICY = {}
POLICY_FALLBACK = 3


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), float(d["bf16_tflops"]), float(d.get("bf16_tflops_sustained", d["bf16_tflops"])), "measured"
    except Exception:
        return 6650.0, 1590.0, 1400.0, "fallback"


class Energy:
    """Board energy over the timed region from NVML's cumulative counter (mJ since driver load;
    SURVEY §8(f) #4, context beside the paper's Wh per subtask)."""

    def __init__(self, index):
        self.h = None
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.e0 = pynvml.nvmlDeviceGetTotalEnergyConsumption(self.h)
            self.t0 = time.perf_counter()
        except Exception:
            self.h = None

    def stop(self):
        if self.h is None:
            return None
        try:
            j = (self.nv.nvmlDeviceGetTotalEnergyConsumption(self.h) - self.e0) / 1000.0  # J
            return j / (time.perf_counter() - self.t0)  # mean board power over the interval, W
        except Exception:
            return None


class Clocks:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    def __init__(self, index):
        self.f = tempfile.NamedTemporaryFile("w+", delete=False, suffix=".csv")
        q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self.p = subprocess.Popen(["nvidia-smi", "-i", str(index), f"--query-gpu={q}", "--format=csv,noheader,nounits",
                                       "-lms", "200"], stdout=self.f, stderr=subprocess.DEVNULL)
        except Exception:
            self.p = None

    def stop(self):
        if self.p is None:
            return None
        self.p.terminate()
        try:
            self.p.wait(timeout=5)
        except Exception:
            self.p.kill()
        self.f.flush()
        rows = []
        with open(self.f.name) as f:
            for line in f:
                parts = [x.strip() for x in line.split(",")]
                if len(parts) >= 9:
                    rows.append(parts)
        os.unlink(self.f.name)
        if not rows:
            return None
        sm = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        reasons = set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in rows:
            for n, v in zip(names, r[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": float(rows[0][2]) if rows[0][2].replace(".", "").isdigit() else None,
                "power_w_max": max(float(r[3]) for r in rows if r[3].replace(".", "").isdigit()) if rows else None,
                "samples": len(rows), "reasons": sorted(reasons)}


def oracle_sample(plan, target_log2):
    from workload import make_plans as MP
    return MP.sub_slice(plan, target_log2)


def run_oracle(sub, steps, warmup):
    from oracle import contract
    from oracle.plan import load
    p = load(sub)
    fl = contract.flops(sub)
    for _ in range(warmup):
        contract.contract(p, 0)
    ts = []
    for _ in range(steps):
        t0 = time.perf_counter()
        contract.contract(p, 0)
        ts.append(time.perf_counter() - t0)
    t = statistics.median(ts)
    return fl, t


def cpu_baseline(plan, target_log2, steps=1, warmup=0):
    from oracle import contract
    sub = oracle_sample(plan, target_log2)
    fl, t = run_oracle(sub, steps, warmup)
    full = contract.flops(plan)
    return {"value": fl / t / 1e12, "unit": "TFLOPS", "cores": _CORES, "kind": "oracle",
            "seconds": t, "sample": f"oracle (numpy complex128, np.tensordot) on slice 0 of the same plan "
                                   f"sub-sliced by {len(sub['sliced']) - len(plan['sliced'])} extra edges "
                                   f"(every intermediate <= 2^{target_log2}); {fl:.3e} flops in {t:.2f} s",
            "extrapolated_full_subtask_s": t * full / fl,
            "extrapolation": f"x {full / fl:.1f} = the full subtask's {full:.3e} flops at the sample's rate "
                             f"(labelled estimate, SURVEY 8(d) d.4)"}, sub


def parity(tn, sub, cfg_kw):
    """The GPU path on the oracle's sub-slice (same plan, same kernels, fewer modes; SURVEY §8(c) c.6
    step 1) against the oracle's complex128 amplitudes: rel-L2, bound 2e-2 (north_star)."""
    from oracle import contract, metrics
    from oracle.plan import load
    ref = contract.contract(load(sub), 0)
    p = tn.Plan(sub, tn.make_config(**cfg_kw))
    got = tn.contract(p, tn.Buffers(p), 0)
    return {"rel_l2_vs_oracle": metrics.rel_l2(got, ref), "bound": 2e-2,
            "sample": f"slice 0 of the plan sub-sliced to max 2^{p.info()['max_stem_log2']} "
                      f"({len(sub['sliced'])} sliced edges), complex-half GPU path vs oracle complex128"}


def bench_sparse(args, plan_json, tn, torch, dist, world, rank, local):
    """C5 (BJ configs[4]): one subtask = the dense stem + the sparse-state tail for S seeded correlated
    subspaces (values of the plan's sparse legs) + top-1 post-selection on the device.
    Replicas over GPUs: rank r runs slice r (weak scaling).  Reported beside the metric:
    the linear XEB of the S post-selected samples of THIS slice (a partial sum, reading C-A25: context,
    not a fidelity estimate) and the parity of the same path on the oracle's sub-slice."""
    import numpy as np
    from paper_2407_00769_b200 import postselect
    dev_stream = torch.cuda.current_stream()
    L = len(plan_json["sparse_legs"])
    rng = np.random.default_rng(args.seed)
    pre = np.sort(rng.choice(2 ** L, size=min(args.subspaces, 2 ** L), replace=False)).astype(np.uint64)
    p = tn.Plan(plan_json, tn.make_config(dtype=tn.TN_CHALF, stem_min_log2=20))
    info = p.info()
    free = torch.cuda.mem_get_info()[0]
    stem_bytes = max(info["stem_bytes"], int(min(free * 0.42, 80 << 30)) // 4096 * 4096)
    bufs = tn.Buffers(p, stem_bytes=stem_bytes)
    n_sl = min(info["n_slices_log2"], 63)
    slice_id = rank % (1 << n_sl) if n_sl else 0
    tn.tn_plan_upload(p, bufs)

    def step():
        tn.tn_stem_contract(p, bufs, slice_id)
        return tn.tn_sample_sparse(p, bufs, pre, k=1)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    clk = Clocks(local)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(dev_stream)
    for _ in range(args.steps):
        amps, top = step()
    e1.record(dev_stream)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clocks = clk.stop()
    t_ms = e0.elapsed_time(e1) / args.steps
    rep = p.report()
    flops_rank = info["stem_flops"] + rep["sparse_flops"]
    if world > 1:
        tt = torch.tensor([t_ms], device="cuda")
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        t_ms = float(tt.item())
    value = flops_rank * world / (t_ms * 1e-3) / 1e12
    chosen = np.abs(amps[np.arange(len(pre)), top[:, 0].astype(np.int64)]) ** 2
    n_qubits = plan_json["circuit"]["n_qubits"]
    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": "TFLOPS", "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": t_ms, "higher_is_better": True,
                "scaling": "weak" if world > 1 else "strong", "vs_baseline": None, "dtype": "f16",
                "data": "synthetic",
                "config": {"workload": WORKLOADS.get(args.plan, args.plan), "plan": f"plans/{args.plan}.json",
                           "slice": "rank r runs slice r (replicas over independent subtasks)",
                           "subspaces": int(len(pre)), "members": int(amps.shape[1]), "sparse_legs": L,
                           "sparse_from_step": rep["sparse_from"], "stem_steps": info["n_stem_steps"],
                           "sparse_chunks": rep["sparse_chunks"], "stem_flops": info["stem_flops"],
                           "sparse_tail_flops": rep["sparse_flops"], "stem_buffers_gib": 2 * stem_bytes / 2 ** 30,
                           "l2": "tail tensors larger than L2"},
                "tflops_per_gpu": value / world, "subtask_ms": t_ms,
                "samples": {"n": int(len(pre)), "xeb_one_slice": postselect.linear_xeb(chosen, n_qubits),
                            "note": "top-1 per subspace of ONE slice's partial amplitudes (C-A25): context only"},
                "gpu_launches": p.info()["n_launches"] * args.steps, "clocks": clocks}
        if world == 1 and not args.no_cpu:
            try:
                from oracle import contract, metrics
                from oracle.plan import load
                from workload import make_plans as MP
                sub = MP.sub_slice(plan_json, args.oracle_log2)
                ref = contract.contract(load(sub), 0)
                sp = sub["sparse_legs"]
                rest = [l for l in sub["open"] if l not in sp]
                blocks = np.transpose(ref, [sub["open"].index(l) for l in sp + rest]).reshape(2 ** len(sp), -1)
                q = tn.Plan(sub, tn.make_config(dtype=tn.TN_CHALF, stem_min_log2=min(20, args.oracle_log2 - 4)))
                qb = tn.Buffers(q)
                tn.tn_plan_upload(q, qb)
                tn.tn_stem_contract(q, qb, 0)
                few = pre[:64]
                got, _ = tn.tn_sample_sparse(q, qb, few, k=1)
                line["parity"] = {"rel_l2_vs_oracle": metrics.rel_l2(got, blocks[few.astype(np.int64)]), "bound": 2e-2,
                                  "sample": f"64 subspaces of slice 0 of the plan sub-sliced to 2^{args.oracle_log2}"}
            except Exception as e:
                line["parity"] = {"error": str(e)}
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--plan", default="c3")
    ap.add_argument("--oracle-log2", type=int, default=26)
    ap.add_argument("--ref-log2", type=int, default=24, help="--impl reference: oracle sample per step")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--replicas", action="store_true", help="N>1: independent slices per GPU (weak scaling)")
    ap.add_argument("--comm", default="int8", choices=["int8", "int4", "fp16", "int8_tensor"])
    ap.add_argument("--policy", type=int, default=-1, help="layout policy (tn.h); -1: the plan's default")
    ap.add_argument("--subspaces", type=int, default=1024, help="sparse-state plans: correlated subspaces")
    ap.add_argument("--quant-from-pct", type=int, default=-1, help="sharded: quantise swaps from this %% of the path")
    ap.add_argument("--seed", type=int, default=0)
    args = ap.parse_args()

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    with open(os.path.join(ROOT, "plans", f"{args.plan}.json")) as f:
        plan_json = json.load(f)

    if args.impl == "reference":
        if rank != 0:
            return
        # each step a bounded sample (the 2^24 sub-slice, ~4 s of host time), so K + W steps fit in
        # a few minutes; the GPU line's cpu_baseline times the larger 2^26 sample once
        sub = oracle_sample(plan_json, args.ref_log2)
        fl, t = run_oracle(sub, args.steps, args.warmup)
        line = {"metric": METRIC, "value": fl / t / 1e12, "unit": "TFLOPS", "n_gpus": args.gpus, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": t * 1e3, "higher_is_better": True, "scaling": "weak",
                "vs_baseline": None, "dtype": "c128", "data": "synthetic", "impl": "reference",
                "config": {"workload": WORKLOADS.get(args.plan, args.plan), "plan": f"plans/{args.plan}.json",
                           "sample": f"sub-sliced to 2^{args.ref_log2}"},
                "cpu_baseline": {"value": fl / t / 1e12, "unit": "TFLOPS", "cores": _CORES, "kind": "oracle",
                                 "sample": f"slice 0 of plans/{args.plan}.json sub-sliced so every intermediate "
                                           f"<= 2^{args.ref_log2}; {fl:.3e} flops"},
                "e2e": {"value": fl / t / 1e12, "unit": "TFLOPS", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
        print(json.dumps(line), flush=True)
        return

    import torch
    import torch.distributed as dist
    from paper_2407_00769_b200 import build as B
    B.build()
    from paper_2407_00769_b200 import tn

    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev_stream = torch.cuda.current_stream()

    if plan_json.get("sparse_legs"):
        return bench_sparse(args, plan_json, tn, torch, dist, world, rank, local)
    sharded = world > 1 and not args.replicas
    comm = tn.Comm(rank, world, local) if sharded else None
    codec = {"int8": tn.TN_COMM_INT8, "int4": tn.TN_COMM_INT4, "int8_tensor": tn.TN_COMM_INT8_TENSOR}.get(
        args.comm, tn.TN_COMM_FP16)
    policy = args.policy if args.policy >= 0 else DEFAULT_POLICY.get(args.plan, POLICY_FALLBACK)
    p = tn.Plan(plan_json, tn.make_config(dtype=tn.TN_CHALF, stem_min_log2=20, comm_codec=codec,
                                          layout_policy=policy, quant_from_pct=args.quant_from_pct), comm=comm)
    info = p.info()
    bufs = tn.Buffers(p)
    n_sl = min(info["n_slices_log2"], 63)
    slice_id = 0 if sharded else (rank % (1 << n_sl) if n_sl else 0)
    tn.tn_plan_upload(p, bufs)

    def step():
        tn.tn_stem_contract(p, bufs, slice_id)
        tn.tn_split_contract(p, bufs)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    p.set_timing(True)
    clk = Clocks(local)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    nrg = Energy(local)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(dev_stream)
    ms_sum = None
    for _ in range(args.steps):
        step()
        # per-phase CUDA events of this step (recorded by the library inside its graph on this stream);
        # reading them waits for the step's last event: one short host sync per step
        msk = p.report().get("ms", [])
        ms_sum = msk if ms_sum is None else [a + b for a, b in zip(ms_sum, msk)]
    e1.record(dev_stream)
    torch.cuda.synchronize()
    watts = nrg.stop()
    if world > 1:
        dist.barrier()
    clocks = clk.stop()
    if world > 1 and watts is not None:  # whole-job power: sum over ranks
        wt = torch.tensor([watts], device="cuda", dtype=torch.float64)
        dist.all_reduce(wt, op=dist.ReduceOp.SUM)
        watts = float(wt.item())
    t_ms = e0.elapsed_time(e1) / args.steps
    rep = p.report()
    launches = p.info()["n_launches"] * args.steps
    p.set_timing(False)
    if world > 1:
        tt = torch.tensor([t_ms], device="cuda")
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        t_ms = float(tt.item())

    # ---- end to end through the public API with host buffers (H2D leaves, D2H amplitudes)
    for _ in range(2):
        tn.contract(p, bufs, slice_id)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        tn.contract(p, bufs, slice_id)
    torch.cuda.synchronize()
    te_ms = (time.perf_counter() - t0) * 1e3 / args.steps
    if world > 1:
        tt = torch.tensor([te_ms], device="cuda")
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        te_ms = float(tt.item())

    # ---- sharded with a codec: its error at full size against the same subtask with fp16 swaps
    comm_err = None
    if sharded and codec != tn.TN_COMM_FP16 and any(st.get("quant") for st in p.report()["steps"]):
        a_q = tn.contract(p, bufs, slice_id)
        p16 = tn.Plan(plan_json, tn.make_config(dtype=tn.TN_CHALF, stem_min_log2=20, comm_codec=tn.TN_COMM_FP16,
                                                layout_policy=policy), comm=comm)
        a_16 = tn.contract(p16, tn.Buffers(p16), slice_id)
        del p16
        import numpy as np
        comm_err = {"rel_l2_vs_fp16_swaps": float(np.linalg.norm(a_q - a_16) / np.linalg.norm(a_16)),
                    "quantised_swaps": sum(1 for st in p.report()["steps"] if st.get("quant")),
                    "note": "full-size subtask, same slice; fp16 swaps move bits (reading C-A32)"}

    # job flops: stem_flops is per rank (a shard does 1/N of the subtask's stem work when sharded;
    # a replica does a whole subtask)
    flops = info["stem_flops"] * world
    value = flops / (t_ms * 1e-3) / 1e12
    hbm, tc_burst, tc_sus, src = peaks()
    # the GEMMs run inside a step of hundreds of ms under the 1000 W cap: the SUSTAINED tensor peak
    # (MEASURED_PEAKS bf16_tflops_sustained, cuBLAS back to back for 4 s) is the roofline denominator
    # (B200_PROFILING: burst for a kernel timed alone, sustained inside a long step); burst reported beside
    tc_peak = tc_sus

    # ---- roofline of the dominant kernel (from the timed region's CUDA events, mean over the K steps)
    ms = [x / args.steps for x in ms_sum] if ms_sum else []
    steps = rep["steps"]
    gemm_ms = perm_ms = 0.0
    gemm_bytes = gemm_flops = t_roof_gemm = perm_bytes = 0.0
    eb = 4
    for i, st in enumerate(steps):
        M, K, N = 2.0 ** st["m"], 2.0 ** st["k"], 2.0 ** st["n"]
        pm, gm = ms[1 + 2 * i], ms[2 + 2 * i]
        perm_ms += pm
        gemm_ms += gm
        by = eb * (M * K + M * N) + 8 * K * N
        fl = 8 * M * K * N
        gemm_bytes += by
        gemm_flops += fl
        t_roof_gemm += max(by / (hbm * 1e9), fl / (tc_peak * 1e12)) * 1e3
        if st.get("pass", st["perm"]):  # (an MN-major step has perm = 1 but runs no pass)
            perm_bytes += 2 * eb * M * K
    final_ms = ms[-1] if ms else 0.0
    if rep.get("final_layout") and final_ms > 0:
        perm_ms += final_ms
        perm_bytes += 2 * eb * 2.0 ** len(rep["final_layout"])
    common_ms = ms[0] if ms else 0.0
    # per GEMM kernel (the library reports which kernel each step ran: "tc2" CTA-pair tcgen05,
    # "tc2_mn" its MN-major form, "tc1" single-CTA tcgen05, "simt", "c64"); the dominant one is the
    # kernel with the most step time.  The GEMM family as a whole is kept beside it.
    fam = {}
    for i, st in enumerate(steps):
        k = st.get("kern") or "gemm"
        k = "gemm_chalf_tc2" if k.startswith("tc2") else {"tc1": "gemm_chalf_tc", "simt": "gemm_chalf_rows",
                                                          "c64": "gemm_c64"}.get(k, k)
        M, K, N = 2.0 ** st["m"], 2.0 ** st["k"], 2.0 ** st["n"]
        f = fam.setdefault(k, {"ms": 0.0, "flops": 0.0, "bytes": 0.0, "launches": 0})
        f["ms"] += ms[2 + 2 * i]
        f["flops"] += 8 * M * K * N
        f["bytes"] += eb * (M * K + M * N) + 8 * K * N
        f["launches"] += 1

    def roof_of(name, ms_, flops_, bytes_):
        if bytes_ / (hbm * 1e9) >= flops_ / (tc_peak * 1e12):
            ach = bytes_ / (ms_ * 1e-3) / 1e9
            return {"kernel": name, "bound": "hbm", "achieved": ach, "peak": hbm, "unit": "GB/s", "frac": ach / hbm}
        ach = flops_ / (ms_ * 1e-3) / 1e12
        return {"kernel": name, "bound": "tensor", "achieved": ach, "peak": tc_peak, "unit": "TFLOP/s",
                "frac": ach / tc_peak, "peak_kind": "sustained (kernel inside a long step)", "peak_burst": tc_burst,
                "frac_burst": ach / tc_burst, "peak_spec": 2250.0, "frac_spec": ach / 2250.0}

    if gemm_ms >= perm_ms:
        dom = max(fam, key=lambda k: fam[k]["ms"])
        d = fam[dom]
        roof = roof_of(dom, d["ms"], d["flops"], d["bytes"])
        roof["launches_per_step"] = d["launches"]
        roof["share_of_gemm_time"] = d["ms"] / gemm_ms if gemm_ms else None
        roof["gemm_family"] = roof_of("all stem GEMMs", gemm_ms, gemm_flops, gemm_bytes)
        roof["gemm_family"]["roofline_time_frac"] = t_roof_gemm / gemm_ms if gemm_ms else None
        roof["per_kernel_ms"] = {k: round(v["ms"], 3) for k, v in sorted(fam.items(), key=lambda x: -x[1]["ms"])}
    else:
        ach = perm_bytes / (perm_ms * 1e-3) / 1e9
        roof = {"kernel": "permute", "bound": "hbm", "achieved": ach, "peak": hbm, "unit": "GB/s", "frac": ach / hbm}
    roof["peak_source"] = src
    # traffic: DRAM bytes (dram__bytes_read + dram__bytes_write) of the same kernel family per
    # subtask, from the committed ncu launch list of this command (profiles/, C3 single GPU only)
    roof["traffic"] = None
    roof["algorithmic_bytes"] = fam[roof["kernel"]]["bytes"] if roof["kernel"] in fam else gemm_bytes
    summ_name = {"c3": "r02_launches_summary.json", "c3_sweep": "r01_launches_summary.json"}.get(args.plan)
    summ = os.path.join(ROOT, "profiles", summ_name) if summ_name else ""
    if roof["kernel"].startswith("gemm") and world == 1 and summ and os.path.exists(summ):
        with open(summ) as fh:
            ps = json.load(fh)["per_subtask"]
        # ncu families (tools/ncu_summary.py): gemm_tc2 = the CTA-pair kernel (both forms)
        key = {"gemm_chalf_tc2": "gemm_tc2", "gemm_chalf_tc": "gemm_tc", "gemm_chalf_rows": "gemm_simt"}.get(roof["kernel"])
        if key in ps:
            roof["traffic"] = ps[key]["dram_bytes"]
            roof["traffic_source"] = f"profiles/{summ_name} (ncu, DRAM bytes per subtask of this kernel's launches)"
    roof["share_of_step"] = {"gemm": gemm_ms / t_ms, "permute": perm_ms / t_ms, "common+prep": common_ms / t_ms}
    # path roofline: sum over stem steps of max(F/P, B_alg/BW) over the measured step
    # time, and the step-shape histogram (log2 K*N -> steps) of the plan
    t_roof_path = 0.0
    shape_hist = {}
    for st in steps:
        M, K, N = 2.0 ** st["m"], 2.0 ** st["k"], 2.0 ** st["n"]
        t_roof_path += max(8 * M * K * N / (tc_peak * 1e12), (4 * (M * K + M * N) + 8 * K * N) / (hbm * 1e9)) * 1e3
        kn = st["k"] + st["n"]
        shape_hist[kn] = shape_hist.get(kn, 0) + 1
    path_roof = {"roofline_ms": t_roof_path, "frac": t_roof_path / t_ms,
                 "peaks": f"{tc_peak:.0f} TF/s sustained, {hbm:.0f} GB/s ({src})",
                 "log2_KN_histogram": {str(k): shape_hist[k] for k in sorted(shape_hist)},
                 "tensor_bound_steps": sum(1 for st in steps if 2 * 2.0 ** (st["k"] + st["n"]) /
                                           (2.0 ** st["k"] + 2.0 ** st["n"]) > tc_peak * 1e3 / hbm)}

    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": "TFLOPS", "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": t_ms, "higher_is_better": True,
                "scaling": "strong" if (sharded or world == 1) else "weak",
                "vs_baseline": None, "dtype": "f16", "data": "synthetic",
                "config": {"workload": WORKLOADS.get(args.plan, args.plan), "plan": f"plans/{args.plan}.json",
                           "slice": ("slice 0 sharded over all ranks (C4), swaps: " + args.comm) if sharded else
                                    "rank r runs slice r (replicas over independent subtasks)",
                           "mode_swaps": rep.get("n_swaps", 0), "epilogue_swaps": rep.get("n_fused_swaps", 0), "swap_bytes_per_rank": rep.get("swap_bytes", 0),
                           "stem_steps": info["n_stem_steps"], "permutes": info["n_permutes"],
                           "max_stem_log2": info["max_stem_log2"], "stem_flops": flops,
                           "layout_policy": policy,
                           "l2": f"inputs larger than L2 (stem tensors up to {info['stem_bytes'] / 2**30:.0f} GiB "
                                 f">> 126 MB)"},
                "tflops_per_gpu": value / world, "subtask_ms": t_ms,
                "breakdown_ms": {"common+prep": common_ms, "permute": perm_ms, "gemm": gemm_ms},
                "roofline": roof, "path_roofline": path_roof,
                "e2e": {"value": flops / (te_ms * 1e-3) / 1e12, "unit": "TFLOPS",
                        "ms_per_step": te_ms, "h2d_bytes_per_step": info["h2d_bytes"],
                        "d2h_bytes_per_step": (4 << info["n_open"]) + 4 * (2 * info["n_stem_steps"] + 4)},
                "gpu_launches": launches, "clocks": clocks, "comm_error": comm_err,
                "energy": None if watts is None else
                {"joules_per_step": watts * t_ms * 1e-3, "wh_per_step": watts * t_ms * 1e-3 / 3600.0,
                 "mean_board_w_per_gpu": watts / world,
                 "source": "nvmlDeviceGetTotalEnergyConsumption delta / wall time over the timed region "
                           "(summed over ranks) x device ms_per_step",
                 "note": "context only (SURVEY 8(f) #4); a step = one subtask (sharded) or one per rank"}}
        if world == 1 and not args.no_cpu:
            try:
                line["cpu_baseline"], sub = cpu_baseline(plan_json, args.oracle_log2)
                line["parity"] = parity(tn, sub, dict(dtype=tn.TN_CHALF, stem_min_log2=min(20, args.oracle_log2 - 4),
                                                      layout_policy=policy))
            except Exception as e:  # the oracle must not take the GPU number down with it
                line.setdefault("cpu_baseline", {"error": str(e)})
                line["parity"] = {"error": str(e)}
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
