"""Build libtn.so in-tree with nvcc for sm_100a (no JIT cache; the .so travels with the repo)."""
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
OUT = os.path.join(HERE, "libtn.so")
SOURCES = ["plan.cpp", "k_permute.cu", "k_common.cu", "k_gemm_simt.cu", "k_gemm_tc.cu", "k_gemm_tc_m0.cu",
           "k_gemm_tc_m1.cu", "k_gemm_tc_m2.cu", "k_gemm_tc_m3.cu", "k_gemm_tc_m4.cu", "k_gemm_tc_m5.cu", "k_gemm_tc2.cu", "k_quant.cu", "k_select.cu", "runtime.cu"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = ["-O3", "-std=c++17", "-lineinfo", "-gencode", "arch=compute_100a,code=sm_100a",
         "-Xcompiler", "-fPIC", "-Xcompiler", "-fvisibility=hidden", "--expt-relaxed-constexpr"]


def _stale():
    if not os.path.exists(OUT):
        return True
    t = os.path.getmtime(OUT)
    for f in os.listdir(CSRC):
        if os.path.getmtime(os.path.join(CSRC, f)) > t:
            return True
    hdr = os.path.join(os.path.dirname(HERE), "include", "tn.h")
    return os.path.getmtime(hdr) > t


def _obj_stale(src, obj):
    """An object is rebuilt when its source or any header (csrc/*.cuh, *.hpp, include/tn.h) is newer."""
    if not os.path.exists(obj):
        return True
    t = os.path.getmtime(obj)
    hdrs = [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".cuh", ".hpp", ".h"))]
    hdrs.append(os.path.join(os.path.dirname(HERE), "include", "tn.h"))
    return any(os.path.getmtime(f) > t for f in [src] + hdrs)


def build(force=False, verbose=False):
    if not force and not _stale():
        return OUT
    objs = []
    os.makedirs(os.path.join(HERE, "build"), exist_ok=True)
    procs = []
    for s in SOURCES:
        src = os.path.join(CSRC, s)
        obj = os.path.join(HERE, "build", s + ".o")
        objs.append(obj)
        if not force and not _obj_stale(src, obj):
            continue
        cmd = [NVCC] + FLAGS + ["-c", src, "-o", obj]
        if s.endswith(".cpp"):
            cmd = [NVCC] + FLAGS + ["-x", "cu", "-c", src, "-o", obj]
        procs.append((s, subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT)))
    for s, p in procs:
        out, _ = p.communicate()
        if verbose or p.returncode:
            sys.stdout.write(out.decode())
        if p.returncode:
            raise RuntimeError(f"nvcc failed on {s}")
    link = [NVCC, "-shared", "-gencode", "arch=compute_100a,code=sm_100a", "-o", OUT] + objs + ["-ldl"]
    r = subprocess.run(link, stdout=subprocess.PIPE, stderr=subprocess.STDOUT)
    if r.returncode:
        sys.stdout.write(r.stdout.decode())
        raise RuntimeError("link failed")
    return OUT


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
