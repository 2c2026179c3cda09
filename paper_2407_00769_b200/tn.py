"""Thin ctypes binding of libtn.so (include/tn.h).  Argument marshalling only: every step of the
contraction runs in the library's CUDA kernels.  PyTorch supplies device memory and streams.

There is no CPU fallback: if libtn.so is missing or a call fails, a TnError is raised.
"""
from __future__ import annotations

import ctypes as C
import json
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libtn.so")

TN_CHALF, TN_CFLOAT = 0, 1
TN_COMM_FP16, TN_COMM_INT8, TN_COMM_INT4, TN_COMM_INT8_TENSOR = 0, 1, 2, 3
ERRORS = {0: "TN_OK", -1: "TN_E_INVALID", -2: "TN_E_PARSE", -3: "TN_E_INFEASIBLE", -4: "TN_E_CAPACITY",
          -5: "TN_E_CUDA", -6: "TN_E_NCCL", -7: "TN_E_UNSUPPORTED"}


class TnError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"{ERRORS.get(code, code)}: {msg}")
        self.code = code


class tn_config(C.Structure):
    _fields_ = [("dtype", C.c_int32), ("stem_min_log2", C.c_int32), ("comm_codec", C.c_int32),
                ("comm_group", C.c_int32), ("stem_capacity_bytes", C.c_uint64), ("split_log2", C.c_int32),
                ("layout_policy", C.c_int32), ("quant_from_pct", C.c_int32), ("virtual_world", C.c_int32),
                ("no_gather", C.c_int32), ("no_fuse_swap_quant", C.c_int32), ("recompute", C.c_int32),
                ("no_fused_swap", C.c_int32)]


class tn_buffers(C.Structure):
    _fields_ = [("d_stem", C.c_void_p * 2), ("stem_bytes", C.c_uint64), ("d_ws", C.c_void_p),
                ("ws_bytes", C.c_uint64)]


class tn_plan_info(C.Structure):
    _fields_ = [("ws_bytes", C.c_uint64), ("stem_bytes", C.c_uint64), ("n_slices_log2", C.c_uint64),
                ("n_stem_steps", C.c_uint64), ("n_permutes", C.c_uint64), ("n_common", C.c_uint64),
                ("stem_flops", C.c_double), ("total_flops", C.c_double), ("stem_bytes_alg", C.c_double),
                ("perm_bytes", C.c_double), ("n_open", C.c_uint64), ("max_stem_log2", C.c_uint64),
                ("h2d_bytes", C.c_uint64), ("split_chunks", C.c_uint64), ("n_launches", C.c_uint64),
                ("n_sparse_legs", C.c_uint64)]


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise TnError(-5, f"{LIB_PATH} not built (run __graft_entry__.build())")
        L = C.CDLL(LIB_PATH)
        vp, u64, i32 = C.c_void_p, C.c_uint64, C.c_int
        L.tn_last_error.restype = C.c_char_p
        L.tn_set_device.argtypes = [C.c_int]
        L.tn_plan_load.argtypes = [C.c_char_p, C.c_size_t, C.POINTER(tn_config), vp, C.POINTER(vp)]
        L.tn_plan_info_get.argtypes = [vp, C.POINTER(tn_plan_info)]
        L.tn_plan_free.argtypes = [vp]
        L.tn_plan_free.restype = None
        L.tn_plan_upload.argtypes = [vp, C.POINTER(tn_buffers), vp]
        L.tn_stem_contract.argtypes = [vp, C.POINTER(tn_buffers), u64, vp]
        L.tn_split_contract.argtypes = [vp, C.POINTER(tn_buffers), vp]
        L.tn_sample_amplitudes.argtypes = [vp, C.POINTER(tn_buffers), vp, C.c_size_t, vp, i32, vp, vp]
        L.tn_report_json.argtypes = [vp, C.c_char_p, C.c_size_t, C.POINTER(C.c_size_t)]
        L.tn_set_timing.argtypes = [vp, i32]
        L.tn_set_graph.argtypes = [vp, i32]
        L.tn_permute.argtypes = [vp, vp, i32, i32, C.POINTER(C.c_int), vp]
        L.tn_gemm_chalf.argtypes = [vp, vp, vp, u64, C.c_uint32, C.c_uint32, vp, vp, vp, vp, vp]
        L.tn_gemm_chalf_gather.argtypes = [vp, vp, vp, i32, i32, C.c_uint32, C.POINTER(C.c_int64),
                                           C.POINTER(C.c_int64), vp, vp, vp, vp, vp]
        L.tn_gemm_cfloat.argtypes = [vp, vp, vp, u64, C.c_uint32, C.c_uint32, vp]
        L.tn_gemm_chalf_batched.argtypes = [vp, vp, vp, u64, C.c_uint32, C.c_uint32, u64, vp, vp, u64, u64,
                                            vp, vp, vp, vp, vp]
        L.tn_gemm_chalf_padded.argtypes = [vp, vp, vp, u64, C.c_uint32, C.c_uint32, u64, vp, i32, u64,
                                           vp, vp, vp, vp, vp]
        L.tn_pad_b.argtypes = [vp, vp, C.c_uint32, C.c_uint32, vp, vp, vp, vp]
        L.tn_pad_b_mn.argtypes = [vp, vp, C.c_uint32, C.c_uint32, vp, vp, vp, vp]
        L.tn_gemm_chalf_mn.argtypes = [vp, vp, vp, u64, C.c_uint32, C.c_uint32, i32, vp, vp, vp, vp, vp]
        L.tn_quant_int8.argtypes = [vp, vp, vp, vp, u64, i32, vp]
        L.tn_dequant_int8.argtypes = [vp, vp, vp, vp, u64, i32, vp]
        L.tn_quant_int8_f16.argtypes = [vp, vp, vp, vp, u64, i32, vp]
        L.tn_dequant_int8_f16.argtypes = [vp, vp, vp, vp, u64, i32, vp]
        L.tn_quant_int4_f16.argtypes = [vp, vp, vp, vp, u64, i32, vp]
        L.tn_permute_quant_f16.argtypes = [vp, vp, vp, vp, i32, vp, i32, i32, vp]
        L.tn_dequant_int4_f16.argtypes = [vp, vp, vp, vp, u64, i32, vp]
        L.tn_quant_int8_exp_f16.argtypes = [vp, vp, vp, vp, u64, u64, C.c_double, vp, vp]
        L.tn_dequant_int8_exp_f16.argtypes = [vp, vp, vp, vp, u64, u64, C.c_double, vp]
        L.tn_comm_unique_id.argtypes = [vp]
        L.tn_comm_init.argtypes = [vp, i32, i32, i32, C.POINTER(vp)]
        L.tn_comm_init_loopback.argtypes = [i32, i32, vp]
        L.tn_comm_free.argtypes = [vp]
        L.tn_comm_free.restype = None
        _lib = L
    return _lib


def set_device(device=None):
    """Make libtn's CUDA runtime use torch's current device (or `device`)."""
    try:
        import torch
        if device is None:
            if not torch.cuda.is_available():
                return
            device = torch.cuda.current_device()
    except ImportError:
        return
    _check(lib().tn_set_device(int(device)))


def _check(code):
    if code != 0:
        raise TnError(code, lib().tn_last_error().decode(errors="replace"))


def _ptr(t):
    return None if t is None else C.c_void_p(t.data_ptr())


def _stream(stream):
    import torch
    s = stream if stream is not None else torch.cuda.current_stream()
    return C.c_void_p(s.cuda_stream)


def make_config(dtype=TN_CHALF, stem_min_log2=20, comm_codec=TN_COMM_INT8, comm_group=128,
                stem_capacity_bytes=0, split_log2=0, layout_policy=3, virtual_world=1, quant_from_pct=-1,
                no_gather=0, no_fuse_swap_quant=0, recompute=0, no_fused_swap=0):
    c = tn_config()
    c.no_fused_swap = no_fused_swap
    c.recompute = recompute
    c.no_gather = no_gather
    c.no_fuse_swap_quant = no_fuse_swap_quant
    c.layout_policy = layout_policy
    c.virtual_world = virtual_world  # host-only lowering for several ranks (no communicator)
    c.quant_from_pct = quant_from_pct
    c.dtype, c.stem_min_log2, c.comm_codec, c.comm_group = dtype, stem_min_log2, comm_codec, comm_group
    c.stem_capacity_bytes, c.split_log2 = stem_capacity_bytes, split_log2
    return c


class Plan:
    """tn_plan_load / tn_plan_info_get / tn_plan_free."""

    def __init__(self, plan, cfg=None, comm=None):
        if isinstance(plan, dict):
            plan = json.dumps(plan)
        if isinstance(plan, str) and not plan.lstrip().startswith("{"):
            with open(plan) as f:
                plan = f.read()
        data = plan.encode() if isinstance(plan, str) else plan
        self._h = C.c_void_p()
        self.cfg = cfg or make_config()
        self.comm = comm  # keep the communicator alive as long as the plan
        set_device()
        _check(lib().tn_plan_load(data, len(data), C.byref(self.cfg), comm.handle if comm is not None else None,
                                  C.byref(self._h)))

    def __del__(self):
        if getattr(self, "_h", None) and _lib is not None:
            _lib.tn_plan_free(self._h)
            self._h = None

    def info(self):
        i = tn_plan_info()
        _check(lib().tn_plan_info_get(self._h, C.byref(i)))
        return {k: getattr(i, k) for k, _ in tn_plan_info._fields_}

    def report(self):
        need = C.c_size_t(0)
        _check(lib().tn_report_json(self._h, None, 0, C.byref(need)))
        buf = C.create_string_buffer(need.value)
        _check(lib().tn_report_json(self._h, buf, need.value, C.byref(need)))
        return json.loads(buf.value.decode())

    def set_timing(self, on=True):
        _check(lib().tn_set_timing(self._h, 1 if on else 0))

    def set_graph(self, on=True):
        _check(lib().tn_set_graph(self._h, 1 if on else 0))


class Buffers:
    """Caller-owned device buffers (torch.empty uint8) lent to the library."""

    def __init__(self, plan: Plan, device="cuda", stem_bytes=None):
        import torch
        info = plan.info()
        sb = max(stem_bytes or info["stem_bytes"], 256)
        self.stem = [torch.empty(sb, dtype=torch.uint8, device=device) for _ in range(2)]
        self.ws = torch.empty(max(info["ws_bytes"], 256), dtype=torch.uint8, device=device)
        self.c = tn_buffers()
        self.c.d_stem[0] = self.stem[0].data_ptr()
        self.c.d_stem[1] = self.stem[1].data_ptr()
        self.c.stem_bytes = sb
        self.c.d_ws = self.ws.data_ptr()
        self.c.ws_bytes = self.ws.numel()


def tn_plan_upload(plan, bufs, stream=None):
    _check(lib().tn_plan_upload(plan._h, C.byref(bufs.c), _stream(stream)))


def tn_stem_contract(plan, bufs, slice_id=0, stream=None):
    _check(lib().tn_stem_contract(plan._h, C.byref(bufs.c), slice_id, _stream(stream)))


def tn_split_contract(plan, bufs, stream=None):
    _check(lib().tn_split_contract(plan._h, C.byref(bufs.c), _stream(stream)))


def tn_sample_amplitudes(plan, bufs, k=0, stream=None):
    """Returns (complex128 numpy array over the open legs, top-k indices or None)."""
    import numpy as np
    n_open = plan.info()["n_open"]
    out = np.empty(2 << n_open, dtype=np.float64)
    top = np.empty(max(k, 1), dtype=np.uint64)
    _check(lib().tn_sample_amplitudes(plan._h, C.byref(bufs.c), None, 0, out.ctypes.data, k,
                                      top.ctypes.data if k > 0 else None, _stream(stream)))
    amps = (out[0::2] + 1j * out[1::2]).reshape((2,) * n_open)
    return amps, (top[:k].copy() if k > 0 else None)


def tn_sample_sparse(plan, bufs, prefixes, k=1, stream=None):
    """Sparse-state batch: amplitudes of the correlated subspaces `prefixes` (values of the split
    legs) and the post-selected member of each.  Returns (complex128 [n_sub, members], top [n_sub, k])."""
    import numpy as np
    info = plan.info()
    # sparse-state plan: subspaces are values of the sparse legs; split plan: values of the split legs
    j = info["n_sparse_legs"] or int(np.log2(info["split_chunks"]))
    members = 1 << (info["n_open"] - j)
    pre = np.ascontiguousarray(np.asarray(prefixes, dtype=np.uint64))
    out = np.empty(2 * len(pre) * members, dtype=np.float64)
    top = np.empty(max(1, len(pre) * max(k, 1)), dtype=np.uint64)
    _check(lib().tn_sample_amplitudes(plan._h, C.byref(bufs.c), pre.ctypes.data, len(pre), out.ctypes.data, k,
                                      top.ctypes.data if k > 0 else None, _stream(stream)))
    amps = (out[0::2] + 1j * out[1::2]).reshape(len(pre), members)
    return amps, (top[:len(pre) * k].reshape(len(pre), k) if k > 0 else None)


def contract(plan, bufs, slice_id=0, stream=None, upload=True):
    """Public one-call API: upload leaves, contract one slice, read the amplitudes."""
    if upload:
        tn_plan_upload(plan, bufs, stream)
    tn_stem_contract(plan, bufs, slice_id, stream)
    tn_split_contract(plan, bufs, stream)
    return tn_sample_amplitudes(plan, bufs, 0, stream)[0]


# ---- kernel-level entry points ----
def tn_permute(dst, src, perm, stream=None):
    n = len(perm)
    arr = (C.c_int * max(n, 1))(*perm)
    eb = src.element_size() * (2 if src.is_complex() else 1)
    if src.dtype.is_complex:
        eb = src.element_size()
    _check(lib().tn_permute(_ptr(dst), _ptr(src), eb, n, arr, _stream(stream)))


def tn_permute_bytes(dst, src, elem_bytes, perm, stream=None):
    n = len(perm)
    arr = (C.c_int * max(n, 1))(*perm)
    _check(lib().tn_permute(_ptr(dst), _ptr(src), elem_bytes, n, arr, _stream(stream)))


def tn_gemm_chalf(c, a, bp, M, K, N, in_max=None, b_bound=None, out_max=None, exp=None, stream=None):
    _check(lib().tn_gemm_chalf(_ptr(c), _ptr(a), _ptr(bp), M, K, N, _ptr(in_max), _ptr(b_bound),
                               _ptr(out_max), _ptr(exp), _stream(stream)))


def tn_gemm_chalf_gather(c, a, bp, mlog, klog, N, m_stride, k_stride, in_max=None, b_bound=None, out_max=None,
                         exp=None, stream=None):
    ms = (C.c_int64 * max(len(m_stride), 1))(*m_stride)
    ks = (C.c_int64 * max(len(k_stride), 1))(*k_stride)
    _check(lib().tn_gemm_chalf_gather(_ptr(c), _ptr(a), _ptr(bp), mlog, klog, N, ms, ks, _ptr(in_max),
                                      _ptr(b_bound), _ptr(out_max), _ptr(exp), _stream(stream)))


def tn_gemm_chalf_batched(c, a, bp, M, K, N, index_a, index_b, n_a, n_b, in_max=None, b_bound=None, out_max=None,
                          exp=None, stream=None):
    """index_a / index_b: int32 CUDA tensors of n_out entries."""
    _check(lib().tn_gemm_chalf_batched(_ptr(c), _ptr(a), _ptr(bp), M, K, N, index_a.numel(), _ptr(index_a),
                                       _ptr(index_b), n_a, n_b, _ptr(in_max), _ptr(b_bound), _ptr(out_max),
                                       _ptr(exp), _stream(stream)))


def tn_gemm_chalf_padded(c, a, bp, M, K, N, table, n_b, in_max=None, b_bound=None, out_max=None, exp=None,
                         stream=None):
    """table: int32 CUDA tensor [n_a, m_r] (-1 = zero block)."""
    n_a, m_r = table.shape
    _check(lib().tn_gemm_chalf_padded(_ptr(c), _ptr(a), _ptr(bp), M, K, N, n_a, _ptr(table), m_r, n_b,
                                      _ptr(in_max), _ptr(b_bound), _ptr(out_max), _ptr(exp), _stream(stream)))


def tn_gemm_cfloat(c, a, b, M, K, N, stream=None):
    _check(lib().tn_gemm_cfloat(_ptr(c), _ptr(a), _ptr(b), M, K, N, _stream(stream)))


def tn_gemm_chalf_mn(c, a, bpm, M, K, N, ma, in_max=None, b_bound=None, out_max=None, exp=None, stream=None):
    _check(lib().tn_gemm_chalf_mn(_ptr(c), _ptr(a), _ptr(bpm), M, K, N, ma, _ptr(in_max), _ptr(b_bound),
                                  _ptr(out_max), _ptr(exp), _stream(stream)))


def tn_pad_b_mn(bpm, b, K, N, b_bound=None, exp=None, scratch=None, stream=None):
    _check(lib().tn_pad_b_mn(_ptr(bpm), _ptr(b), K, N, _ptr(b_bound), _ptr(exp), _ptr(scratch), _stream(stream)))


def tn_pad_b(bp, b, K, N, b_bound=None, exp=None, scratch=None, stream=None):
    _check(lib().tn_pad_b(_ptr(bp), _ptr(b), K, N, _ptr(b_bound), _ptr(exp), _ptr(scratch), _stream(stream)))


def tn_quant_int8(codes, scales, zeros, x, g, stream=None):
    _check(lib().tn_quant_int8(_ptr(codes), _ptr(scales), _ptr(zeros), _ptr(x), x.numel(), g, _stream(stream)))


def tn_quant_int8_f16(codes, scales, zeros, x, g, stream=None):
    _check(lib().tn_quant_int8_f16(_ptr(codes), _ptr(scales), _ptr(zeros), _ptr(x), x.numel(), g, _stream(stream)))


def tn_dequant_int8_f16(y, codes, scales, zeros, g, stream=None):
    _check(lib().tn_dequant_int8_f16(_ptr(y), _ptr(codes), _ptr(scales), _ptr(zeros), y.numel(), g, _stream(stream)))


def tn_permute_quant_f16(codes, scales, zeros, x, perm, g, codec=TN_COMM_INT8, stream=None):
    """x: complex-half stem as a tensor of 2^(n+1) fp16 reals; perm: tn_permute's axes."""
    n = len(perm)
    arr = (C.c_int * max(n, 1))(*perm)
    _check(lib().tn_permute_quant_f16(_ptr(codes), _ptr(scales), _ptr(zeros), _ptr(x), n, arr, g, codec,
                                      _stream(stream)))


def tn_quant_int8_exp_f16(codes, scales, zeros, x, g, e, tmp, stream=None):
    _check(lib().tn_quant_int8_exp_f16(_ptr(codes), _ptr(scales), _ptr(zeros), _ptr(x), x.numel(), g, e, _ptr(tmp),
                                       _stream(stream)))


def tn_dequant_int8_exp_f16(y, codes, scales, zeros, g, e, stream=None):
    _check(lib().tn_dequant_int8_exp_f16(_ptr(y), _ptr(codes), _ptr(scales), _ptr(zeros), y.numel(), g, e,
                                         _stream(stream)))


def tn_quant_int4_f16(packed, scales, zeros, x, g, stream=None):
    _check(lib().tn_quant_int4_f16(_ptr(packed), _ptr(scales), _ptr(zeros), _ptr(x), x.numel(), g, _stream(stream)))


def tn_dequant_int4_f16(y, packed, scales, zeros, g, stream=None):
    _check(lib().tn_dequant_int4_f16(_ptr(y), _ptr(packed), _ptr(scales), _ptr(zeros), y.numel(), g, _stream(stream)))


def tn_dequant_int8(y, codes, scales, zeros, g, stream=None):
    _check(lib().tn_dequant_int8(_ptr(y), _ptr(codes), _ptr(scales), _ptr(zeros), y.numel(), g, _stream(stream)))


class Comm:
    """tn_comm_unique_id / tn_comm_init / tn_comm_free.  The library owns its NCCL communicator;
    torch.distributed (already initialised) only broadcasts the unique id."""

    def __init__(self, rank, world, device):
        import torch.distributed as dist
        L = lib()
        uid = (C.c_uint8 * 128)()
        obj = [None]
        if rank == 0:
            _check(L.tn_comm_unique_id(uid))
            obj = [bytes(uid)]
        if world > 1:
            dist.broadcast_object_list(obj, src=0)
        uid = (C.c_uint8 * 128)(*obj[0])
        self._h = C.c_void_p()
        _check(L.tn_comm_init(uid, rank, world, device, C.byref(self._h)))
        self.rank, self.world = rank, world

    @property
    def handle(self):
        return self._h

    def __del__(self):
        if getattr(self, "_h", None) and _lib is not None:
            _lib.tn_comm_free(self._h)
            self._h = None


class LoopbackComm:
    """tn_comm_init_loopback: `world` virtual ranks on one device (include/tn.h).  Drive each
    rank's plan from its own thread (see run_ranks)."""

    def __init__(self, world, device=0):
        arr = (C.c_void_p * world)()
        _check(lib().tn_comm_init_loopback(world, device, arr))
        self._h = [C.c_void_p(arr[r]) for r in range(world)]
        self.world = world
        self.ranks = [_Rank(self, r) for r in range(world)]

    def __del__(self):
        if getattr(self, "_h", None) and _lib is not None:
            for h in self._h:
                _lib.tn_comm_free(h)
            self._h = None


class _Rank:
    def __init__(self, group, rank):
        self.group, self.rank, self.world = group, rank, group.world

    @property
    def handle(self):
        return self.group._h[self.rank]


def run_ranks(world, fn):
    """Run fn(rank) on `world` threads, one per virtual rank, each with its own CUDA stream;
    returns the per-rank results (re-raises the first exception)."""
    import threading
    import torch
    dev = torch.cuda.current_device()
    out, errs = [None] * world, [None] * world

    def body(r):
        try:
            torch.cuda.set_device(dev)
            with torch.cuda.stream(torch.cuda.Stream()):
                out[r] = fn(r)
                torch.cuda.current_stream().synchronize()
        except BaseException as e:  # noqa: BLE001
            errs[r] = e
    ts = [threading.Thread(target=body, args=(r,)) for r in range(world)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    for e in errs:
        if e is not None:
            raise e
    return out
