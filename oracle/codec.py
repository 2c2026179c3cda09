"""Group quantisation, Eq. 1 and Table 1; CR, Eq. "compress".

Eq. 1:  Q([T]_i) = [T]_i^exp * scale + zero,
        scale = (q_max - q_min) / (max[T]_i - min[T]_i),
        zero  = (q_min max[T]_i - q_max min[T]_i) / (max[T]_i - min[T]_i).
Readings:
* C-A10: x' = sign(x)|x|^exp; max/min are taken over x' (the literal text is inconsistent when
  exp != 1); dequant y' = (code - zero)/scale, y = sign(y')|y'|^(1/exp).
* C-A11: a constant group (max == min) is flagged by scale = 0 and stores the constant as
  zero = x'_c, codes = q_min; dequantisation returns zero when scale == 0 (exact round trip; the
  SPEC's two rules contradict each other and q_min - x'_c is not exact in fp32).
* C-A12: the build's primary codec is int8, per-block groups of g = 128 reals (64 complex,
  interleaved re/im), exp = 1, fp32 scale and zero; the Table-1 presets are also provided.
* C-A13: rounding = round-half-to-even; x'*scale + zero evaluated as an fp32 multiply followed by
  an fp32 add (no fused multiply-add), so the CUDA kernel's codes are bit-comparable.
* C-A14: int4 codes packed two per byte, low nibble = even index.
Everything is float32 (the paper's payload precision), step by step.
"""
import numpy as np

F32 = np.float32

PRESETS = {  # Table 1: (q_min, q_max, exp, group, round)
    "half": (F32(-65504.0), F32(65504.0), 1.0, None, False),
    "int8": (F32(-128.0), F32(127.0), 0.2, None, True),
    "int4": (F32(0.0), F32(15.0), 1.0, 128, True),
    "int8_g128": (F32(-128.0), F32(127.0), 1.0, 128, True),   # build's primary (C-A12)
}


def _signed_pow(x, e):
    x = x.astype(F32)
    if e == 1.0:
        return x
    return (np.sign(x) * np.power(np.abs(x).astype(np.float64), e)).astype(F32)


def group_params(xp, qmin, qmax):
    """scale, zero of Eq. 1 for one group of transformed values xp (float32 arithmetic)."""
    mx = F32(np.max(xp))
    mn = F32(np.min(xp))
    if mx == mn:                       # C-A11
        return F32(0.0), F32(mx)
    den = F32(mx - mn)
    scale = F32(F32(qmax - qmin) / den)
    zero = F32(F32(F32(qmin * mx) - F32(qmax * mn)) / den)
    return scale, zero


def quantize(x, qmin, qmax, exp=1.0, group=None, round_=True):
    """x: flat float32 array.  Returns (codes float32 array, scales, zeros) per group.
    Groups are the rows of x reshaped to [n_groups, g]; every step is elementwise float32 in the
    order of Eq. 1 (max/min per row, then scale, zero, multiply, add, round, clip)."""
    x = np.asarray(x, dtype=F32).reshape(-1)
    g = x.size if group is None else group
    if x.size % g:
        raise ValueError("group size must divide the tensor")
    xp = _signed_pow(x, exp).reshape(-1, g)
    mx = xp.max(axis=1).astype(F32)
    mn = xp.min(axis=1).astype(F32)
    const = mx == mn                                   # degenerate groups (C-A11)
    den = np.where(const, F32(1.0), (mx - mn).astype(F32)).astype(F32)
    scales = (F32(qmax - qmin) / den).astype(F32)
    zeros = ((F32(qmin) * mx).astype(F32) - (F32(qmax) * mn).astype(F32)).astype(F32)
    zeros = (zeros / den).astype(F32)
    scales = np.where(const, F32(0.0), scales).astype(F32)
    zeros = np.where(const, mx, zeros).astype(F32)
    v = (xp * scales[:, None]).astype(F32)             # fp32 multiply (rounded)
    v = (v + zeros[:, None]).astype(F32)               # then fp32 add (rounded); no FMA (C-A13)
    if round_:
        v = np.rint(v)                                 # round half to even
    v = np.where(const[:, None], F32(qmin), v)
    codes = np.clip(v, qmin, qmax).astype(F32).reshape(-1)
    return codes, scales, zeros


def dequantize(codes, scales, zeros, exp=1.0, group=None):
    codes = np.asarray(codes, dtype=F32).reshape(-1)
    g = codes.size if group is None else group
    c = codes.reshape(-1, g)
    scales = np.asarray(scales, dtype=F32)
    zeros = np.asarray(zeros, dtype=F32)
    const = scales == 0                                # degenerate group (C-A11)
    den = np.where(const, F32(1.0), scales).astype(F32)
    y = ((c - zeros[:, None]).astype(F32) / den[:, None]).astype(F32)
    y = np.where(const[:, None], zeros[:, None], y).astype(F32)
    return _signed_pow(y.reshape(-1), 1.0 / exp)


def pack_int4(codes):
    """C-A14: two 4-bit codes per byte, low nibble = even index."""
    c = np.asarray(codes).astype(np.uint8).reshape(-1)
    return (c[0::2] & 0xF) | ((c[1::2] & 0xF) << 4)


def unpack_int4(packed):
    p = np.asarray(packed, dtype=np.uint8)
    out = np.empty(p.size * 2, dtype=np.uint8)
    out[0::2] = p & 0xF
    out[1::2] = p >> 4
    return out


def compression_rate(n_values, bits_per_code, n_groups, scale_bytes=4, zero_bytes=4,
                     orig_bytes_per_value=4):
    """Eq. "compress": (sizeof scales + sizeof zeros + sizeof quant) / sizeof original."""
    quant = n_values * bits_per_code / 8.0
    return (n_groups * scale_bytes + n_groups * zero_bytes + quant) / (n_values * orig_bytes_per_value)
