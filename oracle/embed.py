"""Eq. 6 complex-as-real einsum (§3.3), float64.

Eq. 5/6: append the re/im mode alpha_{N_A+1} to A (its interleaved real view) and pad B from
[B(real, imag)] to [B(real,-imag), B(imag, real)] with a new leading mode gamma_{N_C+1}:
    alpha_1..alpha_NA alpha_{NA+1}, gamma_{NC+1} beta_1..beta_NB alpha_{NA+1} -> gamma_1..gamma_NC gamma_{NC+1}
Reading C-A6: B_P[c, beta..., a]; c=0 -> (Re b, -Im b), c=1 -> (Im b, Re b); the output's trailing
gamma_{NC+1} is (re, im).  Pinned by the paper's worked example.
"""
import numpy as np


def pad_b(b):
    """B_P[c, beta..., a] per Eq. 6 (C-A6)."""
    b = np.asarray(b, dtype=np.complex128)
    bp = np.empty((2,) + b.shape + (2,), dtype=np.float64)
    bp[0, ..., 0] = b.real
    bp[0, ..., 1] = -b.imag
    bp[1, ..., 0] = b.imag
    bp[1, ..., 1] = b.real
    return bp


def real_view(a):
    """A's interleaved real view with trailing mode alpha_{N_A+1} = (re, im)."""
    a = np.asarray(a, dtype=np.complex128)
    return np.stack([a.real, a.imag], axis=-1)


def einsum_complex_as_real(spec, a_real, b_padded):
    """Run Eq. 6 as one real einsum.  ``spec`` is the complex equation 'A,B->C' written with
    single letters; the re/im letters 'Z' (alpha_{N_A+1}) and 'Y' (gamma_{N_C+1}) are appended."""
    lhs, out = spec.split("->")
    sa, sb = lhs.split(",")
    real_spec = f"{sa}Z,Y{sb}Z->{out}Y"
    return np.einsum(real_spec, a_real, b_padded)


def cgemm_real(a_real_mk2, bp):
    """The GEMM form used on the stem: A real [M, 2K] (interleaved), B_P real [2K, 2N] with
    row (k,a), column (n,c) -> C real [M, 2N] interleaved.  ``bp`` is pad_b(B[K,N]) i.e.
    [c, k, n, a]; it is rearranged to [(k,a),(n,c)] by its definition."""
    c, k, n, a = bp.shape
    b2 = np.transpose(bp, (1, 3, 2, 0)).reshape(k * a, n * c)
    return a_real_mk2 @ b2
