"""Kernel-level parity on a B200 through the C-ABI (libtn.so), against the oracle / exact
definitions.  Bit-exact for data movement and the codec; fp tolerances derived in DESIGN.md."""
import numpy as np
import pytest

from oracle import codec, embed

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def env():
    import torch
    from paper_2407_00769_b200 import build as B
    B.build()
    from paper_2407_00769_b200 import tn
    assert torch.cuda.is_available()
    return torch, tn


def _perm_ref_index(out_idx, perm, n):
    """source flat index of destination flat index under numpy transpose(perm) for dims 2"""
    src = 0
    for j in range(n):
        bit = (out_idx >> (n - 1 - j)) & 1
        src |= bit << (n - 1 - perm[j])
    return src


PERMS = {
    "identity": lambda n: list(range(n)),
    "reversal": lambda n: list(range(n))[::-1],
    "swap_last_first": lambda n: [n - 1] + list(range(1, n - 1)) + [0] if n > 1 else [0],
    "outer3_inner3": lambda n: (list(range(n - 3, n)) + list(range(3, n - 3)) + list(range(3))) if n >= 6 else list(range(n))[::-1],
    "bitrev_low8": lambda n: list(range(n - 8)) + list(range(n - 8, n))[::-1] if n >= 8 else list(range(n))[::-1],
}


@pytest.mark.parametrize("elem", [4, 8])
@pytest.mark.parametrize("n", [1, 3, 5, 7, 10, 13, 17, 22])
def test_permute_bit_exact(env, n, elem):
    torch, tn = env
    rng = np.random.default_rng(n * 10 + elem)
    perms = [f(n) for f in PERMS.values()] + [list(rng.permutation(n)) for _ in range(3)]
    x = rng.integers(0, 2 ** 31, size=(1 << n) * (elem // 4), dtype=np.int64).astype(np.int32)
    src = torch.from_numpy(x).cuda()
    ref_view = x.view(np.int32 if elem == 4 else np.int64).reshape((2,) * n) if n else x
    for perm in perms:
        dst = torch.empty_like(src)
        tn.tn_permute_bytes(dst, src, elem, [int(p) for p in perm])
        torch.cuda.synchronize()
        got = dst.cpu().numpy().view(np.int32 if elem == 4 else np.int64)
        exp = np.ascontiguousarray(np.transpose(ref_view, perm)).reshape(-1)
        assert np.array_equal(got, exp), perm


def test_permute_large_sampled_64bit_indexing(env):
    """2^32 complex-half elements (16 GiB): sampled outputs vs the index definition."""
    torch, tn = env
    n = 32
    free, _ = torch.cuda.mem_get_info()
    if free < 40 * 2 ** 30:
        pytest.skip("needs 40 GiB free")
    src = torch.arange(0, 1 << n, dtype=torch.int64, device="cuda").to(torch.int32)  # value = index (mod 2^32)
    dst = torch.empty_like(src)
    rng = np.random.default_rng(0)
    perm = [int(p) for p in rng.permutation(n)]
    tn.tn_permute_bytes(dst, src, 4, perm)
    torch.cuda.synchronize()
    idx = rng.integers(0, 1 << n, size=4096, dtype=np.int64)
    got = dst[torch.from_numpy(idx).cuda()].cpu().numpy().astype(np.int64) & 0xFFFFFFFF
    exp = np.array([_perm_ref_index(int(i), perm, n) for i in idx], dtype=np.int64) & 0xFFFFFFFF
    assert np.array_equal(got, exp)
    del src, dst
    torch.cuda.empty_cache()


def _half_pairs(z):
    return np.stack([z.real, z.imag], -1).astype(np.float16)


@pytest.mark.parametrize("M,K,N", [(1, 8, 8), (128, 8, 8), (300, 16, 8), (1000, 8, 32), (4096 + 37, 32, 64),
                                   (777, 64, 128), (2048, 128, 256), (513, 256, 16), (1024, 512, 512),
                                   (256, 2048, 8), (640, 8, 1024), (1000, 4, 64), (5000, 16, 4),
                                   (3000, 8, 2), (129, 4, 256), (4100, 16, 256),
                                   # CTA-pair kernel (M % 256 == 0, 2N >= 128, 2K >= 64): single k block,
                                   # BN = 128 and 256, more pair tiles than resident pairs
                                   (512, 32, 64), (256, 64, 128), (1536, 32, 512), (65536, 64, 128), (2048, 128, 64),
                                   (1024, 128, 32), (4096, 512, 32),
                                   (16384, 256, 256),
                                   # packed narrow rows (2N = 16 / 32 fp16 per row stored as 128-byte rows)
                                   (4096, 16, 16), (1024, 32, 8), (128, 4, 16)])
def test_gemm_chalf_tensor_core_vs_oracle(env, M, K, N):
    """tcgen05 Eq. 6 GEMM (no scaling) vs the oracle's real-embedding GEMM in fp64 on the same
    fp16 operands.  Error: one fp16 rounding of C (2^-11 relative) + fp32 accumulation."""
    torch, tn = env
    rng = np.random.default_rng(M + K * 7 + N * 13)
    a = (rng.standard_normal((M, K)) + 1j * rng.standard_normal((M, K))) / np.sqrt(2)
    b = (rng.standard_normal((K, N)) + 1j * rng.standard_normal((K, N))) / np.sqrt(2 * K)
    a16 = _half_pairs(a)                                   # [M, K, 2]
    b16 = b.real.astype(np.float16) + 1j * b.imag.astype(np.float16)
    bp = embed.pad_b(b16)                                   # [c, K, N, a] exact in fp16
    bp_km = np.transpose(bp, (2, 0, 1, 3)).reshape(2 * N, 2 * K).astype(np.float16)  # [(n,c), (k,a)]
    ref = embed.cgemm_real(a16.astype(np.float64).reshape(M, 2 * K), bp)            # [M, 2N]
    A = torch.from_numpy(a16.reshape(-1)).cuda()
    BP = torch.from_numpy(bp_km.reshape(-1)).cuda()
    Cc = torch.full((M * 2 * N,), float("nan"), dtype=torch.float16, device="cuda")
    tn.tn_gemm_chalf(Cc, A, BP, M, K, N)
    torch.cuda.synchronize()
    got = Cc.cpu().numpy().astype(np.float64).reshape(M, 2 * N)
    assert np.all(np.isfinite(got))
    err = np.abs(got - ref)
    tol = 2.0 ** -10 * np.abs(ref) + 1e-3 * np.sqrt(np.mean(ref ** 2)) + 1e-7
    assert np.all(err <= tol), float((err / (np.abs(ref) + 1e-9)).max())


def test_gemm_chalf_exact_on_integers(env):
    """Small-integer operands: every product and sum is exact in fp32 and the result fits fp16
    exactly, so the tensor-core result must equal the definition bit for bit."""
    torch, tn = env
    rng = np.random.default_rng(5)
    M, K, N = 1000, 64, 32
    a = rng.integers(-3, 4, (M, K)) + 1j * rng.integers(-3, 4, (M, K))
    b = rng.integers(-2, 3, (K, N)) + 1j * rng.integers(-2, 3, (K, N))
    bp = embed.pad_b(b)
    bp_km = np.transpose(bp, (2, 0, 1, 3)).reshape(2 * N, 2 * K).astype(np.float16)
    A = torch.from_numpy(_half_pairs(a).reshape(-1)).cuda()
    C = torch.empty(M * 2 * N, dtype=torch.float16, device="cuda")
    tn.tn_gemm_chalf(C, A, torch.from_numpy(bp_km.reshape(-1)).cuda(), M, K, N)
    torch.cuda.synchronize()
    got = C.cpu().numpy().astype(np.float64).reshape(M, N, 2)
    ref = a @ b
    assert np.array_equal(got[..., 0], ref.real) and np.array_equal(got[..., 1], ref.imag)


@pytest.mark.parametrize("K,N", [(2, 4), (4, 64), (1, 8), (64, 2), (8, 1), (4, 1), (4, 4), (2, 64), (16, 4), (8, 16), (1, 1), (2, 32),
                                 (8, 4), (8, 8), (4, 32), (16, 8), (4, 8), (16, 2)])
def test_gemm_chalf_simt_small_shapes(env, K, N):
    torch, tn = env
    rng = np.random.default_rng(K * 100 + N)
    M = 777
    a = rng.integers(-3, 4, (M, K)) + 1j * rng.integers(-3, 4, (M, K))
    b = rng.integers(-2, 3, (K, N)) + 1j * rng.integers(-2, 3, (K, N))
    bp_km = np.transpose(embed.pad_b(b), (2, 0, 1, 3)).reshape(2 * N, 2 * K).astype(np.float16)
    C = torch.empty(M * 2 * N, dtype=torch.float16, device="cuda")
    tn.tn_gemm_chalf(C, torch.from_numpy(_half_pairs(a).reshape(-1)).cuda(),
                     torch.from_numpy(bp_km.reshape(-1)).cuda(), M, K, N)
    torch.cuda.synchronize()
    got = C.cpu().numpy().astype(np.float64).reshape(M, N, 2)
    ref = a @ b
    assert np.array_equal(got[..., 0] + 1j * got[..., 1], ref)


@pytest.mark.parametrize("K,N,M", [(8, 8, 2_500_001), (8, 4, 2_000_003), (16, 4, 1_200_007), (4, 32, 600_001)])
def test_gemm_chalf_rows_bulk_ring_wrap(env, K, N, M):
    """Row-streaming steps with K >= 4 run the bulk-copy pipelined kernel: M large enough that every
    CTA wraps its shared-memory ring several times, with a ragged last tile (and a partial row group
    where a thread owns 2 rows); exact on small-integer operands."""
    torch, tn = env
    rng = np.random.default_rng(K * 1000 + N)
    a = rng.integers(-3, 4, (M, K)) + 1j * rng.integers(-3, 4, (M, K))
    b = rng.integers(-2, 3, (K, N)) + 1j * rng.integers(-2, 3, (K, N))
    bp_km = np.transpose(embed.pad_b(b), (2, 0, 1, 3)).reshape(2 * N, 2 * K).astype(np.float16)
    C = torch.full((M * 2 * N,), float("nan"), dtype=torch.float16, device="cuda")
    tn.tn_gemm_chalf(C, torch.from_numpy(_half_pairs(a).reshape(-1)).cuda(),
                     torch.from_numpy(bp_km.reshape(-1)).cuda(), M, K, N)
    torch.cuda.synchronize()
    got = C.cpu().numpy().astype(np.float64).reshape(M, N, 2)
    ref = a @ b
    assert np.array_equal(got[..., 0], ref.real) and np.array_equal(got[..., 1], ref.imag)


@pytest.mark.parametrize("M", [3000, 4096])
def test_pad_b_and_scaled_gemm(env, M):
    """Eq. 6 padding on the device (scale 2^t by the C-A8 rule) vs the oracle's pad_b, then the
    scaled GEMM: exponent recorded, |C| <= 2^14, out_max = max|C| (M = 4096: the CTA-pair kernel)."""
    torch, tn = env
    rng = np.random.default_rng(9)
    K, N = 64, 128
    b = ((rng.standard_normal((K, N)) + 1j * rng.standard_normal((K, N))) * 1e-3).astype(np.complex64)
    B = torch.from_numpy(b.view(np.float32).reshape(-1)).cuda()
    BP = torch.empty(4 * K * N, dtype=torch.float16, device="cuda")
    bound = torch.zeros(1, dtype=torch.float32, device="cuda")
    ex = torch.zeros(2, dtype=torch.int32, device="cuda")
    scratch = torch.zeros(4, dtype=torch.int32, device="cuda")
    tn.tn_pad_b(BP, B, K, N, bound, ex, scratch)
    torch.cuda.synchronize()
    bmax = np.abs(b.view(np.float32)).max()
    p = int(np.frexp(np.float32(bmax))[1])
    t = 14 - p
    assert int(ex[0].item()) == t
    bs = (b.real.astype(np.float32) * np.float32(2.0 ** t)).astype(np.float16) + \
        1j * (b.imag.astype(np.float32) * np.float32(2.0 ** t)).astype(np.float16)
    exp_bp = np.transpose(embed.pad_b(bs), (2, 0, 1, 3)).reshape(2 * N, 2 * K).astype(np.float16)
    got_bp = BP.cpu().numpy().reshape(2 * N, 2 * K)
    assert np.array_equal(got_bp, exp_bp)
    l1 = np.abs(exp_bp.astype(np.float64)).sum(axis=1).max()
    assert abs(bound.item() - l1) <= 1e-5 * l1
    # scaled GEMM
    a = (rng.standard_normal((M, K)) + 1j * rng.standard_normal((M, K))) * 3.0
    a16 = _half_pairs(a)
    in_max = torch.tensor([float(np.abs(a16.astype(np.float32)).max())], device="cuda")
    out_max = torch.zeros(1, dtype=torch.int32, device="cuda")
    C = torch.empty(M * 2 * N, dtype=torch.float16, device="cuda")
    tn.tn_gemm_chalf(C, torch.from_numpy(a16.reshape(-1)).cuda(), BP, M, K, N, in_max, bound, out_max, ex[1:])
    torch.cuda.synchronize()
    e = int(ex[1].item())
    prod = np.float32(in_max.item()) * np.float32(bound.item())
    assert e == 14 - int(np.frexp(prod)[1])
    ref = embed.cgemm_real(a16.astype(np.float64).reshape(M, 2 * K), embed.pad_b(bs)) * 2.0 ** e
    got = C.cpu().numpy().astype(np.float64).reshape(M, 2 * N)
    assert np.abs(got).max() <= 2 ** 14
    assert np.all(np.abs(got - ref) <= 2.0 ** -10 * np.abs(ref) + 1e-3 * np.sqrt(np.mean(ref ** 2)))
    # out_max: max of the scaled fp32 values before the fp16 rounding (so it stays meaningful when the
    # stored values underflow, reading C-A28): within half an fp16 ulp of the stored max
    mx = np.frombuffer(np.int32(out_max.item()).tobytes(), dtype=np.float32)[0]
    assert abs(mx - np.abs(got).max()) <= 2.0 ** -11 * np.abs(got).max()


@pytest.mark.parametrize("M,K,N,ma", [(128, 64, 64, 7), (1024, 64, 128, 7), (4096, 128, 256, 9),
                                      (2048, 512, 512, 8), (1 << 14, 64, 64, 14)])
def test_gemm_chalf_mn_exact(env, M, K, N, ma):
    """The permutation folded into an MN-major operand (tn_gemm_chalf_mn): A stored [M >> ma][K][2^ma]
    (kept modes innermost, the contracted ones next).  Integer operands in [-1, 1]: every product and
    sum is exact, so C equals a @ b bit for bit, and the scaled launch equals the Eq. 6 path
    (tn_gemm_chalf on the explicitly permuted A with B_P) bit for bit, exponent and max included."""
    torch, tn = env
    rng = np.random.default_rng(M + K + N)
    x = rng.integers(-1, 2, (M >> ma, K, 1 << ma)) + 1j * rng.integers(-1, 2, (M >> ma, K, 1 << ma))
    a = np.transpose(x, (0, 2, 1)).reshape(M, K)                     # a[m, k], m = (hi, lo)
    b = rng.integers(-1, 2, (K, N)) + 1j * rng.integers(-1, 2, (K, N))
    B = torch.from_numpy(b.astype(np.complex64).view(np.float32).reshape(-1)).cuda()
    BPM = torch.empty(2 * N * K, dtype=torch.float16, device="cuda")
    scratch = torch.zeros(4, dtype=torch.int32, device="cuda")
    tn.tn_pad_b_mn(BPM, B, K, N, None, None, scratch)
    torch.cuda.synchronize()
    exp_bpm = np.stack([b.real.T, b.imag.T], axis=1).reshape(2 * N, K).astype(np.float16)
    assert np.array_equal(BPM.cpu().numpy().reshape(2 * N, K), exp_bpm)
    X = torch.from_numpy(_half_pairs(x.reshape(1, -1)).reshape(-1)).cuda()
    C = torch.full((M * 2 * N,), float("nan"), dtype=torch.float16, device="cuda")
    tn.tn_gemm_chalf_mn(C, X, BPM, M, K, N, ma)
    torch.cuda.synchronize()
    got = C.cpu().numpy().astype(np.float64).reshape(M, N, 2)
    ref = a @ b
    assert np.array_equal(got[..., 0], ref.real) and np.array_equal(got[..., 1], ref.imag)
    # scaled: the same exponent, values and realised max as the Eq. 6 GEMM on the permuted operand
    bound = torch.zeros(1, dtype=torch.float32, device="cuda")
    ex = torch.zeros(4, dtype=torch.int32, device="cuda")
    tn.tn_pad_b_mn(BPM, B, K, N, bound, ex[0:], scratch)
    BP = torch.empty(4 * K * N, dtype=torch.float16, device="cuda")
    bound2 = torch.zeros(1, dtype=torch.float32, device="cuda")
    tn.tn_pad_b(BP, B, K, N, bound2, ex[1:], scratch)
    in_max = torch.tensor([1.0], device="cuda")
    om1 = torch.zeros(1, dtype=torch.int32, device="cuda")
    om2 = torch.zeros(1, dtype=torch.int32, device="cuda")
    C2 = torch.empty_like(C)
    tn.tn_gemm_chalf_mn(C, X, BPM, M, K, N, ma, in_max, bound, om1, ex[2:])
    tn.tn_gemm_chalf(C2, torch.from_numpy(_half_pairs(a).reshape(-1)).cuda(), BP, M, K, N, in_max, bound2, om2,
                     ex[3:])
    torch.cuda.synchronize()
    assert float(bound.item()) == float(bound2.item())
    assert int(ex[2].item()) == int(ex[3].item())
    assert torch.equal(C, C2)
    assert int(om1.item()) == int(om2.item())


def test_gemm_chalf_mn_rejects_bad_geometry(env):
    torch, tn = env
    t = torch.zeros(16, dtype=torch.float16, device="cuda")
    for M, K, N, ma in ((1024, 32, 64, 7), (1024, 64, 32, 7), (1024, 64, 64, 6), (1000, 64, 64, 7), (64, 64, 64, 7)):
        with pytest.raises(tn.TnError):
            tn.tn_gemm_chalf_mn(t, t, t, M, K, N, ma)


@pytest.mark.parametrize("M,K,N", [(1, 1, 1), (100, 3, 5), (1000, 64, 64), (4097, 128, 33)])
def test_gemm_cfloat(env, M, K, N):
    torch, tn = env
    rng = np.random.default_rng(M)
    a = (rng.standard_normal((M, K)) + 1j * rng.standard_normal((M, K))).astype(np.complex64)
    b = (rng.standard_normal((K, N)) + 1j * rng.standard_normal((K, N))).astype(np.complex64)
    A = torch.from_numpy(a.view(np.float32).reshape(-1)).cuda()
    B = torch.from_numpy(b.view(np.float32).reshape(-1)).cuda()
    C = torch.empty(2 * M * N, dtype=torch.float32, device="cuda")
    tn.tn_gemm_cfloat(C, A, B, M, K, N)
    torch.cuda.synchronize()
    got = C.cpu().numpy().view(np.complex64).reshape(M, N).astype(np.complex128)
    ref = a.astype(np.complex128) @ b.astype(np.complex128)
    assert np.linalg.norm(got - ref) <= 1e-6 * np.linalg.norm(ref)


@pytest.mark.parametrize("g", [128, 64, 256])
def test_quant_int8_bit_exact_vs_oracle_codec(env, g):
    torch, tn = env
    rng = np.random.default_rng(g)
    x = (rng.standard_normal(g * 257) * 10.0 ** rng.uniform(-6, 2)).astype(np.float32)
    x[:g] = 0.37  # a constant group (C-A11)
    X = torch.from_numpy(x).cuda()
    codes = torch.empty(x.size, dtype=torch.int8, device="cuda")
    sc = torch.empty(x.size // g, dtype=torch.float32, device="cuda")
    ze = torch.empty_like(sc)
    tn.tn_quant_int8(codes, sc, ze, X, g)
    y = torch.empty_like(X)
    tn.tn_dequant_int8(y, codes, sc, ze, g)
    torch.cuda.synchronize()
    rc, rs, rz = codec.quantize(x, np.float32(-128), np.float32(127), 1.0, group=g)
    assert np.array_equal(codes.cpu().numpy().astype(np.float32), rc)
    assert np.array_equal(sc.cpu().numpy(), rs) and np.array_equal(ze.cpu().numpy(), rz)
    assert np.array_equal(y.cpu().numpy(), codec.dequantize(rc, rs, rz, 1.0, group=g))


def test_quant_int8_f16_payload_bit_exact(env):
    """The mode-swap codec on complex-half payloads (fp16 reals): codes/scales/zeros bit-exact vs
    the oracle codec on the same float32 values; dequantised fp16 = oracle dequant rounded to fp16."""
    torch, tn = env
    rng = np.random.default_rng(3)
    g = 128
    x = (rng.standard_normal(g * 300) * 2000).astype(np.float16)
    x[g:2 * g] = 0                           # all-zero group
    x[2 * g:3 * g:2] = 0                     # half zeros (interleaved imaginary parts)
    X = torch.from_numpy(x).cuda()
    codes = torch.empty(x.size, dtype=torch.int8, device="cuda")
    sc = torch.empty(x.size // g, dtype=torch.float32, device="cuda")
    ze = torch.empty_like(sc)
    tn.tn_quant_int8_f16(codes, sc, ze, X, g)
    y = torch.empty_like(X)
    tn.tn_dequant_int8_f16(y, codes, sc, ze, g)
    torch.cuda.synchronize()
    rc, rs, rz = codec.quantize(x.astype(np.float32), np.float32(-128), np.float32(127), 1.0, group=g)
    assert np.array_equal(codes.cpu().numpy().astype(np.float32), rc)
    assert np.array_equal(sc.cpu().numpy(), rs) and np.array_equal(ze.cpu().numpy(), rz)
    assert np.array_equal(y.cpu().numpy(), codec.dequantize(rc, rs, rz, 1.0, group=g).astype(np.float16))
    assert np.linalg.norm(y.cpu().numpy().astype(np.float64) - x) <= 0.01 * np.linalg.norm(x.astype(np.float64))


@pytest.mark.parametrize("mlog,klog,N,seed", [(7, 3, 8, 0), (9, 4, 16, 1), (10, 5, 64, 2), (8, 7, 32, 3),
                                              (12, 6, 256, 4), (11, 8, 4, 5), (13, 5, 2, 6), (10, 9, 128, 7)])
def test_gemm_chalf_gathered_a_exact(env, mlog, klog, N, seed):
    """The stem permutation fused into the GEMM load: A[m, k] read at arbitrary per-bit strides of
    the unpermuted stem (k bits 0, 1 fixed contiguous).  Integer operands in [-1, 1] keep every
    product, sum and the fp16 result exact, so the gathered tcgen05 GEMM must equal (transpose,
    then multiply) bit for bit."""
    torch, tn = env
    rng = np.random.default_rng(seed)
    n = mlog + klog
    pos = [int(x) for x in rng.permutation(np.arange(2, n))]
    kpos = [0, 1] + pos[:klog - 2]
    mpos = pos[klog - 2:]
    ms = [1 << p for p in mpos]
    ks = [1 << p for p in kpos]
    x = rng.integers(-1, 2, 1 << n) + 1j * rng.integers(-1, 2, 1 << n)
    mi = np.arange(1 << mlog)
    ki = np.arange(1 << klog)
    moff = sum(((mi >> j) & 1) * ms[j] for j in range(mlog))
    koff = sum(((ki >> j) & 1) * ks[j] for j in range(klog))
    a = x[moff[:, None] + koff[None, :]]                       # [M, K] = the permuted stem
    K = 1 << klog
    b = rng.integers(-1, 2, (K, N)) + 1j * rng.integers(-1, 2, (K, N))
    bp = embed.pad_b(b)
    rows = max(2 * N, 16)
    bp_km = np.zeros((rows, 2 * K), np.float16)
    bp_km[:2 * N] = np.transpose(bp, (2, 0, 1, 3)).reshape(2 * N, 2 * K)
    X = torch.from_numpy(_half_pairs(x.reshape(1, -1)).reshape(-1)).cuda()
    C = torch.full(((1 << mlog) * 2 * N,), float("nan"), dtype=torch.float16, device="cuda")
    tn.tn_gemm_chalf_gather(C, X, torch.from_numpy(bp_km.reshape(-1)).cuda(), mlog, klog, N, ms, ks)
    torch.cuda.synchronize()
    got = C.cpu().numpy().astype(np.float64).reshape(1 << mlog, N, 2)
    ref = a @ b
    assert np.array_equal(got[..., 0], ref.real) and np.array_equal(got[..., 1], ref.imag)


def test_gemm_chalf_gathered_rejects_bad_geometry(env):
    torch, tn = env
    t = torch.zeros(1 << 12, dtype=torch.float16, device="cuda")
    with pytest.raises(tn.TnError):   # M < 128
        tn.tn_gemm_chalf_gather(t, t, t, 6, 3, 8, [1 << j for j in range(3, 9)], [1, 2, 4])
    with pytest.raises(tn.TnError):   # K < 8
        tn.tn_gemm_chalf_gather(t, t, t, 7, 2, 8, [1 << j for j in range(2, 9)], [1, 2])


@pytest.mark.parametrize("runs,N", [("m8k5m5", 32), ("m12k6m2", 64), ("m5k7m4", 16), ("m7k3m1k2m2", 128),
                                    ("m6k9m3", 256), ("m9k4", 8), ("m2k3m5k2m4", 2), ("m10k8", 512)])
def test_gemm_chalf_gathered_word_pieces_exact(env, runs, N):
    """Contracted modes NOT innermost (the middle-of-the-order layouts the grouped C3 plan produces):
    the fused permutation loads single complex elements (4-byte cp.async, mode 4).  Exact integer
    parity with (transpose, then multiply) as above."""
    import re
    torch, tn = env
    kpos, mpos, b = [], [], 0
    for kind, cnt in re.findall(r"([km])(\d+)", runs):
        for _ in range(int(cnt)):
            (kpos if kind == "k" else mpos).append(b)
            b += 1
    mlog, klog, n = len(mpos), len(kpos), b
    rng = np.random.default_rng(n * 17 + N)
    ms = [1 << p for p in mpos]
    ks = [1 << p for p in kpos]
    x = rng.integers(-1, 2, 1 << n) + 1j * rng.integers(-1, 2, 1 << n)
    mi = np.arange(1 << mlog)
    ki = np.arange(1 << klog)
    moff = sum(((mi >> j) & 1) * ms[j] for j in range(mlog))
    koff = sum(((ki >> j) & 1) * ks[j] for j in range(klog))
    a = x[moff[:, None] + koff[None, :]]
    K = 1 << klog
    bm = rng.integers(-1, 2, (K, N)) + 1j * rng.integers(-1, 2, (K, N))
    bp = embed.pad_b(bm)
    bp_km = np.zeros((max(2 * N, 16), 2 * K), np.float16)
    bp_km[:2 * N] = np.transpose(bp, (2, 0, 1, 3)).reshape(2 * N, 2 * K)
    X = torch.from_numpy(_half_pairs(x.reshape(1, -1)).reshape(-1)).cuda()
    C = torch.full(((1 << mlog) * 2 * N,), float("nan"), dtype=torch.float16, device="cuda")
    tn.tn_gemm_chalf_gather(C, X, torch.from_numpy(bp_km.reshape(-1)).cuda(), mlog, klog, N, ms, ks)
    torch.cuda.synchronize()
    got = C.cpu().numpy().astype(np.float64).reshape(1 << mlog, N, 2)
    ref = a @ bm
    assert np.array_equal(got[..., 0], ref.real) and np.array_equal(got[..., 1], ref.imag)


@pytest.mark.parametrize("runs,N", [("k2m8k5m5", 32), ("k3m8k2m5", 16), ("k4m4k4m7", 64), ("k5m7k2m3", 8),
                                    ("k7m9", 256), ("k2m3k3m9", 4), ("k2m7k1m1k3m2", 64), ("k4m2k3m8", 2),
                                    ("k3m1k4m9", 128), ("k2m12k4", 16),
                                    # 128-byte rows, N >= 128, M % 256 == 0: the CTA-pair kernel's N-d box
                                    ("k5m9k2m4", 128), ("k6m8k3m5", 256),
                                    # 6 source runs: adjacent m / k runs outside the box share a TMA dim
                                    ("k5m8k3m2k2m3", 32), ("k5m9k2m1k3m2", 128),
                                    # two contracted modes innermost (core-matrix box) on the CTA-pair kernel
                                    ("k2m8k5m5", 128), ("k2m9k4m3", 256), ("k5m9k2m1k3m2", 32),
                                    # short direct rows: raw box + reshuffle on the CTA-pair kernel
                                    ("k4m8k4m4", 128), ("k3m1k6m9", 128), ("k3m1k3m10", 64)])
def test_gemm_chalf_gathered_runs_exact(env, runs, N):
    """Stem layouts as they occur on the C3 path (runs of contracted k / kept m modes, innermost
    first, kept modes in stored order): these go through the N-dimensional TMA box (swizzled rows
    when >= 3 contracted modes are innermost, interleaved core matrices when 2), the others through
    the cp.async gather.  Exact integer parity as above."""
    import re
    torch, tn = env
    kpos, mpos, b = [], [], 0
    for kind, cnt in re.findall(r"([km])(\d+)", runs):
        for _ in range(int(cnt)):
            (kpos if kind == "k" else mpos).append(b)
            b += 1
    mlog, klog, n = len(mpos), len(kpos), b
    rng = np.random.default_rng(n * 31 + N)
    ms = [1 << p for p in mpos]
    ks = [1 << p for p in kpos]
    x = rng.integers(-1, 2, 1 << n) + 1j * rng.integers(-1, 2, 1 << n)
    mi = np.arange(1 << mlog)
    ki = np.arange(1 << klog)
    moff = sum(((mi >> j) & 1) * ms[j] for j in range(mlog))
    koff = sum(((ki >> j) & 1) * ks[j] for j in range(klog))
    a = x[moff[:, None] + koff[None, :]]
    K = 1 << klog
    bm = rng.integers(-1, 2, (K, N)) + 1j * rng.integers(-1, 2, (K, N))
    bp = embed.pad_b(bm)
    bp_km = np.zeros((max(2 * N, 16), 2 * K), np.float16)
    bp_km[:2 * N] = np.transpose(bp, (2, 0, 1, 3)).reshape(2 * N, 2 * K)
    X = torch.from_numpy(_half_pairs(x.reshape(1, -1)).reshape(-1)).cuda()
    C = torch.full(((1 << mlog) * 2 * N,), float("nan"), dtype=torch.float16, device="cuda")
    tn.tn_gemm_chalf_gather(C, X, torch.from_numpy(bp_km.reshape(-1)).cuda(), mlog, klog, N, ms, ks)
    torch.cuda.synchronize()
    got = C.cpu().numpy().astype(np.float64).reshape(1 << mlog, N, 2)
    ref = a @ bm
    assert np.array_equal(got[..., 0], ref.real) and np.array_equal(got[..., 1], ref.imag)


def test_quant_int4_f16_payload_bit_exact(env):
    """int4 preset (Table 1; reading C-A14 packing) on fp16 payloads: packed codes,
    scales and zeros bit-exact vs the oracle codec; dequantised fp16 = oracle dequant rounded."""
    torch, tn = env
    rng = np.random.default_rng(4)
    g = 128
    x = (rng.standard_normal(g * 300) * 2000).astype(np.float16)
    x[g:2 * g] = 0                           # constant group (C-A11)
    x[2 * g:3 * g:2] = 0
    X = torch.from_numpy(x).cuda()
    packed = torch.empty(x.size // 2, dtype=torch.uint8, device="cuda")
    sc = torch.empty(x.size // g, dtype=torch.float32, device="cuda")
    ze = torch.empty_like(sc)
    tn.tn_quant_int4_f16(packed, sc, ze, X, g)
    y = torch.empty_like(X)
    tn.tn_dequant_int4_f16(y, packed, sc, ze, g)
    torch.cuda.synchronize()
    rc, rs, rz = codec.quantize(x.astype(np.float32), np.float32(0), np.float32(15), 1.0, group=g)
    assert np.array_equal(packed.cpu().numpy(), codec.pack_int4(rc))
    assert np.array_equal(sc.cpu().numpy(), rs) and np.array_equal(ze.cpu().numpy(), rz)
    assert np.array_equal(y.cpu().numpy(), codec.dequantize(rc, rs, rz, 1.0, group=g).astype(np.float16))
    # half a quantisation step per element, plus the fp16 rounding of the dequantised value:
    # |err| <= (max - min) / 30 + ulp_fp16(|x|) per group
    xg = x.astype(np.float64).reshape(-1, g)
    err = np.abs(y.cpu().numpy().astype(np.float64).reshape(-1, g) - xg)
    span = np.ptp(xg, axis=1)
    assert np.all(err.max(axis=1) <= span / 30 * (1 + 1e-5) + np.abs(xg).max(axis=1) * 2.0 ** -10)


def _fusable_perm(rng, n, b):
    """A random axis permutation of a rank-n tensor that keeps the innermost b axes in place."""
    outer = [int(a) for a in rng.permutation(n - b)]
    return outer + list(range(n - b, n))


@pytest.mark.parametrize("n,g,codec_id,seed", [(10, 128, 1, 0), (13, 64, 1, 1), (12, 256, 1, 2), (9, 2, 1, 3),
                                               (16, 128, 1, 4), (11, 128, 2, 5), (14, 32, 2, 6), (7, 128, 1, 7),
                                               (20, 128, 1, 8), (18, 128, 2, 9), (12, 512, 1, 10),
                                               (13, 512, 2, 11), (15, 256, 2, 12)])
def test_permute_quant_fused_bit_exact(env, n, g, codec_id, seed):
    """Sender side of a quantised mode swap with the permutation fused into the codec (north_star
    (5)): codes, scales and zeros of tn_permute_quant_f16 equal the oracle codec applied to the
    numpy-transposed complex-half payload, bit for bit (int8 and packed int4)."""
    torch, tn = env
    rng = np.random.default_rng(seed)
    b = (g // 2).bit_length() - 1
    perm = _fusable_perm(rng, n, b)
    x = (rng.standard_normal((1 << n, 2)) * 10.0 ** rng.uniform(-3, 3)).astype(np.float16)
    x[: 1 << b] = 0.25                       # a constant group of the source (C-A11)
    xt = x.reshape([2] * n + [2]).transpose(perm + [n]).reshape(-1)  # the permuted payload
    X = torch.from_numpy(x.reshape(-1)).cuda()
    reals = 2 << n
    ncode = reals if codec_id == 1 else reals // 2
    codes = torch.empty(ncode, dtype=torch.int8 if codec_id == 1 else torch.uint8, device="cuda")
    sc = torch.empty(reals // g, dtype=torch.float32, device="cuda")
    ze = torch.empty_like(sc)
    tn.tn_permute_quant_f16(codes, sc, ze, X, perm, g, codec_id)
    torch.cuda.synchronize()
    lo, hi = (-128, 127) if codec_id == 1 else (0, 15)
    rc, rs, rz = codec.quantize(xt.astype(np.float32), np.float32(lo), np.float32(hi), 1.0, group=g)
    want = rc if codec_id == 1 else codec.pack_int4(rc)
    got = codes.cpu().numpy()
    assert np.array_equal(got.astype(np.float32) if codec_id == 1 else got, want)
    assert np.array_equal(sc.cpu().numpy(), rs) and np.array_equal(ze.cpu().numpy(), rz)


def test_permute_quant_rejects_unfusable(env):
    """A permutation that moves one of the innermost log2(g/2) axes is refused (TN_E_INVALID)."""
    torch, tn = env
    n = 10
    perm = list(range(n))
    perm[-1], perm[0] = perm[0], perm[-1]
    X = torch.zeros(2 << n, dtype=torch.float16, device="cuda")
    codes = torch.empty(2 << n, dtype=torch.int8, device="cuda")
    sc = torch.empty((2 << n) // 128, dtype=torch.float32, device="cuda")
    with pytest.raises(Exception):
        tn.tn_permute_quant_f16(codes, sc, sc.clone(), X, perm, 128)


@pytest.mark.parametrize("g", [2048, 1 << 16])
def test_quant_int8_exp02_tensor_preset_vs_oracle(env, g):
    """Table 1 int8 preset (entire tensor, exp 0.2; reading C-A10) on fp16 payloads: scales and
    zeros bit-exact vs the oracle codec; codes equal except where the double-precision power rounds to
    the other side of a code boundary (CUDA pow vs libm: at most 1 code, rare); dequantised values vs
    the oracle dequantisation of the GPU's own codes: fp16 rounding of the same fp32 value."""
    torch, tn = env
    rng = np.random.default_rng(5)
    n = 4 * g
    x = (rng.standard_normal(n) * np.exp(rng.uniform(-6, 3, n))).astype(np.float16)
    x[g:2 * g] = np.float16(0.37)                       # constant group (C-A11)
    X = torch.from_numpy(x).cuda()
    codes = torch.empty(n, dtype=torch.int8, device="cuda")
    sc = torch.empty(n // g, dtype=torch.float32, device="cuda")
    ze = torch.empty_like(sc)
    tmp = torch.empty(2 * (n // g), dtype=torch.int32, device="cuda")
    tn.tn_quant_int8_exp_f16(codes, sc, ze, X, g, 0.2, tmp)
    y = torch.empty_like(X)
    tn.tn_dequant_int8_exp_f16(y, codes, sc, ze, g, 0.2)
    torch.cuda.synchronize()
    rc, rs, rz = codec.quantize(x.astype(np.float32), np.float32(-128), np.float32(127), 0.2, group=g)
    assert np.array_equal(sc.cpu().numpy(), rs) and np.array_equal(ze.cpu().numpy(), rz)
    gc = codes.cpu().numpy().astype(np.float32)
    diff = np.abs(gc - rc)
    assert diff.max() <= 1 and np.count_nonzero(diff) <= max(2, n // 100000)
    want = codec.dequantize(gc, rs, rz, 0.2, group=g).astype(np.float16)
    got = y.cpu().numpy()
    close = (got == want) | (np.abs(got.astype(np.float64) - want) <= 2.0 ** -10 * np.abs(want.astype(np.float64)))
    assert close.all()
    assert np.array_equal(got[g:2 * g], x[g:2 * g])       # constant group round-trips exactly


def _sparse_operands(rng, m_a, n_b, M, K, N):
    a = (rng.standard_normal((m_a, M, K)) + 1j * rng.standard_normal((m_a, M, K))) / np.sqrt(2)
    b = (rng.standard_normal((n_b, K, N)) + 1j * rng.standard_normal((n_b, K, N))) / np.sqrt(2 * K)
    a16 = a.real.astype(np.float16) + 1j * a.imag.astype(np.float16)
    b16 = b.real.astype(np.float16) + 1j * b.imag.astype(np.float16)
    A = np.stack([a16.real, a16.imag], axis=-1).astype(np.float16).reshape(-1)
    bp = np.stack([np.transpose(embed.pad_b(b16[j]), (2, 0, 1, 3)).reshape(2 * N, 2 * K) for j in range(n_b)])
    return a16, b16, A, bp.astype(np.float16).reshape(-1)


def _close(got, ref):
    tol = 2.0 ** -10 * np.abs(ref) + 1e-3 * np.sqrt(np.mean(np.abs(ref) ** 2)) + 1e-7
    bad = np.abs(got - ref) > tol
    if bad.any():
        print("mismatches", int(bad.sum()), "of", bad.size, "first at", np.argwhere(bad)[:4].tolist())
    return not bad.any()


@pytest.mark.parametrize("M,K,N", [(128, 8, 8), (256, 64, 16), (512, 32, 128), (128, 256, 64)])
def test_gemm_chalf_batched_vs_oracle_gather(env, M, K, N):
    """Fig. 5 bottom: C[n] = A[Index_A[n]] x B[Index_B[n]] in one tcgen05 launch vs the
    oracle's gather_contract (oracle/sparse.py) on the same fp16 operands; Index_A with the paper's
    repeat pattern [0, 0, 1, 1, 1, 3, 4, ...]."""
    from oracle import sparse
    torch, tn = env
    rng = np.random.default_rng(M + K + N)
    m_a, n_b = 6, 5
    ia = np.array([0, 0, 1, 1, 1, 3, 4, 5, 5, 2], dtype=np.int32)
    ib = rng.integers(0, n_b, size=ia.size).astype(np.int32)
    a16, b16, A, BP = _sparse_operands(rng, m_a, n_b, M, K, N)
    ref = sparse.gather_contract(a16, b16, ia, ib)                       # [n, M, N] complex128
    C = torch.full((ia.size * M * N * 2,), float("nan"), dtype=torch.float16, device="cuda")
    tn.tn_gemm_chalf_batched(C, torch.from_numpy(A).cuda(), torch.from_numpy(BP).cuda(), M, K, N,
                             torch.from_numpy(ia).cuda(), torch.from_numpy(ib).cuda(), m_a, n_b)
    torch.cuda.synchronize()
    g = C.cpu().numpy().astype(np.float64).reshape(ia.size, M, N, 2)
    assert _close(g[..., 0] + 1j * g[..., 1], ref)


@pytest.mark.parametrize("M,K,N", [(128, 16, 32), (256, 64, 32), (128, 32, 256), (256, 128, 64)])
def test_gemm_chalf_padded_index_vs_oracle(env, M, K, N):
    """Fig. 5 top: the padded 2-d index of Index_B (m_r = max repeat of Index_A, -1 padding,
    built by the oracle's build_padded_index) drives C_P = A x B_P on the GPU; the extracted valid
    blocks equal the oracle's padded_contract and gather_contract (same fp16 operands); the padding
    blocks are exact zeros."""
    from oracle import sparse
    torch, tn = env
    rng = np.random.default_rng(7 * M + K + N)
    m_a, n_b = 5, 4
    ia = np.array([0, 0, 1, 1, 1, 3, 4], dtype=np.int64)                 # the paper's example: m_r = 3
    ib = rng.integers(0, n_b, size=ia.size)
    table, m_r = sparse.build_padded_index(ia, ib, m_a)
    assert m_r == 3
    a16, b16, A, BP = _sparse_operands(rng, m_a, n_b, M, K, N)
    ref = sparse.padded_contract(a16, b16, ia, ib)
    assert np.allclose(ref, sparse.gather_contract(a16, b16, ia, ib))
    C = torch.full((m_a * M * m_r * N * 2,), float("nan"), dtype=torch.float16, device="cuda")
    tn.tn_gemm_chalf_padded(C, torch.from_numpy(A).cuda(), torch.from_numpy(BP).cuda(), M, K, N,
                            torch.from_numpy(table.astype(np.int32)).cuda(), n_b)
    torch.cuda.synchronize()
    g = C.cpu().numpy().astype(np.float64).reshape(m_a, M, m_r, N, 2)
    cp = g[..., 0] + 1j * g[..., 1]                                       # C_P[a, m, r, n]
    occ = np.zeros(m_a, dtype=np.int64)
    got = []
    for i in ia:                                                          # extract valid blocks
        got.append(cp[i, :, occ[i], :])
        occ[i] += 1
    assert _close(np.stack(got), ref)
    for a in range(m_a):
        for r in range(m_r):
            if table[a, r] < 0:
                assert np.all(cp[a, :, r, :] == 0)
