// SIMT stem GEMMs.
// * gemm_c64: the complex64 (TN_CFLOAT) stem GEMM C[M,N] = A[M,K] B[K,N] with true fp32 FMA
//   (reading c.5: TF32 would miss the 1e-5 bound).  64x64 complex tile, 256 threads, 4x4 per
//   thread, operands staged through shared memory.
// * gemm_chalf_simt: complex-half stem steps whose K or N is below the tcgen05 minimum
//   (2K or 2N < 16): memory-bound, thread per output element, fp32 accumulation, B read from the
//   same Eq. 6 padded B_P the tensor-core path uses, same power-of-two output scaling (C-A8).
#include <cstring>

#include "common.cuh"

namespace tn {

constexpr int TM = 64, TN_ = 64, TK = 8;

__global__ void __launch_bounds__(256) gemm_c64_kernel(float2* __restrict__ C, const float2* __restrict__ A,
                                                       const float2* __restrict__ B, uint64_t M, int K, int N,
                                                       const OutMap om, uint64_t m_base, const float* in_max,
                                                       const float* b_bound, uint32_t* out_max, int* exp_slot) {
  // power-of-two output scale (reading C-A8, also for complex64: one-slice partial amplitudes of a
  // 53-qubit network fall below fp32's normal range, 1e-38, long before the root)
  int e = 0;
  if (in_max && b_bound) e = scale_exp_for(in_max[0] * b_bound[0]);
  if (exp_slot && blockIdx.x == 0 && blockIdx.y == 0 && threadIdx.x == 0 && m_base == 0) *exp_slot = e;
  const float sc = ldexpf(1.f, e);
  float mx = 0.f;
  __shared__ float2 As[TK][TM + 1];
  __shared__ float2 Bs[TK][TN_];
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  const uint64_t m0 = (uint64_t)blockIdx.y * TM;
  const int n0 = blockIdx.x * TN_;
  float2 acc[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j] = make_float2(0.f, 0.f);
  for (int k0 = 0; k0 < K; k0 += TK) {
    for (int i = threadIdx.x; i < TM * TK; i += 256) {
      int r = i / TK, c = i % TK;
      uint64_t gm = m0 + r;
      int gk = k0 + c;
      As[c][r] = (gm < M && gk < K) ? A[gm * K + gk] : make_float2(0.f, 0.f);
    }
    for (int i = threadIdx.x; i < TK * TN_; i += 256) {
      int r = i / TN_, c = i % TN_;
      int gk = k0 + r, gn = n0 + c;
      Bs[r][c] = (gk < K && gn < N) ? B[(uint64_t)gk * N + gn] : make_float2(0.f, 0.f);
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < TK; ++kk) {
      float2 a[4], b[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) a[i] = As[kk][ty * 4 + i];
#pragma unroll
      for (int j = 0; j < 4; ++j) b[j] = Bs[kk][tx + 16 * j];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          acc[i][j].x = fmaf(a[i].x, b[j].x, fmaf(-a[i].y, b[j].y, acc[i][j].x));
          acc[i][j].y = fmaf(a[i].x, b[j].y, fmaf(a[i].y, b[j].x, acc[i][j].y));
        }
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    uint64_t gm = m0 + ty * 4 + i;
    if (gm >= M) continue;
    const int64_t mo = om.identity ? 0 : outmap_m(om, m_base + gm);
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      int gn = n0 + tx + 16 * j;
      if (gn < N) {
        const float2 v = make_float2(acc[i][j].x * sc, acc[i][j].y * sc);
        mx = fmaxf(mx, fmaxf(fabsf(v.x), fabsf(v.y)));
        if (om.identity)
          C[gm * N + gn] = v;
        else
          C[mo + outmap_n(om, gn)] = v;
      }
    }
  }
  if (out_max) {
#pragma unroll
    for (int o = 16; o; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    if ((threadIdx.x & 31) == 0) atomicMax(out_max, __float_as_uint(mx));
  }
}

void launch_gemm_c64(float2* c, const float2* a, const float2* b, uint64_t M, uint32_t K, uint32_t N,
                     const OutMap* om_in, cudaStream_t s, const float* in_max, const float* b_bound, uint32_t* out_max,
                     int* exp_slot) {
  g_last_kern = "c64";
  OutMap om = om_in ? *om_in : identity_map(M, N);
  uint64_t gy = (M + TM - 1) / TM;
  if (gy > 65535ull * 1024) throw TnError{TN_E_UNSUPPORTED, "gemm_c64: M too large"};
  dim3 grid((N + TN_ - 1) / TN_, 1, 1);
  // fold huge M into grid.y chunks
  const uint64_t maxy = 65535;
  for (uint64_t y0 = 0; y0 < gy; y0 += maxy) {
    uint64_t ny = std::min<uint64_t>(maxy, gy - y0);
    grid.y = (unsigned)ny;
    uint64_t moff = y0 * TM;
    gemm_c64_kernel<<<grid, 256, 0, s>>>(om.identity ? c + moff * N : c, a + moff * K, b, M - moff, (int)K, (int)N, om,
                                         moff, in_max, b_bound, out_max, exp_slot);
  }
  TN_CUDA(cudaGetLastError());
}

OutMap identity_map(uint64_t M, uint32_t N) {
  OutMap o;
  memset(&o, 0, sizeof(o));
  o.identity = 1;
  int mb = 0, nb = 0;
  while ((1ull << mb) < M) ++mb;
  while ((1u << nb) < N) ++nb;
  o.mbits = mb;
  o.nbits = nb;
  for (int j = 0; j < mb && j < kMaxModes; ++j) o.ms[j] = (int64_t)N << j;
  for (int j = 0; j < nb && j < 24; ++j) o.ns[j] = (int64_t)1 << j;
  return o;
}

__device__ __forceinline__ void atomic_max_pos2(uint32_t* addr, float v) { atomicMax(addr, __float_as_uint(v)); }

// Memory-bound complex-half stem steps with small K*N (K <= 8 and N <= 4, or K <= 4): a CTA
// streams a contiguous tile of T rows of A (16-byte vector loads) into shared memory, computes the
// T x N outputs with B (complex fp32, from the Eq. 6 padded B_P) in shared memory, and writes them
// in output order: consecutive threads -> consecutive outputs (coalesced; vector stores when the
// output layout keeps the lowest n bits contiguous).
constexpr int kTileCplx = 4096;   // complex elements of A per CTA tile

__global__ void __launch_bounds__(256) gemm_chalf_simt_kernel(__half2* __restrict__ C, const __half2* __restrict__ A,
                                                              const __half* __restrict__ BP, uint64_t M, int K, int N,
                                                              int rows_log, int run, const float* in_max,
                                                              const float* b_bound, uint32_t* out_max, int* exp_slot,
                                                              const OutMap om) {
  __shared__ __align__(16) __half2 sA[kTileCplx];
  __shared__ float2 sB[2048];
  const bool smem_b = K * N <= 2048;
  int e = 0;
  if (in_max && in_max[0] < 0.f) return;  // scale re-run not needed (runtime.cu redo)
  if (in_max && b_bound) e = scale_exp_for(in_max[0] * b_bound[0]);
  if (exp_slot && blockIdx.x == 0 && threadIdx.x == 0) *exp_slot = e;
  const float sc = ldexpf(1.f, e);
  const int K2 = 2 * K;
  for (int i = threadIdx.x; smem_b && i < K * N; i += blockDim.x) {
    int k = i / N, n = i - k * N;
    // B_P row (n,0) holds (Re b, -Im b); row (n,1) holds (Im b, Re b)
    sB[i] = make_float2(__half2float(BP[(size_t)(2 * n) * K2 + 2 * k]), __half2float(BP[(size_t)(2 * n + 1) * K2 + 2 * k]));
  }
  const int T = 1 << rows_log;  // rows per tile
  int nlog = 0;
  while ((1 << nlog) < N) ++nlog;
  const int vlog = run < 2 ? run : 2;  // vector of 2^vlog outputs when contiguous
  const int V = 1 << vlog;
  const uint64_t tiles = (M + T - 1) >> rows_log;
  float mx = 0.f;
  for (uint64_t tile = blockIdx.x; tile < tiles; tile += gridDim.x) {
    const uint64_t m0 = tile << rows_log;
    const int rows = (int)((M - m0) < (uint64_t)T ? (M - m0) : (uint64_t)T);
    __syncthreads();  // sB ready / previous tile consumed
    const int cnt = rows * K;
    const uint4* src = reinterpret_cast<const uint4*>(A + m0 * K);
    if ((cnt & 3) == 0) {
      for (int i = threadIdx.x; i < (cnt >> 2); i += blockDim.x) reinterpret_cast<uint4*>(sA)[i] = src[i];
    } else {
      for (int i = threadIdx.x; i < cnt; i += blockDim.x) sA[i] = A[m0 * K + i];
    }
    __syncthreads();
    const int outs = rows * N;
    for (int g = threadIdx.x; g < (outs >> vlog); g += blockDim.x) {
      const int o0 = g << vlog;
      const int r = o0 >> nlog, n0 = o0 & (N - 1);
      uint32_t pk[4];
      for (int v = 0; v < V; ++v) {
        float cr = 0.f, ci = 0.f;
        for (int k = 0; k < K; ++k) {
          float2 a = __half22float2(sA[r * K + k]);
          float2 b = smem_b ? sB[k * N + n0 + v]
                            : make_float2(__half2float(BP[(size_t)(2 * (n0 + v)) * K2 + 2 * k]),
                                          __half2float(BP[(size_t)(2 * (n0 + v) + 1) * K2 + 2 * k]));
          cr = fmaf(a.x, b.x, fmaf(-a.y, b.y, cr));
          ci = fmaf(a.x, b.y, fmaf(a.y, b.x, ci));
        }
        __half2 h = __floats2half2_rn(cr * sc, ci * sc);
        mx = fmaxf(mx, fmaxf(fabsf(cr * sc), fabsf(ci * sc)));  // fp32 max (see gemm_tc.cuh epilogue)
        pk[v] = *reinterpret_cast<uint32_t*>(&h);
      }
      const uint64_t m = m0 + r;
      int64_t base;
      if (om.identity) {
        base = (int64_t)(m * N + n0);
      } else {
        base = 0;
        uint64_t mm = m;
        while (mm) {
          int j = __ffsll((long long)mm) - 1;
          base += om.ms[j];
          mm &= mm - 1;
        }
        for (int j = vlog; j < om.nbits; ++j)
          if ((n0 >> j) & 1) base += om.ns[j];
      }
      uint32_t* dst = reinterpret_cast<uint32_t*>(C) + base;
      if (V == 4)
        *reinterpret_cast<uint4*>(dst) = make_uint4(pk[0], pk[1], pk[2], pk[3]);
      else if (V == 2)
        *reinterpret_cast<uint2*>(dst) = make_uint2(pk[0], pk[1]);
      else
        dst[0] = pk[0];
    }
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  if (out_max && (threadIdx.x & 31) == 0) atomic_max_pos2(out_max, mx);
}

// Row-streaming variant for K*N <= 128 (K <= 16, N <= 32; see rows_ok): each thread owns RPT
// consecutive rows of A (RPT*K complex-half contiguous, 16-byte vector loads), keeps the RPT*N
// outputs in registers and, for a row-major output, stores them as one contiguous run with 256-bit
// stores (one full 32-byte sector per instruction and lane; RPT is chosen so a thread writes >= 32
// B when registers allow).  No shared memory for A, no barriers; the grid-stride loop keeps many
// rows in flight.
template <int K, int N>
struct RowsCfg {
  // K <= 2 (outer-product-like, write-bound): >= 64 output bytes per thread; larger K: >= 32 bytes
  // with <= 16 complex of A in registers (measured on C3: more rows per thread slowed K >= 4)
  static constexpr int kRptWant = K <= 2 ? (N >= 16 ? 1 : 16 / N) : (N >= 8 ? 1 : 8 / N);
  static constexpr int kRptRegs = K <= 2 ? 32 / K : (16 / K >= 1 ? 16 / K : 1);
  static constexpr int kRpt = kRptWant < kRptRegs ? kRptWant : kRptRegs;
};

template <int K, int N>
__global__ void __launch_bounds__(256) gemm_chalf_rows_kernel(uint32_t* __restrict__ C, const __half2* __restrict__ A,
                                                              const __half* __restrict__ BP, uint64_t M, int contiguous,
                                                              const float* in_max, const float* b_bound,
                                                              uint32_t* out_max, int* exp_slot, const OutMap om) {
  constexpr int R = RowsCfg<K, N>::kRpt;
  __shared__ float2 sB[K * N];
  int e = 0;
  if (in_max && in_max[0] < 0.f) return;  // scale re-run not needed (runtime.cu redo)
  if (in_max && b_bound) e = scale_exp_for(in_max[0] * b_bound[0]);
  if (exp_slot && blockIdx.x == 0 && threadIdx.x == 0) *exp_slot = e;
  const float sc = ldexpf(1.f, e);
  for (int i = threadIdx.x; i < K * N; i += blockDim.x) {
    int k = i / N, n = i - k * N;
    sB[i] = make_float2(__half2float(BP[(size_t)(2 * n) * 2 * K + 2 * k]), __half2float(BP[(size_t)(2 * n + 1) * 2 * K + 2 * k]));
  }
  __syncthreads();
  float mx = 0.f;
  const uint64_t groups = (M + R - 1) / R;
  for (uint64_t g = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; g < groups; g += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t m0 = g * R;
    const bool full = m0 + R <= M;
    float2 a[R * K];
    const __half2* ar = A + m0 * K;
    if constexpr ((R * K) % 8 == 0) {
      if (full) {
        // 256-bit loads: a lane's 32-byte piece is one full sector per instruction
#pragma unroll
        for (int q = 0; q < R * K / 8; ++q) {
          uint32_t w[8];
          asm volatile("ld.global.nc.L1::no_allocate.v8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                       : "=r"(w[0]), "=r"(w[1]), "=r"(w[2]), "=r"(w[3]), "=r"(w[4]), "=r"(w[5]), "=r"(w[6]), "=r"(w[7])
                       : "l"(reinterpret_cast<const uint32_t*>(ar) + 8 * q));
#pragma unroll
          for (int j = 0; j < 8; ++j) a[8 * q + j] = __half22float2(*reinterpret_cast<__half2*>(&w[j]));
        }
      } else {
#pragma unroll
        for (int k = 0; k < R * K; ++k) a[k] = (m0 + k / K < M) ? __half22float2(ar[k]) : make_float2(0.f, 0.f);
      }
    } else if constexpr ((R * K) % 4 == 0) {
      if (full) {
#pragma unroll
        for (int q = 0; q < R * K / 4; ++q) {
          uint4 v = __ldg(reinterpret_cast<const uint4*>(ar) + q);
          a[4 * q] = __half22float2(*reinterpret_cast<__half2*>(&v.x));
          a[4 * q + 1] = __half22float2(*reinterpret_cast<__half2*>(&v.y));
          a[4 * q + 2] = __half22float2(*reinterpret_cast<__half2*>(&v.z));
          a[4 * q + 3] = __half22float2(*reinterpret_cast<__half2*>(&v.w));
        }
      } else {
#pragma unroll
        for (int k = 0; k < R * K; ++k) a[k] = (m0 + k / K < M) ? __half22float2(ar[k]) : make_float2(0.f, 0.f);
      }
    } else {
#pragma unroll
      for (int k = 0; k < R * K; ++k) a[k] = (m0 + k / K < M) ? __half22float2(ar[k]) : make_float2(0.f, 0.f);
    }
    uint32_t out[R * N];
#pragma unroll
    for (int r = 0; r < R; ++r)
#pragma unroll
      for (int n = 0; n < N; ++n) {
        float cr = 0.f, ci = 0.f;
#pragma unroll
        for (int k = 0; k < K; ++k) {
          float2 b = sB[k * N + n];
          cr = fmaf(a[r * K + k].x, b.x, fmaf(-a[r * K + k].y, b.y, cr));
          ci = fmaf(a[r * K + k].x, b.y, fmaf(a[r * K + k].y, b.x, ci));
        }
        __half2 h = __floats2half2_rn(cr * sc, ci * sc);
        if (r == 0 || m0 + r < M) mx = fmaxf(mx, fmaxf(fabsf(cr * sc), fabsf(ci * sc)));  // fp32 max
        out[r * N + n] = *reinterpret_cast<uint32_t*>(&h);
      }
    if (om.identity && full) {
      // the thread's R*N outputs are one contiguous run
      uint32_t* dst = C + m0 * N;
      if constexpr (R * N >= 8) {
#pragma unroll
        for (int q = 0; q < R * N; q += 8)
          asm volatile("st.global.v8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(dst + q), "r"(out[q]), "r"(out[q + 1]),
                       "r"(out[q + 2]), "r"(out[q + 3]), "r"(out[q + 4]), "r"(out[q + 5]), "r"(out[q + 6]),
                       "r"(out[q + 7])
                       : "memory");
      } else if constexpr (R * N == 4) {
        *reinterpret_cast<uint4*>(dst) = make_uint4(out[0], out[1], out[2], out[3]);
      } else if constexpr (R * N == 2) {
        *reinterpret_cast<uint2*>(dst) = make_uint2(out[0], out[1]);
      } else {
        dst[0] = out[0];
      }
      continue;
    }
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const uint64_t m = m0 + r;
      if (m >= M) break;
      int64_t base;
      if (om.identity) {
        base = (int64_t)(m * N);
      } else {
        base = 0;
        uint64_t mm = m;
        while (mm) {
          int j = __ffsll((long long)mm) - 1;
          base += om.ms[j];
          mm &= mm - 1;
        }
      }
      uint32_t* dst = C + base;
      if (contiguous) {
        if constexpr (N >= 4) {
#pragma unroll
          for (int q = 0; q < N / 4; ++q)
            reinterpret_cast<uint4*>(dst)[q] =
                make_uint4(out[r * N + 4 * q], out[r * N + 4 * q + 1], out[r * N + 4 * q + 2], out[r * N + 4 * q + 3]);
        } else if constexpr (N == 2) {
          *reinterpret_cast<uint2*>(dst) = make_uint2(out[r * N], out[r * N + 1]);
        } else {
          dst[0] = out[r * N];
        }
      } else {
#pragma unroll
        for (int n = 0; n < N; ++n) {
          int64_t o = 0;
          for (int j = 0; j < om.nbits; ++j)
            if ((n >> j) & 1) o += om.ns[j];
          dst[o] = out[r * N + n];
        }
      }
    }
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  if (out_max && (threadIdx.x & 31) == 0) atomic_max_pos2(out_max, mx);
}

template <int K, int N>
static void launch_rows(__half2* c, const __half2* a, const __half* bp, uint64_t M, int contiguous, const float* in_max,
                        const float* b_bound, uint32_t* out_max, int* exp_slot, const OutMap& om, cudaStream_t s) {
  constexpr int R = RowsCfg<K, N>::kRpt;
  uint64_t blocks = std::min<uint64_t>(((M + R - 1) / R + 255) / 256, 148ull * 16);
  if (blocks == 0) blocks = 1;
  gemm_chalf_rows_kernel<K, N><<<(unsigned)blocks, 256, 0, s>>>(reinterpret_cast<uint32_t*>(c), a, bp, M, contiguous,
                                                                in_max, b_bound, out_max, exp_slot, om);
}

template <int K>
static bool dispatch_rows_n(uint32_t N, __half2* c, const __half2* a, const __half* bp, uint64_t M, int contiguous,
                            const float* in_max, const float* b_bound, uint32_t* out_max, int* exp_slot,
                            const OutMap& om, cudaStream_t s) {
  switch (N) {
    case 1: launch_rows<K, 1>(c, a, bp, M, contiguous, in_max, b_bound, out_max, exp_slot, om, s); return true;
    case 2: launch_rows<K, 2>(c, a, bp, M, contiguous, in_max, b_bound, out_max, exp_slot, om, s); return true;
    case 4: launch_rows<K, 4>(c, a, bp, M, contiguous, in_max, b_bound, out_max, exp_slot, om, s); return true;
    case 8: launch_rows<K, 8>(c, a, bp, M, contiguous, in_max, b_bound, out_max, exp_slot, om, s); return true;
  }
  if constexpr (K <= 8) {
    if (N == 16) {
      launch_rows<K, 16>(c, a, bp, M, contiguous, in_max, b_bound, out_max, exp_slot, om, s);
      return true;
    }
  }
  if constexpr (K <= 4) {
    if (N == 32) {
      launch_rows<K, 32>(c, a, bp, M, contiguous, in_max, b_bound, out_max, exp_slot, om, s);
      return true;
    }
  }
  return false;
}

// Shapes the row-streaming kernel covers (the lowering's tensor-core rule mirrors this, plan.cpp).
static bool rows_ok(uint32_t K, uint32_t N) { return K <= 16 && N <= 32 && K * N <= 128; }

void launch_gemm_chalf_simt(__half2* c, const __half2* a, const __half* bp, uint64_t M, uint32_t K, uint32_t N,
                            const float* in_max, const float* b_bound, uint32_t* out_max, int* exp_slot,
                            const OutMap* om_in, cudaStream_t s) {
  g_last_kern = "simt";
  if (K > (uint32_t)kTileCplx) throw TnError{TN_E_UNSUPPORTED, "SIMT complex-half GEMM: K > 4096"};
  OutMap om = om_in ? *om_in : identity_map(M, N);
  int nlog = 0;
  while ((1u << nlog) < N) ++nlog;
  int run = 0;
  if (om.identity)
    run = nlog;
  else
    while (run < om.nbits && om.ns[run] == ((int64_t)1 << run)) ++run;
  if (rows_ok(K, N)) {
    const int contiguous = run >= nlog;
    bool ok = false;
    switch (K) {
      case 16: ok = dispatch_rows_n<16>(N, c, a, bp, M, contiguous, in_max, b_bound, out_max, exp_slot, om, s); break;
      case 1: ok = dispatch_rows_n<1>(N, c, a, bp, M, contiguous, in_max, b_bound, out_max, exp_slot, om, s); break;
      case 2: ok = dispatch_rows_n<2>(N, c, a, bp, M, contiguous, in_max, b_bound, out_max, exp_slot, om, s); break;
      case 4: ok = dispatch_rows_n<4>(N, c, a, bp, M, contiguous, in_max, b_bound, out_max, exp_slot, om, s); break;
      case 8: ok = dispatch_rows_n<8>(N, c, a, bp, M, contiguous, in_max, b_bound, out_max, exp_slot, om, s); break;
    }
    if (ok) {
      TN_CUDA(cudaGetLastError());
      return;
    }
  }
  // rows per tile: A tile of <= kTileCplx complex, at least one row
  int rows_log = 0;
  while ((2ull << rows_log) * K <= (uint64_t)kTileCplx && (2ull << rows_log) <= 1024) ++rows_log;
  uint64_t tiles = (M + (1ull << rows_log) - 1) >> rows_log;
  uint64_t blocks = std::min<uint64_t>(tiles, 148ull * 8);
  if (blocks == 0) blocks = 1;
  gemm_chalf_simt_kernel<<<(unsigned)blocks, 256, 0, s>>>(c, a, bp, M, (int)K, (int)N, rows_log, run, in_max, b_bound,
                                                           out_max, exp_slot, om);
  TN_CUDA(cudaGetLastError());
}

// Gather-batched complex-half GEMM for the small steps of the sparse-state tail (K < 4, N < 8 or
// fewer than 128 rows per entry, where the tcgen05 batched launch does not apply): thread per output
// element, C[b][m][n] = 2^e sum_k A[ia[b]][m][k] B_ib[b][k][n] with B read from its Eq. 6 B_P block
// (Re b at row 2n, column 2k; Im b at row 2n+1), fp32 accumulation, same scale rule and max record as
// the other stem GEMMs.  One launch per tail step instead of one per batch entry.
__global__ void __launch_bounds__(256) gemm_chalf_batched_simt_kernel(
    __half2* __restrict__ C, const __half2* __restrict__ A, const __half* __restrict__ BP, uint64_t M, int K, int N,
    uint64_t n_out, const int* __restrict__ ia, const int* __restrict__ ib, uint64_t b_blk_halfs,
    const float* in_max, const float* b_bound, uint32_t* out_max, int* exp_slot) {
  if (in_max && in_max[0] < 0.f) return;  // scale re-run not needed (runtime.cu redo)
  int e = 0;
  if (in_max && b_bound) e = scale_exp_for(in_max[0] * b_bound[0]);
  if (exp_slot && blockIdx.x == 0 && threadIdx.x == 0) *exp_slot = e;
  const float sc = ldexpf(1.f, e);
  const int K2 = 2 * K;
  const uint64_t per = M * (uint64_t)N, total = per * n_out;
  float mx = 0.f;
  for (uint64_t idx = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; idx < total;
       idx += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t b = idx / per, r = idx % per, m = r / N;
    const int n = (int)(r % N);
    const __half2* a = A + ((uint64_t)ia[b] * M + m) * K;
    const __half* bp = BP + (uint64_t)ib[b] * b_blk_halfs;
    float cr = 0.f, ci = 0.f;
    for (int k = 0; k < K; ++k) {
      const float2 av = __half22float2(a[k]);
      const float br = __half2float(bp[(size_t)(2 * n) * K2 + 2 * k]);
      const float bi = __half2float(bp[(size_t)(2 * n + 1) * K2 + 2 * k]);
      cr = fmaf(av.x, br, fmaf(-av.y, bi, cr));
      ci = fmaf(av.x, bi, fmaf(av.y, br, ci));
    }
    C[idx] = __floats2half2_rn(cr * sc, ci * sc);
    mx = fmaxf(mx, fmaxf(fabsf(cr * sc), fabsf(ci * sc)));
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  if (out_max && (threadIdx.x & 31) == 0) atomic_max_pos2(out_max, mx);
}

void launch_gemm_chalf_batched_simt(__half2* c, const __half2* a, const __half* bp, uint64_t M, uint32_t K, uint32_t N,
                                    uint64_t n_out, const int* ia, const int* ib, uint64_t b_blk_halfs,
                                    const float* in_max, const float* b_bound, uint32_t* out_max, int* exp_slot,
                                    cudaStream_t s) {
  const uint64_t total = M * N * n_out;
  if (total == 0) return;
  const uint64_t blocks = std::min<uint64_t>((total + 255) / 256, 148ull * 16);
  gemm_chalf_batched_simt_kernel<<<(unsigned)blocks, 256, 0, s>>>(c, a, bp, M, (int)K, (int)N, n_out, ia, ib, b_blk_halfs,
                                                                  in_max, b_bound, out_max, exp_slot);
  TN_CUDA(cudaGetLastError());
}

}  // namespace tn
