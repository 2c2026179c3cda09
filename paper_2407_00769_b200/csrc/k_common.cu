// Common-type contractions and stem-operand preparation.
//
// * contract_c64: one pairwise contraction of MB-scale non-stem tensors ("Common Type"),
//   Eq. 3 with arbitrary strided operands (slicing = a base offset), complex64
//   with fp32 accumulation.  Thread per output element; the reduce index walks a Gray code so each
//   iteration changes one stride.
// * gather_kn: lay a branch tensor out as the dense [K][N] operand of its stem step.
// * pad_b: Eq. 6 padding (reading C-A6) to the fp16 K-major B_P [2N][2K] with an exact
//   power-of-two scale (reading C-A8), and the column 1-norm bound used to scale the step output.
// * c64_to_chalf: stem entry, complex64 -> interleaved fp16 with an exact power-of-two scale.
#include <cstring>

#include "common.cuh"

namespace tn {

__device__ __forceinline__ void atomic_max_pos(uint32_t* addr, float v) {
  // v >= 0: IEEE bit patterns of non-negative floats order like unsigned integers
  atomicMax(addr, __float_as_uint(v));
}

__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

__global__ void contract_c64_kernel(const ContractArgs args, uint64_t n_out_elems) {
  const uint64_t nred = 1ull << args.n_red;
  const float2* A = args.a + slice_offset(args.sa);
  const float2* B = args.b + slice_offset(args.sb);
  for (uint64_t o = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; o < n_out_elems;
       o += (uint64_t)gridDim.x * blockDim.x) {
    int64_t oa = 0, ob = 0;
    for (int j = 0; j < args.n_out; ++j)
      if (o >> j & 1) {
        oa += args.out_sa[j];
        ob += args.out_sb[j];
      }
    float2 acc = make_float2(0.f, 0.f);
    uint64_t g = 0;
    for (uint64_t r = 0; r < nred; ++r) {
      if (r) {
        int j = __ffsll((long long)r) - 1;  // Gray code: bit j flips
        g ^= 1ull << j;
        if (g >> j & 1) {
          oa += args.red_sa[j];
          ob += args.red_sb[j];
        } else {
          oa -= args.red_sa[j];
          ob -= args.red_sb[j];
        }
      }
      float2 x = A[oa], y = B[ob];
      acc.x = fmaf(x.x, y.x, fmaf(-x.y, y.y, acc.x));
      acc.y = fmaf(x.x, y.y, fmaf(x.y, y.x, acc.y));
    }
    args.c[o] = acc;
  }
}

// Level-batched common phase: every contraction of one tree level (independent of each other) in
// one launch.  Block b of the launch belongs to node i with start[i] <= b < start[i+1] and works on
// that node's outputs [(b - start[i]) * 256, ...) with a grid stride of the node's block count.
__global__ void contract_c64_level_kernel(const ContractArgs* __restrict__ args, const uint32_t* __restrict__ start,
                                          int nnodes) {
  int lo = 0, hi = nnodes - 1;
  while (lo < hi) {  // last node whose start <= blockIdx.x
    const int mid = (lo + hi + 1) >> 1;
    if (start[mid] <= blockIdx.x) lo = mid; else hi = mid - 1;
  }
  const ContractArgs& a = args[lo];
  const uint32_t nb = start[lo + 1] - start[lo], b = blockIdx.x - start[lo];
  const uint64_t n_out = 1ull << a.n_out, nred = 1ull << a.n_red;
  const float2* A = a.a + slice_offset(a.sa);
  const float2* B = a.b + slice_offset(a.sb);
  for (uint64_t o = b * (uint64_t)blockDim.x + threadIdx.x; o < n_out; o += (uint64_t)nb * blockDim.x) {
    int64_t oa = 0, ob = 0;
    for (int j = 0; j < a.n_out; ++j)
      if (o >> j & 1) {
        oa += a.out_sa[j];
        ob += a.out_sb[j];
      }
    float2 acc = make_float2(0.f, 0.f);
    uint64_t g = 0;
    for (uint64_t r = 0; r < nred; ++r) {
      if (r) {
        int j = __ffsll((long long)r) - 1;  // Gray code: bit j flips
        g ^= 1ull << j;
        if (g >> j & 1) {
          oa += a.red_sa[j];
          ob += a.red_sb[j];
        } else {
          oa -= a.red_sa[j];
          ob -= a.red_sb[j];
        }
      }
      float2 x = A[oa], y = B[ob];
      acc.x = fmaf(x.x, y.x, fmaf(-x.y, y.y, acc.x));
      acc.y = fmaf(x.x, y.y, fmaf(x.y, y.x, acc.y));
    }
    a.c[o] = acc;
  }
}

void launch_contract_c64_level(const ContractArgs* d_args, const uint32_t* d_start, int nnodes, uint32_t blocks,
                               cudaStream_t s) {
  if (nnodes <= 0 || blocks == 0) return;
  contract_c64_level_kernel<<<blocks, 256, 0, s>>>(d_args, d_start, nnodes);
  TN_CUDA(cudaGetLastError());
}

void launch_contract_c64(const ContractArgs& a, cudaStream_t s) {
  uint64_t n = 1ull << a.n_out;
  int threads = 256;
  uint64_t blocks = (n + threads - 1) / threads;
  if (blocks > 148 * 16) blocks = 148 * 16;
  contract_c64_kernel<<<(unsigned)blocks, threads, 0, s>>>(a, n);
  TN_CUDA(cudaGetLastError());
}

__global__ void gather_kn_kernel(const GatherArgs g) {
  const uint64_t n = 1ull << (g.klog + g.nlog);
  const float2* src = g.src + slice_offset(g.ss);
  const uint64_t nmask = (1ull << g.nlog) - 1;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x) {
    uint64_t k = i >> g.nlog, nn = i & nmask;
    int64_t off = 0;
    for (int j = 0; j < g.klog; ++j)
      if (k >> j & 1) off += g.sk[j];
    for (int j = 0; j < g.nlog; ++j)
      if (nn >> j & 1) off += g.sn[j];
    g.dst[i] = src[off];
  }
}

void launch_gather_kn(const GatherArgs& g, cudaStream_t s) {
  uint64_t n = 1ull << (g.klog + g.nlog);
  uint64_t blocks = (n + 255) / 256;
  if (blocks > 148 * 16) blocks = 148 * 16;
  gather_kn_kernel<<<(unsigned)blocks, 256, 0, s>>>(g);
  TN_CUDA(cudaGetLastError());
}

template <typename T>
__global__ void max_abs_kernel(const T* __restrict__ x, uint64_t n, uint32_t* out) {
  float m = 0.f;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x)
    m = fmaxf(m, fabsf((float)x[i]));
  m = warp_max(m);
  if ((threadIdx.x & 31) == 0) atomic_max_pos(out, m);
}

void launch_max_abs_f32(const float* x, uint64_t n, uint32_t* out_bits, cudaStream_t s) {
  uint64_t blocks = (n + 255) / 256;
  if (blocks > 148 * 8) blocks = 148 * 8;
  if (blocks == 0) blocks = 1;
  max_abs_kernel<float><<<(unsigned)blocks, 256, 0, s>>>(x, n, out_bits);
  TN_CUDA(cudaGetLastError());
}

void launch_max_abs_f16(const __half* x, uint64_t n, uint32_t* out_bits, cudaStream_t s) {
  uint64_t blocks = (n + 255) / 256;
  if (blocks > 148 * 8) blocks = 148 * 8;
  if (blocks == 0) blocks = 1;
  max_abs_kernel<__half><<<(unsigned)blocks, 256, 0, s>>>(x, n, out_bits);
  TN_CUDA(cudaGetLastError());
}

// One warp per column n of B: writes rows (n,0) and (n,1) of B_P [2N][2K].
__global__ void pad_b_kernel(__half* __restrict__ bp, const float2* __restrict__ b, int klog, int nlog,
                             const uint32_t* bmax_bits, float* b_bound, int* exp_slot) {
  const int K = 1 << klog, N = 1 << nlog;
  const int t = bmax_bits ? scale_exp_for(__uint_as_float(*bmax_bits)) : 0;
  if (exp_slot && blockIdx.x == 0 && threadIdx.x == 0) *exp_slot = t;
  const float sc = ldexpf(1.f, t);
  const int warps = blockDim.x >> 5, lane = threadIdx.x & 31;
  for (int n = blockIdx.x * warps + (threadIdx.x >> 5); n < N; n += gridDim.x * warps) {
    float l1 = 0.f;
    __half2* r0 = reinterpret_cast<__half2*>(bp + (size_t)(2 * n) * 2 * K);
    __half2* r1 = reinterpret_cast<__half2*>(bp + (size_t)(2 * n + 1) * 2 * K);
    for (int k = lane; k < K; k += 32) {
      float2 v = b[(size_t)k * N + n];
      __half re = __float2half_rn(v.x * sc), im = __float2half_rn(v.y * sc);
      __half nim = __hneg(im);
      r0[k] = __halves2half2(re, nim);   // c=0: (Re b, -Im b)
      r1[k] = __halves2half2(im, re);    // c=1: (Im b,  Re b)
      l1 += fabsf(__half2float(re)) + fabsf(__half2float(im));
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) l1 += __shfl_xor_sync(0xffffffffu, l1, o);
    if (lane == 0 && b_bound) atomic_max_pos(reinterpret_cast<uint32_t*>(b_bound), l1);
  }
}

void launch_pad_b(__half* bp, const float2* b, int klog, int nlog, const uint32_t* bmax_bits,
                  float* b_bound, int* exp_slot, cudaStream_t s) {
  int N = 1 << nlog;
  int blocks = (N + 7) / 8;
  if (blocks > 148 * 4) blocks = 148 * 4;
  pad_b_kernel<<<blocks, 256, 0, s>>>(bp, b, klog, nlog, bmax_bits, b_bound, exp_slot);
  TN_CUDA(cudaGetLastError());
}

// One warp per column n of B: rows (n,0) = Re b[:, n] and (n,1) = Im b[:, n] of B' [2N][K] (the
// MN-major GEMM's operand, k_gemm_tc2.cu); the bound is the same column 1-norm as pad_b_kernel's.
__global__ void pad_b_mn_kernel(__half* __restrict__ bpm, const float2* __restrict__ b, int klog, int nlog,
                                const uint32_t* bmax_bits, float* b_bound, int* exp_slot) {
  const int K = 1 << klog, N = 1 << nlog;
  const int t = bmax_bits ? scale_exp_for(__uint_as_float(*bmax_bits)) : 0;
  if (exp_slot && blockIdx.x == 0 && threadIdx.x == 0) *exp_slot = t;
  const float sc = ldexpf(1.f, t);
  const int warps = blockDim.x >> 5, lane = threadIdx.x & 31;
  for (int n = blockIdx.x * warps + (threadIdx.x >> 5); n < N; n += gridDim.x * warps) {
    float l1 = 0.f;
    __half* r0 = bpm + (size_t)(2 * n) * K;
    __half* r1 = bpm + (size_t)(2 * n + 1) * K;
    for (int k = lane; k < K; k += 32) {
      float2 v = b[(size_t)k * N + n];
      __half re = __float2half_rn(v.x * sc), im = __float2half_rn(v.y * sc);
      r0[k] = re;
      r1[k] = im;
      l1 += fabsf(__half2float(re)) + fabsf(__half2float(im));
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) l1 += __shfl_xor_sync(0xffffffffu, l1, o);
    if (lane == 0 && b_bound) atomic_max_pos(reinterpret_cast<uint32_t*>(b_bound), l1);
  }
}

void launch_pad_b_mn(__half* bpm, const float2* b, int klog, int nlog, const uint32_t* bmax_bits, float* b_bound,
                     int* exp_slot, cudaStream_t s) {
  int N = 1 << nlog;
  int blocks = (N + 7) / 8;
  if (blocks > 148 * 4) blocks = 148 * 4;
  pad_b_mn_kernel<<<blocks, 256, 0, s>>>(bpm, b, klog, nlog, bmax_bits, b_bound, exp_slot);
  TN_CUDA(cudaGetLastError());
}

// B' = blockdiag(B_P, ..., B_P) (fold copies): B' [max(f 2N, 16)][f 2K] fp16 from B_P [2N][2K]
__global__ void fold_b_kernel(__half* __restrict__ bf, const __half* __restrict__ bp, int k2, int n2, int f,
                              uint64_t rows) {
  const uint64_t cols = (uint64_t)f * k2, total = rows * cols;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < total; i += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t r = i / cols, c = i % cols;
    const uint64_t bi = r / n2, bj = c / k2;
    bf[i] = (r < (uint64_t)f * n2 && bi == bj) ? bp[(r % n2) * k2 + (c % k2)] : __float2half_rn(0.f);
  }
}

void launch_fold_b(__half* bf, const __half* bp, int klog, int nlog, int f, cudaStream_t s) {
  const int k2 = 2 << klog, n2 = 2 << nlog;
  const uint64_t rows = std::max<uint64_t>((uint64_t)f * n2, 16);
  const uint64_t total = rows * (uint64_t)f * k2;
  const int blocks = (int)std::min<uint64_t>((total + 255) / 256, 148 * 4);
  fold_b_kernel<<<blocks, 256, 0, s>>>(bf, bp, k2, n2, f, rows);
  TN_CUDA(cudaGetLastError());
}

__global__ void c64_to_chalf_kernel(__half2* __restrict__ dst, const float2* __restrict__ src, uint64_t n,
                                    const uint32_t* max_bits, int* exp_slot, uint32_t* out_max) {
  const int e = max_bits ? scale_exp_for(__uint_as_float(*max_bits)) : 0;
  if (exp_slot && blockIdx.x == 0 && threadIdx.x == 0) *exp_slot = e;
  const float sc = ldexpf(1.f, e);
  float m = 0.f;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x) {
    float2 v = src[i];
    __half2 h = __floats2half2_rn(v.x * sc, v.y * sc);
    dst[i] = h;
    float2 hf = __half22float2(h);
    m = fmaxf(m, fmaxf(fabsf(hf.x), fabsf(hf.y)));
  }
  m = warp_max(m);
  if (out_max && (threadIdx.x & 31) == 0) atomic_max_pos(out_max, m);
}

void launch_c64_to_chalf(__half2* dst, const float2* src, uint64_t n, const uint32_t* max_bits, int* exp_slot,
                         uint32_t* out_max_bits, cudaStream_t s) {
  uint64_t blocks = (n + 255) / 256;
  if (blocks > 148 * 8) blocks = 148 * 8;
  if (blocks == 0) blocks = 1;
  c64_to_chalf_kernel<<<(unsigned)blocks, 256, 0, s>>>(dst, src, n, max_bits, exp_slot, out_max_bits);
  TN_CUDA(cudaGetLastError());
}

// complex64 path (C-A8 for fp32): column bound of B and the scaled stem entry
__global__ void colnorm_c64_kernel(const float2* __restrict__ b, int klog, int nlog, float* b_bound) {
  const int K = 1 << klog, N = 1 << nlog;
  const int warps = blockDim.x >> 5, lane = threadIdx.x & 31;
  for (int n = blockIdx.x * warps + (threadIdx.x >> 5); n < N; n += gridDim.x * warps) {
    float l1 = 0.f;
    for (int k = lane; k < K; k += 32) {
      const float2 v = b[(size_t)k * N + n];
      l1 += fabsf(v.x) + fabsf(v.y);
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) l1 += __shfl_xor_sync(0xffffffffu, l1, o);
    if (lane == 0) atomic_max_pos(reinterpret_cast<uint32_t*>(b_bound), l1);
  }
}

void launch_colnorm_c64(const float2* b, int klog, int nlog, float* b_bound, cudaStream_t s) {
  const int N = 1 << nlog;
  int blocks = (N + 7) / 8;
  if (blocks > 148 * 4) blocks = 148 * 4;
  colnorm_c64_kernel<<<blocks, 256, 0, s>>>(b, klog, nlog, b_bound);
  TN_CUDA(cudaGetLastError());
}

__global__ void c64_scale_kernel(float2* __restrict__ dst, const float2* __restrict__ src, uint64_t n,
                                 const uint32_t* max_bits, int* exp_slot, uint32_t* out_max) {
  const int e = max_bits ? scale_exp_for(__uint_as_float(*max_bits)) : 0;
  if (exp_slot && blockIdx.x == 0 && threadIdx.x == 0) *exp_slot = e;
  const float sc = ldexpf(1.f, e);
  float m = 0.f;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    const float2 v = make_float2(src[i].x * sc, src[i].y * sc);
    dst[i] = v;
    m = fmaxf(m, fmaxf(fabsf(v.x), fabsf(v.y)));
  }
  m = warp_max(m);
  if (out_max && (threadIdx.x & 31) == 0) atomic_max_pos(out_max, m);
}

void launch_c64_scale(float2* dst, const float2* src, uint64_t n, const uint32_t* max_bits, int* exp_slot,
                      uint32_t* out_max_bits, cudaStream_t s) {
  uint64_t blocks = (n + 255) / 256;
  if (blocks > 148 * 8) blocks = 148 * 8;
  if (blocks == 0) blocks = 1;
  c64_scale_kernel<<<(unsigned)blocks, 256, 0, s>>>(dst, src, n, max_bits, exp_slot, out_max_bits);
  TN_CUDA(cudaGetLastError());
}

__global__ void set_u64_kernel(uint64_t* p, uint64_t v) { *p = v; }

void launch_set_u64(uint64_t* p, uint64_t v, cudaStream_t s) {
  set_u64_kernel<<<1, 1, 0, s>>>(p, v);
  TN_CUDA(cudaGetLastError());
}

// Loopback transport (runtime.cu): max over the virtual ranks' 1-float slots, written to `dst`.
// The slots hold non-negative float bits (atomicMax order); a concurrent reader of `dst` sees its
// old value or the maximum, both valid bounds for every rank.
__global__ void max_slots_kernel(float* dst, MaxSlots src) {
  float m = 0.f;
  for (int r = 0; r < src.n; ++r) m = fmaxf(m, *src.p[r]);
  *dst = m;
}

void launch_max_slots(float* dst, const MaxSlots& src, cudaStream_t s) {
  max_slots_kernel<<<1, 1, 0, s>>>(dst, src);
  TN_CUDA(cudaGetLastError());
}

// Scale re-run decision (reading C-A28, revised): a GEMM's output exponent comes from a bound
// (max|A| x max column 1-norm of B_P) so |C| <= 2^14 is guaranteed, but heavy cancellation can leave
// the actual max |C| far below it and push the fp16 output into subnormals / zero.  When the realised
// max (out_max, already scaled) is below 2^(14 - bits), the GEMM is run again from the same input
// with an input max smaller by exactly 2^delta (delta = the exponent that brings out_max near 2^14),
// i.e. an output exponent larger by delta; otherwise the re-run launch exits at once (-1).
// The re-run's outputs are exactly the first pass's fp32 values times 2^delta, so the realised max is
// updated here (no second max reduction, and no second all-reduce across ranks).
__global__ void redo_check_kernel(uint32_t* out_max, const float* in_max, float* redo_in, int bits) {
  const float m = __uint_as_float(*out_max);
  const int d = scale_exp_for(m);
  const bool redo = m > 0.f && d >= bits;
  *redo_in = redo ? ldexpf(*in_max, -d) : -1.f;
  if (redo) *out_max = __float_as_uint(ldexpf(m, d));
}

void launch_redo_check(uint32_t* out_max, const float* in_max, float* redo_in, int bits, cudaStream_t s) {
  redo_check_kernel<<<1, 1, 0, s>>>(out_max, in_max, redo_in, bits);
  TN_CUDA(cudaGetLastError());
}

void launch_copy_c64(float2* dst, const float2* src, uint64_t n, cudaStream_t s) {
  TN_CUDA(cudaMemcpyAsync(dst, src, n * sizeof(float2), cudaMemcpyDeviceToDevice, s));
}

}  // namespace tn
