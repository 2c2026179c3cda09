// SIMT stem GEMMs.
// * gemm_c64: the complex64 (TN_CFLOAT) stem GEMM C[M,N] = A[M,K] B[K,N] with true fp32 FMA
//   (reading c.5: TF32 would miss the 1e-5 bound).  64x64 complex tile, 256 threads, 4x4 per
//   thread, operands staged through shared memory.
// * gemm_chalf_simt: complex-half stem steps whose K or N is below the tcgen05 minimum
//   (2K or 2N < 16): memory-bound, thread per output element, fp32 accumulation, B read from the
//   same Eq. 6 padded B_P the tensor-core path uses, same power-of-two output scaling (C-A8).
#include "common.cuh"

namespace tn {

constexpr int TM = 64, TN_ = 64, TK = 8;

__global__ void __launch_bounds__(256) gemm_c64_kernel(float2* __restrict__ C, const float2* __restrict__ A,
                                                       const float2* __restrict__ B, uint64_t M, int K, int N) {
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
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      int gn = n0 + tx + 16 * j;
      if (gn < N) C[gm * N + gn] = acc[i][j];
    }
  }
}

void launch_gemm_c64(float2* c, const float2* a, const float2* b, uint64_t M, uint32_t K, uint32_t N,
                     cudaStream_t s) {
  uint64_t gy = (M + TM - 1) / TM;
  if (gy > 65535ull * 1024) throw TnError{TN_E_UNSUPPORTED, "gemm_c64: M too large"};
  dim3 grid((N + TN_ - 1) / TN_, 1, 1);
  // fold huge M into grid.y chunks
  const uint64_t maxy = 65535;
  for (uint64_t y0 = 0; y0 < gy; y0 += maxy) {
    uint64_t ny = std::min<uint64_t>(maxy, gy - y0);
    grid.y = (unsigned)ny;
    uint64_t moff = y0 * TM;
    gemm_c64_kernel<<<grid, 256, 0, s>>>(c + moff * N, a + moff * K, b, M - moff, (int)K, (int)N);
  }
  TN_CUDA(cudaGetLastError());
}

__device__ __forceinline__ void atomic_max_pos2(uint32_t* addr, float v) { atomicMax(addr, __float_as_uint(v)); }

__global__ void __launch_bounds__(256) gemm_chalf_simt_kernel(__half2* __restrict__ C, const __half2* __restrict__ A,
                                                              const __half* __restrict__ BP, uint64_t M, int K, int N,
                                                              const float* in_max, const float* b_bound,
                                                              uint32_t* out_max, int* exp_slot) {
  int e = 0;
  if (in_max && b_bound) e = scale_exp_for(in_max[0] * b_bound[0]);
  if (exp_slot && blockIdx.x == 0 && threadIdx.x == 0) *exp_slot = e;
  const float sc = ldexpf(1.f, e);
  const uint64_t total = M * (uint64_t)N;
  const int K2 = 2 * K;
  float mx = 0.f;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < total;
       i += (uint64_t)gridDim.x * blockDim.x) {
    uint64_t m = i / N;
    int n = (int)(i - m * N);
    const __half2* a = A + m * K;
    const __half* b0 = BP + (size_t)(2 * n) * K2;      // (Re b, -Im b) pairs
    const __half* b1 = BP + (size_t)(2 * n + 1) * K2;  // (Im b,  Re b) pairs
    float cr = 0.f, ci = 0.f;
    for (int k = 0; k < K; ++k) {
      float2 av = __half22float2(a[k]);
      float br = __half2float(b0[2 * k]), bi = __half2float(b1[2 * k]);
      cr = fmaf(av.x, br, fmaf(-av.y, bi, cr));
      ci = fmaf(av.x, bi, fmaf(av.y, br, ci));
    }
    __half2 h = __floats2half2_rn(cr * sc, ci * sc);
    C[i] = h;
    float2 hf = __half22float2(h);
    mx = fmaxf(mx, fmaxf(fabsf(hf.x), fabsf(hf.y)));
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  if (out_max && (threadIdx.x & 31) == 0) atomic_max_pos2(out_max, mx);
}

void launch_gemm_chalf_simt(__half2* c, const __half2* a, const __half* bp, uint64_t M, uint32_t K, uint32_t N,
                            const float* in_max, const float* b_bound, uint32_t* out_max, int* exp_slot,
                            cudaStream_t s) {
  uint64_t total = M * (uint64_t)N;
  uint64_t blocks = (total + 255) / 256;
  if (blocks > 148 * 16) blocks = 148 * 16;
  if (blocks == 0) blocks = 1;
  gemm_chalf_simt_kernel<<<(unsigned)blocks, 256, 0, s>>>(c, a, bp, M, (int)K, (int)N, in_max, b_bound, out_max,
                                                           exp_slot);
  TN_CUDA(cudaGetLastError());
}

}  // namespace tn
