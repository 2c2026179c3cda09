// Post-selection (keep the most probable member of each correlated subspace;
// reading C-A23: ties go to the lexicographically smallest bitstring, i.e. the smallest MEMBER
// index in member (open-leg) order, whatever the storage layout).  One CTA per subspace scans its
// 2^r complex-half amplitudes (probability |a|^2 in fp32; the subspace's power-of-two scale does
// not change the argmax), maps each layout index to its member index (bit permutation), and
// reduces (p, member) with ties to the smaller member.  A NaN probability ranks below every number.
#include "common.cuh"

namespace tn {

__device__ __forceinline__ bool better(float p, uint64_t o, float bp, uint64_t bo) {
  return p > bp || (p == bp && o < bo);
}

__global__ void top1_chalf_kernel(const __half2* __restrict__ amps, uint64_t members, const __grid_constant__ MemberMap mm,
                                  uint64_t* __restrict__ top) {
  const __half2* a = amps + blockIdx.x * members;
  float best = -2.f;  // below the NaN rank (-1): every subspace yields a valid member
  uint64_t bo = ~0ull;
  for (uint64_t i = threadIdx.x; i < members; i += blockDim.x) {
    float2 v = __half22float2(a[i]);
    float pr = v.x * v.x + v.y * v.y;
    if (pr != pr) pr = -1.f;
    uint64_t o = 0;
    for (int t = 0; t < mm.r; ++t) o |= ((i >> mm.src_bit[t]) & 1ull) << (mm.r - 1 - t);
    if (better(pr, o, best, bo)) {
      best = pr;
      bo = o;
    }
  }
  __shared__ float sp[32];
  __shared__ uint64_t si[32];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
  for (int off = 16; off; off >>= 1) {
    float op = __shfl_xor_sync(0xffffffffu, best, off);
    uint64_t oo = __shfl_xor_sync(0xffffffffu, bo, off);
    if (better(op, oo, best, bo)) {
      best = op;
      bo = oo;
    }
  }
  if (lane == 0) {
    sp[w] = best;
    si[w] = bo;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int k = 1; k < (int)(blockDim.x >> 5); ++k)
      if (better(sp[k], si[k], best, bo)) {
        best = sp[k];
        bo = si[k];
      }
    top[blockIdx.x] = bo;
  }
}

void launch_top1_chalf(const __half2* amps, uint64_t n_sub, uint64_t members, const MemberMap& mm, uint64_t* top,
                       cudaStream_t s) {
  if (n_sub == 0) return;
  top1_chalf_kernel<<<(unsigned)n_sub, 256, 0, s>>>(amps, members, mm, top);
  TN_CUDA(cudaGetLastError());
}

}  // namespace tn
