// Post-selection (keep the most probable member of each correlated subspace;
// reading C-A23: ties go to the smaller index).  One CTA per subspace scans its 2^q complex-half
// amplitudes (probability |a|^2 in fp32; the subspace's power-of-two scale does not change the
// argmax) and reduces (p, index) with ties to the smaller index.
#include "common.cuh"

namespace tn {

__global__ void top1_chalf_kernel(const __half2* __restrict__ amps, uint64_t members, uint64_t* __restrict__ top) {
  const __half2* a = amps + blockIdx.x * members;
  float best = -1.f;
  uint64_t bi = ~0ull;
  for (uint64_t i = threadIdx.x; i < members; i += blockDim.x) {
    float2 v = __half22float2(a[i]);
    float pr = v.x * v.x + v.y * v.y;
    if (pr > best) {  // increasing i per thread: strict > keeps the smaller index on ties
      best = pr;
      bi = i;
    }
  }
  __shared__ float sp[32];
  __shared__ uint64_t si[32];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    float op = __shfl_xor_sync(0xffffffffu, best, o);
    uint64_t oi = __shfl_xor_sync(0xffffffffu, bi, o);
    if (op > best || (op == best && oi < bi)) {
      best = op;
      bi = oi;
    }
  }
  if (lane == 0) {
    sp[w] = best;
    si[w] = bi;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int k = 1; k < (int)(blockDim.x >> 5); ++k)
      if (sp[k] > best || (sp[k] == best && si[k] < bi)) {
        best = sp[k];
        bi = si[k];
      }
    top[blockIdx.x] = bi;
  }
}

void launch_top1_chalf(const __half2* amps, uint64_t n_sub, uint64_t members, uint64_t* top, cudaStream_t s) {
  if (n_sub == 0) return;
  top1_chalf_kernel<<<(unsigned)n_sub, 256, 0, s>>>(amps, members, top);
  TN_CUDA(cudaGetLastError());
}

}  // namespace tn
