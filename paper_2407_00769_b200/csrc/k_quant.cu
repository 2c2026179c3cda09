// Eq. 1 group quantisation for mode-swap payloads, int8, exp = 1,
// readings C-A10..C-A13: per group of g reals, scale = 255/(max-min),
// zero = (q_min*max - q_max*min)/(max-min), code = rint(x*scale + zero) evaluated as an fp32
// multiply then an fp32 add (no FMA) so codes are bit-identical to the oracle (oracle/codec.py);
// constant groups: scale = 0, zero = the constant (C-A11).  One warp per group.
#include <algorithm>
#include <cstdlib>
#include <vector>

#include "common.cuh"

namespace tn {

__device__ __forceinline__ float to_f32(float v) { return v; }
__device__ __forceinline__ float to_f32(__half v) { return __half2float(v); }
__device__ __forceinline__ void from_f32(float& d, float v) { d = v; }
__device__ __forceinline__ void from_f32(__half& d, float v) { d = __float2half_rn(v); }

// Sender-side fusion of the mode-swap permutation (north_star (5): "quantise/
// dequantise fused into the permutation kernel").  When the permutation keeps the innermost
// log2(g/2) complex modes in place, every quantisation group of the permuted (send) layout is a
// contiguous run of g reals in the source, so the codec reads it straight from the unpermuted
// stem: group gi of the output starts at complex offset sum_j bit_j(gi) 2^sbit[j].  The codes,
// scales and zeros are bit-identical to permute-then-quantise (same values, same groups); the
// permutation pass (8 bytes per complex-half element) disappears.  The 32 lanes of the warp that
// owns a group each evaluate up to two index bits and OR-reduce them (the bits are distinct).
__device__ __forceinline__ uint64_t group_base(uint64_t gi, int g, const GroupPerm& gp, int lane) {
  if (gp.nb < 0) return gi * (uint64_t)g;
  uint64_t c = 0;
  if (lane < gp.nb && ((gi >> lane) & 1)) c = 1ull << gp.sbit[lane];
  if (lane + 32 < gp.nb && ((gi >> (lane + 32)) & 1)) c |= 1ull << gp.sbit[lane + 32];
  const uint32_t lo = __reduce_or_sync(0xffffffffu, (uint32_t)c);
  const uint32_t hi = __reduce_or_sync(0xffffffffu, (uint32_t)(c >> 32));
  return ((((uint64_t)hi << 32) | lo)) * 2;  // complex offset -> real offset
}

template <typename T>
__global__ void quant_int8_kernel(int8_t* __restrict__ codes, float* __restrict__ scales, float* __restrict__ zeros,
                                  const T* __restrict__ x, uint64_t n_groups, int g,
                                  const __grid_constant__ GroupPerm gp) {
  const int lane = threadIdx.x & 31;
  const uint64_t warps = (uint64_t)gridDim.x * (blockDim.x >> 5);
  for (uint64_t gi = blockIdx.x * (uint64_t)(blockDim.x >> 5) + (threadIdx.x >> 5); gi < n_groups; gi += warps) {
    const T* xs = x + group_base(gi, g, gp, lane);
    float mx = -INFINITY, mn = INFINITY;
    for (int i = lane; i < g; i += 32) {
      float v = to_f32(xs[i]);
      mx = fmaxf(mx, v);
      mn = fminf(mn, v);
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
      mn = fminf(mn, __shfl_xor_sync(0xffffffffu, mn, o));
    }
    float scale, zero;
    if (mx == mn) {
      scale = 0.f;
      zero = mx;
    } else {
      float den = __fsub_rn(mx, mn);
      scale = __fdiv_rn(255.f, den);
      zero = __fdiv_rn(__fsub_rn(__fmul_rn(-128.f, mx), __fmul_rn(127.f, mn)), den);
    }
    if (lane == 0) {
      scales[gi] = scale;
      zeros[gi] = zero;
    }
    int8_t* cs = codes + gi * g;
    for (int i = lane; i < g; i += 32) {
      float c;
      if (scale == 0.f) {
        c = -128.f;
      } else {
        c = rintf(__fadd_rn(__fmul_rn(to_f32(xs[i]), scale), zero));
        c = fminf(fmaxf(c, -128.f), 127.f);
      }
      cs[i] = (int8_t)(int)c;
    }
  }
}

template <typename T>
__global__ void dequant_int8_kernel(T* __restrict__ y, const int8_t* __restrict__ codes,
                                    const float* __restrict__ scales, const float* __restrict__ zeros, uint64_t n,
                                    int g) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    uint64_t gi = i / g;
    float s = scales[gi], z = zeros[gi];
    from_f32(y[i], (s == 0.f) ? z : __fdiv_rn(__fsub_rn((float)codes[i], z), s));
  }
}

// Vectorised codec for g = 128, 256 or 512 reals: every lane owns 16 consecutive reals of one group
// (two 16-byte loads, one 16-byte int8 / 8-byte int4 store), so g/16 lanes share a group and a warp
// quantises 32*16/g groups at once — the per-group scalar work (min/max reduction, the two IEEE
// divisions, the group's source offset) is issued once per warp for several groups.  U trips of
// loads are in flight per warp to cover HBM latency.  (The scalar one-group-per-warp loop above was
// issue-bound at 1.6 TB/s.)  Same fp32 operations per element as the scalar kernels, so codes,
// scales and zeros are identical.
template <int G, int U, bool INT4>
__global__ void __launch_bounds__(256) quant_vec_half_kernel(uint8_t* __restrict__ out, float* __restrict__ scales,
                                                             float* __restrict__ zeros, const __half* __restrict__ x,
                                                             uint64_t n_groups, const __grid_constant__ GroupPerm gp) {
  constexpr int LPG = G / 16, GPW = 32 / LPG;  // lanes per group, groups per warp
  const int lane = threadIdx.x & 31, sl = lane % LPG, sub = lane / LPG;
  const uint64_t warps = (uint64_t)gridDim.x * (blockDim.x >> 5);
  const uint64_t wid = blockIdx.x * (uint64_t)(blockDim.x >> 5) + (threadIdx.x >> 5);
  for (uint64_t g0 = wid * (GPW * U); g0 < n_groups; g0 += warps * (GPW * U)) {
    uint4 v[U][2];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint64_t gi = g0 + u * GPW + sub;
      uint64_t base;
      if (gp.nb < 0) {
        base = gi * G;
      } else {
        uint64_t c = 0;
        for (int j = sl; j < gp.nb; j += LPG)
          if ((gi >> j) & 1) c |= 1ull << gp.sbit[j];
        uint32_t lo = (uint32_t)c, hi = (uint32_t)(c >> 32);
#pragma unroll
        for (int o = LPG / 2; o; o >>= 1) {
          lo |= __shfl_xor_sync(0xffffffffu, lo, o);
          hi |= __shfl_xor_sync(0xffffffffu, hi, o);
        }
        base = ((((uint64_t)hi << 32) | lo)) * 2;
      }
      if (gi < n_groups) {
        const uint4* p = reinterpret_cast<const uint4*>(x + base + sl * 16);
        v[u][0] = __ldcs(p);
        v[u][1] = __ldcs(p + 1);
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint64_t gi = g0 + u * GPW + sub;
      float f[16];
      float mx = -INFINITY, mn = INFINITY;
#pragma unroll
      for (int h = 0; h < 8; ++h) {
        const uint32_t w = h < 4 ? (&v[u][0].x)[h] : (&v[u][1].x)[h - 4];
        const __half2 p = *reinterpret_cast<const __half2*>(&w);
        f[2 * h] = __low2float(p);
        f[2 * h + 1] = __high2float(p);
        mx = fmaxf(mx, fmaxf(f[2 * h], f[2 * h + 1]));
        mn = fminf(mn, fminf(f[2 * h], f[2 * h + 1]));
      }
#pragma unroll
      for (int o = LPG / 2; o; o >>= 1) {
        mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
        mn = fminf(mn, __shfl_xor_sync(0xffffffffu, mn, o));
      }
      if (gi >= n_groups) continue;
      constexpr float qmin = INT4 ? 0.f : -128.f, qmax = INT4 ? 15.f : 127.f;
      float scale, zero;
      if (mx == mn) {
        scale = 0.f;
        zero = mx;
      } else {
        const float den = __fsub_rn(mx, mn);
        scale = __fdiv_rn(qmax - qmin, den);
        zero = __fdiv_rn(__fsub_rn(__fmul_rn(qmin, mx), __fmul_rn(qmax, mn)), den);
      }
      if (sl == 0) {
        scales[gi] = scale;
        zeros[gi] = zero;
      }
      uint32_t q[16];
#pragma unroll
      for (int e = 0; e < 16; ++e) {
        // rint then clamp to [qmin, qmax] == round-to-nearest-even convert with saturation
        // (cvt.rni.sat) for every finite value; int4 saturates to u8, then to 15
        const float t = __fadd_rn(__fmul_rn(f[e], scale), zero);
        uint32_t r;
        if (INT4) {
          asm("cvt.rni.sat.u8.f32 %0, %1;" : "=r"(r) : "f"(t));
          r = min(r, 15u);
        } else {
          asm("cvt.rni.sat.s8.f32 %0, %1;" : "=r"(r) : "f"(t));
          r &= 0xffu;
        }
        q[e] = scale != 0.f ? r : (INT4 ? 0u : 0x80u);
      }
      if (INT4) {
        uint2 w;
        w.x = q[0] | (q[1] << 4) | (q[2] << 8) | (q[3] << 12) | (q[4] << 16) | (q[5] << 20) | (q[6] << 24) | (q[7] << 28);
        w.y = q[8] | (q[9] << 4) | (q[10] << 8) | (q[11] << 12) | (q[12] << 16) | (q[13] << 20) | (q[14] << 24) |
              (q[15] << 28);
        __stcs(reinterpret_cast<uint2*>(out + gi * (G / 2) + sl * 8), w);
      } else {
        uint4 w;
        w.x = q[0] | (q[1] << 8) | (q[2] << 16) | (q[3] << 24);
        w.y = q[4] | (q[5] << 8) | (q[6] << 16) | (q[7] << 24);
        w.z = q[8] | (q[9] << 8) | (q[10] << 16) | (q[11] << 24);
        w.w = q[12] | (q[13] << 8) | (q[14] << 16) | (q[15] << 24);
        __stcs(reinterpret_cast<uint4*>(out + gi * G + sl * 16), w);
      }
    }
  }
}

// experiment knob: TN_QUANT_SCALAR=1 keeps the one-group-per-warp scalar codec
static bool quant_scalar_knob() {
  static const bool v = getenv("TN_QUANT_SCALAR") != nullptr;
  return v;
}

template <bool INT4>
static bool launch_quant_vec_half(uint8_t* out, float* scales, float* zeros, const __half* x, uint64_t n, int g,
                                  cudaStream_t s, const GroupPerm* gp) {
  if ((g != 128 && g != 256 && g != 512) || (reinterpret_cast<uintptr_t>(x) & 15) ||
      (reinterpret_cast<uintptr_t>(out) & 15))
    return false;
  constexpr int U = 2;
  const uint64_t groups = n / g;
  const uint64_t per_block = 8ull * U * (512 / g);
  const uint64_t blocks = std::min<uint64_t>((groups + per_block - 1) / per_block, 148ull * 8);
  if (blocks == 0) return true;
  const GroupPerm p = gp ? *gp : GroupPerm{};
  if (g == 128)
    quant_vec_half_kernel<128, U, INT4><<<(unsigned)blocks, 256, 0, s>>>(out, scales, zeros, x, groups, p);
  else if (g == 256)
    quant_vec_half_kernel<256, U, INT4><<<(unsigned)blocks, 256, 0, s>>>(out, scales, zeros, x, groups, p);
  else
    quant_vec_half_kernel<512, U, INT4><<<(unsigned)blocks, 256, 0, s>>>(out, scales, zeros, x, groups, p);
  TN_CUDA(cudaGetLastError());
  return true;
}

// Vectorised dequantisation for g = 128, 256 or 512: each thread expands 16 codes of one group (one
// 16-byte int8 / 8-byte int4 load) into 16 fp16 reals (two 16-byte stores); y = (code - zero) /
// scale per element, the IEEE division of the scalar kernels, so the outputs are identical.
template <int G, bool INT4>
__global__ void __launch_bounds__(256) dequant_vec_half_kernel(__half* __restrict__ y, const uint8_t* __restrict__ in,
                                                               const float* __restrict__ scales,
                                                               const float* __restrict__ zeros, uint64_t n16) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n16; i += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t gi = i / (G / 16);
    const float sc = __ldg(scales + gi), z = __ldg(zeros + gi);
    float c[16];
    if (INT4) {
      const uint2 w = __ldcs(reinterpret_cast<const uint2*>(in + i * 8));
#pragma unroll
      for (int e = 0; e < 8; ++e) c[e] = (float)((w.x >> (4 * e)) & 0xF);
#pragma unroll
      for (int e = 0; e < 8; ++e) c[8 + e] = (float)((w.y >> (4 * e)) & 0xF);
    } else {
      const uint4 w = __ldcs(reinterpret_cast<const uint4*>(in + i * 16));
      const uint32_t ws[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
      for (int e = 0; e < 16; ++e) c[e] = (float)(int8_t)((ws[e >> 2] >> (8 * (e & 3))) & 0xFF);
    }
    uint32_t o[8];
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      const float a = (sc == 0.f) ? z : __fdiv_rn(__fsub_rn(c[2 * e], z), sc);
      const float b = (sc == 0.f) ? z : __fdiv_rn(__fsub_rn(c[2 * e + 1], z), sc);
      const __half2 h = __halves2half2(__float2half_rn(a), __float2half_rn(b));
      o[e] = *reinterpret_cast<const uint32_t*>(&h);
    }
    uint4* dst = reinterpret_cast<uint4*>(y + i * 16);
    __stcs(dst, make_uint4(o[0], o[1], o[2], o[3]));
    __stcs(dst + 1, make_uint4(o[4], o[5], o[6], o[7]));
  }
}

template <bool INT4>
static bool launch_dequant_vec_half(__half* y, const uint8_t* in, const float* scales, const float* zeros, uint64_t n,
                                    int g, cudaStream_t s) {
  if ((g != 128 && g != 256 && g != 512) || quant_scalar_knob() || (reinterpret_cast<uintptr_t>(y) & 15) ||
      (reinterpret_cast<uintptr_t>(in) & 15))
    return false;
  const uint64_t n16 = n / 16;
  const uint64_t blocks = std::min<uint64_t>((n16 + 255) / 256, 148ull * 8);
  if (blocks == 0) return true;
  if (g == 128)
    dequant_vec_half_kernel<128, INT4><<<(unsigned)blocks, 256, 0, s>>>(y, in, scales, zeros, n16);
  else if (g == 256)
    dequant_vec_half_kernel<256, INT4><<<(unsigned)blocks, 256, 0, s>>>(y, in, scales, zeros, n16);
  else
    dequant_vec_half_kernel<512, INT4><<<(unsigned)blocks, 256, 0, s>>>(y, in, scales, zeros, n16);
  TN_CUDA(cudaGetLastError());
  return true;
}

void launch_quant_int8(int8_t* codes, float* scales, float* zeros, const float* x, uint64_t n, int g,
                       cudaStream_t s) {
  if (g <= 0 || n % g) throw TnError{TN_E_INVALID, "quant: n must be a multiple of the group size"};
  uint64_t groups = n / g;
  uint64_t blocks = (groups + 7) / 8;
  if (blocks > 148 * 16) blocks = 148 * 16;
  if (blocks == 0) return;
  quant_int8_kernel<float><<<(unsigned)blocks, 256, 0, s>>>(codes, scales, zeros, x, groups, g, GroupPerm{});
  TN_CUDA(cudaGetLastError());
}

void launch_dequant_int8(float* y, const int8_t* codes, const float* scales, const float* zeros, uint64_t n, int g,
                         cudaStream_t s) {
  if (g <= 0 || n % g) throw TnError{TN_E_INVALID, "dequant: n must be a multiple of the group size"};
  uint64_t blocks = (n + 255) / 256;
  if (blocks > 148 * 16) blocks = 148 * 16;
  if (blocks == 0) return;
  dequant_int8_kernel<float><<<(unsigned)blocks, 256, 0, s>>>(y, codes, scales, zeros, n, g);
  TN_CUDA(cudaGetLastError());
}

// complex-half payload of a mode swap: the interleaved fp16 reals are the codec's input (their exact
// float32 values), and the dequantised values are rounded back to fp16
void launch_quant_int8_half(int8_t* codes, float* scales, float* zeros, const __half* x, uint64_t n, int g,
                            cudaStream_t s, const GroupPerm* gp) {
  if (g <= 0 || n % g) throw TnError{TN_E_INVALID, "quant: n must be a multiple of the group size"};
  if (!quant_scalar_knob() &&
      launch_quant_vec_half<false>(reinterpret_cast<uint8_t*>(codes), scales, zeros, x, n, g, s, gp))
    return;
  uint64_t groups = n / g;
  uint64_t blocks = std::min<uint64_t>((groups + 7) / 8, 148ull * 16);
  if (blocks == 0) return;
  quant_int8_kernel<__half><<<(unsigned)blocks, 256, 0, s>>>(codes, scales, zeros, x, groups, g, gp ? *gp : GroupPerm{});
  TN_CUDA(cudaGetLastError());
}

void launch_dequant_int8_half(__half* y, const int8_t* codes, const float* scales, const float* zeros, uint64_t n,
                              int g, cudaStream_t s) {
  if (g <= 0 || n % g) throw TnError{TN_E_INVALID, "dequant: n must be a multiple of the group size"};
  if (launch_dequant_vec_half<false>(y, reinterpret_cast<const uint8_t*>(codes), scales, zeros, n, g, s)) return;
  uint64_t blocks = std::min<uint64_t>((n + 255) / 256, 148ull * 16);
  if (blocks == 0) return;
  dequant_int8_kernel<__half><<<(unsigned)blocks, 256, 0, s>>>(y, codes, scales, zeros, n, g);
  TN_CUDA(cudaGetLastError());
}

// int4 preset of Table 1: q in [0, 15], exp = 1, groups of g reals (reading C-A14: two
// codes per byte, low nibble = even index).  scale = 15/(max-min), zero = (0*max - 15*min)/(max-min)
// in the same fp32 operation order as the int8 codec; degenerate groups: scale 0, zero = the
// constant, codes 0 (q_min).  One warp per group, each lane packs pairs of reals.
__global__ void quant_int4_half_kernel(uint8_t* __restrict__ packed, float* __restrict__ scales,
                                       float* __restrict__ zeros, const __half* __restrict__ x, uint64_t n_groups,
                                       int g, const __grid_constant__ GroupPerm gp) {
  const int lane = threadIdx.x & 31;
  const uint64_t warps = (uint64_t)gridDim.x * (blockDim.x >> 5);
  for (uint64_t gi = blockIdx.x * (uint64_t)(blockDim.x >> 5) + (threadIdx.x >> 5); gi < n_groups; gi += warps) {
    const __half* xs = x + group_base(gi, g, gp, lane);
    float mx = -INFINITY, mn = INFINITY;
    for (int i = lane; i < g; i += 32) {
      float v = __half2float(xs[i]);
      mx = fmaxf(mx, v);
      mn = fminf(mn, v);
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
      mn = fminf(mn, __shfl_xor_sync(0xffffffffu, mn, o));
    }
    float scale, zero;
    if (mx == mn) {
      scale = 0.f;
      zero = mx;
    } else {
      float den = __fsub_rn(mx, mn);
      scale = __fdiv_rn(15.f, den);
      zero = __fdiv_rn(__fsub_rn(__fmul_rn(0.f, mx), __fmul_rn(15.f, mn)), den);
    }
    if (lane == 0) {
      scales[gi] = scale;
      zeros[gi] = zero;
    }
    uint8_t* ps = packed + gi * (g / 2);
    for (int i = lane; i < g / 2; i += 32) {
      uint32_t q[2];
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        float c = 0.f;
        if (scale != 0.f) {
          c = rintf(__fadd_rn(__fmul_rn(__half2float(xs[2 * i + h]), scale), zero));
          c = fminf(fmaxf(c, 0.f), 15.f);
        }
        q[h] = (uint32_t)c;
      }
      ps[i] = (uint8_t)(q[0] | (q[1] << 4));
    }
  }
}

__global__ void dequant_int4_half_kernel(__half* __restrict__ y, const uint8_t* __restrict__ packed,
                                         const float* __restrict__ scales, const float* __restrict__ zeros,
                                         uint64_t n, int g) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; 2 * i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    const uint8_t b = packed[i];
    const uint64_t gi = (2 * i) / g;
    const float s = scales[gi], z = zeros[gi];
    const float c0 = (float)(b & 0xF), c1 = (float)(b >> 4);
    y[2 * i] = __float2half_rn((s == 0.f) ? z : __fdiv_rn(__fsub_rn(c0, z), s));
    y[2 * i + 1] = __float2half_rn((s == 0.f) ? z : __fdiv_rn(__fsub_rn(c1, z), s));
  }
}

void launch_quant_int4_half(uint8_t* packed, float* scales, float* zeros, const __half* x, uint64_t n, int g,
                            cudaStream_t s, const GroupPerm* gp) {
  if (g <= 0 || (g & 1) || n % g) throw TnError{TN_E_INVALID, "int4 quant: n must be a multiple of an even group size"};
  if (!quant_scalar_knob() && launch_quant_vec_half<true>(packed, scales, zeros, x, n, g, s, gp))
    return;
  uint64_t groups = n / g;
  uint64_t blocks = std::min<uint64_t>((groups + 7) / 8, 148ull * 16);
  if (blocks == 0) return;
  quant_int4_half_kernel<<<(unsigned)blocks, 256, 0, s>>>(packed, scales, zeros, x, groups, g, gp ? *gp : GroupPerm{});
  TN_CUDA(cudaGetLastError());
}

void launch_dequant_int4_half(__half* y, const uint8_t* packed, const float* scales, const float* zeros, uint64_t n,
                              int g, cudaStream_t s) {
  if (g <= 0 || (g & 1) || n % g) throw TnError{TN_E_INVALID, "int4 dequant: n must be a multiple of an even group size"};
  if (launch_dequant_vec_half<true>(y, packed, scales, zeros, n, g, s)) return;
  uint64_t blocks = std::min<uint64_t>((n / 2 + 255) / 256, 148ull * 16);
  if (blocks == 0) return;
  dequant_int4_half_kernel<<<(unsigned)blocks, 256, 0, s>>>(y, packed, scales, zeros, n, g);
  TN_CUDA(cudaGetLastError());
}

// Group permutation of a fused permute + quantise (see group_base): the permutation `perm` of a
// rank-n complex tensor (output axis j = input axis perm[j], axis 0 outermost, the tn_permute
// convention) fuses when it keeps the innermost log2(g/2) axes in place.  Returns false otherwise.
bool make_group_perm(GroupPerm& gp, int n, const int* perm, int g) {
  if (g < 2 || (g & (g - 1)) || n < 0 || n > 46) return false;
  int b = 0;
  while ((2 << b) < g) ++b;  // g/2 = 2^b complex elements per group
  if (b > n) return false;
  std::vector<int> p_of_q(n);  // destination bit q comes from source bit p_of_q[q]
  for (int j = 0; j < n; ++j) p_of_q[n - 1 - j] = n - 1 - perm[j];
  for (int q = 0; q < b; ++q)
    if (p_of_q[q] != q) return false;
  gp.nb = n - b;
  if (gp.nb > 48) return false;
  for (int j = 0; j < gp.nb; ++j) gp.sbit[j] = (int8_t)p_of_q[j + b];
  return true;
}

// ---- Table 1 int8 preset (int8, group = the entire tensor, exp 0.2), readings C-A10/C-A13 ----
// x' = sign(x)|x|^exp (evaluated in double, rounded to fp32, as the oracle's _signed_pow); scale and
// zero of Eq. 1 from max/min of x' over the group; code = rint(x' scale + zero) (fp32 multiply then
// add); dequant y' = (code - zero)/scale, y = sign(y')|y'|^(1/exp), rounded to fp16.  In a mode swap
// the "entire tensor" is each destination chunk (groups never straddle destinations).
// x -> x' is monotone, so max/min of x' over a group are the transforms of max/min of x: pass 1
// reduces max/min of the fp16 values per group (order-preserving integer atomics), pass 2 encodes.
__device__ __forceinline__ float spow(float x, double e) {
  const float r = (float)pow((double)fabsf(x), e);
  return x < 0.f ? -r : (x > 0.f ? r : 0.f);
}
__device__ __forceinline__ uint32_t f2ord(float f) {
  const uint32_t u = __float_as_uint(f);
  return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}
__device__ __forceinline__ float ord2f(uint32_t u) {
  return __uint_as_float((u & 0x80000000u) ? (u & 0x7fffffffu) : ~u);
}

// tiles of T reals (T = min(2048, g), g a power of two): every tile lies in one group
__global__ void __launch_bounds__(256) minmax_groups_half_kernel(const __half* __restrict__ x, uint64_t n, int tile_log2,
                                                                 int g_log2, uint32_t* __restrict__ mx_ord,
                                                                 uint32_t* __restrict__ mn_ord) {
  const uint64_t T = 1ull << tile_log2, tiles = n >> tile_log2;
  for (uint64_t t = blockIdx.x; t < tiles; t += gridDim.x) {
    float mx = -INFINITY, mn = INFINITY;
    for (uint64_t i = threadIdx.x; i < T; i += blockDim.x) {
      const float v = __half2float(x[(t << tile_log2) + i]);
      mx = fmaxf(mx, v);
      mn = fminf(mn, v);
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
      mn = fminf(mn, __shfl_xor_sync(0xffffffffu, mn, o));
    }
    if ((threadIdx.x & 31) == 0) {
      const uint64_t gi = (t << tile_log2) >> g_log2;
      atomicMax(mx_ord + gi, f2ord(mx));
      atomicMin(mn_ord + gi, f2ord(mn));
    }
  }
}

__global__ void init_minmax_kernel(uint32_t* mx_ord, uint32_t* mn_ord, uint64_t ng) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < ng; i += (uint64_t)gridDim.x * blockDim.x) {
    mx_ord[i] = 0u;           // below every ordered float
    mn_ord[i] = 0xffffffffu;  // above every ordered float
  }
}

__device__ __forceinline__ void group_scale_zero(uint32_t mxo, uint32_t mno, double e, float& scale, float& zero) {
  const float mx = spow(ord2f(mxo), e), mn = spow(ord2f(mno), e);
  if (mx == mn) {
    scale = 0.f;
    zero = mx;
  } else {
    const float den = __fsub_rn(mx, mn);
    scale = __fdiv_rn(255.f, den);
    zero = __fdiv_rn(__fsub_rn(__fmul_rn(-128.f, mx), __fmul_rn(127.f, mn)), den);
  }
}

__global__ void __launch_bounds__(256) quant_exp_half_kernel(int8_t* __restrict__ codes, float* __restrict__ scales,
                                                             float* __restrict__ zeros, const __half* __restrict__ x,
                                                             uint64_t n, int g_log2, double e,
                                                             const uint32_t* __restrict__ mx_ord,
                                                             const uint32_t* __restrict__ mn_ord) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t gi = i >> g_log2;
    float scale, zero;
    group_scale_zero(mx_ord[gi], mn_ord[gi], e, scale, zero);
    if ((i & ((1ull << g_log2) - 1)) == 0) {
      scales[gi] = scale;
      zeros[gi] = zero;
    }
    float c = -128.f;
    if (scale != 0.f) {
      c = rintf(__fadd_rn(__fmul_rn(spow(__half2float(x[i]), e), scale), zero));
      c = fminf(fmaxf(c, -128.f), 127.f);
    }
    codes[i] = (int8_t)(int)c;
  }
}

__global__ void __launch_bounds__(256) dequant_exp_half_kernel(__half* __restrict__ y, const int8_t* __restrict__ codes,
                                                               const float* __restrict__ scales,
                                                               const float* __restrict__ zeros, uint64_t n, int g_log2,
                                                               double inv_e) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t gi = i >> g_log2;
    const float s = scales[gi], z = zeros[gi];
    const float yp = (s == 0.f) ? z : __fdiv_rn(__fsub_rn((float)codes[i], z), s);
    y[i] = __float2half_rn(spow(yp, inv_e));
  }
}

static int log2_exact(uint64_t g) {
  if (g == 0 || (g & (g - 1))) return -1;
  int b = 0;
  while ((1ull << b) < g) ++b;
  return b;
}

void launch_quant_int8_exp_half(int8_t* codes, float* scales, float* zeros, const __half* x, uint64_t n, uint64_t g,
                                double e, uint32_t* d_tmp, cudaStream_t s) {
  const int gl = log2_exact(g);
  if (gl < 0 || n % g || !(e > 0.0)) throw TnError{TN_E_INVALID, "int8 exp codec: g must be a power of two dividing n, exp > 0"};
  if (n == 0) return;
  const uint64_t ng = n / g;
  uint32_t* mx = d_tmp;
  uint32_t* mn = d_tmp + ng;
  const unsigned gb = (unsigned)std::min<uint64_t>((ng + 255) / 256, 148ull * 8);
  init_minmax_kernel<<<gb, 256, 0, s>>>(mx, mn, ng);
  const int tl = std::min(gl, 11);
  const uint64_t tiles = n >> tl;
  minmax_groups_half_kernel<<<(unsigned)std::min<uint64_t>(tiles, 148ull * 16), 256, 0, s>>>(x, n, tl, gl, mx, mn);
  quant_exp_half_kernel<<<(unsigned)std::min<uint64_t>((n + 255) / 256, 148ull * 16), 256, 0, s>>>(codes, scales, zeros, x,
                                                                                                  n, gl, e, mx, mn);
  TN_CUDA(cudaGetLastError());
}

void launch_dequant_int8_exp_half(__half* y, const int8_t* codes, const float* scales, const float* zeros, uint64_t n,
                                  uint64_t g, double e, cudaStream_t s) {
  const int gl = log2_exact(g);
  if (gl < 0 || n % g || !(e > 0.0)) throw TnError{TN_E_INVALID, "int8 exp codec: g must be a power of two dividing n, exp > 0"};
  if (n == 0) return;
  dequant_exp_half_kernel<<<(unsigned)std::min<uint64_t>((n + 255) / 256, 148ull * 16), 256, 0, s>>>(y, codes, scales,
                                                                                                    zeros, n, gl, 1.0 / e);
  TN_CUDA(cudaGetLastError());
}

}  // namespace tn
