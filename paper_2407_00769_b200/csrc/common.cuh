// Shared device helpers and kernel launch declarations of libtn.
#pragma once
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <string>

#include "plan.hpp"

namespace tn {

#define TN_CUDA(call)                                                                       \
  do {                                                                                      \
    cudaError_t e_ = (call);                                                                \
    if (e_ != cudaSuccess)                                                                  \
      throw ::tn::TnError{TN_E_CUDA, std::string(#call) + ": " + cudaGetErrorString(e_)};   \
  } while (0)

constexpr int kMaxModes = 48;

// Offset of a sliced leaf view, computed on the device from the slice id (C-A20): every
// sliced label of the leaf contributes bit `bit[t]` of the slice id times its stride.  Reading the
// slice id from device memory lets one captured CUDA graph serve every slice.
struct SliceOff {
  const uint64_t* slice;         // device slot holding the slice id (nullptr: no sliced labels)
  int n;
  int bit[8];
  int64_t stride[8];
};

__host__ __device__ inline int64_t slice_offset(const SliceOff& so) {
#ifdef __CUDA_ARCH__
  if (!so.slice || so.n == 0) return 0;
  const uint64_t id = *so.slice;
  int64_t off = 0;
  for (int t = 0; t < so.n; ++t)
    if ((id >> so.bit[t]) & 1) off += so.stride[t];
  return off;
#else
  return 0;
#endif
}

// Strides (in complex elements) of a strided complex64 view with every mode of dimension 2.
struct ContractArgs {
  const float2* a;               // A base (the slice offset is added on the device)
  const float2* b;               // B base
  SliceOff sa, sb;
  float2* c;                     // C (dense, row-major in out order)
  int n_out, n_red;              // output bits, reduce bits
  int64_t out_sa[kMaxModes];     // per output bit (bit j = output axis n_out-1-j): stride in A (0 if absent)
  int64_t out_sb[kMaxModes];
  int64_t red_sa[kMaxModes];     // per reduce bit
  int64_t red_sb[kMaxModes];
};

// Gather a complex64 view into a dense [K][N] matrix (row-major), optional fp16 padding output.
struct GatherArgs {
  const float2* src;
  SliceOff ss;
  float2* dst;                   // dense [K][N] complex64
  int klog, nlog;
  int64_t sk[kMaxModes];         // stride of k-bit j (bit j of k = axis klog-1-j of R)
  int64_t sn[kMaxModes];
};

// Output address map of a stem GEMM: C[m, n] lives at
//   sum_j bit_j(m) * ms[j] + sum_j bit_j(n) * ns[j]   (complex elements)
// identity != 0 means plain row-major [M][N] (ms[j] = N << j, ns[j] = 1 << j).
// Mode swap done by the epilogue of the GEMM before it (Alg. 1; runtime.cu
// fused_swap_target): output element C[m, n] belongs to swap member v, formed from nsw of its
// coordinate bits (is_n[t] ? bit bit[t] of the complex column n : bit bit[t] of the row m, giving
// bit vbit[t] of v), and is stored at base[v] — member v's rank's receive buffer, at this rank's
// chunk — at the coordinates with those bits removed.  The launcher honours it only for TMA-store
// epilogues whose store boxes keep the member bits constant (m bits >= 7, n bits >= 5) and sets
// honored; otherwise it stores locally and the runtime exchanges through the transport.
struct PeerTarget {
  int nsw;
  int is_n[3], bit[3], vbit[3];
  void* base[8];
  int honored;
};

struct OutMap {
  int mbits, nbits, identity;
  int transposed;                // C[n][m]: n outermost, m innermost (ns[j] = M << j, ms[j] = 1 << j)
  int64_t ms[kMaxModes];
  int64_t ns[24];
  PeerTarget* peer;              // host only (nullptr: local output)
  int fold_t;                    // 2: a row-folded GEMM (f = 2, N = 16) writing the unfolded C^T [16][2 M]
};

struct PermArgs {
  int n;                         // total bits
  int u;                         // tile bits
  int o;                         // number of tile bits that are output-innermost (write order)
  int64_t tile_in[16];           // input strides of tile bits (read order; first = input innermost)
  int64_t tile_out[16];          // output strides of tile bits (read order)
  int wr_map[16];                // write order bit j -> read-order tile bit index
  int64_t outer_in[64];
  int64_t outer_out[64];
};

// Which GEMM kernel family the last stem-GEMM launch on this host thread used ("tc2", "tc2_mn",
// "tc1", "simt", "c64"; reporting only: tn_report_json's per-step "kern")
extern thread_local const char* g_last_kern;

// ---- launchers (all asynchronous on `s`) ----
// Member chunks of a mode swap through peer memory: output bytes [v chunk_bytes, (v+1) chunk_bytes)
// of a permutation go to base[v] (member v's receive buffer at this rank's chunk) instead of dst.
struct PeerChunks {
  uint64_t chunk_bytes;
  void* base[8];
  // bit routing (nsw > 0, replaces the chunk routing): output element O goes to member v whose bit
  // vbit[t] is O's bit pos[t] (bit positions in elem_bytes units, from the innermost); that bit is
  // replaced by mebit[t] and the element lands at base[v] + O' (base = the start of the buffer)
  int nsw;
  int pos[3], vbit[3], mebit[3];
};
void launch_permute(void* dst, const void* src, int elem_bytes, int n, const int* perm, cudaStream_t s,
                    const PeerChunks* pc = nullptr);
void launch_contract_c64(const ContractArgs& a, cudaStream_t s);
// one launch for the contractions of one tree level (device arrays: args[nnodes], start[nnodes + 1]
// = first block of each node, start[nnodes] = blocks)
void launch_contract_c64_level(const ContractArgs* d_args, const uint32_t* d_start, int nnodes, uint32_t blocks,
                               cudaStream_t s);
void launch_gather_kn(const GatherArgs& g, cudaStream_t s);
void launch_max_abs_f32(const float* x, uint64_t n, uint32_t* out_bits, cudaStream_t s);
void launch_max_abs_f16(const __half* x, uint64_t n, uint32_t* out_bits, cudaStream_t s);
// B' of the MN-major GEMM: rows (n, c') = c'-part of b[k][n] (k contiguous), fp16, the same scale,
// exponent slot and column 1-norm bound as launch_pad_b
void launch_pad_b_mn(__half* bpm, const float2* b, int klog, int nlog, const uint32_t* bmax_bits, float* b_bound,
                     int* exp_slot, cudaStream_t s);
// B' = blockdiag(B_P x f) fp16 [max(f 2N, 16)][f 2K] (row folding, StemStep::fold)
void launch_fold_b(__half* bf, const __half* bp, int klog, int nlog, int f, cudaStream_t s);
// B [K][N] c64 -> B_P fp16 [2N][2K] with scale 2^t (t from *bmax_bits), bound, exp
void launch_pad_b(__half* bp, const float2* b, int klog, int nlog, const uint32_t* bmax_bits,
                  float* b_bound, int* exp_slot, cudaStream_t s);
// complex64 -> complex-half with scale from max (entry of the stem)
void launch_c64_to_chalf(__half2* dst, const float2* src, uint64_t n, const uint32_t* max_bits,
                         int* exp_slot, uint32_t* out_max_bits, cudaStream_t s);
// fused mode-swap permutation for the codecs (k_quant.cu): nb < 0 = identity (groups in order)
struct GroupPerm {
  int nb = -1;      // group-index bits
  int8_t sbit[48];  // source complex-bit position of group-index bit j
};
bool make_group_perm(GroupPerm& gp, int n, const int* perm, int g);
void launch_quant_int4_half(uint8_t* packed, float* scales, float* zeros, const __half* x, uint64_t n, int g,
                            cudaStream_t s, const GroupPerm* gp = nullptr);
void launch_dequant_int4_half(__half* y, const uint8_t* packed, const float* scales, const float* zeros, uint64_t n,
                              int g, cudaStream_t s);
void launch_set_u64(uint64_t* p, uint64_t v, cudaStream_t s);
struct MaxSlots {
  int n;
  const float* p[8];
};
void launch_max_slots(float* dst, const MaxSlots& src, cudaStream_t s);
void launch_redo_check(uint32_t* out_max, const float* in_max, float* redo_in, int bits, cudaStream_t s);
void launch_copy_c64(float2* dst, const float2* src, uint64_t n, cudaStream_t s);
void launch_gemm_c64(float2* c, const float2* a, const float2* b, uint64_t M, uint32_t K, uint32_t N,
                     const OutMap* om, cudaStream_t s, const float* in_max = nullptr, const float* b_bound = nullptr,
                     uint32_t* out_max = nullptr, int* exp_slot = nullptr);
// complex64 operand B [K][N]: *b_bound = max over n of sum_k (|Re B| + |Im B|) (float bits, atomicMax)
void launch_colnorm_c64(const float2* b, int klog, int nlog, float* b_bound, cudaStream_t s);
// complex64 stem entry: dst = src * 2^e, e from *max_bits (as launch_c64_to_chalf); out max recorded
void launch_c64_scale(float2* dst, const float2* src, uint64_t n, const uint32_t* max_bits, int* exp_slot,
                      uint32_t* out_max_bits, cudaStream_t s);
void launch_gemm_chalf_simt(__half2* c, const __half2* a, const __half* bp, uint64_t M, uint32_t K,
                            uint32_t N, const float* in_max, const float* b_bound,
                            uint32_t* out_max, int* exp_slot, const OutMap* om, cudaStream_t s);
// Strided A operand of a tcgen05 GEMM (the stem permutation fused into the load): A[m, k] at
// a + sum_j bit_j(m) ms[j] + sum_j bit_j(k) ks[j] complex elements; requires ks[0] = 1, ks[1] = 2.
struct AGather {
  int mlog, klog;
  int64_t ms[kMaxModes];
  int64_t ks[24];
};
void launch_gemm_chalf_tc(__half* c, const __half* a, const __half* bp, uint64_t M, uint32_t K2,
                          uint32_t N2, const float* in_max, const float* b_bound, uint32_t* out_max,
                          int* exp_slot, const OutMap* om, cudaStream_t s, const AGather* ag = nullptr);
int gather_mode_of(const AGather& ag);  // k_gemm_tc.cu: the gathered-A path (plan.cpp cost model)
// MN-major A (k_gemm_tc2.cu): A stored [M >> ma][K][2^ma] complex-half (2^ma kept rows innermost),
// bpm = B' [2N][K] (launch_pad_b_mn); no permutation pass.
// Split form (kl, mm > 0): A stored [M >> (ma + mm)][K >> kl][2^mm][2^kl][2^ma] (a run of mm kept
// modes between the contracted ones; output rows in stored order m_hi, m_mid, m_lo).
bool mn_gemm_supported(uint64_t M, uint32_t K, uint32_t N, int ma, const OutMap* om, int kl = 0, int mm = 0);
void launch_gemm_chalf_mn(__half* c, const __half* a, const __half* bpm, uint64_t M, uint32_t K, uint32_t N, int ma,
                          const float* in_max, const float* b_bound, uint32_t* out_max, int* exp_slot,
                          const OutMap* om, cudaStream_t s, int kl = 0, int mm = 0);
// Gather-batched tcgen05 GEMM (Fig. 5; see BatchArgs in gemm_tc.cuh): n_out
// entries of M rows (M % 128 == 0).  Index variant (pad_r == 0): C[b] = A[ia[b]] x B_P[ib[b]].
// Padded 2-d index (pad_r > 0, n_out = n_a): C_P[a] = A[a] x [B_P[table[a pad_r + r]]]_r, rows of
// C_P are pad_r blocks of 2N reals, table < 0 -> zero block.  ia/ib/table are device int32 arrays.
struct BatchSpec {
  int pad_r = 0;
  const int* ia = nullptr;
  const int* ib = nullptr;
  const int* table = nullptr;
  uint64_t n_out = 0, n_a = 0, n_b = 0;
};
void launch_gemm_chalf_batched_simt(__half2* c, const __half2* a, const __half* bp, uint64_t M, uint32_t K, uint32_t N,
                                    uint64_t n_out, const int* ia, const int* ib, uint64_t b_blk_halfs,
                                    const float* in_max, const float* b_bound, uint32_t* out_max, int* exp_slot,
                                    cudaStream_t s);
void launch_gemm_chalf_tc_batched(__half* c, const __half* a, const __half* bp, uint64_t M, uint32_t K2, uint32_t N2,
                                  const float* in_max, const float* b_bound, uint32_t* out_max, int* exp_slot,
                                  const BatchSpec& bs, cudaStream_t s);
OutMap identity_map(uint64_t M, uint32_t N);
// member (open-leg order) index of a stored amplitude: bit (r-1-t) of the member index is bit
// src_bit[t] of the layout index
struct MemberMap {
  int r;
  int8_t src_bit[64];
};
void launch_top1_chalf(const __half2* amps, uint64_t n_sub, uint64_t members, const MemberMap& mm, uint64_t* top,
                       cudaStream_t s);
void launch_quant_int8(int8_t* codes, float* scales, float* zeros, const float* x, uint64_t n, int g,
                       cudaStream_t s);
void launch_dequant_int8(float* y, const int8_t* codes, const float* scales, const float* zeros,
                         uint64_t n, int g, cudaStream_t s);
void launch_quant_int8_half(int8_t* codes, float* scales, float* zeros, const __half* x, uint64_t n, int g,
                            cudaStream_t s, const GroupPerm* gp = nullptr);
void launch_dequant_int8_half(__half* y, const int8_t* codes, const float* scales, const float* zeros, uint64_t n,
                              int g, cudaStream_t s);
// Table 1 int8 preset (exp != 1, large power-of-two groups); d_tmp holds 2 * n/g uint32
void launch_quant_int8_exp_half(int8_t* codes, float* scales, float* zeros, const __half* x, uint64_t n, uint64_t g,
                                double e, uint32_t* d_tmp, cudaStream_t s);
void launch_dequant_int8_exp_half(__half* y, const int8_t* codes, const float* scales, const float* zeros, uint64_t n,
                                  uint64_t g, double e, cudaStream_t s);

// ---- device helpers ----
__host__ __device__ inline int64_t outmap_m(const OutMap& o, uint64_t m) {
  int64_t a = 0;
  for (int j = 0; j < o.mbits; ++j)
    if ((m >> j) & 1) a += o.ms[j];
  return a;
}
__host__ __device__ inline int64_t outmap_n(const OutMap& o, uint64_t n) {
  int64_t a = 0;
  for (int j = 0; j < o.nbits; ++j)
    if ((n >> j) & 1) a += o.ns[j];
  return a;
}
// power-of-two exponent e so that prod * 2^e < 2^14 (prod > 0); 0 if prod == 0 or not finite.
__host__ __device__ inline int scale_exp_for(float prod) {
  if (!(prod > 0.f) || !(prod < 3.0e38f)) return 0;
  int p;
  frexpf(prod, &p);  // prod = f * 2^p, f in [0.5, 1)  => prod < 2^p
  int e = 14 - p;
  if (e > 120) e = 120;
  if (e < -120) e = -120;
  return e;
}

}  // namespace tn
