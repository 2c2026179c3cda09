// CTA-pair (cta_group::2) variant of the complex-half stem GEMM (gemm_tc.cuh), for the steps whose
// A operand is plain (stored order, no fused gather) and whose output is row-major or transposed.
//
// Same operation (Eq. 6: C = A_real x B_P in fp16 with fp32 accumulation and an
// exact power-of-two output scale, readings C-A7/C-A8); what changes is the tile shape.  A cluster
// of two CTAs on neighbouring SMs computes one 256 x BN tile with tcgen05.mma.cta_group::2: each CTA
// stages its own 128 rows of A and HALF of the B tile (BN/2 rows), and the leader's MMA reads both
// CTAs' shared memory.  Per SM and per k block that is 128 x 64 (A) + BN/2 x 64 (B) staged bytes for
// 128 x BN x 64 MACs, instead of 128 x 64 + BN x 64 for the single-CTA tile: 1/3 fewer bytes through
// TMA and shared memory per MAC at BN = 256.  Shared-memory traffic (TMA writes + UMMA reads), not
// the tensor pipe, is what held the single-CTA kernel near 62 % of the measured fp16 peak on the
// compute-bound steps.
//
// Roles (384 threads per CTA, both CTAs):
//   warp 0   : TMA producer for this CTA's halves; the loads complete on the LEADER's full barrier
//              (.cta_group::2 form), whose expected byte count the leader posts for both CTAs
//   warp 1   : (leader only) MMA issuer; tcgen05.commit multicasts to both CTAs' empty / tfull
//   warp 2   : TMEM allocator (cta_group::2, both CTAs)
//   warps 4-11: epilogue, two warpgroups alternating tiles, each CTA drains its own 128 TMEM lanes
//              (= its 128 rows) and tells the leader through a remote mbarrier arrive
#pragma once
#include "gemm_tc.cuh"

namespace tn {
namespace tc2 {

using namespace tc;

template <int BN>
struct Cfg2 {
  static constexpr int KB = 64;
  static constexpr int kABytes = BM * KB * 2;        // this CTA's 128 rows of A
  static constexpr int kBBytes = (BN / 2) * KB * 2;  // this CTA's half of the B tile
  static constexpr int kStageBytes = kABytes + kBBytes;
  static constexpr int kNBuf = 2;                    // 64-column staging buffers per epilogue group
  static constexpr int kCBytes = 2 * kNBuf * BM * 128;
  static constexpr int kTable = 1024;                // barriers + TMEM slot
  static constexpr int kMaxSmem = 232448;
  static constexpr int kStagesRaw = (kMaxSmem - 1024 - kTable - kCBytes) / kStageBytes;
  static constexpr int kStages = kStagesRaw > 16 ? 16 : kStagesRaw;
  static constexpr int kStageArea = (kStages * kStageBytes + 1023) / 1024 * 1024;
  static constexpr int kSmem = kStageArea + kCBytes + 1024 + kTable;
  static_assert(kSmem <= kMaxSmem, "shared memory budget");
  static_assert(kStages >= 3, "pipeline depth");
  static constexpr int kNAcc = 512 / BN;
  // M = 256 (the pair), N = BN, fp16 x fp16 -> fp32, both K-major
  static constexpr uint32_t kIdesc = (1u << 4) | ((uint32_t)(BN >> 3) << 17) | ((uint32_t)(256 >> 4) << 24);
  static constexpr uint32_t kIdescMN = kIdesc | (1u << 15);  // A MN-major (bit 15)
};

// MN-major A (complex rows interleaved, see the kernel comment): SWIZZLE_128B atoms of 64 rows (128 B)
// x 8 k; the two 64-row atoms of a stage sit LBO = 64 k x 128 B = 8 KB apart, consecutive 8-k groups
// SBO = 1 KB apart (canonical Major-MN SW128 layout ((8 x 16 B, m), (8, k)) : ((16 B, LBO), (128 B, SBO)))
__device__ __forceinline__ uint64_t smem_desc_mn_sw128(const void* p) {
  uint64_t addr = smem_u32(p);
  uint64_t d = 0;
  d |= (addr & 0x3FFFFull) >> 4;
  d |= (uint64_t)(8192 >> 4) << 16;
  d |= (uint64_t)(1024 >> 4) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)2 << 61;
  return d;
}

__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}

// shared::cluster address of the same shared-memory object in CTA `rank` of the cluster
__device__ __forceinline__ uint32_t map_rank(const void* p, uint32_t rank) {
  uint32_t out;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(out) : "r"(smem_u32(p)), "r"(rank));
  return out;
}

__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

// TMA tile load into this CTA's shared memory whose completion is signalled on an mbarrier that may
// live in the peer CTA (the leader's full barrier)
__device__ __forceinline__ void tma_load_2d_pair(void* dst, const CUtensorMap* map, uint32_t bar_cluster, int c0,
                                                 int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, "
      "%3}], [%4];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(bar_cluster)
      : "memory");
}

// The same with an L2 eviction-priority hint (createpolicy): the streamed A operand evict_first, the
// B_P tile every m pair re-reads evict_last, so the A stream does not push B out of L2
__device__ __forceinline__ void tma_load_2d_pair_hint(void* dst, const CUtensorMap* map, uint32_t bar_cluster, int c0,
                                                      int c1, uint64_t pol) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.tile.mbarrier::complete_tx::bytes.L2::cache_hint "
      "[%0], [%1, {%2, %3}], [%4], %5;" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(bar_cluster), "l"(pol)
      : "memory");
}

__device__ __forceinline__ uint64_t l2_policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t l2_policy_evict_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}

// N-dimensional form (2..5 dims, coordinates innermost first): the fused stem permutation of a
// gathered-A step (NdArgs, gemm_tc.cuh) loaded per CTA of the pair
__device__ __forceinline__ void tma_load_nd_pair(void* dst, const CUtensorMap* map, uint32_t bar_cluster, int nd,
                                                 const int* c) {
  const uint32_t d = smem_u32(dst);
  const uint64_t m = reinterpret_cast<uint64_t>(map);
  if (nd == 2)
    asm volatile("cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
                 ::"r"(d), "l"(m), "r"(c[0]), "r"(c[1]), "r"(bar_cluster) : "memory");
  else if (nd == 3)
    asm volatile("cp.async.bulk.tensor.3d.cta_group::2.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];"
                 ::"r"(d), "l"(m), "r"(c[0]), "r"(c[1]), "r"(c[2]), "r"(bar_cluster) : "memory");
  else if (nd == 4)
    asm volatile("cp.async.bulk.tensor.4d.cta_group::2.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], [%6];"
                 ::"r"(d), "l"(m), "r"(c[0]), "r"(c[1]), "r"(c[2]), "r"(c[3]), "r"(bar_cluster) : "memory");
  else
    asm volatile("cp.async.bulk.tensor.5d.cta_group::2.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5, %6}], [%7];"
                 ::"r"(d), "l"(m), "r"(c[0]), "r"(c[1]), "r"(c[2]), "r"(c[3]), "r"(c[4]), "r"(bar_cluster) : "memory");
}

__device__ __forceinline__ void mma_f16_pair(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                             uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
}

// arrive (once) on the mbarrier at this offset in both CTAs of the pair when the leader's
// previously issued MMAs have completed
__device__ __forceinline__ void mma_commit_pair(uint64_t* bar) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
          smem_u32(bar)),
      "h"((uint16_t)0x3)
      : "memory");
}

__device__ __forceinline__ void mbar_arrive_cluster(uint32_t bar_cluster) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(bar_cluster) : "memory");
}

// Pair tile i of this cluster -> (m-pair, n-block); false past the end.  order 0: tile t = pair + i *
// npairs, n fastest (clusters with neighbouring ids share the A rows).  order 1: each cluster runs every
// n-block of its own m-pairs in turn, so the re-reads of its A rows stay in its own die's L2 (with order 0
// the clusters sharing an m-pair can sit on both dies: ncu showed 2.3x the A bytes from DRAM at K = N = 2^10).
__device__ __forceinline__ bool tc2_tile(uint32_t i, uint32_t pair, uint32_t npairs, uint32_t num_mp,
                                         uint32_t num_n, int order, int& mp, int& nb) {
  if (order == 1) {
    const uint32_t m = pair + (i / num_n) * npairs;
    mp = (int)m;
    nb = (int)(i % num_n);
    return m < num_mp;
  }
  const uint64_t t = (uint64_t)pair + (uint64_t)i * npairs;
  mp = (int)(t / num_n);
  nb = (int)(t % num_n);
  return t < (uint64_t)num_mp * num_n;
}

// epi: 0 = row-major C tile [128 rows][64-column subtiles] (TMA store box {64, 128}),
//      4 = transposed C^T (layout policy 3, box {128 m, 32 n} at global row m_base + m0)
//
// kMN: the stem permutation of a step whose stored order is [m_hi | contracted k | m_lo] (m_lo >= 7
// modes innermost) folded into the operand layout instead of a permutation pass.  With m innermost
// the real/imaginary parts interleave along m, so the real GEMM is taken over ROWS (m, c):
//   A'[(m,c)][k] = c-part of A[m,k]  (MN-major: 128 A' rows = 64 complex m are 256 contiguous bytes
//   per k, loaded as two 3-D TMA boxes {64 halves, 64 k, 1} of the map [m_hi][k][2 m_lo]),
//   B'[(n,c')][k] = c'-part of b[k,n] (K-major, tn_pad_b_mn),
//   C'[(m,c)][(n,c')] = sum_k A' B'^T,  Re C = C'[(m,0)][(n,0)] - C'[(m,1)][(n,1)],
//                                       Im C = C'[(m,0)][(n,1)] + C'[(m,1)][(n,0)]
// — the same 4 M K N real MACs as Eq. 6, with the complex combination moved
// from B_P's sign pattern to the epilogue: TMEM lanes 2j / 2j+1 hold the two parts of complex row j,
// neighbouring threads swap half of their columns (shfl.xor 1) and each writes 8 of every 16
// complex outputs.  Each CTA's tile is 64 complex rows (the pair: 128), K blocks are 64 complex k.
// Output row permutation of an MN-major step (the kept modes above its 64-row tile written in
// next-use order, plan.cpp): store row = sum_j bit_j(m) << p[j] (p[j] = j for j < 6)
struct RowPerm {
  int on, nb;
  int8_t p[64];
};

__device__ __forceinline__ uint64_t row_perm(const RowPerm& rp, uint64_t m) {
  uint64_t r = m & 63;
  for (int j = 6; j < rp.nb; ++j) r |= ((m >> j) & 1ull) << rp.p[j];
  return r;
}

template <int BN, bool kMN = false>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kThreads, 1)
    gemm_chalf_tc2_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                          const __grid_constant__ CUtensorMap tmC, uint32_t num_mp, uint32_t num_n, int K2,
                          const float* in_max, const float* b_bound, uint32_t* out_max, int* exp_slot, int epi,
                          uint64_t m_base, int order, const __grid_constant__ PeerStore ps,
                          const __grid_constant__ NdArgs nda, int mn_ma, const __grid_constant__ RowPerm rp,
                          int l2_hints, int a_inter) {
  // complex rows per CTA tile, per pair tile
  constexpr int kRows = kMN ? BM / 2 : BM;
  using C = Cfg2<BN>;
  constexpr int KB = C::KB;
  // "no re-run needed" signal of the scale re-run: both CTAs read the same value and leave together
  if (in_max && in_max[0] < 0.f) return;
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* smem = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~(uintptr_t)1023);
  unsigned char* sA = smem;
  unsigned char* sB = smem + C::kStages * C::kABytes;
  unsigned char* sC = smem + C::kStageArea;
  uint64_t* full = reinterpret_cast<uint64_t*>(sC + C::kCBytes);
  uint64_t* empty = full + C::kStages;
  uint64_t* tfull = empty + C::kStages;
  uint64_t* tempty = tfull + C::kNAcc;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + C::kNAcc);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = cluster_rank();
  const uint32_t pair = blockIdx.x >> 1, npairs = gridDim.x >> 1;
  const int num_k = (K2 + KB - 1) / KB;

  if (warp == 0 && lane == 0) {
    for (int s = 0; s < C::kStages; ++s) {
      mbar_init(&full[s], 1);   // leader: its own arrive.expect_tx (bytes of both CTAs)
      mbar_init(&empty[s], 1);  // one multicast commit per use
    }
    for (int a = 0; a < C::kNAcc; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], 2);  // leader: one arrive per CTA's epilogue group
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmA)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmB)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmC)) : "memory");
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(tmem_slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  tc_fence_before();
  cluster_sync();  // barriers initialised and TMEM allocated in both CTAs
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      // ===== TMA producer (both CTAs): this CTA's A rows and B half, completing on the leader =====
      int s = 0;
      uint32_t ph = 0;
      const bool hints = l2_hints != 0;
      const uint64_t pol_a = hints ? l2_policy_evict_first() : 0, pol_b = hints ? l2_policy_evict_last() : 0;
      int mp, nb;
      for (uint32_t i = 0; tc2_tile(i, pair, npairs, num_mp, num_n, order, mp, nb); ++i) {
        const int a_row = mp * 2 * kRows + (int)rank * kRows;
        const int b_row = nb * BN + (int)rank * (BN / 2);
        int cm[5] = {0, 0, 0, 0, 0};  // N-d A: row part of the box coordinates (global row)
        if (!kMN && nda.nd > 0) nd_coords_rows(nda, m_base + (uint64_t)a_row, cm);
        for (int kb = 0; kb < num_k; ++kb) {
          mbar_wait(&empty[s], ph ^ 1);
          if (rank == 0) mbar_expect_tx(&full[s], 2 * C::kStageBytes);
          const uint32_t fb = map_rank(&full[s], 0);
          if constexpr (kMN) {
            const uint64_t gr = m_base + (uint64_t)a_row;
            if (nda.nd == 5) {
              // split block: (m_lo halves, k_lo, m_mid, k_hi, m_hi)
              const int kl = nda.kj0[0], mm = nda.mj0[0];
              const uint64_t r = gr >> mn_ma;
              const int k0 = kb * KB;
              int cc[5] = {(int)(2 * (gr & ((1ull << mn_ma) - 1))), k0 & ((1 << kl) - 1), (int)(r & ((1ull << mm) - 1)),
                           k0 >> kl, (int)(r >> mm)};
              tma_load_nd_pair(sA + s * C::kABytes, &tmA, fb, 5, cc);
              cc[0] += 64;
              tma_load_nd_pair(sA + s * C::kABytes + C::kABytes / 2, &tmA, fb, 5, cc);
            } else {
              int cc[3] = {(int)(2 * (gr & ((1ull << mn_ma) - 1))), kb * KB, (int)(gr >> mn_ma)};
              tma_load_nd_pair(sA + s * C::kABytes, &tmA, fb, 3, cc);
              cc[0] += 64;
              tma_load_nd_pair(sA + s * C::kABytes + C::kABytes / 2, &tmA, fb, 3, cc);
            }
          } else if (nda.nd > 0) {
            int cc[5];
            nd_coords_k(nda, (uint32_t)kb * (KB / 2), cm, cc);
            tma_load_nd_pair(sA + s * C::kABytes, &tmA, fb, nda.nd, cc);
          } else if (hints) {
            tma_load_2d_pair_hint(sA + s * C::kABytes, &tmA, fb, kb * KB, a_row, pol_a);
          } else {
            tma_load_2d_pair(sA + s * C::kABytes, &tmA, fb, kb * KB, a_row);
          }
          if (hints)
            tma_load_2d_pair_hint(sB + s * C::kBBytes, &tmB, fb, kb * KB, b_row, pol_b);
          else
            tma_load_2d_pair(sB + s * C::kBBytes, &tmB, fb, kb * KB, b_row);
          if (++s == C::kStages) {
            s = 0;
            ph ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0 && rank == 0) {
      // ===== MMA issuer (leader): M = 256 over both CTAs' A rows, N = BN over both B halves =====
      int s = 0;
      uint32_t ph = 0;
      int mp, nb;
      for (uint32_t i = 0; tc2_tile(i, pair, npairs, num_mp, num_n, order, mp, nb); ++i) {
        const uint32_t acc = i % C::kNAcc, aph = (i / C::kNAcc) & 1;
        mbar_wait(&tempty[acc], aph ^ 1);
        tc_fence_after();
        const uint32_t tmem_d = tmem_base + acc * BN;
        for (int kb = 0; kb < num_k; ++kb) {
          mbar_wait(&full[s], ph);
          tc_fence_after();
          const uint64_t bd = smem_desc_sw<KB>(sB + s * C::kBBytes);
          if constexpr (kMN) {
            // 16 k = two 8-k groups = 2 KB further along the MN-major atoms (>>4 => +128)
            const uint64_t ad = smem_desc_mn_sw128(sA + s * C::kABytes);
#pragma unroll
            for (int kk = 0; kk < KB / 16; ++kk)
              mma_f16_pair(tmem_d, ad + 128 * kk, bd + 2 * kk, C::kIdescMN, (kb | kk) != 0);
          } else if (a_inter) {
            // A landed by the N-d box in the no-swizzle core-matrix layout (gathered steps whose two
            // innermost stored modes are the only contracted modes there): 16 k = two 2048-byte
            // columns of core matrices (>>4 => +256)
            const uint64_t ad = smem_desc_interleaved(sA + s * C::kABytes);
#pragma unroll
            for (int kk = 0; kk < KB / 16; ++kk)
              mma_f16_pair(tmem_d, ad + 256 * kk, bd + 2 * kk, C::kIdesc, (kb | kk) != 0);
          } else {
            const uint64_t ad = smem_desc_sw<KB>(sA + s * C::kABytes);
#pragma unroll
            for (int kk = 0; kk < KB / 16; ++kk)
              mma_f16_pair(tmem_d, ad + 2 * kk, bd + 2 * kk, C::kIdesc, (kb | kk) != 0);
          }
          mma_commit_pair(&empty[s]);
          if (++s == C::kStages) {
            s = 0;
            ph ^= 1;
          }
        }
        mma_commit_pair(&tfull[acc]);
      }
    }
  } else if (warp >= 4) {
    // ===== epilogue (both CTAs): TMEM lanes = this CTA's 128 rows of the pair tile =====
    const int grp = (warp - 4) >> 2;
    const int ew = warp & 3;
    const int row = ew * 32 + lane;
    const int etid = threadIdx.x - 128 - 128 * grp;
    unsigned char* sCg = sC + grp * (C::kNBuf * BM * 128);
    int e = 0;
    if (in_max && b_bound) e = scale_exp_for(in_max[0] * b_bound[0]);
    if (exp_slot && blockIdx.x == 0 && grp == 0 && etid == 0) *exp_slot = e;
    const float sc = ldexpf(1.f, e);
    float mx = 0.f;
    uint32_t gsub = 0;
    int mp, nb;
    for (uint32_t i = grp; tc2_tile(i, pair, npairs, num_mp, num_n, order, mp, nb); i += 2) {
      const uint32_t acc = i % C::kNAcc, aph = (i / C::kNAcc) & 1;
      const int m0 = mp * 2 * kRows + (int)rank * kRows, n0 = nb * BN;
      mbar_wait(&tfull[acc], aph);
      tc_fence_after();
      const uint32_t taddr = tmem_base + ((uint32_t)(ew * 32) << 16) + acc * BN;
#pragma unroll 1
      for (int sub = 0; sub < BN; sub += 64, ++gsub) {
        unsigned char* sbuf = sCg + (gsub % C::kNBuf) * (BM * 128);
        if (etid == 0) asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(C::kNBuf - 1) : "memory");
        named_bar(1 + grp, 128);
        uint32_t r[2][32];
        tmem_ld_32x32b_x32(taddr + sub, r[0]);
        tmem_ld_32x32b_x32(taddr + sub + 32, r[1]);
        tmem_ld_wait();
        if (sub + 64 >= BN) {
          // this CTA's half of the accumulator drained: tell the leader's MMA (one arrive per group)
          tc_fence_before();
          named_bar(1 + grp, 128);
          if (etid == 0) mbar_arrive_cluster(map_rank(&tempty[acc], 0));
        }
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int c = sub + 32 * h;
          if constexpr (kMN) {
            // lanes 2j (re part of complex row j) and 2j+1 (im part): the even lane finishes columns
            // 0..7 of these 16 complex columns, the odd lane 8..15, each with its partner's half
            const int odd = lane & 1, jr = row >> 1;
            float pv[16];
#pragma unroll
            for (int q = 0; q < 16; ++q)
              pv[q] = __shfl_xor_sync(0xffffffffu, __uint_as_float(odd ? r[h][q] : r[h][16 + q]), 1);  // static indices: no local memory
            uint32_t pk[8];
#pragma unroll
            for (int q = 0; q < 8; ++q) {
              // x_c'[part]: even: own = part 0 (cols 2q, 2q+1), partner = part 1; odd: own = part 1 at
              // 16 + 2q, partner = part 0
              const float a0 = odd ? pv[2 * q] : __uint_as_float(r[h][2 * q]);            // C'[(m,0)][(n,0)]
              const float a1 = odd ? pv[2 * q + 1] : __uint_as_float(r[h][2 * q + 1]);    // C'[(m,0)][(n,1)]
              const float b0 = odd ? __uint_as_float(r[h][16 + 2 * q]) : pv[2 * q];        // C'[(m,1)][(n,0)]
              const float b1 = odd ? __uint_as_float(r[h][17 + 2 * q]) : pv[2 * q + 1];    // C'[(m,1)][(n,1)]
              const float re = (a0 - b1) * sc, im = (a1 + b0) * sc;
              __half2 hv = __floats2half2_rn(re, im);
              mx = fmaxf(mx, fmaxf(fabsf(re), fabsf(im)));
              pk[q] = *reinterpret_cast<uint32_t*>(&hv);
            }
            // complex columns (c & 63) / 2 + 8 odd + q of the 32-column subtile, complex row jr
            const int q0 = ((c & 63) >> 1) + 8 * odd;
            if (epi == 4) {
              const uint32_t sb = smem_u32(sbuf);
#pragma unroll
              for (int q = 0; q < 8; ++q) sts32(sb + 4u * ((q0 + q) * kRows + jr), pk[q]);
            } else {
              const uint32_t srow = smem_u32(sbuf) + jr * 128;
#pragma unroll
              for (int q = 0; q < 2; ++q) {
                const int chunk = ((q0 >> 2) + q) ^ (jr & 7);
                sts128(srow + chunk * 16, pk[4 * q], pk[4 * q + 1], pk[4 * q + 2], pk[4 * q + 3]);
              }
            }
          } else {
            uint32_t pk[16];
#pragma unroll
            for (int j = 0; j < 16; ++j) {
              const float x0 = __uint_as_float(r[h][2 * j]) * sc, x1 = __uint_as_float(r[h][2 * j + 1]) * sc;
              __half2 hv = __floats2half2_rn(x0, x1);
              mx = fmaxf(mx, fmaxf(fabsf(x0), fabsf(x1)));
              pk[j] = *reinterpret_cast<uint32_t*>(&hv);
            }
            if (epi == 4) {
              const uint32_t sb = smem_u32(sbuf);
              const int q0 = (c & 63) >> 1;
#pragma unroll
              for (int j = 0; j < 16; ++j) sts32(sb + 4u * ((q0 + j) * BM + row), pk[j]);
            } else {
              const uint32_t srow = smem_u32(sbuf) + row * 128;
              const int cb = (c & 63) >> 3;
#pragma unroll
              for (int q = 0; q < 4; ++q) {
                const int chunk = (cb + q) ^ (row & 7);
                sts128(srow + chunk * 16, pk[4 * q], pk[4 * q + 1], pk[4 * q + 2], pk[4 * q + 3]);
              }
            }
          }
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        named_bar(1 + grp, 128);
        if (etid == 0) {
          if (ps.on) {
            // fused mode swap: the box goes to the swap member owning it (PeerStore)
            uint64_t gm = m_base + (uint64_t)m0;
            uint32_t nc = (uint32_t)(n0 + sub) >> 1;
            const int v = peer_coords(ps, gm, nc);
            if (epi == 4)
              tma_store_2d(&ps.maps[v], sbuf, (int)gm, (int)nc);
            else
              tma_store_2d(&ps.maps[v], sbuf, (int)(2 * nc), (int)gm);
          } else if (kMN && rp.on) {
            const uint64_t gm = row_perm(rp, m_base + (uint64_t)m0);
            if (epi == 4)
              tma_store_2d(&tmC, sbuf, (int)gm, (n0 + sub) >> 1);
            else
              tma_store_2d(&tmC, sbuf, n0 + sub, (int)gm);
          } else if (epi == 4) {
            tma_store_2d(&tmC, sbuf, (int)(m_base + (uint64_t)m0), (n0 + sub) >> 1);
          } else {
            tma_store_2d(&tmC, sbuf, n0 + sub, m0);
          }
          asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        }
      }
    }
    if (lane == 0) {
      asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
      if (ps.on) peer_store_fence();
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    if (out_max && lane == 0) atomicMax(out_max, __float_as_uint(mx));
  }
  // neither CTA leaves (or frees TMEM) while the pair may still signal its barriers or write its TMEM
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  if (warp == 2) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(tmem_base));
}

}  // namespace tc2
}  // namespace tn
