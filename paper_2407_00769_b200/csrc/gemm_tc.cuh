// Shared implementation of the tcgen05 complex-half GEMM (included by k_gemm_tc*.cu; each
// k_gemm_tc_m<G>.cu instantiates one A-operand mode so the variants compile in parallel).
#pragma once
// Complex-half stem GEMM on the 5th-generation tensor cores.
//
// Eq. 6: C[m,(n,c)] = sum_{(k,a)} A_real[m,(k,a)] * B_P[(k,a),(n,c)], i.e. the
// complex contraction of the stem A (interleaved fp16 re/im, read AS STORED — P:502 "include an
// extra mode for tensor B, as it is smaller than tensor A") with the padded B_P
// [[Re b,-Im b],[Im b, Re b]] is ONE real fp16 GEMM [M,2K] x [2K,2N] -> [M,2N] whose output is
// again interleaved complex.  fp32 accumulation in TMEM (reading C-A7), one round-to-nearest to
// fp16 in the epilogue with an exact power-of-two scale (reading C-A8).
//
// sm_100a design: persistent warp-specialised kernel, one CTA per SM (grid = min(tiles, #SMs)).
//   warp 0   : TMA producer — A tile [128 x 64] and B tile [BN x 64] per stage, 128B swizzle,
//              mbarrier full/empty ring of STAGES
//   warp 1   : MMA issuer — one elected thread issues tcgen05.mma.cta_group::1.kind::f16
//              (M=128, N=BN, K=16), accumulators in TMEM (512 columns: 2 x 256 ... 16 x 32),
//              tcgen05.commit -> mbarriers
//   warp 2   : TMEM allocator
//   warps 4-11: epilogue, two warpgroups; group g drains every other tile —
//              tcgen05.ld 32x32b -> scale -> fp16 -> 128B-swizzled smem ring -> TMA store; running
//              max |C| for the next step's scale.  Two groups keep two warps per SM sub-partition
//              converting, which output-heavy shapes (small K, large N) need to reach HBM write speed
#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdlib>
#include <mutex>
#include <type_traits>

#include "common.cuh"

#ifndef TN_RAW_CAP
#define TN_RAW_CAP 8
#endif
namespace tn {

namespace tc {

constexpr int BM = 128;
constexpr int kThreads = 384;        // 4 role warps + 2 epilogue warpgroups
constexpr int kThreadsGather = 512;  // + 4 warps gathering A (fused permutation)
constexpr int kGatherWarps = 4;

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// epilogue staging stores with 32-bit shared addresses (the generic 64-bit stores cost address
// arithmetic per store)
__device__ __forceinline__ void sts32(uint32_t addr, uint32_t v) {
  asm volatile("st.shared.b32 [%0], %1;" ::"r"(addr), "r"(v) : "memory");
}
__device__ __forceinline__ void sts128(uint32_t addr, uint32_t a, uint32_t b, uint32_t c, uint32_t d) {
  asm volatile("st.shared.v4.b32 [%0], {%1,%2,%3,%4};" ::"r"(addr), "r"(a), "r"(b), "r"(c), "r"(d) : "memory");
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  uint32_t addr = smem_u32(bar);
  asm volatile(
      "{\n\t.reg .pred P1;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
      "@!P1 bra WAIT_%=;\n\t}" ::"r"(addr),
      "r"(parity)
      : "memory");
}

__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
          smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(smem_u32(bar))
      : "memory");
}

// N-dimensional TMA tile load (3..5 dims; coordinates innermost first)
__device__ __forceinline__ void tma_load_nd(void* dst, const CUtensorMap* map, uint64_t* bar, int nd, const int* c) {
  const uint32_t d = smem_u32(dst), b = smem_u32(bar);
  const uint64_t m = reinterpret_cast<uint64_t>(map);
  if (nd == 3)
    asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];"
                 ::"r"(d), "l"(m), "r"(c[0]), "r"(c[1]), "r"(c[2]), "r"(b) : "memory");
  else if (nd == 4)
    asm volatile("cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], [%6];"
                 ::"r"(d), "l"(m), "r"(c[0]), "r"(c[1]), "r"(c[2]), "r"(c[3]), "r"(b) : "memory");
  else if (nd == 5)
    asm volatile("cp.async.bulk.tensor.5d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5, %6}], [%7];"
                 ::"r"(d), "l"(m), "r"(c[0]), "r"(c[1]), "r"(c[2]), "r"(c[3]), "r"(c[4]), "r"(b) : "memory");
  else
    asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
                 ::"r"(d), "l"(m), "r"(c[0]), "r"(c[1]), "r"(b) : "memory");
}

__device__ __forceinline__ void tma_store_2d_hint(const CUtensorMap* map, const void* src, int c0, int c1,
                                                  uint64_t policy) {
  asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group.L2::cache_hint [%0, {%1, %2}], [%3], %4;" ::"l"(
                   reinterpret_cast<uint64_t>(map)),
               "r"(c0), "r"(c1), "r"(smem_u32(src)), "l"(policy)
               : "memory");
}

__device__ __forceinline__ void tma_store_2d(const CUtensorMap* map, const void* src, int c0, int c1) {
  asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];" ::"l"(
                   reinterpret_cast<uint64_t>(map)),
               "r"(c0), "r"(c1), "r"(smem_u32(src))
               : "memory");
}

// SM100 UMMA shared-memory matrix descriptor, K-major, rows of KB fp16 = 2*KB bytes swizzled at that
// width: start>>4 [0,14) | LBO>>4 [16,30) (unused for swizzled K-major) | SBO>>4 [32,46) = 8 rows
// between 8-row groups | version 1 [46,48) | base offset 0 | layout [61,64): SWIZZLE_128B = 2,
// SWIZZLE_64B = 4, SWIZZLE_32B = 6.
template <int KB>
__device__ __forceinline__ uint64_t smem_desc_sw(const void* p) {
  constexpr uint64_t kRow = 2 * KB;
  constexpr uint64_t kLayout = KB == 64 ? 2 : (KB == 32 ? 4 : 6);
  uint64_t addr = smem_u32(p);
  uint64_t d = 0;
  d |= (addr & 0x3FFFFull) >> 4;
  d |= (uint64_t)1 << 16;
  d |= (uint64_t)((8 * kRow) >> 4) << 32;
  d |= (uint64_t)1 << 46;
  d |= kLayout << 61;
  return d;
}

// K-major, no swizzle ("interleaved" core matrices of 8 rows x 16 B): rows 16 B apart, 8-row groups
// SBO = 128 B apart, 16-byte K pieces LBO = 128 rows x 16 B = 2048 B apart (layout type 0)
__device__ __forceinline__ uint64_t smem_desc_interleaved(const void* p) {
  uint64_t addr = smem_u32(p);
  uint64_t d = 0;
  d |= (addr & 0x3FFFFull) >> 4;
  d |= (uint64_t)(2048 >> 4) << 16;
  d |= (uint64_t)(128 >> 4) << 32;
  d |= (uint64_t)1 << 46;
  return d;
}

__device__ __forceinline__ void mma_f16(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                        uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
}

__device__ __forceinline__ void mma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}

__device__ __forceinline__ void tmem_ld_32x32b_x32(uint32_t taddr, uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
        "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
        "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
}

__device__ __forceinline__ void tmem_ld_wait() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

__device__ __forceinline__ void named_bar(int id, int n) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}

// KB: fp16 elements of K per stage (the TMA box and swizzle width): 64, or 2K when 2K < 64 so that
// small-K steps neither stage nor zero-fill 3/4 empty boxes and keep more tiles in flight.
// AMODE: the A-operand mode of the kernel (3 = raw landing slots, 4 = 4-byte gather with a bigger table).
template <int BN, int KB, int AMODE = 0>
struct Cfg {
  static constexpr int kABytes = BM * KB * 2;
  static constexpr int kBBytes = BN * KB * 2;
  static constexpr int kStageBytes = kABytes + kBBytes;
  static constexpr int kCSub = (BN + 63) / 64;            // 64-column store subtiles
  static constexpr int kMaxSmem = 232448;                 // 227 KB opt-in dynamic shared memory per CTA
  static constexpr int kTable = AMODE == 4 ? 4096 : 2048; // barriers + gather table
  static constexpr bool kDeep = AMODE == 5;               // plain TMA A, deep pipeline (see kNBuf)
  // raw TMA landing slots (A mode 3): they are the A bytes in flight from HBM, so as many as fit
  // (<= 8) next to 2 pipeline stages and 2 staging buffers per epilogue group
  static constexpr int kNBufOld = ((220 * 1024 - 2 * 4 * BM * 128) / kStageBytes >= 4) ? 4 : 2;
  static constexpr int kRawFit = (220 * 1024 - 2 * kNBufOld * BM * 128 - 2 * kStageBytes) / kABytes;
  static constexpr int kRaw = AMODE != 3 ? 0 : (kRawFit > TN_RAW_CAP ? TN_RAW_CAP : (kRawFit < 2 ? 2 : kRawFit));
  static constexpr int kRawBytes = kRaw * kABytes;
  static constexpr int kFixed = 1024 /*align*/ + kTable + kRawBytes;
  static constexpr int stages_for(int nbuf) {
    return (kMaxSmem - kFixed - 2 * nbuf * BM * 128) / kStageBytes;
  }
  // output staging ring (64-column subtiles) per epilogue group.  Deep variant (AMODE 5, K-heavy
  // steps, chosen at launch): as few buffers as keep the most pipeline stages — the A operand is the
  // bytes in flight from HBM, and a tile's epilogue is rare next to its k loop (BN = 256: 4 stages
  // with one buffer instead of 3 with two).  Otherwise: 4 buffers (more TMA stores in flight) when
  // that still leaves >= 4 stages, else 2.
  static constexpr int kNBufDeep = stages_for(1) > stages_for(2) ? 1 : (stages_for(2) > stages_for(4) ? 2 : 4);
  static constexpr int kNBuf = kDeep ? kNBufDeep : kNBufOld;
  static constexpr int kCTma = 2 * kNBuf * BM * 128;      // 128B-swizzled staging for TMA stores, 2 groups
  static constexpr int kCBytes = kCTma;
  // round-1 budget (220 KB for stages + staging) unless deep
  static constexpr int kStagesRaw = kDeep ? stages_for(kNBuf) : (220 * 1024 - kCBytes - kRawBytes) / kStageBytes;
  static constexpr int kStages = kStagesRaw > 24 ? 24 : kStagesRaw;
  // the TMA-store staging (128B swizzle) must start 1024-aligned: pad the stage area
  static constexpr int kStageArea = (kStages * kStageBytes + 1023) / 1024 * 1024;
  static constexpr int kSmem = kStageArea + kCBytes + kRawBytes + 1024 /*align*/ + kTable;
  static_assert(kSmem <= kMaxSmem, "shared memory budget");
  static_assert(kStages >= 2, "pipeline depth");
  // TMEM accumulators: as many as fit in 512 columns (<= 16), so the MMA runs ahead of the
  // epilogue by several tiles when a tile is small (small K, small N)
  static constexpr int kAccStride = BN < 32 ? 32 : BN;
  static constexpr int kNAcc = (512 / kAccStride) > 16 ? 16 : (512 / kAccStride);
  static constexpr uint32_t kIdesc = (1u << 4) | ((uint32_t)(BN >> 3) << 17) | ((uint32_t)(BM >> 4) << 24);
};

}  // namespace tc

// Scatter epilogue description (output layout = any bit placement of m and n, see OutMap):
// C[m, n] goes to sum_j bit_j(m) ms[j] + sum_j bit_j(n) ns[j] (complex elements).  Each epilogue
// thread owns one row of the tile and stores its values straight from registers in contiguous
// vectors along the lowest n bits whose strides are 1, 2, 4, ... (no shared-memory staging).
// Tile rasterisation for scatter layouts: tile index bit b sets bit vbit_idx[b] of the m-block
// (vbit_is_m[b] = 1) or of the n-block; bits are ordered by output stride so tiles that fill the
// same output lines run concurrently on neighbouring CTAs and their partial sectors merge in L2.
struct ScatterArgs {
  int on;
  int mbits, nbits;
  int nv;
  int8_t vbit_is_m[64];
  int8_t vbit_idx[64];
  int64_t ms[kMaxModes];
  int64_t ns[24];
};

__device__ __forceinline__ void tile_coords(const ScatterArgs& sa, uint32_t t, uint32_t num_n, int BMv, int BNv,
                                            int& m0, int& n0) {
  if (sa.on) {
    uint32_t mb = 0, nb = 0;
    for (int b = 0; b < sa.nv; ++b)
      if ((t >> b) & 1) {
        if (sa.vbit_is_m[b])
          mb |= 1u << sa.vbit_idx[b];
        else
          nb |= 1u << sa.vbit_idx[b];
      }
    m0 = (int)(mb * BMv);
    n0 = (int)(nb * BNv);
  } else {
    m0 = (int)((t / num_n) * BMv);
    n0 = (int)((t % num_n) * BNv);
  }
}

// Gathered A operand (the stem permutation fused into the GEMM load): A[m, k] (complex-half) sits at
// a + sum_j bit_j(m) ms[j] + sum_j bit_j(k) ks[j] (complex elements) with ks[0] = 1, ks[1] = 2, so
// every 16-byte piece of a K-major smem row is 4 contiguous complex values.  A stage (128 rows x
// KB fp16) is nvb = 7 + log2(KB/8) "vector bits" (row bits and 16-byte chunk bits); they are sorted
// by source stride on the host so the 32 lanes of a warp read the lowest-stride (most contiguous)
// combinations.
struct AGatherArgs {
  const uint32_t* a;
  uint64_t m_base;  // row offset of this launch chunk
  int mlog, klog, nvb;
  int fence;           // consumer-side proxy fence (TN_GATHER_FENCE; off: CUTLASS's cp.async->UMMA pipelines use none)
  int8_t vb_is_k[16];  // vector bit b: 16-byte chunk bit (k bit 2 + idx) or row bit (m bit idx)
  int8_t vb_idx[16];
  int64_t ms[kMaxModes];
  int64_t ks[24];
};

// Gathered A through one N-dimensional TMA box (the fused stem permutation when the source's bit
// runs allow, <= 5 dims): dim d's coordinate = bits [j0, j0 + nb) of the tile's start row
// (kind 0), of its start k index (kind 1), or 0 (kind 2: box-only dim).  nd == 0: plain 2-D A map.
struct NdArgs {
  int nd;
  // dim d's coordinate = ((row >> mj0) & mmask) << msh | ((k >> kj0) & kmask) << ksh  (row, k =
  // the tile's start row and start k index; a zero mask drops that part)
  int8_t mj0[5], msh[5], kj0[5], ksh[5];
  uint32_t mmask[5], kmask[5];
  // mode 3 (raw box + reshuffle): the raw box's 16-byte pieces are enumerated as
  // p = XOR of lane_pat[b] over the lane's bits b, XOR it_pat[i] over the iteration's bits i (a
  // basis of GF(2)^npb chosen on the host so that every 8-lane phase touches 8 distinct 16-byte bank
  // slots on both the raw read and the stage write).  Piece p sits at raw byte 16 p and goes to
  // byte dst(p) of the interleaved stage; dst is GF(2)-linear (each piece bit owns one address
  // bit), so it is carried as lane_dst / it_dst the same way.
  int npb;
  uint16_t lane_pat[5], it_pat[8];
  uint32_t lane_dst[5], it_dst[8];
};

// Gather-batched operands (§3.4.2 Fig. 5): the launch computes several
// independent products of identical shape.  Entry b of the output (M rows of C, M a multiple of 128):
//   index variant (pad_r == 0):  C[b] = A[ia[b]] x B_P[ib[b]]            (Fig. 5 bottom, A_I x B_I)
//   padded 2-d index (pad_r > 0): C_P[b] = A[b] x [B_P[t_0] | ... | B_P[t_{pad_r-1}]],
//                                 t_r = table[b * pad_r + r], t_r < 0 -> a zero block (Fig. 5 top)
// A entry a = rows [a M, (a+1) M) of the A map, B_P block j = rows [j b_rows, (j+1) b_rows) of the B
// map (b_rows = max(2N, 16)), C entry b = rows [b M, (b+1) M) of the C map (padded: pad_r b_rows
// columns).  Indices are read on the device, so one launch (or one captured graph) serves any
// batch; A is never materialised as A_I (a repeated A entry is re-read from L2 by neighbouring tiles).
struct BatchArgs {
  int on;
  int pad_r;
  const int* ia;
  const int* ib;
  const int* table;
  uint32_t m_tiles;   // 128-row tiles per entry
  uint64_t rows;      // M
  uint32_t b_rows;    // rows of one B_P block
};

// Kernel-side form of a PeerTarget (common.cuh): the output store boxes go straight to the swap
// members' receive buffers.  Entries are sorted so that, per coordinate, bits are removed from the
// highest down (removing a higher bit leaves the lower bit indices valid).  maps[v]: member v's
// destination chunk, row-major [M'][2N'] fp16 (box {64, 128}) or transposed C^T [N'][M'] (box
// {128, 32}), M' / N' = M / N with the member bits removed.
struct PeerStore {
  int on, nsw;
  int8_t is_n[4], bit[4], vbit[4];
  CUtensorMap maps[8];
};

namespace tc {

// Member index of a store box at (row m, complex column n) and its coordinates in that member's
// chunk (the member bits removed).
__device__ __forceinline__ int peer_coords(const PeerStore& ps, uint64_t& m, uint32_t& n) {
  int v = 0;
  for (int t = 0; t < ps.nsw; ++t) {
    const int b = ps.bit[t];
    if (ps.is_n[t]) {
      v |= (int)((n >> b) & 1u) << ps.vbit[t];
      n = (n & ((1u << b) - 1u)) | ((n >> (b + 1)) << b);
    } else {
      v |= (int)((m >> b) & 1ull) << ps.vbit[t];
      m = (m & ((1ull << b) - 1ull)) | ((m >> (b + 1)) << b);
    }
  }
  return v;
}

// After the last peer store of a thread: its bulk stores have completed (wait_group 0); make them
// visible at system scope before the kernel ends (the swap's barrier follows on the stream).
__device__ __forceinline__ void peer_store_fence() {
  asm volatile("fence.proxy.async.global;" ::: "memory");
  asm volatile("fence.acq_rel.sys;" ::: "memory");
}

// Tile t -> C tile (m0 row, n0 column), A row and B row of its operands, skip = zero tile.
__device__ __forceinline__ void batch_tile(const BatchArgs& ba, uint32_t t, uint32_t num_n, int BNv, int& m0, int& n0,
                                           int& a_row, int& b_row, bool& skip) {
  const uint32_t per = ba.m_tiles * num_n;
  const uint32_t b = t / per, rem = t % per, mt = rem / num_n, nt = rem % num_n;
  m0 = (int)(b * ba.rows + (uint64_t)mt * BM);
  n0 = (int)(nt * BNv);
  skip = false;
  if (ba.pad_r > 0) {
    const uint32_t per_r = ba.b_rows / BNv, r = nt / per_r, w = nt % per_r;
    const int j = __ldg(ba.table + (uint64_t)b * ba.pad_r + r);
    skip = j < 0;
    a_row = m0;
    b_row = (int)((skip ? 0 : j) * ba.b_rows + w * BNv);
  } else {
    a_row = (int)((uint64_t)__ldg(ba.ia + b) * ba.rows + (uint64_t)mt * BM);
    b_row = (int)((uint64_t)__ldg(ba.ib + b) * ba.b_rows + nt * BNv);
  }
}

__device__ __forceinline__ void cp_async16(uint32_t smem_addr, const void* gmem) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_addr), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async4(uint32_t smem_addr, const void* gmem) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(smem_addr), "l"(gmem) : "memory");
}

// Row / k parts of the N-d box coordinates: the TMA thread evaluates the row part once per tile
// and the k part once per stage (a handful of shifts, so the single issuing thread keeps up).
__device__ __forceinline__ void nd_coords_rows(const NdArgs& nda, uint64_t row, int (&cm)[5]) {
#pragma unroll
  for (int d = 0; d < 5; ++d) cm[d] = (int)(((uint32_t)(row >> nda.mj0[d]) & nda.mmask[d]) << nda.msh[d]);
}
__device__ __forceinline__ void nd_coords_k(const NdArgs& nda, uint32_t k, const int (&cm)[5], int (&cc)[5]) {
#pragma unroll
  for (int d = 0; d < 5; ++d) cc[d] = cm[d] | (int)(((k >> nda.kj0[d]) & nda.kmask[d]) << nda.ksh[d]);
}

// kAMode: 0 = A by TMA (2-D map, or N-d box when nda.nd > 0; swizzled rows), 1 = A gathered by
// cp.async producer warps, 2 = A by N-d TMA box into the no-swizzle (interleaved) K-major layout,
// 3 = A by an N-d TMA box in source order into a raw slot, reshuffled by warp 3 (16-byte pieces)
// into the interleaved layout
template <int BN, int KB, int kAMode>
__global__ void __launch_bounds__((kAMode == 1 || kAMode == 4) ? kThreadsGather : kThreads, 1)
    gemm_chalf_tc_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                         const __grid_constant__ CUtensorMap tmC, uint32_t num_m, uint32_t num_n, int K2,
                         const float* in_max, const float* b_bound, uint32_t* out_max, int* exp_slot,
                         const __grid_constant__ ScatterArgs sc_args, uint32_t* out_scatter, uint64_t rows,
                         uint32_t n_cols, const __grid_constant__ AGatherArgs ga,
                         const __grid_constant__ NdArgs nda, int epi_stg, const __grid_constant__ BatchArgs ba,
                         const __grid_constant__ PeerStore ps) {
  // 1: cp.async gather of 16-byte pieces (4 consecutive complex k); 4: of 4-byte pieces (single
  // complex elements, any layout: the stem permutation of a step whose contracted modes sit in the
  // middle of the stored order, fused into the load)
  constexpr bool kGather = kAMode == 1 || kAMode == 4;
  constexpr bool kWord = kAMode == 4;
  constexpr bool kInter = kAMode == 2 || kAMode == 3;
  using C = Cfg<BN, KB, kAMode>;
  // a negative input max is the "no re-run needed" signal of the scale re-run (runtime.cu redo)
  if (in_max && in_max[0] < 0.f) return;
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* smem = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~(uintptr_t)1023);
  unsigned char* sA = smem;
  unsigned char* sB = smem + C::kStages * C::kABytes;
  unsigned char* sC = smem + C::kStageArea;  // 1024-aligned (SW128 staging)
  unsigned char* sRaw = sC + C::kCBytes;
  uint64_t* full = reinterpret_cast<uint64_t*>(sRaw + C::kRawBytes);
  uint64_t* empty = full + C::kStages;
  uint64_t* tfull = empty + C::kStages;
  uint64_t* tempty = tfull + C::kNAcc;
  uint64_t* raw_full = tempty + C::kNAcc;
  uint64_t* raw_empty = raw_full + 8;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(raw_empty + 8);
  struct GTab {
    int64_t off;
    int rc;
    int pad;
  };
  GTab* gtab = reinterpret_cast<GTab*>(reinterpret_cast<unsigned char*>(full) + 1024);  // gather table

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t num_tiles = num_m * num_n;
  const int num_k = (K2 + KB - 1) / KB;
  const int last_kk = ((K2 - (num_k - 1) * KB) + 15) / 16;  // MMAs in the last k block

  if (warp == 0 && lane == 0) {
    for (int s = 0; s < C::kStages; ++s) {
      // gather / reshuffle: the TMA (B) arrive + the A producer warp's arrive
      mbar_init(&full[s], kGather ? 2 : (kAMode == 3 ? 3 : 1));
      mbar_init(&empty[s], 1);
    }
    for (int r = 0; r < 8; ++r) {
      mbar_init(&raw_full[r], 1);
      mbar_init(&raw_empty[r], 2);  // both reshuffle warps
    }
    for (int a = 0; a < C::kNAcc; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], 128);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmA)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmB)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmC)) : "memory");
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(tmem_slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      // ===== TMA producer =====
      int s = 0;
      uint32_t ph = 0;
      const uint32_t reuse_dist = (uint32_t)C::kStages * gridDim.x;  // tile that last filled this slot
      uint32_t qa = 0;  // stage counter (raw A slots)
      for (uint32_t t = blockIdx.x; t < num_tiles; t += gridDim.x) {
        int m0, n0, a_row, b_row;
        bool skip = false;
        if (ba.on) {
          batch_tile(ba, t, num_n, BN, m0, n0, a_row, b_row, skip);
        } else {
          tile_coords(sc_args, t, num_n, BM, BN, m0, n0);
          a_row = m0;
          b_row = n0;
        }
        int cm[5] = {0, 0, 0, 0, 0};  // row part of the N-d box coordinates (once per tile)
        if (nda.nd > 0) nd_coords_rows(nda, ga.m_base + (uint64_t)m0, cm);
        // single k-block: the slot still holds B of the tile kStages iterations ago; skip the B
        // load when that tile had the same n-block (always when N fits one tile)
        bool b_resident = false;
        if (!ba.on && num_k == 1 && t >= blockIdx.x + reuse_dist) {
          int pm, pn;
          tile_coords(sc_args, t - reuse_dist, num_n, BM, BN, pm, pn);
          b_resident = pn == n0;
        }
        for (int kb = 0; kb < num_k; ++kb, ++qa) {
          if constexpr (kAMode == 3) {
            // A: the raw box (source order) into raw slot qa % kRaw, for warps 2-3 to reshuffle
            const int r = (int)(qa % C::kRaw);
            mbar_wait(&raw_empty[r], ((qa / C::kRaw) & 1) ^ 1);
            mbar_expect_tx(&raw_full[r], C::kABytes);
            int cc[5];
            nd_coords_k(nda, (uint32_t)kb * (KB / 2), cm, cc);
            tma_load_nd(sRaw + r * C::kABytes, &tmA, &raw_full[r], nda.nd, cc);
          }
          mbar_wait(&empty[s], ph ^ 1);
          if (skip) {  // zero tile of the padded 2-d index: nothing to load, the MMA is skipped
            mbar_arrive(&full[s]);
          } else if (kGather || kAMode == 3) {  // A comes from the gather / reshuffle warps
            if (b_resident) {
              mbar_arrive(&full[s]);
            } else {
              mbar_expect_tx(&full[s], C::kBBytes);
              tma_load_2d(sB + s * C::kBBytes, &tmB, &full[s], kb * KB, n0);
            }
          } else {
            mbar_expect_tx(&full[s], b_resident ? C::kABytes : C::kStageBytes);
            if (nda.nd > 0) {
              int cc[5];
              nd_coords_k(nda, (uint32_t)kb * (KB / 2), cm, cc);
              tma_load_nd(sA + s * C::kABytes, &tmA, &full[s], nda.nd, cc);
            } else {
              tma_load_2d(sA + s * C::kABytes, &tmA, &full[s], kb * KB, a_row);
            }
            if (!b_resident) tma_load_2d(sB + s * C::kBBytes, &tmB, &full[s], kb * KB, b_row);
          }
          if (++s == C::kStages) {
            s = 0;
            ph ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      // ===== MMA issuer =====
      int s = 0;
      uint32_t ph = 0;
      uint32_t i = 0;
      for (uint32_t t = blockIdx.x; t < num_tiles; t += gridDim.x, ++i) {
        const uint32_t acc = i % C::kNAcc, aph = (i / C::kNAcc) & 1;
        bool skip = false;
        if (ba.on && ba.pad_r > 0) {
          int m0, n0, ar, br;
          batch_tile(ba, t, num_n, BN, m0, n0, ar, br, skip);
        }
        mbar_wait(&tempty[acc], aph ^ 1);
        tc_fence_after();
        const uint32_t tmem_d = tmem_base + acc * C::kAccStride;
        for (int kb = 0; kb < num_k; ++kb) {
          mbar_wait(&full[s], ph);
          tc_fence_after();
          if (skip) {  // zero tile: release the stage, no MMA
            mma_commit(&empty[s]);
            if (++s == C::kStages) {
              s = 0;
              ph ^= 1;
            }
            continue;
          }
          if (kGather && ga.fence) asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // experiment knob
          const int nkk = (kb == num_k - 1) ? last_kk : KB / 16;
          const uint64_t ad = kInter ? smem_desc_interleaved(sA + s * C::kABytes)
                                     : smem_desc_sw<KB>(sA + s * C::kABytes);
          const uint64_t bd = smem_desc_sw<KB>(sB + s * C::kBBytes);
          for (int kk = 0; kk < nkk; ++kk) {
            // advance 16 fp16 along K: 32 bytes inside a swizzle atom (>>4 => +2), or two
            // 2048-byte core-matrix columns in the interleaved layout (>>4 => +256)
            mma_f16(tmem_d, ad + (kInter ? 256 : 2) * kk, bd + 2 * kk, C::kIdesc, (kb | kk) != 0);
          }
          mma_commit(&empty[s]);
          if (++s == C::kStages) {
            s = 0;
            ph ^= 1;
          }
        }
        mma_commit(&tfull[acc]);
      }
    }
  } else if (kAMode == 3 && (warp == 2 || warp == 3)) {
    if constexpr (kAMode == 3) {
    // ===== A reshuffle (warps 2 and 3, alternate iterations): raw slot (source order) ->
    // interleaved K-major stage, 16-byte pieces, bank-conflict-free enumeration (NdArgs)
    const int h = warp - 2;
    uint32_t raw_lane = 0, dst_lane = 0;
#pragma unroll
    for (int b = 0; b < 5; ++b)
      if ((lane >> b) & 1) {
        raw_lane ^= (uint32_t)nda.lane_pat[b] << 4;
        dst_lane ^= nda.lane_dst[b];
      }
    const int n_it = 1 << (nda.npb - 5);
    uint2* itab = reinterpret_cast<uint2*>(gtab);  // (raw byte, stage byte) per iteration
    if (h == 0 && lane < n_it) {
      uint32_t rr = 0, dd = 0;
      for (int b = 0; b < nda.npb - 5; ++b)
        if ((lane >> b) & 1) {
          rr ^= (uint32_t)nda.it_pat[b] << 4;
          dd ^= nda.it_dst[b];
        }
      itab[lane] = make_uint2(rr, dd);
    }
    asm volatile("bar.sync 3, 64;" ::: "memory");  // both reshuffle warps see the table
    const uint32_t raw_u32 = smem_u32(sRaw), a_u32 = smem_u32(sA);
    uint32_t q = 0;
    for (uint32_t t = blockIdx.x; t < num_tiles; t += gridDim.x) {
      for (int kb = 0; kb < num_k; ++kb, ++q) {
        const int r = (int)(q % C::kRaw);
        const int s = (int)(q % C::kStages);
        mbar_wait(&raw_full[r], (q / C::kRaw) & 1);
        mbar_wait(&empty[s], ((q / C::kStages) & 1) ^ 1);
        const uint32_t src = raw_u32 + r * C::kABytes, dst = a_u32 + s * C::kABytes;
        // batches of 8 pieces: all 8 loads in flight before the 8 stores (the LDS->STS latency,
        // not bandwidth, bounded the single-piece loop)
        for (int it0 = h; it0 < n_it; it0 += 16) {
          uint4 v[8];
          uint32_t dd[8];
#pragma unroll
          for (int u = 0; u < 8; ++u) {
            const int it = it0 + 2 * u;
            if (it < n_it) {
              const uint2 e = itab[it];
              dd[u] = dst + (dst_lane ^ e.y);
              asm volatile("ld.shared.v4.b32 {%0,%1,%2,%3}, [%4];"
                           : "=r"(v[u].x), "=r"(v[u].y), "=r"(v[u].z), "=r"(v[u].w)
                           : "r"(src + (raw_lane ^ e.x)));
            }
          }
#pragma unroll
          for (int u = 0; u < 8; ++u)
            if (it0 + 2 * u < n_it)
              asm volatile("st.shared.v4.b32 [%0], {%1,%2,%3,%4};" ::"r"(dd[u]), "r"(v[u].x), "r"(v[u].y), "r"(v[u].z),
                           "r"(v[u].w)
                           : "memory");
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic writes -> UMMA reads
        __syncwarp();
        if (lane == 0) {
          mbar_arrive(&full[s]);
          mbar_arrive(&raw_empty[r]);
        }
      }
    }
    }
  } else if (kGather && warp >= 12) {
    // ===== A gather (fused stem permutation): warp g fills the ring slots s = g mod 4 with
    // cp.async 16-byte pieces at arbitrary source strides, up to 4 stages in flight per warp
    // (commit groups); a stage is published by wait_group + proxy fence + mbarrier arrive
    const int g = warp - 12;
    constexpr int kCB = KB / 8;                 // 16-byte chunks per row
    constexpr int kLogCB = kCB == 8 ? 3 : (kCB == 4 ? 2 : 1);
    constexpr int kPieces = kWord ? KB / 2 : kCB;  // pieces per row (complex elements or 16-byte chunks)
    constexpr int kIters = BM * kPieces / 32;   // pieces per lane per stage
    // piece v = it * 32 + lane; vector bits 0..4 come from the lane, 5.. from it.  Offsets and
    // (row, chunk) of both parts are tile-independent: lane part in registers, it part in a
    // 32-entry smem table (one broadcast load per piece)
    int64_t off_lane = 0;
    int r_lane = 0, c_lane = 0;
    int64_t off_it = 0;
    int r_it = 0, c_it = 0;
    for (int b = 0; b < 5 && b < ga.nvb; ++b) {
      if (!((lane >> b) & 1)) continue;
      off_lane += ga.vb_is_k[b] ? ga.ks[(kWord ? 0 : 2) + ga.vb_idx[b]] : ga.ms[ga.vb_idx[b]];
      r_lane |= ga.vb_is_k[b] ? 0 : (1 << ga.vb_idx[b]);
      c_lane |= ga.vb_is_k[b] ? (1 << ga.vb_idx[b]) : 0;
    }
    for (int it = lane; it < kIters; it += 32) {  // iteration part of the piece index (bits >= 5)
      off_it = 0;
      r_it = c_it = 0;
      for (int b = 5; b < ga.nvb; ++b) {
        if (!((it >> (b - 5)) & 1)) continue;
        off_it += ga.vb_is_k[b] ? ga.ks[(kWord ? 0 : 2) + ga.vb_idx[b]] : ga.ms[ga.vb_idx[b]];
        r_it |= ga.vb_is_k[b] ? 0 : (1 << ga.vb_idx[b]);
        c_it |= ga.vb_is_k[b] ? (1 << ga.vb_idx[b]) : 0;
      }
      gtab[it].off = off_it;
      gtab[it].rc = (r_it << 8) | c_it;
    }
    __syncwarp();
    const uint32_t sA_u32 = smem_u32(sA);
    // this warp owns ring slots g, g+4, ...; it keeps up to `depth` of them in flight (cp.async
    // groups), completing the oldest (wait_group + proxy fence + arrive) before reusing a slot
    const int owned = C::kStages > g ? (C::kStages - 1 - g) / kGatherWarps + 1 : 0;
    const int depth = owned < 4 ? owned : 4;
    uint32_t pend = 0;  // ring of pending slots, 8 bits each, oldest in the low byte
    int npend = 0;
    auto complete_oldest = [&]() {
      switch (npend - 1) {  // wait until only the npend-1 youngest groups are outstanding
        case 0: asm volatile("cp.async.wait_group 0;" ::: "memory"); break;
        case 1: asm volatile("cp.async.wait_group 1;" ::: "memory"); break;
        case 2: asm volatile("cp.async.wait_group 2;" ::: "memory"); break;
        default: asm volatile("cp.async.wait_group 3;" ::: "memory"); break;
      }
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic (cp.async) -> async proxy (UMMA)
      __syncwarp();
      if (lane == 0) mbar_arrive(&full[pend & 0xff]);
      pend >>= 8;
      --npend;
    };
    uint32_t q = 0;
    int64_t mbase = 0;
    for (uint32_t t = blockIdx.x; t < num_tiles; t += gridDim.x) {
      int m0, n0;
      tile_coords(sc_args, t, num_n, BM, BN, m0, n0);
      bool have_m = false;
      for (int kb = 0; kb < num_k; ++kb, ++q) {
        // each ring slot always belongs to the same gather warp, so its phases are waited in order
        const int s = (int)(q % C::kStages);
        if (s % kGatherWarps != g) continue;
        const uint32_t ph = (q / C::kStages) & 1;
        if (!have_m) {  // m bits >= 7 of the tile's first row
          mbase = 0;
          const uint64_t mrow = ga.m_base + (uint64_t)m0;
          for (int j = 7; j < ga.mlog; ++j)
            if ((mrow >> j) & 1) mbase += ga.ms[j];
          have_m = true;
        }
        int64_t base = mbase + off_lane;
        const uint32_t kc = (uint32_t)kb * (KB / 2);  // complex k index of the box start
        for (int j = 2 + kLogCB; j < ga.klog; ++j)
          if ((kc >> j) & 1) base += ga.ks[j];
        if (npend == depth) complete_oldest();
        mbar_wait(&empty[s], ph ^ 1);
        const uint32_t stage = sA_u32 + s * C::kABytes;
        const uint32_t* src = ga.a + base;
#pragma unroll 8
        for (int it = 0; it < kIters; ++it) {
          const GTab e = gtab[it];
          const int r = r_lane | (e.rc >> 8), c = c_lane | (e.rc & 0xff);
          // swizzled K-major row (SW128 / SW64 / SW32 as the TMA box would have written it)
          const int sw = KB == 64 ? (r & 7) : (KB == 32 ? ((r >> 1) & 3) : ((r >> 2) & 1));
          if constexpr (kWord)
            cp_async4(stage + r * (2 * KB) + ((((c >> 2) ^ sw)) << 4) + ((c & 3) << 2), src + e.off);
          else
            cp_async16(stage + r * (2 * KB) + ((c ^ sw) << 4), src + e.off);
        }
        asm volatile("cp.async.commit_group;" ::: "memory");
        pend |= (uint32_t)s << (8 * npend);
        ++npend;
      }
    }
    while (npend > 0) complete_oldest();
  } else if (warp >= 4) {
    // ===== epilogue: two independent warpgroups, group g drains the tiles i = g mod 2
    const int grp = (warp - 4) >> 2;
    const int ew = warp & 3;  // TMEM lane quarter this warp may access
    const int row = ew * 32 + lane;
    const int etid = threadIdx.x - 128 - 128 * grp;
    unsigned char* sCg = sC + grp * (C::kNBuf * BM * 128);
    int e = 0;
    if (in_max && b_bound) e = scale_exp_for(in_max[0] * b_bound[0]);
    if (exp_slot && blockIdx.x == 0 && grp == 0 && etid == 0) *exp_slot = e;
    const float sc = ldexpf(1.f, e);
    float mx = 0.f;
    const bool scat = sc_args.on != 0;
    // scatter mode: run = number of lowest n bits whose output strides are 1, 2, 4, ...: each
    // thread stores its row's values in contiguous vectors of 2^run complex (<= 16)
    int run = 0;
    if (scat)
      while (run < 4 && run < sc_args.nbits && sc_args.ns[run] == ((int64_t)1 << run)) ++run;
    uint32_t gsub = 0;  // staging subtiles used so far (ring position)
    for (uint32_t t = blockIdx.x + grp * gridDim.x, i = grp; t < num_tiles; t += 2 * gridDim.x, i += 2) {
      const uint32_t acc = i % C::kNAcc, aph = (i / C::kNAcc) & 1;
      int m0, n0;
      bool skip = false;
      if (ba.on) {
        int ar, br;
        batch_tile(ba, t, num_n, BN, m0, n0, ar, br, skip);
      } else {
        tile_coords(sc_args, t, num_n, BM, BN, m0, n0);
      }
      mbar_wait(&tfull[acc], aph);
      tc_fence_after();
      const uint32_t taddr = tmem_base + ((uint32_t)(ew * 32) << 16) + acc * C::kAccStride;
      int64_t row_off = 0;
      const bool row_ok = (uint64_t)(m0 + row) < rows;
      if (scat) {
        const uint64_t mg = (uint64_t)(m0 + row);
        for (int j = 0; j < sc_args.mbits; ++j)
          if ((mg >> j) & 1) row_off += sc_args.ms[j];
      }
#pragma unroll 1
      for (int sub = 0; sub < BN; sub += 64, ++gsub) {
        unsigned char* sbuf = sCg + (gsub % C::kNBuf) * (BM * 128);
        if (!scat && epi_stg == 3) {
          // per-warp stores: this warp's 32 rows of the slot are free once its own store has read them
          if (lane == 0) asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(C::kNBuf - 1) : "memory");
          __syncwarp();
        } else if (!scat && epi_stg != 1) {
          // ring slot free? (the TMA store that used it kNBuf subtiles ago has read it)
          if (etid == 0) asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(C::kNBuf - 1) : "memory");
          named_bar(1 + grp, 128);
        }
        // both 32-column halves of the subtile in flight before one wait
        uint32_t r[2][32];
        tmem_ld_32x32b_x32(taddr + sub, r[0]);
        if (sub + 32 < BN) tmem_ld_32x32b_x32(taddr + sub + 32, r[1]);
        tmem_ld_wait();
        if (sub + 64 >= BN) {
          // accumulator drained -> MMA may reuse it (before the stores are issued)
          tc_fence_before();
          mbar_arrive(&tempty[acc]);
        }
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int c = sub + 32 * h;
          if (c >= BN) break;
          uint32_t pk[16];
          // complex values of this 32-column chunk that exist (N < 8 pads B_P with zero rows)
          const int nleft = (int)n_cols - ((n0 + c) >> 1);
          const int nvalid = nleft < 16 ? (nleft > 0 ? nleft : 0) : 16;
          // (two copies of the loop: the common case — all 16 columns real, no zero block — without
          // the per-value selects, which cost ~25 % of the epilogue's issue slots on output-heavy steps)
          auto convert = [&](auto all_valid) {
#pragma unroll
            for (int j = 0; j < 16; ++j) {
              float x0 = __uint_as_float(r[h][2 * j]) * sc, x1 = __uint_as_float(r[h][2 * j + 1]) * sc;
              if constexpr (!decltype(all_valid)::value) {
                if (skip) x0 = x1 = 0.f;  // zero block of the padded 2-d index (TMEM was not written)
              }
              __half2 hv = __floats2half2_rn(x0, x1);
              // the max of the scaled fp32 values (not of their fp16 roundings): it stays meaningful when
              // cancellation pushes the stored values into fp16 subnormals or zero (scale re-run, redo_check)
              if (decltype(all_valid)::value || j < nvalid) mx = fmaxf(mx, fmaxf(fabsf(x0), fabsf(x1)));
              pk[j] = *reinterpret_cast<uint32_t*>(&hv);
            }
          };
          if (nvalid == 16 && !skip)
            convert(std::true_type{});
          else
            convert(std::false_type{});
          if (scat) {
            if (row_ok) {
              const uint64_t nb = (uint64_t)((n0 + c) >> 1);  // a multiple of 16: bits 0..3 are q's
              const int V = 1 << run;
              // the 16 columns' offsets = this chunk's base (its n bits >= 4, once per chunk) + the
              // offset of q's bits 0..3 (compile-time q, four strides in registers): a couple of adds
              // per store instead of a loop over every n bit
              int64_t nbase = row_off;
              for (int j = 4; j < sc_args.nbits; ++j)
                if ((nb >> j) & 1) nbase += sc_args.ns[j];
              const int64_t ns0 = run <= 0 && sc_args.nbits > 0 ? sc_args.ns[0] : 0;
              const int64_t ns1 = run <= 1 && sc_args.nbits > 1 ? sc_args.ns[1] : 0;
              const int64_t ns2 = run <= 2 && sc_args.nbits > 2 ? sc_args.ns[2] : 0;
              const int64_t ns3 = run <= 3 && sc_args.nbits > 3 ? sc_args.ns[3] : 0;
              // q and v are compile-time (full unroll) so pk stays in registers
#pragma unroll
              for (int q = 0; q < 16; ++q) {
                if ((q & (V - 1)) || q >= nvalid) continue;
                const int64_t off = nbase + ((q & 1) ? ns0 : 0) + ((q & 2) ? ns1 : 0) + ((q & 4) ? ns2 : 0) +
                                    ((q & 8) ? ns3 : 0);
                uint32_t* dst = out_scatter + off;
                if (V >= 8) {
                  // 256-bit stores (STG.256): one full 32-byte sector per instruction and thread
#pragma unroll
                  for (int v = 0; v < 16; v += 8)
                    if (v < V && q + v + 7 < 16)
                      asm volatile("st.global.v8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(dst + v), "r"(pk[q + v]),
                                   "r"(pk[q + v + 1]), "r"(pk[q + v + 2]), "r"(pk[q + v + 3]), "r"(pk[q + v + 4]),
                                   "r"(pk[q + v + 5]), "r"(pk[q + v + 6]), "r"(pk[q + v + 7])
                                   : "memory");
                } else if (V == 4) {
                  if (q + 3 < 16) *reinterpret_cast<uint4*>(dst) = make_uint4(pk[q], pk[q + 1], pk[q + 2], pk[q + 3]);
                } else if (V == 2) {
                  if (q + 1 < 16) *reinterpret_cast<uint2*>(dst) = make_uint2(pk[q], pk[q + 1]);
                } else {
                  *dst = pk[q];
                }
              }
            }
          } else if (BN == 64 && epi_stg == 6) {
            // row-folded GEMM (f = 2) with a transposed output: tile row p holds output rows 2p + h
            // (h = this 32-column half) for 16 complex columns; staged as C^T [16 n][256 m], one
            // TMA box of 1 KB rows
            const uint32_t sb = smem_u32(sbuf);
#pragma unroll
            for (int j = 0; j < 16; ++j) sts32(sb + 4u * (j * (2 * BM) + 2 * row + h), pk[j]);
          } else if (epi_stg == 4) {
            // transposed store C[n][m] (layout policy 3): stage the subtile as [32 complex n][128 m]
            // (each warp writes 32 consecutive words per column: no bank conflict), then one TMA box
            const uint32_t sb = smem_u32(sbuf);
            const int q0 = (c & 63) >> 1;  // first complex column of these 32 real columns
#pragma unroll
            for (int j = 0; j < 16; ++j) sts32(sb + 4u * ((q0 + j) * BM + row), pk[j]);
          } else if (BN < 64 && epi_stg == 5) {
            // packed narrow rows: 64 / BN output rows (BN fp16 each) share one 128-byte staging row,
            // stored as rows of 128 B (the TMA engine's per-row cost made 32/64-byte rows its limit)
            constexpr int kFo = BN < 64 ? 64 / BN : 1;
            const int prow = row / kFo, part = row % kFo;
            const uint32_t srow = smem_u32(sbuf) + prow * 128;
#pragma unroll
            for (int q = 0; q < BN / 8; ++q) {
              const int chunk = (part * (BN / 8) + q) ^ (prow & 7);
              sts128(srow + chunk * 16, pk[4 * q], pk[4 * q + 1], pk[4 * q + 2], pk[4 * q + 3]);
            }
          } else {
            const uint32_t srow = smem_u32(sbuf) + row * 128;
            const int cb = (c & 63) >> 3;  // first 16-byte chunk of these 32 columns
#pragma unroll
            for (int q = 0; q < 4; ++q) {
              if ((c & 63) + q * 8 < BN || BN >= 64) {
                const int chunk = (cb + q) ^ (row & 7);
                sts128(srow + chunk * 16, pk[4 * q], pk[4 * q + 1], pk[4 * q + 2], pk[4 * q + 3]);
              }
            }
          }
        }
        if (!scat && epi_stg == 1) {
          // coalesced stores from the staged subtile: 8 threads per 128-byte row segment, each warp
          // instruction writes 4 full lines (LSU path instead of the TMA store engine)
          named_bar(1 + grp, 128);
          const uint32_t pitch = num_n * BN;  // halfs per output row
          const int ncol = (int)(2 * n_cols);
#pragma unroll 4
          for (int it = 0; it < 8; ++it) {
            const int id = it * 128 + etid;
            const int rr = id >> 3, cc = id & 7;
            const int col = n0 + sub + cc * 8;
            if ((uint64_t)(m0 + rr) < rows && col < ncol && (BN >= 64 || sub + cc * 8 < BN)) {
              const uint4 v = *reinterpret_cast<const uint4*>(sbuf + rr * 128 + ((cc ^ (rr & 7)) << 4));
              __half* gp = reinterpret_cast<__half*>(out_scatter) + (uint64_t)(m0 + rr) * pitch + col;
              *reinterpret_cast<uint4*>(gp) = v;
            }
          }
          named_bar(1 + grp, 128);  // the ring slot may be rewritten
        } else if (!scat && epi_stg == 3) {
          // experiment: each warp stores its own 32 x 64 box (no group barrier per subtile)
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          __syncwarp();
          if (lane == 0) {
            tma_store_2d(&tmC, sbuf + ew * 32 * 128, n0 + sub, m0 + ew * 32);
            asm volatile("cp.async.bulk.commit_group;" ::: "memory");
          }
        } else if (!scat) {
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          named_bar(1 + grp, 128);
          if (etid == 0) {
            if (epi_stg == 2) {  // experiment: streaming output, evict-first in L2
              uint64_t pol;
              asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
              tma_store_2d_hint(&tmC, sbuf, n0 + sub, m0, pol);
            } else if (ps.on) {
              // fused mode swap: the box goes to the swap member owning it (PeerStore)
              uint64_t gm = ga.m_base + (uint64_t)m0;
              uint32_t nc = (uint32_t)(n0 + sub) >> 1;
              const int v = peer_coords(ps, gm, nc);
              if (epi_stg == 4)
                tma_store_2d(&ps.maps[v], sbuf, (int)gm, (int)nc);
              else if (BN < 64 && epi_stg == 5)
                tma_store_2d(&ps.maps[v], sbuf, 0, (int)(gm / (64 / BN)));
              else
                tma_store_2d(&ps.maps[v], sbuf, (int)(2 * nc), (int)gm);
            } else if (BN < 64 && epi_stg == 5) {
              tma_store_2d(&tmC, sbuf, 0, m0 / (64 / BN));  // [rows / (64 / BN)][64 fp16] map
            } else if (BN == 64 && epi_stg == 6) {
              tma_store_2d(&tmC, sbuf, (int)(2 * (ga.m_base + (uint64_t)m0)), 0);  // C^T map, box {256 m, 16 n}
            } else if (epi_stg == 4) {
              // box {128 m (inner, global row), 32 complex n} of the C^T map
              tma_store_2d(&tmC, sbuf, (int)(ga.m_base + (uint64_t)m0), (n0 + sub) >> 1);
            } else {
              tma_store_2d(&tmC, sbuf, n0 + sub, m0);
            }
            asm volatile("cp.async.bulk.commit_group;" ::: "memory");
          }
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
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 2) {
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem_base));
  }
}

}  // namespace tc

// ---- host side ----
static PFN_cuTensorMapEncodeTiled_v12000 get_encode() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  });
  if (!fn) throw TnError{TN_E_CUDA, "cuTensorMapEncodeTiled unavailable"};
  return fn;
}

static CUtensorMap make_map_2d(const void* base, uint64_t inner, uint64_t outer, uint32_t box_inner,
                               uint32_t box_outer) {
  // swizzle width = the box row (64 fp16 = 128 B, 32 = 64 B, 16 = 32 B), matching smem_desc_sw
  const CUtensorMapSwizzle sw = box_inner >= 64 ? CU_TENSOR_MAP_SWIZZLE_128B
                                : (box_inner == 32 ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_32B);
  CUtensorMap m;
  cuuint64_t dims[2] = {inner, outer};
  cuuint64_t strides[1] = {inner * 2};
  cuuint32_t box[2] = {box_inner, box_outer};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = get_encode()(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, const_cast<void*>(base), dims, strides, box, estr,
                            CU_TENSOR_MAP_INTERLEAVE_NONE, sw,
                            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) throw TnError{TN_E_CUDA, "cuTensorMapEncodeTiled failed (" + std::to_string((int)r) + ")"};
  return m;
}

// C^T [N complex][M complex] as 4-byte elements (one complex-half value each), box {128 m, 32 n}
// (N < 32: {128 m, N n}, the tile's single n block)
static CUtensorMap make_map_t(const void* base, uint64_t M, uint64_t N, uint32_t box_m = tc::BM) {
  CUtensorMap m;
  cuuint64_t dims[2] = {M, N};
  cuuint64_t strides[1] = {M * 4};
  cuuint32_t box[2] = {box_m, (cuuint32_t)std::min<uint64_t>(N, 32)};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = get_encode()(&m, CU_TENSOR_MAP_DATA_TYPE_UINT32, 2, const_cast<void*>(base), dims, strides, box, estr,
                            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) throw TnError{TN_E_CUDA, "cuTensorMapEncodeTiled (C^T) failed (" + std::to_string((int)r) + ")"};
  return m;
}

// Fused mode swap (PeerTarget, common.cuh): the store maps of the swap members, or on = 0 when this
// launch's epilogue cannot do it (scatter or direct stores, batched launches, member bits inside a
// store box).  pt->honored tells the runtime whether the exchange happened here.
static PeerStore make_peer_store(PeerTarget* pt, bool tma_epi, bool transposed, uint64_t M, uint32_t N2_real,
                                 uint32_t box_rows = tc::BM, int pack = 1) {
  PeerStore ps;
  memset(&ps, 0, sizeof(ps));
  if (!pt) return ps;
  pt->honored = 0;
  if (!tma_epi || pt->nsw <= 0 || pt->nsw > 3) return ps;
  const uint64_t Nc = N2_real / 2;
  struct E {
    int is_n, bit, vbit;
  };
  std::vector<E> es;
  int mrem = 0, nrem = 0;
  for (int t = 0; t < pt->nsw; ++t) {
    const int b = pt->bit[t];
    if (pt->is_n[t]) {
      if (b < 5 || (1ull << b) >= Nc || pack > 1) return ps;  // a 32-column store box would span two members
      ++nrem;
    } else {
      if ((1 << b) < (int)box_rows || (1ull << b) >= M) return ps;   // a row box would span two members
      ++mrem;
    }
    es.push_back({pt->is_n[t], b, pt->vbit[t]});
  }
  std::sort(es.begin(), es.end(), [](const E& x, const E& y) { return x.is_n != y.is_n ? x.is_n < y.is_n : x.bit > y.bit; });
  const uint64_t Mp = M >> mrem, Np = Nc >> nrem;
  if (Mp >= (1ull << 31) || 2 * Np >= (1ull << 31)) return ps;
  for (int v = 0; v < (1 << pt->nsw); ++v)
    ps.maps[v] = transposed ? make_map_t(pt->base[v], Mp, Np, box_rows)
                 : pack > 1 ? make_map_2d(pt->base[v], 64, Mp / pack, 64, box_rows / pack)
                            : make_map_2d(pt->base[v], 2 * Np, Mp, 64, box_rows);
  ps.nsw = pt->nsw;
  for (int t = 0; t < ps.nsw; ++t) {
    ps.is_n[t] = (int8_t)es[t].is_n;
    ps.bit[t] = (int8_t)es[t].bit;
    ps.vbit[t] = (int8_t)es[t].vbit;
  }
  ps.on = 1;
  pt->honored = 1;
  return ps;
}

static int num_sms() {
  int dev = 0, n = 0;
  TN_CUDA(cudaGetDevice(&dev));
  TN_CUDA(cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev));
  return n;
}

// Gathered A as one N-dimensional TMA box (<= 5 dims).  Logical bits of a stage: complex k bits
// and m (row) bits with source positions log2(stride).  w = number of k bits sitting at source bits
// 0..w-1.  w >= 3: rows of 2^min(w,5) complex (32/64/128 B, swizzled like the 2-D path), box =
// [row][m0..m6].  w == 2: no-swizzle core matrices, box = [k0 k1 m0..m6 | k2..k(1+cb)] so the smem
// image is [k piece][row][16 B].  Each tensor dim is a maximal run of logical successors at
// consecutive source bits (box bits first, <= 8 per dim); more than 5 dims -> not representable.
struct NdPlan {
  int interleaved = 0, KB = 0, nd = 0;
  uint64_t dim[5], stride[5];
  uint32_t box[5];
  NdArgs args;
};

static CUtensorMap make_map_nd(const void* base, const NdPlan& np) {
  CUtensorMap m;
  cuuint64_t dims[5], strides[4];
  cuuint32_t box[5], estr[5];
  for (int d = 0; d < np.nd; ++d) {
    dims[d] = np.dim[d];
    box[d] = np.box[d];
    estr[d] = 1;
    if (d) strides[d - 1] = np.stride[d];
  }
  const int row_bytes = (int)np.box[0] * 4;
  const CUtensorMapSwizzle sw = np.interleaved ? CU_TENSOR_MAP_SWIZZLE_NONE
                                : (row_bytes >= 128 ? CU_TENSOR_MAP_SWIZZLE_128B
                                   : (row_bytes == 64 ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_32B));
  CUresult r = get_encode()(&m, CU_TENSOR_MAP_DATA_TYPE_UINT32, np.nd, const_cast<void*>(base), dims, strides, box,
                            estr, CU_TENSOR_MAP_INTERLEAVE_NONE, sw, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) throw TnError{TN_E_CUDA, "cuTensorMapEncodeTiled (N-d gather) failed (" + std::to_string((int)r) + ")"};
  return m;
}

// CTA-pair variant (gemm_tc2.cuh, k_gemm_tc2.cu)
bool tc2_enabled();
void launch_tc2(int BN, const CUtensorMap& ma, const CUtensorMap& mb, const CUtensorMap& mc, uint32_t num_mp,
                uint32_t num_n, int K2, const float* in_max, const float* b_bound, uint32_t* out_max, int* exp_slot,
                int epi, uint64_t m_base, const PeerStore& ps, const NdArgs& nda, cudaStream_t s, int a_inter = 0);

template <int BN, int KB, int G>
static void launch_bn(__half* c, const __half* a, const __half* bp, uint64_t M, uint32_t K2, uint32_t N2_real,
                      const float* in_max, const float* b_bound, uint32_t* out_max, int* exp_slot, const OutMap* om,
                      cudaStream_t s, const AGather* ag, const NdPlan* np, const BatchSpec* bs) {
  const uint32_t N2 = std::max<uint32_t>(N2_real, 16);  // B_P has at least 16 (zero-padded) rows
  using C = tc::Cfg<BN, KB, G>;
  {
    // the dynamic shared-memory opt-in is per device: remember it per device ordinal (a process may
    // drive several devices, e.g. one thread per GPU)
    static std::mutex mu;
    static uint64_t done = 0;
    int dev = 0;
    TN_CUDA(cudaGetDevice(&dev));
    std::lock_guard<std::mutex> lk(mu);
    if (dev >= 64 || !((done >> dev) & 1)) {
      TN_CUDA(cudaFuncSetAttribute(tc::gemm_chalf_tc_kernel<BN, KB, G>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   C::kSmem));
      if (dev < 64) done |= 1ull << dev;
    }
  }
  AGatherArgs gargs;
  memset(&gargs, 0, sizeof(gargs));
  NdArgs nda;
  memset(&nda, 0, sizeof(nda));
  if (np) nda = np->args;
  if (G == 1 || G == 4) {
    // vector bits of a stage: 7 row bits + log2(KB/8) chunk bits (G = 4: log2(KB/2) complex k bits),
    // by source stride (lanes take the 5 smallest: the most contiguous reads)
    gargs.a = reinterpret_cast<const uint32_t*>(a);
    static const bool fence_env = getenv("TN_GATHER_FENCE") != nullptr;
    gargs.fence = fence_env ? 1 : 0;
    gargs.mlog = ag->mlog;
    gargs.klog = ag->klog;
    for (int j = 0; j < kMaxModes; ++j) gargs.ms[j] = ag->ms[j];
    for (int j = 0; j < 24; ++j) gargs.ks[j] = ag->ks[j];
    struct VB {
      int64_t stride;
      int is_k, idx;
    };
    std::vector<VB> vb;
    for (int j = 0; j < 7; ++j) vb.push_back({ag->ms[j], 0, j});
    const int cb = G == 4 ? (KB == 64 ? 5 : (KB == 32 ? 4 : 3)) : (KB == 64 ? 3 : (KB == 32 ? 2 : 1));
    for (int j = 0; j < cb; ++j) vb.push_back({ag->ks[(G == 4 ? 0 : 2) + j], 1, j});
    std::stable_sort(vb.begin(), vb.end(), [](const VB& x, const VB& y) { return x.stride < y.stride; });
    gargs.nvb = (int)vb.size();
    for (int b = 0; b < gargs.nvb; ++b) {
      gargs.vb_is_k[b] = (int8_t)vb[b].is_k;
      gargs.vb_idx[b] = (int8_t)vb[b].idx;
    }
  }
  ScatterArgs sa;
  memset(&sa, 0, sizeof(sa));
  const uint32_t n_cols = N2_real / 2;
  // transposed output C[n][m] (layout policy 3): TMA stores of [32 n][128 m] boxes of a C^T map when
  // the tile geometry allows (whole 128-row tiles; whole 64-column subtiles, or N = 8 / 16 complex
  // columns in one tile and one narrower box), else the scatter path
  const bool transposed = om && om->transposed && M % tc::BM == 0 &&
                          (N2_real % 64 == 0 || N2_real == 16 || N2_real == 32) && M < (1ull << 31) &&
                          !getenv("TN_NO_TSTORE");
  OutMap ident;
  static const bool direct_env = getenv("TN_DIRECT_EPI") != nullptr;  // experiment knob
  if ((N2_real < 16 || direct_env) && (!om || om->identity)) {  // TMA stores need 16-byte rows
    ident = identity_map(M, N2_real / 2);
    om = &ident;
    ident.identity = 0;
  }
  if (om && !om->identity && !transposed) {
    sa.on = 1;
    sa.mbits = om->mbits;
    sa.nbits = om->nbits;
    {
      // m-block bits (m bits >= 7) and n-block bits (complex n bits >= log2(BN/2)), by output stride
      int cb = 0;
      while ((1 << cb) < BN / 2) ++cb;
      struct VB {
        int64_t stride;
        int is_m, idx;
      };
      std::vector<VB> vb;
      // only the m bits inside one launch chunk (chunks cover 2^30 rows or fewer, see below)
      const uint64_t chunk_rows = std::min<uint64_t>(1ull << 30, ((1ull << 31) / (N2 / BN)) * tc::BM);
      int cl2 = 0;
      while ((1ull << cl2) < chunk_rows) ++cl2;
      for (int j = 7; j < std::min(om->mbits, cl2); ++j) vb.push_back({om->ms[j], 1, j - 7});
      for (int j = cb; j < om->nbits; ++j) vb.push_back({om->ns[j], 0, j - cb});
      std::stable_sort(vb.begin(), vb.end(), [](const VB& x, const VB& y) { return x.stride < y.stride; });
      sa.nv = (int)vb.size();
      if (sa.nv > 31) throw TnError{TN_E_UNSUPPORTED, "too many tile bits"};
      for (int b = 0; b < sa.nv; ++b) {
        sa.vbit_is_m[b] = (int8_t)vb[b].is_m;
        sa.vbit_idx[b] = (int8_t)vb[b].idx;
      }
    }
    for (int j = 0; j < kMaxModes; ++j) sa.ms[j] = om->ms[j];
    for (int j = 0; j < 24; ++j) sa.ns[j] = om->ns[j];
  }
  if (bs) {
    // gather-batched launch (Fig. 5): one launch over every entry, plain 2-D maps over all entries
    if (G != 0 || np || (om && !om->identity) || N2_real < 16 || M % tc::BM)
      throw TnError{TN_E_INVALID, "batched GEMM: needs M % 128 == 0, 2N >= 16, identity output, plain A"};
    BatchArgs ba;
    memset(&ba, 0, sizeof(ba));
    ba.on = 1;
    ba.pad_r = bs->pad_r;
    ba.ia = bs->ia;
    ba.ib = bs->ib;
    ba.table = bs->table;
    ba.m_tiles = (uint32_t)(M / tc::BM);
    ba.rows = M;
    ba.b_rows = N2;
    const uint32_t cols = bs->pad_r > 0 ? (uint32_t)bs->pad_r * N2 : N2;  // C columns per row
    if (N2 % BN) throw TnError{TN_E_INVALID, "batched GEMM: B block rows must be a multiple of the tile"};
    // the epilogue stages 64-column subtiles and stores them with a 64-wide TMA box: a C row narrower
    // than one tile is clipped by the map, a padded row of several narrow blocks would be overwritten
    if (bs->pad_r > 1 && N2 < 64) throw TnError{TN_E_INVALID, "padded 2-d index: needs N >= 32"};
    const uint64_t a_rows = (uint64_t)bs->n_a * M, c_rows = (uint64_t)bs->n_out * M;
    const uint64_t b_rows_all = (uint64_t)bs->n_b * N2;
    if (a_rows >= (1ull << 31) || c_rows >= (1ull << 31) || b_rows_all >= (1ull << 31))
      throw TnError{TN_E_UNSUPPORTED, "batched GEMM: more than 2^31 rows"};
    CUtensorMap ma = make_map_2d(a, K2, a_rows, KB, tc::BM);
    CUtensorMap mbm = make_map_2d(bp, K2, b_rows_all, KB, BN);
    CUtensorMap mc = make_map_2d(c, cols, c_rows, 64, tc::BM);
    const uint32_t num_n = cols / BN;
    const uint64_t tiles = (uint64_t)bs->n_out * ba.m_tiles * num_n;
    if (tiles == 0) return;
    if (tiles >= (1ull << 32)) throw TnError{TN_E_UNSUPPORTED, "batched GEMM: too many tiles"};
    const int grid = (int)std::min<uint64_t>(tiles, (uint64_t)num_sms());
    ScatterArgs sa0;
    memset(&sa0, 0, sizeof(sa0));
    AGatherArgs g0;
    memset(&g0, 0, sizeof(g0));
    NdArgs n0;
    memset(&n0, 0, sizeof(n0));
    g_last_kern = "tc1";
    tc::gemm_chalf_tc_kernel<BN, KB, G><<<grid, tc::kThreads, C::kSmem, s>>>(
        ma, mbm, mc, (uint32_t)(tiles / num_n), num_n, (int)K2, in_max, b_bound, out_max, exp_slot, sa0,
        reinterpret_cast<uint32_t*>(c), c_rows, cols / 2, g0, n0, 0, ba, PeerStore{});
    TN_CUDA(cudaGetLastError());
    return;
  }
  CUtensorMap mb = make_map_2d(bp, K2, N2_real, KB, BN);  // rows >= 2N: TMA zero fill
  // output store mode: 0 = one 128-row TMA store per subtile after a group barrier.  Experiments
  // (TN_STG_EPI): 1 = LSU stores from the staged subtile (slower); 2 = evict-first L2 hint (mixed);
  // 3 = each warp stores its own 32 rows with no group barrier (3-4 % faster on standalone
  // output-heavy GEMMs, but no net change over the C3 plan's N >= 2^8 steps: 23.84 -> 23.71 ms)
  static const int stg_env = getenv("TN_STG_EPI") ? atoi(getenv("TN_STG_EPI")) : 0;
  const int epi_stg = stg_env;
  // TMA coordinates are int32: process M in chunks of at most 2^30 rows
  const uint32_t num_n = N2 / BN;
  const uint64_t chunk = std::min<uint64_t>(1ull << 30, ((1ull << 31) / num_n) * tc::BM);
  // packed narrow rows (epilogue mode 5): a row-major output whose rows are 32 or 64 bytes is staged
  // and TMA-stored as rows of 128 B (64 / BN output rows each)
  // row-folded GEMM (f = 2, 16 complex columns per output row) whose output is transposed C^T
  // (epilogue mode 6): the caller marks it with OutMap::fold_t = 2; M, N2_real are the folded shape
  const bool fold_t = om && om->fold_t == 2 && BN == 64 && N2_real == 64 && !bs && M % tc::BM == 0;
  if (om && om->fold_t && !fold_t) throw TnError{TN_E_INVALID, "folded transposed output: unsupported geometry"};
  static const bool no_pack = getenv("TN_NO_PACK") != nullptr;  // A/B knob
  const bool packed = BN < 64 && !no_pack && !sa.on && !bs && epi_stg == 0 && !transposed && (!om || om->identity) &&
                      N2_real == (uint32_t)BN && M % tc::BM == 0;
  const PeerStore ps = make_peer_store(om ? om->peer : nullptr, !sa.on && epi_stg == 0 && (transposed || (om && om->identity)),
                                       transposed, M, N2_real, tc::BM, packed ? 64 / BN : 1);
  if constexpr ((G == 0 || G == 2) && KB == 64 && BN >= 64) {
    // plain A, row-major or transposed output, whole 256-row pair tiles: the CTA-pair kernel (half
    // the B tile staged per SM: fewer shared-memory bytes per MAC on the compute-bound steps)
    // (also the gathered steps whose permutation is one N-d TMA box of 128-byte swizzled rows: the
    // producer computes the box coordinates from the global row, the stage image is the same)
    // (G = 2: the N-d box lands in the no-swizzle core-matrix layout; TN_TC2_INTER=0 keeps it on tc1)
    static const bool inter_ok = !getenv("TN_TC2_INTER") || atoi(getenv("TN_TC2_INTER")) != 0;
    const bool nd_ok = G == 2 ? (inter_ok && np && np->nd > 0 && np->interleaved && np->KB == 64)
                              : (!np || (np->nd > 0 && !np->interleaved && np->KB == 64));
    // (a row-major output with BN = 128 and K <= 64 complex stays single-CTA: mubench M = 2^25, k5 n6
    // 2.16 vs 2.95 ms, k6 n6 2.60 vs 3.38 ms; from BN = 256 or K >= 128 the pair kernel is equal or
    // faster; transposed outputs: C3 step 29, m26 k5 n6, no better on the single-CTA kernel)
    // (BN = 64: only K-heavy steps, K >= 128 complex, e.g. C3 step 31 m16 k16 n5)
    const bool pair_wins = BN >= 128 ? (BN >= 256 || K2 >= 256 || transposed) : K2 >= 256;
    if (nd_ok && pair_wins && !sa.on && epi_stg == 0 && M % 256 == 0 && N2_real % BN == 0 && chunk % 256 == 0 &&
        tc2_enabled()) {
      CUtensorMap mb2 = make_map_2d(bp, K2, N2_real, KB, BN / 2);
      for (uint64_t m_off = 0; m_off < M; m_off += chunk) {
        const uint64_t mm = std::min<uint64_t>(chunk, M - m_off);
        CUtensorMap ma = np ? make_map_nd(a, *np) : make_map_2d(a + m_off * K2, K2, mm, KB, tc::BM);
        CUtensorMap mc = transposed ? make_map_t(c, M, N2_real / 2) : make_map_2d(c + m_off * N2, N2, mm, 64, tc::BM);
        launch_tc2(BN, ma, mb2, mc, (uint32_t)(mm / 256), num_n, (int)K2, in_max, b_bound, out_max,
                   m_off ? nullptr : exp_slot, transposed ? 4 : 0, m_off, ps, nda, s, G == 2 ? 1 : 0);
      }
      return;
    }
  }
  for (uint64_t m_off = 0; m_off < M; m_off += chunk) {
    uint64_t mm = std::min<uint64_t>(chunk, M - m_off);
    // (cp.async gather: the A map is unused; N-d: the whole stem, coordinates from the global row)
    // plain TMA A (modes 0 and 5): a 2-D map over this chunk's rows; the gathers (1, 4) do not use it
    constexpr bool kPlainA = G == 0 || G == 5;
    CUtensorMap ma = np ? make_map_nd(a, *np)
                        : make_map_2d(kPlainA ? a + m_off * K2 : a, K2, kPlainA ? mm : tc::BM, KB, tc::BM);
    gargs.m_base = m_off;
    CUtensorMap mc = fold_t     ? make_map_t(c, 2 * M, 16, 2 * tc::BM)
                     : transposed ? make_map_t(c, M, N2_real / 2)
                     : packed   ? make_map_2d(c + m_off * N2, 64, mm * N2 / 64, 64, tc::BM * BN / 64)
                                : make_map_2d(c + m_off * N2, N2, mm, 64, epi_stg == 3 ? 32 : tc::BM);
    // scatter: base of this chunk's rows in the OutMap; row-major: the chunk's first row (STG epilogue)
    uint32_t* out_sc = reinterpret_cast<uint32_t*>(c) + (sa.on ? outmap_m(*om, m_off) : m_off * (N2 / 2));
    uint32_t num_m = (uint32_t)((mm + tc::BM - 1) / tc::BM);
    uint64_t tiles = (uint64_t)num_m * num_n;
    int grid = (int)std::min<uint64_t>(tiles, (uint64_t)num_sms());
    // the exponent is recorded once (first chunk); later chunks reuse the same inputs
    g_last_kern = "tc1";
    tc::gemm_chalf_tc_kernel<BN, KB, G><<<grid, (G == 1 || G == 4) ? tc::kThreadsGather : tc::kThreads, C::kSmem, s>>>(
        ma, mb, mc, num_m, num_n, (int)K2, in_max, b_bound, out_max, m_off ? nullptr : exp_slot, sa, out_sc, mm,
        n_cols, gargs, nda, fold_t ? 6 : (transposed ? 4 : (packed ? 5 : epi_stg)), BatchArgs{}, ps);
    TN_CUDA(cudaGetLastError());
  }
}

template <int KB, int G>
static void launch_k(__half* c, const __half* a, const __half* bp, uint64_t M, uint32_t K2, uint32_t N2,
                     const float* in_max, const float* b_bound, uint32_t* out_max, int* exp_slot, const OutMap* om,
                     cudaStream_t s, const AGather* ag, const NdPlan* np, const BatchSpec* bs) {
  static const uint32_t bn_cap = getenv("TN_MAX_BN") ? (uint32_t)atoi(getenv("TN_MAX_BN")) : 256;  // tuning knob
  const uint32_t nsel = std::min<uint32_t>(N2 < 16 ? 16 : N2, bn_cap);
  switch (nsel) {
    case 16: launch_bn<16, KB, G>(c, a, bp, M, K2, N2, in_max, b_bound, out_max, exp_slot, om, s, ag, np, bs); break;
    case 32: launch_bn<32, KB, G>(c, a, bp, M, K2, N2, in_max, b_bound, out_max, exp_slot, om, s, ag, np, bs); break;
    case 64: launch_bn<64, KB, G>(c, a, bp, M, K2, N2, in_max, b_bound, out_max, exp_slot, om, s, ag, np, bs); break;
    case 128: launch_bn<128, KB, G>(c, a, bp, M, K2, N2, in_max, b_bound, out_max, exp_slot, om, s, ag, np, bs); break;
    default: launch_bn<256, KB, G>(c, a, bp, M, K2, N2, in_max, b_bound, out_max, exp_slot, om, s, ag, np, bs); break;
  }
}

template <int G>
void launch_kb(int KB, __half* c, const __half* a, const __half* bp, uint64_t M, uint32_t K2, uint32_t N2,
                      const float* in_max, const float* b_bound, uint32_t* out_max, int* exp_slot, const OutMap* om,
                      cudaStream_t s, const AGather* ag, const NdPlan* np, const BatchSpec* bs) {
  switch (KB) {
    case 64: launch_k<64, G>(c, a, bp, M, K2, N2, in_max, b_bound, out_max, exp_slot, om, s, ag, np, bs); break;
    case 32: launch_k<32, G>(c, a, bp, M, K2, N2, in_max, b_bound, out_max, exp_slot, om, s, ag, np, bs); break;
    default: launch_k<16, G>(c, a, bp, M, K2, N2, in_max, b_bound, out_max, exp_slot, om, s, ag, np, bs); break;
  }
}

}  // namespace tn
