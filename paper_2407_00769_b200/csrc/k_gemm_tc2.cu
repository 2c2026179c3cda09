// Launcher of the CTA-pair (cta_group::2) tcgen05 GEMM; the kernel and its design are in
// gemm_tc2.cuh, the choice between it and the single-CTA kernel in gemm_tc.cuh (launch_bn).
#include "gemm_tc2.cuh"

namespace tn {

bool tc2_enabled() {
  static const bool on = !getenv("TN_TC2") || atoi(getenv("TN_TC2")) != 0;
  return on;
}

template <int BN, bool kMN>
static void launch_tc2_t(const CUtensorMap& ma, const CUtensorMap& mb, const CUtensorMap& mc, uint32_t num_mp,
                         uint32_t num_n, int K2, const float* in_max, const float* b_bound, uint32_t* out_max,
                         int* exp_slot, int epi, uint64_t m_base, const PeerStore& ps, const NdArgs& nda,
                         int mn_ma, const tc2::RowPerm& rp, cudaStream_t s, int a_inter = 0) {
  using C = tc2::Cfg2<BN>;
  // per device: the shared-memory opt-in and how many CTA pairs can be resident at once (an odd SM
  // count per GPC leaves SMs without a partner, so this can be below #SMs / 2)
  static std::mutex mu;
  static int max_pairs[64] = {0};  // (per instantiation)
  int dev = 0;
  TN_CUDA(cudaGetDevice(&dev));
  int pairs;
  {
    std::lock_guard<std::mutex> lk(mu);
    if (dev >= 64 || max_pairs[dev] == 0) {
      TN_CUDA(cudaFuncSetAttribute(tc2::gemm_chalf_tc2_kernel<BN, kMN>, cudaFuncAttributeMaxDynamicSharedMemorySize, C::kSmem));
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(2 * 128, 1, 1);
      cfg.blockDim = dim3(tc::kThreads, 1, 1);
      cfg.dynamicSmemBytes = C::kSmem;
      int n = 0;
      TN_CUDA(cudaOccupancyMaxActiveClusters(&n, tc2::gemm_chalf_tc2_kernel<BN, kMN>, &cfg));
      if (n <= 0) throw TnError{TN_E_CUDA, "CTA-pair GEMM: no resident cluster"};
      if (dev < 64) max_pairs[dev] = n;
      pairs = n;
    } else {
      pairs = max_pairs[dev];
    }
  }
  const uint64_t tiles = (uint64_t)num_mp * num_n;
  if (tiles == 0) return;
  // tile order (tc2_tile): per-cluster m-pairs (order 1) only when every cluster's A rows fit in L2
  // together (K2 x 256 rows x 2 B x pairs <= 40 MB, i.e. K <= 2^9) and there are enough m-pairs to
  // keep every cluster busy; otherwise n fastest across clusters (order 0: the clusters sharing an
  // m-pair read its A rows at the same time).  Measured on C3 step 30 (m21 k11 n11): order 0 49-52
  // ms vs order 1 55-56 ms; mubench M = 2^21, K = N = 2^10: DRAM reads 19 GB vs 33 GB (A = 8.6 GB).
  // TN_TC2_ORDER = 0 / 1 forces either (A/B knob)
  static const int order_env = getenv("TN_TC2_ORDER") ? atoi(getenv("TN_TC2_ORDER")) : -1;
  const bool a_fits_l2 = (uint64_t)K2 * 256 * 2 * (uint64_t)pairs <= (40ull << 20);
  const int order = order_env >= 0 ? order_env : (a_fits_l2 && num_mp >= 8ull * (uint64_t)pairs ? 1 : 0);
  const uint64_t busy = order == 1 ? std::min<uint64_t>(num_mp, (uint64_t)pairs) : std::min<uint64_t>(tiles, (uint64_t)pairs);
  const int grid = 2 * (int)busy;
  g_last_kern = kMN ? "tc2_mn" : "tc2";
  // L2 eviction hints on the A / B loads (A evict_first, B evict_last; TN_L2_HINTS=1, A/B knob): measured
  // worse — C3 step 30's shape read 158.8 GB from DRAM with them vs 141.3 GB without (the clusters that
  // share an m pair re-read its A rows from L2), M = 2^21 K = 2^9 N = 2^10 8.5 vs 6.3 ms — so off
  static const int hints_env = getenv("TN_L2_HINTS") ? atoi(getenv("TN_L2_HINTS")) : 0;
  tc2::gemm_chalf_tc2_kernel<BN, kMN><<<grid, tc::kThreads, C::kSmem, s>>>(ma, mb, mc, num_mp, num_n, K2, in_max, b_bound,
                                                                      out_max, exp_slot, epi, m_base, order, ps, nda, mn_ma, rp, hints_env, a_inter);
  TN_CUDA(cudaGetLastError());
}

void launch_tc2(int BN, const CUtensorMap& ma, const CUtensorMap& mb, const CUtensorMap& mc, uint32_t num_mp,
                uint32_t num_n, int K2, const float* in_max, const float* b_bound, uint32_t* out_max, int* exp_slot,
                int epi, uint64_t m_base, const PeerStore& ps, const NdArgs& nda, cudaStream_t s, int a_inter) {
  if (BN == 256)
    launch_tc2_t<256, false>(ma, mb, mc, num_mp, num_n, K2, in_max, b_bound, out_max, exp_slot, epi, m_base, ps, nda,
                             0, tc2::RowPerm{}, s, a_inter);
  else if (BN == 128)
    launch_tc2_t<128, false>(ma, mb, mc, num_mp, num_n, K2, in_max, b_bound, out_max, exp_slot, epi, m_base, ps, nda,
                             0, tc2::RowPerm{}, s, a_inter);
  else if (BN == 64)
    launch_tc2_t<64, false>(ma, mb, mc, num_mp, num_n, K2, in_max, b_bound, out_max, exp_slot, epi, m_base, ps, nda,
                            0, tc2::RowPerm{}, s, a_inter);
  else
    throw TnError{TN_E_INVALID, "CTA-pair GEMM: BN must be 64, 128 or 256"};
}

// MN-major A (gemm_tc2.cuh, kMN): the stem stored as [M >> ma][K][2^ma] complex (the step's kept
// modes m_lo = 2^ma innermost, then its contracted modes, then the other kept modes) contracted
// without a permutation pass.  bpm = B' [2N][K] fp16 (tn_pad_b_mn).  K2 (the kernel's k count)
// is K: one stage = 64 complex k.
// Output of an MN-major step: 0 = row-major C[m][n], 1 = transposed C[n][m], each optionally with
// its m bits >= 6 permuted (rp: the kept modes above the 64-row tile in next-use order); -1 = other.
static int mn_out_kind(const OutMap* om, uint64_t M, uint32_t N, tc2::RowPerm* rp) {
  tc2::RowPerm r;
  memset(&r, 0, sizeof(r));
  int kind = 0;
  if (om && !om->identity) {
    if (om->transposed) {
      kind = 1;
    } else {
      // row-permuted identity (ns = 1 << j, ms = N << p_j) or transposed (ns = M << j, ms = 1 << p_j)
      bool ident = true, trans = true;
      for (int j = 0; j < om->nbits; ++j) {
        ident = ident && om->ns[j] == ((int64_t)1 << j);
        trans = trans && om->ns[j] == ((int64_t)M << j);
      }
      if (!ident && !trans) return -1;
      kind = ident ? 0 : 1;
      const int64_t unit = ident ? (int64_t)N : 1;
      uint64_t seen = 0;
      r.nb = om->mbits;
      if (r.nb > 64) return -1;
      for (int j = 0; j < om->mbits; ++j) {
        const int64_t st = om->ms[j];
        if (st <= 0 || st % unit) return -1;
        const int64_t q = st / unit;
        if (q & (q - 1)) return -1;
        int p = 0;
        while (((int64_t)1 << p) < q) ++p;
        if (p >= om->mbits || ((seen >> p) & 1) || (j < 6 && p != j)) return -1;
        seen |= 1ull << p;
        r.p[j] = (int8_t)p;
      }
      r.on = 1;
    }
  }
  if (rp) *rp = r;
  return kind;
}

bool mn_gemm_supported(uint64_t M, uint32_t K, uint32_t N, int ma, const OutMap* om, int kl, int mm) {
  if (!tc2_enabled() || ma < 7 || K < 64 || (K & (K - 1)) || N < 64 || (N & (N - 1)) || M % 128 || M >= (1ull << 31))
    return false;
  if (mn_out_kind(om, M, N, nullptr) < 0) return false;
  if ((kl > 0) != (mm > 0) || kl < 0 || mm < 0 || (1ull << kl) >= K) return false;
  return (1ull << (ma + mm)) <= M;
}

void launch_gemm_chalf_mn(__half* c, const __half* a, const __half* bpm, uint64_t M, uint32_t K, uint32_t N, int ma,
                          const float* in_max, const float* b_bound, uint32_t* out_max, int* exp_slot,
                          const OutMap* om, cudaStream_t s, int kl, int mm) {
  if (!mn_gemm_supported(M, K, N, ma, om, kl, mm)) throw TnError{TN_E_INVALID, "MN-major GEMM: unsupported geometry"};
  tc2::RowPerm rp;
  const bool transposed = mn_out_kind(om, M, N, &rp) == 1;
  const uint32_t N2 = 2 * N;
  const int BN = N2 >= 256 ? 256 : 128;
  CUtensorMap ma_map;
  NdArgs nda;
  memset(&nda, 0, sizeof(nda));
  if (kl > 0) {
    // split block: 5-d map (m_lo halves, k_lo, m_mid, k_hi, m_hi), box {64, min(64, 2^kl), 1,
    // 64 / that, 1}: the same 64 rows of 128 B (local k = k_lo + 2^kl k_hi) as the 3-d box
    const uint64_t klo = 1ull << kl, khi = K >> kl, mmid = 1ull << mm;
    cuuint64_t dims[5] = {2ull << ma, klo, mmid, khi, M >> (ma + mm)};
    cuuint64_t strides[4] = {4ull << ma, (4ull << ma) * klo, (4ull << ma) * klo * mmid, (4ull << ma) * klo * mmid * khi};
    const cuuint32_t bk = (cuuint32_t)std::min<uint64_t>(64, klo);
    cuuint32_t box[5] = {64, bk, 1, 64 / bk, 1};
    cuuint32_t estr[5] = {1, 1, 1, 1, 1};
    CUresult r = get_encode()(&ma_map, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 5, const_cast<__half*>(a), dims, strides, box,
                              estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                              CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) throw TnError{TN_E_CUDA, "cuTensorMapEncodeTiled (split MN-major A) failed"};
    nda.nd = 5;
    nda.kj0[0] = (int8_t)kl;
    nda.mj0[0] = (int8_t)mm;
  } else {
    cuuint64_t dims[3] = {2ull << ma, K, M >> ma};
    cuuint64_t strides[2] = {4ull << ma, (4ull << ma) * K};
    cuuint32_t box[3] = {64, 64, 1};
    cuuint32_t estr[3] = {1, 1, 1};
    CUresult r = get_encode()(&ma_map, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 3, const_cast<__half*>(a), dims, strides, box,
                              estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                              CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) throw TnError{TN_E_CUDA, "cuTensorMapEncodeTiled (MN-major A) failed"};
  }
  const CUtensorMap mb = make_map_2d(bpm, K, N2, 64, BN / 2);
  const CUtensorMap mc = transposed ? make_map_t(c, M, N, 64) : make_map_2d(c, N2, M, 64, 64);
  // (peer stores only for an unpermuted output: a fused swap's member bits are output-row bits)
  const PeerStore ps = make_peer_store(om ? om->peer : nullptr, !rp.on, transposed, M, N2, 64);
  const uint32_t num_mp = (uint32_t)(M / 128), num_n = N2 / BN;
  if (BN == 256)
    launch_tc2_t<256, true>(ma_map, mb, mc, num_mp, num_n, (int)K, in_max, b_bound, out_max, exp_slot,
                            transposed ? 4 : 0, 0, ps, nda, ma, rp, s);
  else
    launch_tc2_t<128, true>(ma_map, mb, mc, num_mp, num_n, (int)K, in_max, b_bound, out_max, exp_slot,
                            transposed ? 4 : 0, 0, ps, nda, ma, rp, s);
}

}  // namespace tn
