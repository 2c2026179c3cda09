// Launcher of the CTA-pair (cta_group::2) tcgen05 GEMM; the kernel and its design are in
// gemm_tc2.cuh, the choice between it and the single-CTA kernel in gemm_tc.cuh (launch_bn).
#include "gemm_tc2.cuh"

namespace tn {

bool tc2_enabled() {
  static const bool on = !getenv("TN_TC2") || atoi(getenv("TN_TC2")) != 0;
  return on;
}

template <int BN>
static void launch_tc2_t(const CUtensorMap& ma, const CUtensorMap& mb, const CUtensorMap& mc, uint32_t num_mp,
                         uint32_t num_n, int K2, const float* in_max, const float* b_bound, uint32_t* out_max,
                         int* exp_slot, int epi, uint64_t m_base, const PeerStore& ps, cudaStream_t s) {
  using C = tc2::Cfg2<BN>;
  // per device: the shared-memory opt-in and how many CTA pairs can be resident at once (an odd SM
  // count per GPC leaves SMs without a partner, so this can be below #SMs / 2)
  static std::mutex mu;
  static int max_pairs[64] = {0};
  int dev = 0;
  TN_CUDA(cudaGetDevice(&dev));
  int pairs;
  {
    std::lock_guard<std::mutex> lk(mu);
    if (dev >= 64 || max_pairs[dev] == 0) {
      TN_CUDA(cudaFuncSetAttribute(tc2::gemm_chalf_tc2_kernel<BN>, cudaFuncAttributeMaxDynamicSharedMemorySize, C::kSmem));
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(2 * 128, 1, 1);
      cfg.blockDim = dim3(tc::kThreads, 1, 1);
      cfg.dynamicSmemBytes = C::kSmem;
      int n = 0;
      TN_CUDA(cudaOccupancyMaxActiveClusters(&n, tc2::gemm_chalf_tc2_kernel<BN>, &cfg));
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
  tc2::gemm_chalf_tc2_kernel<BN><<<grid, tc::kThreads, C::kSmem, s>>>(ma, mb, mc, num_mp, num_n, K2, in_max, b_bound,
                                                                      out_max, exp_slot, epi, m_base, order, ps);
  TN_CUDA(cudaGetLastError());
}

void launch_tc2(int BN, const CUtensorMap& ma, const CUtensorMap& mb, const CUtensorMap& mc, uint32_t num_mp,
                uint32_t num_n, int K2, const float* in_max, const float* b_bound, uint32_t* out_max, int* exp_slot,
                int epi, uint64_t m_base, const PeerStore& ps, cudaStream_t s) {
  if (BN == 256)
    launch_tc2_t<256>(ma, mb, mc, num_mp, num_n, K2, in_max, b_bound, out_max, exp_slot, epi, m_base, ps, s);
  else if (BN == 128)
    launch_tc2_t<128>(ma, mb, mc, num_mp, num_n, K2, in_max, b_bound, out_max, exp_slot, epi, m_base, ps, s);
  else
    throw TnError{TN_E_INVALID, "CTA-pair GEMM: BN must be 128 or 256"};
}

}  // namespace tn
