// Complex-half stem GEMM on the 5th-generation tensor cores: operand-mode
// selection (plain TMA A, gathered A through N-d TMA boxes / raw box + reshuffle / cp.async) and
// dispatch.  The kernel itself is in gemm_tc.cuh; see its header comment for the design.
#include <cstdio>

#include "gemm_tc.cuh"

namespace tn {

extern template void launch_kb<0>(int, __half*, const __half*, const __half*, uint64_t, uint32_t, uint32_t,
                                  const float*, const float*, uint32_t*, int*, const OutMap*, cudaStream_t,
                                  const AGather*, const NdPlan*, const BatchSpec*);
extern template void launch_kb<1>(int, __half*, const __half*, const __half*, uint64_t, uint32_t, uint32_t,
                                  const float*, const float*, uint32_t*, int*, const OutMap*, cudaStream_t,
                                  const AGather*, const NdPlan*, const BatchSpec*);
extern template void launch_kb<2>(int, __half*, const __half*, const __half*, uint64_t, uint32_t, uint32_t,
                                  const float*, const float*, uint32_t*, int*, const OutMap*, cudaStream_t,
                                  const AGather*, const NdPlan*, const BatchSpec*);
extern template void launch_kb<3>(int, __half*, const __half*, const __half*, uint64_t, uint32_t, uint32_t,
                                  const float*, const float*, uint32_t*, int*, const OutMap*, cudaStream_t,
                                  const AGather*, const NdPlan*, const BatchSpec*);
extern template void launch_kb<4>(int, __half*, const __half*, const __half*, uint64_t, uint32_t, uint32_t,
                                  const float*, const float*, uint32_t*, int*, const OutMap*, cudaStream_t,
                                  const AGather*, const NdPlan*, const BatchSpec*);
extern template void launch_kb<5>(int, __half*, const __half*, const __half*, uint64_t, uint32_t, uint32_t,
                                  const float*, const float*, uint32_t*, int*, const OutMap*, cudaStream_t,
                                  const AGather*, const NdPlan*, const BatchSpec*);

static bool build_nd(const AGather& ag, NdPlan& out) {
  int pm[kMaxModes], pk[24];
  auto lg = [](int64_t v) {
    int r = 0;
    while ((1ll << r) < v) ++r;
    return ((1ll << r) == v) ? r : -1;
  };
  for (int j = 0; j < ag.mlog; ++j)
    if ((pm[j] = lg(ag.ms[j])) < 0) return false;
  for (int j = 0; j < ag.klog; ++j)
    if ((pk[j] = lg(ag.ks[j])) < 0) return false;
  if (ag.klog < 3 || pk[0] != 0 || pk[1] != 1 || ag.mlog < 7) return false;
  int w = 0;
  while (w < ag.klog && pk[w] == w) ++w;
  const bool inter = w < 3;
  const int W = inter ? 2 : std::min(w, 5);
  const int cb = inter ? std::min(3, ag.klog - 2) : 0;
  out.interleaved = inter ? 1 : 0;
  out.KB = inter ? (8 << cb) : (2 << W);
  auto src = [&](int kind, int j) { return kind == 0 ? pm[j] : pk[j]; };
  auto inbox = [&](int kind, int j) { return kind == 0 ? j < 7 : (inter ? j < 2 + cb : j < W); };
  auto succ = [&](int kind, int j, int& nk, int& nj) {
    if (inter && kind == 1 && j == 1) {  // k1 -> m0 (the 16-byte piece, then the rows)
      nk = 0;
      nj = 0;
      return true;
    }
    nk = kind;
    nj = j + 1;
    return nj < (kind == 0 ? ag.mlog : ag.klog);
  };
  std::vector<std::pair<int, int>> boxseq;
  if (inter) {
    boxseq = {{1, 0}, {1, 1}};
    for (int j = 0; j < 7; ++j) boxseq.push_back({0, j});
    for (int j = 2; j < 2 + cb; ++j) boxseq.push_back({1, j});
  } else {
    for (int j = 0; j < W; ++j) boxseq.push_back({1, j});
    for (int j = 0; j < 7; ++j) boxseq.push_back({0, j});
  }
  std::vector<char> used_m(ag.mlog, 0), used_k(ag.klog, 0);
  auto used = [&](int kind, int j) -> char& { return kind == 0 ? used_m[j] : used_k[j]; };
  std::vector<std::vector<std::pair<int, int>>> dims;
  auto grow = [&](int kind, int j) {
    std::vector<std::pair<int, int>> d{{kind, j}};
    used(kind, j) = 1;
    int nb = inbox(kind, j) ? 1 : 0;
    int ck = kind, cj = j, nk, nj;
    while (succ(ck, cj, nk, nj) && !used(nk, nj) && src(nk, nj) == src(ck, cj) + 1) {
      if (inbox(nk, nj)) {
        if (nb == 8 || !inbox(ck, cj)) break;
        ++nb;
      }
      d.push_back({nk, nj});
      used(nk, nj) = 1;
      ck = nk;
      cj = nj;
    }
    dims.push_back(d);
  };
  for (auto& b : boxseq)
    if (!used(b.first, b.second)) grow(b.first, b.second);
  for (int j = 0; j < ag.mlog; ++j)
    if (!used_m[j]) grow(0, j);
  for (int j = 0; j < ag.klog; ++j)
    if (!used_k[j]) grow(1, j);
  // Outside the box, two runs that are adjacent in the source (one m run, one k run, in either
  // order) share one tensor dim: its coordinate is the m part | the k part shifted past it (NdArgs
  // keeps one m and one k part per dim).  E.g. [k5 | m11 | k8 | m2 | k3 | m3] (6 runs) becomes
  // 4 dims {k5}{m11}{k8 m2}{k3 m3}.
  auto all_out = [&](const std::vector<std::pair<int, int>>& d) {
    for (auto& b : d)
      if (inbox(b.first, b.second)) return false;
    return true;
  };
  auto one_kind = [&](const std::vector<std::pair<int, int>>& d) {
    for (auto& b : d)
      if (b.first != d[0].first) return false;
    return true;
  };
  for (bool merged = true; merged && dims.size() > 5;) {
    merged = false;
    for (size_t a = 0; a < dims.size() && !merged; ++a)
      for (size_t b = 0; b < dims.size() && !merged; ++b) {
        if (a == b || !all_out(dims[a]) || !all_out(dims[b]) || !one_kind(dims[a]) || !one_kind(dims[b]) ||
            dims[a][0].first == dims[b][0].first)
          continue;
        const auto& lo = dims[a];
        const auto& hi = dims[b];
        if (src(hi[0].first, hi[0].second) != src(lo.back().first, lo.back().second) + 1) continue;
        std::vector<std::pair<int, int>> m = lo;
        m.insert(m.end(), hi.begin(), hi.end());
        dims[a] = m;
        dims.erase(dims.begin() + b);
        merged = true;
      }
  }
  if (dims.size() > 5) return false;
  // box dims must tile the box sequence in order (each a contiguous segment)
  size_t pos = 0;
  for (auto& d : dims) {
    for (auto& b : d) {
      if (!inbox(b.first, b.second)) break;
      if (pos >= boxseq.size() || boxseq[pos] != b) return false;
      ++pos;
    }
  }
  if (pos != boxseq.size()) return false;
  out.nd = (int)dims.size();
  memset(&out.args, 0, sizeof(out.args));
  out.args.nd = out.nd;
  for (int d = 0; d < out.nd; ++d) {
    const auto& v = dims[d];
    int nbox = 0;
    bool mixed = false;
    for (auto& b : v) {
      nbox += inbox(b.first, b.second) ? 1 : 0;
      mixed |= b.first != v[0].first;
    }
    if (v.size() > 32) return false;
    out.dim[d] = 1ull << v.size();
    out.stride[d] = 4ull << src(v[0].first, v[0].second);
    out.box[d] = 1u << nbox;
    if (mixed && nbox != 0 && nbox != (int)v.size()) return false;  // a mixed dim lies inside or outside the box
    if (nbox == 0) {
      // outside the box: one run of consecutive j per kind (two when merged above), each the
      // coordinate bits [offset, offset + length) of the dim
      int off = 0;
      for (size_t q = 0; q < v.size();) {
        size_t e = q + 1;
        while (e < v.size() && v[e].first == v[q].first && v[e].second == v[e - 1].second + 1) ++e;
        const int len = (int)(e - q);
        const uint32_t mask = len >= 32 ? 0xffffffffu : ((1u << len) - 1);
        if (v[q].first == 0) {
          if (out.args.mmask[d]) return false;
          out.args.mj0[d] = (int8_t)v[q].second;
          out.args.mmask[d] = mask;
          out.args.msh[d] = (int8_t)off;
        } else {
          if (out.args.kmask[d]) return false;
          out.args.kj0[d] = (int8_t)v[q].second;
          out.args.kmask[d] = mask;
          out.args.ksh[d] = (int8_t)off;
        }
        off += len;
        q = e;
      }
    } else if (nbox != (int)v.size()) {  // the dim's bits are consecutive j of one kind
      const uint32_t mask = v.size() >= 32 ? 0xffffffffu : ((1u << v.size()) - 1);
      if (v[0].first == 0) {
        out.args.mj0[d] = (int8_t)v[0].second;
        out.args.mmask[d] = mask;
      } else {
        out.args.kj0[d] = (int8_t)v[0].second;
        out.args.kmask[d] = mask;
      }
    }
  }
  if (out.stride[0] != 4) return false;
  for (int d = 1; d < out.nd; ++d)
    if (out.stride[d] % 16) return false;
  return true;
}

// Mode 3: the stage's box taken in SOURCE order (dims = runs of source bits: box bits first, then
// the outer bits up to the next box bit; <= 8 box bits per dim), landed raw and reshuffled into the
// interleaved layout by 16-byte pieces.  Inner rows are as long as the source allows (up to 1 KB).
static bool build_raw(const AGather& ag, NdPlan& out) {
  const int n = ag.mlog + ag.klog;
  if (ag.klog < 3 || ag.mlog < 7 || n > 64) return false;
  std::vector<int> kind(n, -1), jj(n, -1);
  auto lg = [](int64_t v) {
    int r = 0;
    while ((1ll << r) < v) ++r;
    return ((1ll << r) == v) ? r : -1;
  };
  for (int j = 0; j < ag.mlog; ++j) {
    const int p = lg(ag.ms[j]);
    if (p < 0 || p >= n || kind[p] >= 0) return false;
    kind[p] = 0;
    jj[p] = j;
  }
  for (int j = 0; j < ag.klog; ++j) {
    const int p = lg(ag.ks[j]);
    if (p < 0 || p >= n || kind[p] >= 0) return false;
    kind[p] = 1;
    jj[p] = j;
  }
  if (kind[0] != 1 || jj[0] != 0 || kind[1] != 1 || jj[1] != 1) return false;
  const int cb = std::min(3, ag.klog - 2);
  uint32_t pdst[16];
  auto inbox = [&](int p) { return kind[p] == 0 ? jj[p] < 7 : jj[p] < 2 + cb; };
  std::vector<std::vector<int>> dims;  // source positions
  for (int p = 0; p < n; ++p) {
    bool fresh = dims.empty();
    if (!fresh && inbox(p)) {
      const auto& d = dims.back();
      int nb = 0;
      for (int x : d) nb += inbox(x) ? 1 : 0;
      if (!inbox(d.back()) || nb == 8) fresh = true;
    }
    if (fresh)
      dims.push_back({p});
    else
      dims.back().push_back(p);
  }
  if (dims.size() > 5) return false;
  out.interleaved = 1;
  out.KB = 8 << cb;
  out.nd = (int)dims.size();
  memset(&out.args, 0, sizeof(out.args));
  out.args.nd = out.nd;
  int npb = 0;
  for (int d = 0; d < out.nd; ++d) {
    const auto& v = dims[d];
    if (v.size() > 32) return false;
    int nbox = 0;
    for (int x : v) nbox += inbox(x) ? 1 : 0;
    out.dim[d] = 1ull << v.size();
    out.stride[d] = 4ull << v[0];
    out.box[d] = 1u << nbox;
    // piece bits = box bits except k0, k1 (the 16-byte piece itself); each owns one stage byte bit
    for (int t = 0; t < nbox; ++t) {
      const int x = v[t];
      if (kind[x] == 1 && jj[x] < 2) continue;
      if (npb >= 12) return false;
      pdst[npb++] = kind[x] == 0 ? (16u << jj[x]) : (2048u << (jj[x] - 2));
    }
    // coordinate: the outer bits form at most one run of rows and one run of k (consecutive j)
    bool has_m = false, has_k = false;
    for (int t = nbox; t < (int)v.size(); ++t) {
      const int x = v[t];
      const bool isk = kind[x] == 1;
      bool& has = isk ? has_k : has_m;
      int8_t& j0 = isk ? out.args.kj0[d] : out.args.mj0[d];
      int8_t& sh = isk ? out.args.ksh[d] : out.args.msh[d];
      uint32_t& mask = isk ? out.args.kmask[d] : out.args.mmask[d];
      if (!has) {
        has = true;
        j0 = (int8_t)jj[x];
        sh = (int8_t)t;
        mask = 1;
      } else {
        const int nbits = __builtin_popcount(mask);
        if (j0 + nbits != jj[x] || sh + nbits != t) return false;  // a second run of this kind
        mask = (mask << 1) | 1u;
      }
    }
  }
  out.args.npb = npb;
  if (npb != 7 + cb || npb < 5 || npb > 13) return false;
  // Enumeration basis over GF(2)^npb (piece-bit masks).  Lanes 0-2 each flip one raw slot bit
  // (raw bytes 16/32/64) and one stage slot bit (stage bytes 16/32/64 = rows m0..m2), so in every
  // 8-lane phase both the reads and the writes hit 8 distinct 16-byte bank slots.
  auto dst_of = [&](uint32_t mask) {
    uint32_t d = 0;
    for (int i = 0; i < npb; ++i)
      if ((mask >> i) & 1) d ^= pdst[i];
    return d;
  };
  int dm[3] = {-1, -1, -1};
  for (int i = 0; i < npb; ++i)
    for (int t = 0; t < 3; ++t)
      if (pdst[i] == (16u << t)) dm[t] = i;
  std::vector<uint32_t> basis;  // reduced copies for the rank test
  auto add_if_indep = [&](uint32_t m) {
    uint32_t r = m;
    for (uint32_t b : basis)
      if ((r ^ b) < r) r ^= b;
    if (!r) return false;
    basis.push_back(r);
    std::sort(basis.begin(), basis.end(), [](uint32_t x, uint32_t y) { return x > y; });
    return true;
  };
  uint32_t lane[5], its[8];
  int nl = 0;
  bool diag = dm[0] >= 0 && dm[1] >= 0 && dm[2] >= 0;
  if (diag) {
    // raw-slot and stage-slot projections of the three lane patterns must both be invertible
    uint32_t rawp[3], dstp[3];
    for (int t = 0; t < 3; ++t) {
      lane[t] = (1u << t) | (1u << dm[t]);
      rawp[t] = lane[t] & 7u;
      dstp[t] = (dst_of(lane[t]) >> 4) & 7u;
    }
    auto inv3 = [](const uint32_t* v) {
      uint32_t a = v[0], b = v[1], c = v[2];
      return a && b && c && a != b && a != c && b != c && (a ^ b) != c;
    };
    diag = inv3(rawp) && inv3(dstp);
  }
  if (diag) {
    for (int t = 0; t < 3; ++t)
      if (!add_if_indep(lane[t])) return false;
    nl = 3;
  }
  for (int i = 0; nl < 5 && i < npb; ++i)
    if (add_if_indep(1u << i)) lane[nl++] = 1u << i;
  int ni = 0;
  for (int i = 0; i < npb; ++i)
    if (add_if_indep(1u << i)) its[ni++] = 1u << i;
  if (nl != 5 || nl + ni != npb) return false;
  for (int b = 0; b < 5; ++b) {
    out.args.lane_pat[b] = (uint16_t)lane[b];
    out.args.lane_dst[b] = dst_of(lane[b]);
  }
  for (int b = 0; b < ni; ++b) {
    out.args.it_pat[b] = (uint16_t)its[b];
    out.args.it_dst[b] = dst_of(its[b]);
  }
  for (int d = 1; d < out.nd; ++d)
    if (out.stride[d] % 16) return false;
  return true;
}


// The A-operand path a gathered step will take (the same choice as launch_gemm_chalf_tc, without the
// A/B knobs): 0 direct N-d box (rows >= 128 B), 2 core-matrix box, 3 raw box + reshuffle, 1 cp.async
// 16-byte pieces, 4 cp.async 4-byte pieces.  For the lowering's cost model (plan.cpp).
int gather_mode_of(const AGather& ag) {
  if (ag.ks[0] != 1 || ag.ks[1] != 2) return 4;
  NdPlan np, rp;
  const bool direct = build_nd(ag, np), raw = build_raw(ag, rp);
  const bool wide = direct && (int)(np.box[0] * 4) >= 128;
  if (direct && (wide || !raw)) return np.interleaved ? 2 : 0;
  return raw ? 3 : 1;
}

int gather_mode_of_strides(int mlog, int klog, const int64_t* ms, const int64_t* ks) {
  AGather ag;
  memset(&ag, 0, sizeof(ag));
  ag.mlog = mlog;
  ag.klog = klog;
  for (int j = 0; j < mlog && j < kMaxModes; ++j) ag.ms[j] = ms[j];
  for (int j = 0; j < klog && j < 24; ++j) ag.ks[j] = ks[j];
  return gather_mode_of(ag);
}

void launch_gemm_chalf_tc(__half* c, const __half* a, const __half* bp, uint64_t M, uint32_t K2, uint32_t N2,
                          const float* in_max, const float* b_bound, uint32_t* out_max, int* exp_slot,
                          const OutMap* om, cudaStream_t s, const AGather* ag) {
  if (K2 < 8 || N2 < 2 || (K2 & (K2 - 1)) || (N2 & (N2 - 1)))
    throw TnError{TN_E_INVALID, "tcgen05 GEMM needs power-of-two 2K >= 8, 2N >= 2"};
  if (M == 0) return;
  const int kb_plain = K2 >= 64 ? 64 : (K2 >= 32 ? 32 : 16);
  if (ag) {
    // the gathered load needs whole 128-row tiles and K-boxes of at least 16 fp16
    if (M % tc::BM || K2 < 16 || (uint64_t)1 << ag->mlog != M || (2u << ag->klog) != K2)
      throw TnError{TN_E_INVALID, "gathered-A GEMM: unsupported operand geometry"};
    static const int force_word = getenv("TN_GATHER_WORD") ? atoi(getenv("TN_GATHER_WORD")) : 0;  // test knob
    if (ag->ks[0] != 1 || ag->ks[1] != 2 || force_word) {
      // contracted modes not innermost (the middle of the stored order): 4-byte cp.async pieces
      launch_kb<4>(kb_plain, c, a, bp, M, K2, N2, in_max, b_bound, out_max, exp_slot, om, s, ag, nullptr, nullptr);
      return;
    }
    // A/B knobs: TN_GATHER_MODE = 1 (cp.async), 2 (direct N-d box), 3 (raw box + reshuffle)
    static const int force = getenv("TN_GATHER_MODE") ? atoi(getenv("TN_GATHER_MODE")) : 0;
    NdPlan np, rp;
    const bool direct = force != 1 && force != 3 && build_nd(*ag, np);
    const bool raw = force != 1 && force != 2 && build_raw(*ag, rp);
    // A direct box unless its TMA rows are shorter than 128 B: there the raw box (rows as long as the
    // source runs allow) plus the smem reshuffle wins (round-1 C3 step 50, m28 k5 n5, 32-byte rows:
    // 22.5 -> 13.5 ms; m21 k9 n6: 1.63 -> 1.18 ms; 64-byte rows: see raw_below); at 128 B the direct
    // box is faster.
    // Raw box when no direct one exists (<= 5 dims); else cp.async.
    // 128: 64-byte rows also take the raw box.  In isolation at full clock the two tie at 64 B, but
    // inside the power-capped subtask (SM clock ~1.2-1.4 GHz) the direct box's per-row TMA cost
    // dominates: C3 step 4 (m24 k8 n7, 64-byte rows) 8.0-10.8 ms raw vs 12.9-13.0 ms direct.
    static const int raw_below = getenv("TN_RAW_BELOW") ? atoi(getenv("TN_RAW_BELOW")) : 128;  // tuning knob
    const bool direct_wide = direct && (int)(np.box[0] * 4) >= raw_below;
    static const bool dbg = getenv("TN_GATHER_DEBUG") != nullptr;
    if (dbg) {
      fprintf(stderr, "gather mlog %d klog %d: direct %d (inter %d KB %d nd %d box0 %u) raw %d (KB %d nd %d box0 %u)\n",
              ag->mlog, ag->klog, (int)direct, np.interleaved, np.KB, np.nd, direct ? np.box[0] : 0, (int)raw, rp.KB,
              rp.nd, raw ? rp.box[0] : 0);
    }
    if (direct && (direct_wide || !raw)) {
      // one N-d TMA box per stage (coordinates per dim from the global row)
      if (np.interleaved)
        launch_kb<2>(np.KB, c, a, bp, M, K2, N2, in_max, b_bound, out_max, exp_slot, om, s, ag, &np, nullptr);
      else
        launch_kb<0>(np.KB, c, a, bp, M, K2, N2, in_max, b_bound, out_max, exp_slot, om, s, ag, &np, nullptr);
      return;
    }
    if (raw) {
      launch_kb<3>(rp.KB, c, a, bp, M, K2, N2, in_max, b_bound, out_max, exp_slot, om, s, ag, &rp, nullptr);
      return;
    }
    launch_kb<1>(kb_plain, c, a, bp, M, K2, N2, in_max, b_bound, out_max, exp_slot, om, s, ag, nullptr, nullptr);
    return;
  }
  // plain TMA A: the deep-pipeline variant (one output staging buffer per epilogue group, more stages)
  // for K-heavy steps; TN_STAGE_DEEP = 0 / 1 forces either (A/B knob)
  static const int deep_env = getenv("TN_STAGE_DEEP") ? atoi(getenv("TN_STAGE_DEEP")) : -1;
  // (tools/mubench.py A/B, M = 2^23: deep = shallow within noise for K >= 2^8, 1.1-1.3x slower for
  // K <= 2^7 — the pipeline depth is not what holds the MMA back, so it stays off by default)
  const bool deep = deep_env > 0;
  if (deep && kb_plain == 64)
    launch_kb<5>(kb_plain, c, a, bp, M, K2, N2, in_max, b_bound, out_max, exp_slot, om, s, nullptr, nullptr, nullptr);
  else
    launch_kb<0>(kb_plain, c, a, bp, M, K2, N2, in_max, b_bound, out_max, exp_slot, om, s, nullptr, nullptr, nullptr);
}

void launch_gemm_chalf_tc_batched(__half* c, const __half* a, const __half* bp, uint64_t M, uint32_t K2, uint32_t N2,
                                  const float* in_max, const float* b_bound, uint32_t* out_max, int* exp_slot,
                                  const BatchSpec& bs, cudaStream_t s) {
  if (K2 < 8 || (K2 & (K2 - 1)) || N2 < 16 || (N2 & (N2 - 1)))
    throw TnError{TN_E_INVALID, "batched GEMM: K >= 4 and N >= 8 powers of two"};
  if (bs.pad_r > 0 ? (!bs.table || bs.n_out != bs.n_a) : (!bs.ia || !bs.ib))
    throw TnError{TN_E_INVALID, "batched GEMM: index arrays missing"};
  const int kb = K2 >= 64 ? 64 : (K2 >= 32 ? 32 : 16);
  launch_kb<0>(kb, c, a, bp, M, K2, N2, in_max, b_bound, out_max, exp_slot, nullptr, s, nullptr, nullptr, &bs);
}

}  // namespace tn
