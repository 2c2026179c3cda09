// Plan parsing, validation and lowering (host only).  SURVEY §8(a) a.1, §8(b).
//
// Lowering decides, per stem step i (Alg. 1 "performer computation of currEin"):
//   R_i = contracted labels (stem ∩ branch, Eq. 3 delta = alpha ∩ beta),
//   kept = stem \ R_i, new = branch \ R_i (Eq. 4),
//   whether a standalone permutation is needed (R_i not already the innermost block),
//   the GEMM geometry M = 2^|kept|, K = 2^|R_i|, N = 2^|new|, and the output layout kept ++ new.
// Layout policy (B200 design): labels are ordered by next use, furthest first
// (outermost), so the labels the next steps contract tend to be innermost and no pass is needed.
#include "plan.hpp"

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <limits>
#include <map>
#include <set>
#include <sstream>
#include <unordered_map>

#include "json.hpp"

namespace tn {

static TnError err(int code, const std::string& m) { return TnError{code, m}; }

static int as_int(const tnjson::Value& v, const char* what) {
  if (!v.is_num()) throw err(TN_E_PARSE, std::string(what) + ": expected a number");
  double d = v.num;
  if (d != std::floor(d) || d < 0 || d > 2e9) throw err(TN_E_INVALID, std::string(what) + ": bad integer");
  return (int)d;
}

static std::vector<int> int_list(const tnjson::Value* v, const char* what) {
  std::vector<int> out;
  if (!v) return out;
  if (!v->is_arr()) throw err(TN_E_PARSE, std::string(what) + ": expected a list");
  for (auto& x : v->arr) out.push_back(as_int(x, what));
  return out;
}

static Plan* load_plan_fixed(const char* json, size_t len, const tn_config* cfg_in, int world, int split_min = -1);

// Steps the MN-major fold may not take in this lowering (load_plan_mn's search), and steps whose
// layout-policy-3 output choice (row-major vs transposed) is inverted (its hill climb)
static thread_local const std::set<int>* g_mn_forbid = nullptr;
static thread_local const std::set<int>* g_tr_flip = nullptr;

// Lowering cost for the searches: bytes of permutation passes plus the extra cost of the gathered A
// loads, as A bytes times a per-path factor measured against a plain read (raw box + reshuffle
// ~0.3, cp.async 16-byte pieces ~1, 4-byte pieces ~3: tools/gather_bench.py)
static double plan_cost(const Plan& p) {
  double c = p.perm_bytes;
  for (const StemStep& st : p.steps) {
    if (!st.gather_a || st.a_m_stride.empty()) continue;
    const int mode = gather_mode_of_strides(st.mlog, st.klog, st.a_m_stride.data(), st.a_k_stride.data());
    const double f = mode == 3 ? 0.3 : mode == 1 ? 1.0 : mode == 4 ? 3.0 : 0.0;
    c += f * 4.0 * std::ldexp(1.0, st.mlog + st.klog);
  }
  return c;
}

// The MN-major fold keeps a step's kept modes in stored order, which changes every later layout: a
// fold can cost more passes downstream than it saves.  The lowering is repeated with folds
// forbidden (each folded step of an explored lowering, depth first, <= 24 lowerings of ~10 ms) and
// the one with the fewest permutation-pass bytes is kept (first found on ties).  On C3 the ranking
// of four variants by pass bytes (73.6 / 86.4 / 90.7 / 103 GB) matched their measured subtask times
// (257.5 / 263.7 / 267.8 / 275.3 ms, 3 interleaved reps).  TN_MN_SEARCH=0: the greedy lowering.
static Plan* load_plan_mn(const char* json, size_t len, const tn_config* cfg, int world, int split_min) {
  std::set<int> forbid;
  g_mn_forbid = &forbid;
  struct Reset {
    ~Reset() { g_mn_forbid = nullptr; }
  } reset;
  std::unique_ptr<Plan> best(load_plan_fixed(json, len, cfg, world, split_min));
  static const bool off = getenv("TN_MN_SEARCH") && atoi(getenv("TN_MN_SEARCH")) == 0;
  auto taken = [](const Plan& p) {
    std::set<int> t;
    for (size_t i = 0; i < p.steps.size(); ++i)
      if (p.steps[i].mn) t.insert((int)i);
    return t;
  };
  if (off) return best.release();
  std::vector<std::pair<std::set<int>, std::set<int>>> stack{{forbid, taken(*best)}};
  std::set<std::set<int>> seen{forbid};
  int evals = 1;
  while (!stack.empty() && evals < 24) {
    const auto top = stack.back();
    stack.pop_back();
    for (int t : top.second) {
      std::set<int> f2 = top.first;
      f2.insert(t);
      if (!seen.insert(f2).second || evals >= 24) continue;
      forbid = f2;
      std::unique_ptr<Plan> q(load_plan_fixed(json, len, cfg, world, split_min));
      ++evals;
      stack.push_back({f2, taken(*q)});
      if (plan_cost(*q) < plan_cost(*best)) best = std::move(q);
    }
  }
  // then (TN_TR_SEARCH=1, opt-in) a hill climb over the transposed-output choices with the chosen folds
  // fixed: invert one choice at a time, keep it when the cost drops.  It lowers the modelled cost
  // (C3: 4 GPUs 24.7 vs 28.1 GB of passes) but measured no faster (1 GPU 248.8 vs 244.6 ms, 4 GPUs
  // 80.6 vs 80.6 ms, 3 interleaved reps each) for ~0.5 s more per plan load, hence off
  static const bool tr_off = !getenv("TN_TR_SEARCH") || atoi(getenv("TN_TR_SEARCH")) == 0;
  if (tr_off) return best.release();
  std::set<int> mn_taken = taken(*best), f_best;
  forbid.clear();
  for (size_t i = 0; i < best->steps.size(); ++i)
    if (!mn_taken.count((int)i)) forbid.insert((int)i);  // the same folds as the best plan
  std::set<int> flips;
  g_tr_flip = &flips;
  struct ResetTr {
    ~ResetTr() { g_tr_flip = nullptr; }
  } reset_tr;
  double c_best = plan_cost(*best);
  for (int pass = 0; pass < 2; ++pass) {
    bool improved = false;
    std::vector<int> pts;
    for (size_t i = 0; i < best->steps.size(); ++i)
      if (best->steps[i].tr_choice) pts.push_back((int)i);
    for (int s : pts) {
      std::set<int> f2 = flips;
      if (!f2.insert(s).second) f2.erase(s);
      flips = f2;
      std::unique_ptr<Plan> q(load_plan_fixed(json, len, cfg, world, split_min));
      const double c = plan_cost(*q);
      if (c < c_best && taken(*q) == mn_taken) {
        best = std::move(q);
        c_best = c;
        improved = true;
      } else {
        if (!f2.count(s)) flips.insert(s); else flips.erase(s);  // undo
      }
    }
    if (!improved) break;
  }
  return best.release();
}

// A split tail on a sharded stem must start after the last mode swap (each rank chunks its own
// shard; a swap would need every chunk of every rank).  The swap schedule does not depend on where
// the tail starts, so a lowering whose tail would contain a swap is redone with the tail starting
// right after it.
static Plan* load_plan_split(const char* json, size_t len, const tn_config* cfg, int world) {
  int split_min = -1;
  for (int pass = 0; pass < 64; ++pass) {
    try {
      return load_plan_mn(json, len, cfg, world, split_min);
    } catch (const TnError& e) {
      const std::string key = "split-retry:";
      if (e.msg.compare(0, key.size(), key) != 0) throw;
      const int s = std::stoi(e.msg.substr(key.size()));
      if (s <= split_min) throw err(TN_E_INFEASIBLE, "split: cannot place the tail after the mode swaps");
      split_min = s;
    }
  }
  throw err(TN_E_INFEASIBLE, "split: cannot place the tail after the mode swaps");
}

// cfg.split_log2 = -1 (auto): "the number of chunks is determined by the current remaining
// capacity of the GPU memory" (reading C-A19: the smallest power of two that fits).  The lowering is
// tried with j = 0, 1, 2, ... split legs; the first whose buffers fit stem_capacity_bytes wins.
// Without a capacity (0) there is nothing to fit: no split.
Plan* load_plan(const char* json, size_t len, const tn_config* cfg_in, int world) {
  if (!cfg_in || cfg_in->split_log2 >= 0) return load_plan_split(json, len, cfg_in, world);
  tn_config c = *cfg_in;
  if (c.stem_capacity_bytes == 0) {
    c.split_log2 = 0;
    return load_plan_split(json, len, &c, world);
  }
  std::string last = "no split count fits";
  for (int j = 0; j <= 16; ++j) {
    c.split_log2 = j;
    try {
      return load_plan_split(json, len, &c, world);
    } catch (const TnError& e) {
      if (e.code != TN_E_INFEASIBLE) throw;
      last = e.msg;
      if (e.msg.find("fewer open legs") != std::string::npos) break;
    }
  }
  throw err(TN_E_CAPACITY, "split auto: no power-of-two chunk count fits stem_capacity_bytes (" + last + ")");
}

static Plan* load_plan_fixed(const char* json, size_t len, const tn_config* cfg_in, int world, int split_min) {
  tnjson::Value root;
  try {
    root = tnjson::parse(json, len);
  } catch (const tnjson::ParseError& e) {
    throw err(TN_E_PARSE, e.what());
  }
  if (!root.is_obj()) throw err(TN_E_PARSE, "plan: expected an object");
  std::unique_ptr<Plan> P(new Plan());
  Plan& p = *P;
  tn_config cfg{};
  cfg.dtype = TN_CHALF;
  cfg.stem_min_log2 = 20;
  cfg.comm_codec = TN_COMM_INT8;
  cfg.comm_group = 128;
  cfg.split_log2 = 0;
  if (cfg_in) cfg = *cfg_in;
  if (cfg.stem_min_log2 < 0) cfg.stem_min_log2 = 20;
  if (cfg.dtype != TN_CHALF && cfg.dtype != TN_CFLOAT) throw err(TN_E_INVALID, "cfg.dtype");
  if (cfg.comm_group <= 0) cfg.comm_group = 128;
  if (cfg.comm_codec < TN_COMM_FP16 || cfg.comm_codec > TN_COMM_INT8_TENSOR) throw err(TN_E_INVALID, "cfg.comm_codec");
  if (cfg.comm_codec != TN_COMM_FP16 && cfg.comm_codec != TN_COMM_INT8_TENSOR &&
      (cfg.comm_group < 16 || (cfg.comm_group & (cfg.comm_group - 1))))
    throw err(TN_E_INVALID, "cfg.comm_group must be a power of two >= 16 for the group codecs");
  p.cfg = cfg;
  if (world != 1 && world != 2 && world != 4 && world != 8) throw err(TN_E_UNSUPPORTED, "world must be 1, 2, 4 or 8");
  p.world = world;
  while ((1 << p.shard_log2) < world) p.shard_log2++;

  // ---- tensors
  const tnjson::Value* ts = root.get("tensors");
  if (!ts || !ts->is_arr() || ts->arr.empty()) throw err(TN_E_PARSE, "plan: 'tensors' missing");
  for (auto& t : ts->arr) {
    Leaf lf;
    lf.labels = int_list(t.get("labels"), "tensors.labels");
    const tnjson::Value* d = t.get("data");
    if (!d || !d->is_arr()) throw err(TN_E_PARSE, "tensors.data missing");
    if (lf.labels.size() > 40) throw err(TN_E_UNSUPPORTED, "leaf rank > 40");
    size_t want = (size_t)2 << lf.labels.size();
    if (d->arr.size() != want)
      throw err(TN_E_INVALID, "tensors.data length != 2*2^rank (all dims must be 2)");
    lf.data.reserve(want);
    for (auto& x : d->arr) {
      if (!x.is_num()) throw err(TN_E_PARSE, "tensors.data: number expected");
      lf.data.push_back(x.num);
    }
    std::set<int> u(lf.labels.begin(), lf.labels.end());
    if (u.size() != lf.labels.size()) throw err(TN_E_INVALID, "duplicate label within a tensor");
    p.leaves.push_back(std::move(lf));
  }
  p.open = int_list(root.get("open"), "open");
  p.sliced = int_list(root.get("sliced"), "sliced");
  if (p.sliced.size() > 4096) throw err(TN_E_UNSUPPORTED, "more than 4096 sliced labels");
  const tnjson::Value* tr = root.get("tree");
  std::vector<std::pair<int, int>> pairs;
  if (tr) {
    if (!tr->is_arr()) throw err(TN_E_PARSE, "tree: expected a list");
    for (auto& pr : tr->arr) {
      if (!pr.is_arr() || pr.arr.size() != 2) throw err(TN_E_PARSE, "tree: pairs expected");
      pairs.emplace_back(as_int(pr.arr[0], "tree"), as_int(pr.arr[1], "tree"));
    }
  }
  std::vector<int> stem_in = int_list(root.get("stem"), "stem");
  p.sparse_legs = int_list(root.get("sparse_legs"), "sparse_legs");

  // ---- label validation: no hyper-edges; open legs appear once; closed labels twice
  std::map<int, int> count;
  for (auto& lf : p.leaves)
    for (int l : lf.labels) count[l]++;
  std::set<int> open_set(p.open.begin(), p.open.end());
  if (open_set.size() != p.open.size()) throw err(TN_E_INVALID, "duplicate open label");
  for (auto& kv : count) {
    bool is_open = open_set.count(kv.first) > 0;
    if (kv.second > 2) throw err(TN_E_INVALID, "label " + std::to_string(kv.first) + " is a hyper-edge");
    if (is_open && kv.second != 1) throw err(TN_E_INVALID, "open label must appear once");
    if (!is_open && kv.second != 2) throw err(TN_E_INVALID, "closed label " + std::to_string(kv.first) + " must appear twice");
  }
  for (int l : p.open)
    if (!count.count(l)) throw err(TN_E_INVALID, "open label not in any tensor");
  std::set<int> sl_set;
  for (int l : p.sliced) {
    if (!count.count(l) || open_set.count(l)) throw err(TN_E_INVALID, "sliced label must be a closed edge");
    if (!sl_set.insert(l).second) throw err(TN_E_INVALID, "duplicate sliced label");
  }
  // sparse-state legs: open legs whose values are given per correlated subspace
  std::set<int> sparse_set;
  for (int l : p.sparse_legs)
    if (!open_set.count(l) || !sparse_set.insert(l).second)
      throw err(TN_E_INVALID, "sparse_legs must be distinct open legs");
  if (p.sparse_legs.size() > 63) throw err(TN_E_UNSUPPORTED, "more than 63 sparse legs");

  // ---- nodes
  const int nl = (int)p.leaves.size();
  if ((int)pairs.size() != nl - 1) throw err(TN_E_INVALID, "tree must have n_tensors-1 pairs");
  p.nodes.resize(nl + pairs.size());
  for (int i = 0; i < nl; ++i) {
    Node& n = p.nodes[i];
    n.kind = NODE_LEAF;
    for (int l : p.leaves[i].labels)
      if (!sl_set.count(l)) n.labels.push_back(l);
  }
  std::vector<char> used(p.nodes.size(), 0);
  for (size_t k = 0; k < pairs.size(); ++k) {
    int id = nl + (int)k;
    int u = pairs[k].first, v = pairs[k].second;
    if (u >= id || v >= id || u == v) throw err(TN_E_INVALID, "tree: not in SSA order");
    if (used[u] || used[v]) throw err(TN_E_INVALID, "tree: node used twice");
    used[u] = used[v] = 1;
    Node& n = p.nodes[id];
    n.u = u;
    n.v = v;
    n.kind = NODE_COMMON;
    const auto& lu = p.nodes[u].labels;
    const auto& lv = p.nodes[v].labels;
    std::set<int> su(lu.begin(), lu.end()), sv(lv.begin(), lv.end());
    for (int l : lu)
      if (!sv.count(l)) n.labels.push_back(l);
    for (int l : lv)
      if (!su.count(l)) n.labels.push_back(l);
    std::set<int> un(su);
    un.insert(sv.begin(), sv.end());
    if (un.size() > 62) throw err(TN_E_INFEASIBLE, "contraction with more than 62 modes");
    n.cost = std::ldexp(1.0, (int)un.size());
    n.sub_cost = p.nodes[u].sub_cost + p.nodes[v].sub_cost + n.cost;
  }
  p.root = (int)p.nodes.size() - 1;
  {
    std::set<int> rl(p.nodes[p.root].labels.begin(), p.nodes[p.root].labels.end());
    if (rl != open_set) throw err(TN_E_INVALID, "root labels != open legs");
  }

  // ---- stem (C-A18)
  if (!stem_in.empty()) {
    for (int id : stem_in)
      if (id < 0 || id >= (int)p.nodes.size()) throw err(TN_E_INVALID, "stem: bad node id");
    if (stem_in.back() != p.root) throw err(TN_E_INVALID, "stem must end at the root");
    for (size_t i = 1; i < stem_in.size(); ++i) {
      const Node& n = p.nodes[stem_in[i]];
      if (n.u != stem_in[i - 1] && n.v != stem_in[i - 1]) throw err(TN_E_INVALID, "stem: not a path");
    }
    p.stem = stem_in;
  } else {
    int k = p.root;
    std::vector<int> path{k};
    while (p.nodes[k].u >= 0) {
      const Node& n = p.nodes[k];
      k = (p.nodes[n.u].sub_cost >= p.nodes[n.v].sub_cost) ? n.u : n.v;
      path.push_back(k);
    }
    std::reverse(path.begin(), path.end());
    p.stem = path;
  }

  // ---- stem entry: first stem node with >= 2^stem_min_log2 elements
  p.stem_entry = -1;
  int entry_idx = -1;
  for (size_t i = 0; i < p.stem.size(); ++i) {
    // the entry is an internal node: its complex64 result lives in the workspace and is converted
    // into stem buffer 0 (a leaf would need a strided gather of a sliced view first)
    if (p.nodes[p.stem[i]].u >= 0 && (int)p.nodes[p.stem[i]].labels.size() >= cfg.stem_min_log2) {
      entry_idx = (int)i;
      break;
    }
  }
  if (entry_idx >= 0 && entry_idx == (int)p.stem.size() - 1 && p.nodes[p.stem[entry_idx]].u >= 0) {
    // the entry is the root itself: still a valid (zero-step) stem; keep it common instead
    entry_idx = -1;
  }
  // A huge entry would itself be a common-type (complex64 SIMT) contraction: enter one node earlier
  // instead, so that contraction becomes the first stem GEMM (C3: a 2^28 entry built from a 2^16 stem
  // node and a 2^20 branch costs ~12 ms as a common contraction, 0.4 ms as a tcgen05 step).
  while (entry_idx > 0 && (int)p.nodes[p.stem[entry_idx]].labels.size() > cfg.stem_min_log2 + 2) {
    const Node& prev = p.nodes[p.stem[entry_idx - 1]];
    if (prev.u < 0 || (int)prev.labels.size() < std::max(cfg.stem_min_log2 - 8, 1)) break;
    --entry_idx;
  }
  if (entry_idx >= 0) {
    p.stem_entry = p.stem[entry_idx];
    for (size_t i = entry_idx + 1; i < p.stem.size(); ++i) p.nodes[p.stem[i]].kind = NODE_STEM;
  }
  for (int id = nl; id < (int)p.nodes.size(); ++id)
    if (p.nodes[id].kind == NODE_COMMON) p.common_order.push_back(id);

  // ---- next use of each label along the stem
  const int INF = std::numeric_limits<int>::max();
  std::unordered_map<int, int> next_use;
  std::vector<int> step_nodes;
  if (entry_idx >= 0)
    for (size_t i = entry_idx + 1; i < p.stem.size(); ++i) step_nodes.push_back(p.stem[i]);
  {
    // a label is contracted at the step whose branch shares it with the stem
    std::vector<int> prev_layout = p.nodes[p.stem_entry >= 0 ? p.stem_entry : p.root].labels;
    int prev = p.stem_entry;
    for (size_t s = 0; s < step_nodes.size(); ++s) {
      const Node& n = p.nodes[step_nodes[s]];
      int br = (n.u == prev) ? n.v : n.u;
      for (int l : p.nodes[br].labels) next_use[l] = (int)s;  // branch-side first appearance
      prev = step_nodes[s];
    }
  }
  for (int l : p.open) next_use.erase(l);  // open legs are never contracted
  // ---- sparse-state tail ("sparse state occurs in the final stage"): from the first stem step
  // whose branch holds a sparse leg, every stem tensor is a batch over the distinct values its sparse
  // legs take among the requested subspaces (a slice per batch entry: fixing the legs like slicing
  // fixes an edge), contracted with gather-batched GEMMs (Fig. 5).  The dense lowering below
  // therefore ignores sparse legs; the branches keep them as batch modes of their B_P blocks.
  if (!sparse_set.empty()) {
    if (entry_idx < 0) throw err(TN_E_UNSUPPORTED, "sparse legs need stem steps");
    for (int l : p.nodes[p.stem_entry].labels)
      if (sparse_set.count(l)) throw err(TN_E_UNSUPPORTED, "sparse legs must enter the stem through branches (the stem entry holds one)");
    if (cfg.split_log2 != 0) throw err(TN_E_UNSUPPORTED, "split tail together with sparse legs (the sparse batch is chunked instead)");
    if (world > 1) throw err(TN_E_UNSUPPORTED, "sparse-state batch on a sharded stem (run replicas)");
    int prev = p.stem_entry;
    for (size_t s = 0; s < step_nodes.size() && p.sparse_from < 0; ++s) {
      const Node& n = p.nodes[step_nodes[s]];
      int br = (n.u == prev) ? n.v : n.u;
      for (int l : p.nodes[br].labels)
        if (sparse_set.count(l)) p.sparse_from = (int)s;
      prev = step_nodes[s];
    }
    if (p.sparse_from < 0) throw err(TN_E_INVALID, "no stem step holds a sparse leg");
    // common-type nodes that hold a sparse leg may only feed the tail as branches: the stem before
    // the tail must be free of them (checked per step below)
  }
  // ---- split-type tail: 2^j chunks fix j open legs.  The chosen legs are
  // the open legs that enter the stem earliest (longest tail); they sort outermost in every layout.
  std::set<int> split_set;
  if (cfg.recompute && cfg.split_log2 != 0) throw err(TN_E_INVALID, "recompute needs split_log2 = 0");
  if (cfg.recompute && !sparse_set.empty()) throw err(TN_E_UNSUPPORTED, "recompute together with sparse legs");
  if ((cfg.split_log2 > 0 || cfg.recompute) && entry_idx >= 0) {
    std::map<int, int> first_app;  // open leg -> first stem step whose INPUT holds it
    for (int l : p.nodes[p.stem_entry].labels) first_app[l] = 0;
    {
      int prev = p.stem_entry;
      for (size_t s = 0; s < step_nodes.size(); ++s) {
        const Node& n = p.nodes[step_nodes[s]];
        int br = (n.u == prev) ? n.v : n.u;
        for (int l : p.nodes[br].labels)
          if (!first_app.count(l)) first_app[l] = (int)s + 1;
        prev = step_nodes[s];
      }
    }
    std::vector<int> cand(p.open.begin(), p.open.end());
    std::stable_sort(cand.begin(), cand.end(), [&](int a, int b) { return first_app[a] < first_app[b]; });
    int nsplit = cfg.split_log2;
    int from_min = split_min;
    if (cfg.recompute) {
      // recomputation on halves: halve right before the step producing the largest stem
      // tensor, along an open leg (a free mode that survives to the end, so the halves concatenate)
      // already held by the stem there
      nsplit = 1;
      std::vector<int> sz(step_nodes.size());
      for (size_t s = 0; s < step_nodes.size(); ++s) sz[s] = (int)p.nodes[step_nodes[s]].labels.size();
      const int peak = (int)(std::max_element(sz.begin(), sz.end()) - sz.begin());
      cand.erase(std::remove_if(cand.begin(), cand.end(), [&](int l) { return first_app[l] > peak; }), cand.end());
      if (cand.empty()) throw err(TN_E_INFEASIBLE, "recompute: no open leg in the stem before its largest tensor");
      std::stable_sort(cand.begin(), cand.end(), [&](int a, int b) { return first_app[a] > first_app[b]; });
      from_min = std::max(from_min, peak);
      p.recompute_from = peak;
    }
    if ((int)cand.size() < nsplit) throw err(TN_E_INFEASIBLE, "split: fewer open legs than split modes");
    for (int t = 0; t < nsplit; ++t) {
      split_set.insert(cand[t]);
      p.split_modes.push_back(cand[t]);
      p.split_from = std::max(p.split_from, first_app[cand[t]]);
    }
    p.split_from = std::max(p.split_from, from_min);
    p.split_log2 = nsplit;
    if (p.split_from >= (int)step_nodes.size()) throw err(TN_E_INFEASIBLE, "split: no tail step holds the split modes");
  }
  auto nu = [&](int l) {
    if (split_set.count(l)) return INF;  // split modes outermost, then the other open legs
    auto it = next_use.find(l);
    return it == next_use.end() ? INF - 1 : it->second;
  };

  // ---- steps
  // Layout policy (tn.h tn_config.layout_policy).  Public 0 (default): every GEMM writes
  // kept ++ new (identity output, TMA-store epilogue); a step whose contracted modes are not the
  // innermost block gets its permutation fused into the GEMM's A load (gathered A) or, when that is
  // impossible, a standalone permutation pass ("reorder then GEMM").  Public 2: every GEMM
  // writes the NEXT step's contracted modes innermost (scatter epilogue), so no permutation is ever
  // needed.  Public 1: scatter only when a thread's stores are >= 64 B contiguous, else as 0.
  // Internal numbering (below): 1 = public 0, 0 = public 1, 2 = public 2.
  const int policy = cfg.layout_policy == 0 ? 1 : (cfg.layout_policy == 1 ? 0 : cfg.layout_policy);
  const int eb = (cfg.dtype == TN_CHALF) ? 4 : 8;
  uint64_t smax = 0, payload_bytes = 0;
  if (entry_idx >= 0) {
    // branch label sets and contracted sets R_s (stem ∩ branch) along the stem
    std::vector<std::set<int>> Rsets(step_nodes.size());
    {
      std::set<int> cur(p.nodes[p.stem_entry].labels.begin(), p.nodes[p.stem_entry].labels.end());
      int prev = p.stem_entry;
      for (size_t s = 0; s < step_nodes.size(); ++s) {
        const Node& n = p.nodes[step_nodes[s]];
        int br = (n.u == prev) ? n.v : n.u;
        for (int l : p.nodes[br].labels)
          if (!sparse_set.count(l)) (cur.count(l) ? Rsets[s] : cur).insert(l);
        for (int l : Rsets[s]) cur.erase(l);
        prev = step_nodes[s];
      }
    }
    auto by_next_use = [&](std::vector<int>& v) {
      std::stable_sort(v.begin(), v.end(), [&](int a, int b) { return nu(a) > nu(b); });
    };
    // order a set of labels as [others by next use desc] ++ [those in `inner`]
    auto order_with_inner = [&](const std::vector<int>& all, const std::set<int>& inner) {
      std::vector<int> outer, in;
      for (int l : all) (inner.count(l) ? in : outer).push_back(l);
      by_next_use(outer);
      outer.insert(outer.end(), in.begin(), in.end());
      return outer;
    };
    if ((policy == 0 || policy == 2 || policy == 3) && !step_nodes.empty()) {
      // the entry is a common node whose device layout we choose: R_1 innermost
      Node& e = p.nodes[p.stem_entry];
      e.labels = order_with_inner(e.labels, Rsets[0]);
    }
    // ---- sharding: the stem's log2(world) outermost modes index the GPU.  Shard
    // modes are the entry labels used furthest in the future (never-contracted open legs first).
    std::vector<int> shard;
    if (p.shard_log2 > 0) {
      Node& e = p.nodes[p.stem_entry];
      // split modes must stay local (each rank chunks its own shard of the tail): never shard them
      std::vector<int> cand;
      for (int l : e.labels)
        if (!split_set.count(l)) cand.push_back(l);
      std::stable_sort(cand.begin(), cand.end(), [&](int a, int b) { return nu(a) > nu(b); });
      if ((int)cand.size() <= p.shard_log2) throw err(TN_E_INFEASIBLE, "stem entry has too few modes to shard");
      shard.assign(cand.begin(), cand.begin() + p.shard_log2);
      std::vector<int> lay = shard;
      for (int l : e.labels)
        if (std::find(shard.begin(), shard.end(), l) == shard.end()) lay.push_back(l);
      e.labels = lay;
      p.shard0 = shard;
    }
    std::vector<int> L = p.nodes[p.stem_entry].labels;
    L.erase(L.begin(), L.begin() + shard.size());  // local layout (shard modes are rank bits)
    smax = 1ull << L.size();
    int prev = p.stem_entry;
    for (size_t s = 0; s < step_nodes.size(); ++s) {
      StemStep st;
      st.node = step_nodes[s];
      const Node& n = p.nodes[st.node];
      st.branch = (n.u == prev) ? n.v : n.u;
      st.sparse = (p.sparse_from >= 0 && (int)s >= p.sparse_from) ? 1 : 0;
      std::vector<int> B;  // dense branch labels (sparse legs are the B_P block index)
      for (int l : p.nodes[st.branch].labels) (sparse_set.count(l) ? st.b_sparse : B).push_back(l);
      if (!st.sparse && !st.b_sparse.empty()) throw err(TN_E_INVALID, "sparse leg in a stem branch before the sparse tail");
      std::set<int> bs(B.begin(), B.end());
      if (!shard.empty()) {
        // Alg. 1: a contracted shard mode forces an all-to-all mode swap first.
        st.shard_before = shard;
        std::vector<int> out_pos;
        for (size_t j = 0; j < shard.size(); ++j)
          if (bs.count(shard[j])) out_pos.push_back((int)j);
        if (!out_pos.empty()) {
          // swap in the local modes used furthest in the future (reading C-A17: furthest next use;
          // only the contracted shard modes are swapped)
          std::vector<int> cand;
          for (int l : L)
            if (!bs.count(l) && !split_set.count(l)) cand.push_back(l);
          std::stable_sort(cand.begin(), cand.end(), [&](int a, int b) { return nu(a) > nu(b); });
          if (cand.size() < out_pos.size()) throw err(TN_E_INFEASIBLE, "partition modes run out (swap)");
          // prefer modes the previous GEMM's epilogue can route (runtime.cu fused_swap_target: whole
          // store boxes per member, m bits >= 7 / n bits >= 5 of its output) among the modes whose next
          // use ties with the last of the sx C-A17 picks (TN_SWAP_PICK=0: plain C-A17 order).  (Among
          // the 2 sx furthest, ignoring ties, C3 at 2 ranks got 4 swaps / 15.0 GB per rank instead of
          // 3 / 10.7 GB.)
          static const bool pick_env = !getenv("TN_SWAP_PICK") || atoi(getenv("TN_SWAP_PICK")) != 0;
          if (pick_env && !p.steps.empty() && p.steps.back().tensor_core && cfg.dtype == TN_CHALF) {
            const StemStep& pv = p.steps.back();
            auto routable = [&](int l) {
              const auto it = std::find(L.begin(), L.end(), l);
              if (it == L.end()) return false;
              const int pos = (int)(L.end() - it) - 1;  // bit position from the innermost
              const bool ident = pv.out_identity, tr = pv.out_transposed;
              if (ident) return pos >= pv.nlog + 7 || (pos >= 5 && pos < pv.nlog);
              if (tr) return (pos >= 7 && pos < pv.mlog) || pos >= pv.mlog + 5;
              return false;
            };
            const int last = nu(cand[out_pos.size() - 1]);
            size_t top = 0;
            while (top < cand.size() && nu(cand[top]) >= last) ++top;
            std::stable_partition(cand.begin(), cand.begin() + top, routable);
          }
          st.swap = true;
          // quantise only in the later stages of the path (earlier errors accumulate), C-A26
          {
            const int pct = cfg.quant_from_pct < 0 ? 65 : cfg.quant_from_pct;
            st.quant = cfg.dtype == TN_CHALF &&
                       (cfg.comm_codec == TN_COMM_INT8 || cfg.comm_codec == TN_COMM_INT4 ||
                        cfg.comm_codec == TN_COMM_INT8_TENSOR) &&
                       100.0 * (double)s >= pct * (double)step_nodes.size();
          }
          st.swap_out_pos = out_pos;
          st.swap_in.assign(cand.begin(), cand.begin() + out_pos.size());
          // sender layout: swap_in outermost (chunk v of the outer bits goes to member v)
          std::vector<int> snd = st.swap_in;
          for (int l : L)
            if (std::find(st.swap_in.begin(), st.swap_in.end(), l) == st.swap_in.end()) snd.push_back(l);
          st.send_layout = snd;
          if (snd != L) {
            st.send_perm = true;
            for (int l : snd) st.send_perm_axes.push_back((int)(std::find(L.begin(), L.end(), l) - L.begin()));
            // the codec can read the unpermuted stem when each group (g/2 complex) stays contiguous
            int gb = 0;
            while (cfg.comm_group > 1 && (2 << gb) < cfg.comm_group) ++gb;
            const int nl = (int)snd.size();
            bool inner = st.quant && cfg.comm_codec != TN_COMM_INT8_TENSOR && !cfg.no_fuse_swap_quant && gb <= nl &&
                         (cfg.comm_group & (cfg.comm_group - 1)) == 0;
            for (int q = 0; inner && q < gb; ++q) inner = st.send_perm_axes[nl - 1 - q] == nl - 1 - q;
            st.fuse_quant = inner;
          }
          // after the exchange: the swapped-out shard modes become the outermost local modes
          std::vector<int> lay;
          for (int j : out_pos) lay.push_back(shard[j]);
          lay.insert(lay.end(), snd.begin() + out_pos.size(), snd.end());
          for (size_t t = 0; t < out_pos.size(); ++t) shard[out_pos[t]] = st.swap_in[t];
          L = lay;
          p.n_swaps++;
          if (st.quant) {
            // codes + fp32 scales + zeros of the whole local stem are staged in one stem buffer
            // (runtime.cu mode_swap): size the buffers for it (matters for small groups / stems)
            const uint64_t reals = 2ull << L.size();
            const uint64_t ng = cfg.comm_codec == TN_COMM_INT8_TENSOR ? (1ull << out_pos.size())
                                                                      : reals / (uint64_t)cfg.comm_group;
            const uint64_t cb = align_up(cfg.comm_codec == TN_COMM_INT4 ? reals / 2 : reals, 256);
            payload_bytes = std::max<uint64_t>(payload_bytes, cb + 3 * align_up(8 * ng, 256));
          }
          const double n_local = std::ldexp(1.0, (int)L.size());
          const double frac = 1.0 - std::ldexp(1.0, -(int)out_pos.size());
          const double per = !st.quant ? (cfg.dtype == TN_CHALF ? 4.0 : 8.0)
                             : cfg.comm_codec == TN_COMM_INT8_TENSOR ? 2.0
                                                                     : ((cfg.comm_codec == TN_COMM_INT4 ? 1.0 : 2.0) +
                                                                        16.0 / cfg.comm_group);
          p.swap_bytes += frac * n_local * per;
        }
        st.shard_after = shard;
      }
      st.in_layout = L;
      std::vector<int> R, kept;
      for (int l : L) (bs.count(l) ? R : kept).push_back(l);
      // is R the innermost block of L?
      bool suffix = true;
      for (size_t j = 0; j < R.size(); ++j)
        if (!bs.count(L[L.size() - R.size() + j])) suffix = false;
      if ((int)s == p.split_from && !split_set.empty()) {
        // entering the split tail: the split modes must be the outermost block (one permutation
        // pass if they are not; kept modes sort by next use with the split modes first)
        std::set<int> pre(L.begin(), L.begin() + std::min(L.size(), split_set.size()));
        if (pre != split_set) suffix = false;
      }
      if (!suffix) {
        // a permutation the GEMM's A load will absorb (gathered-A tcgen05 step, see the fused-
        // permutation pass below) keeps the kept modes in stored order: the m bits then form long
        // source runs, so the gather is a few-dimensional TMA box with 1 KB rows
        const int kl = (int)R.size(), nl = (int)(B.size() - R.size());
        const bool rows_k = kl <= 4 && nl <= 5 && kl + nl <= 7;
        const bool tc_k = cfg.dtype == TN_CHALF && kl >= 2 && !rows_k &&
                          ((kl >= 3 && nl >= 3) || kl >= 4 || kl + nl > 11);
        // 16-byte pieces: the two innermost stored modes are contracted.  4-byte pieces (any layout,
        // e.g. the contracted modes in the middle of the stored order): the warp's lanes still read
        // 32 contiguous complex when the 5 innermost stored modes are tile bits (the 7 innermost kept
        // modes = m bits 0..6, or the min(5, K bits) innermost contracted modes of a stage)
        // 4-byte gather is opt-in: measured 2-4x slower than pass + TMA GEMM on the C3 steps (per-thread
        // cp.async.4 requests cap it near 1.2 TB/s aggregate), kept for layouts nothing else can read
        static const bool no_word = getenv("TN_WORD_GATHER") == nullptr;
        bool word_ok = !no_word && L.size() >= 5 && kept.size() >= 7;
        if (word_ok) {
          std::set<int> tile;
          for (size_t q = kept.size() - 7; q < kept.size(); ++q) tile.insert(kept[q]);
          for (int q = kl - std::min(5, kl); q < kl; ++q) tile.insert(R[q]);
          for (size_t q = L.size() - 5; word_ok && q < L.size(); ++q) word_ok = tile.count(L[q]) > 0;
        }
        const bool fusable = !cfg.no_gather && !st.sparse && tc_k && kl >= 3 && kept.size() >= 7 && L.size() >= 2 &&
                             ((bs.count(L[L.size() - 1]) && bs.count(L[L.size() - 2])) || word_ok) &&
                             (split_set.empty() || (int)s < p.split_from);
        // MN-major operand: stored order [kept | R | >= 7 kept], K >= 64, N >= 64 (2N >= 128: the
        // CTA-pair kernel's B tile), complex-half, not in a split tail or sparse tail
        {
          int ma = 0;
          while (ma < (int)L.size() && !bs.count(L[L.size() - 1 - ma])) ++ma;
          // only where a pass would be expensive (>= 2^28 elements): the fold keeps the kept modes in
          // stored order, which forgoes the pass's next-use ordering of them for the later steps
          static const int mn_min = getenv("TN_MN_MIN_LOG2") ? atoi(getenv("TN_MN_MIN_LOG2")) : 28;  // tuning knob
          const bool geo = ma >= 7 && kl >= 6 && nl >= 6 && (int)kept.size() >= 8 && (int)L.size() >= mn_min;
          bool block = geo;
          for (int q = 0; block && q < kl; ++q) block = bs.count(L[L.size() - 1 - ma - q]) > 0;
          // split block: [.. | R_hi | m_mid | R_lo | m_lo], one kept run inside the contracted modes
          // (5-d A map).  Opt-in (TN_MN_SPLIT=1): exact, and it cuts C3's modelled pass bytes from
          // 73.6 to 47.8 GB on one GPU, but the MN-major kernel is slower than pass + plain GEMM on
          // several of the steps it then takes (C3 steps 20 / 21 / 24: 10.0 / 10.9 / 11.0 vs 7.6 /
          // 7.3 / 6.0 ms), so the subtask measured 260.9-263.7 vs 249.1-261.6 ms (3 interleaved reps);
          // the search's cost counts pass bytes only
          int split_kl = 0, split_mm = 0;
          static const bool split_on = getenv("TN_MN_SPLIT") && atoi(getenv("TN_MN_SPLIT")) != 0;
          if (geo && !block && split_on) {
            int pos = (int)L.size() - 1 - ma, q1 = 0, mm = 0, q2 = 0;
            while (pos >= 0 && bs.count(L[pos])) ++q1, --pos;
            while (pos >= 0 && !bs.count(L[pos])) ++mm, --pos;
            while (pos >= 0 && bs.count(L[pos])) ++q2, --pos;
            if (q1 >= 1 && mm >= 1 && q1 + q2 == kl) {
              block = true;
              split_kl = q1;
              split_mm = mm;
            }
          }
          static const bool mn_off = getenv("TN_NO_MN") != nullptr;  // A/B knob
          // TN_MN_STEPS="i,j,..." (experiment knob): only these step indices may take the fold
          static const char* mn_steps = getenv("TN_MN_STEPS");
          if (mn_steps) {
            const std::string lst = std::string(",") + mn_steps + ",";
            block = block && lst.find("," + std::to_string(s) + ",") != std::string::npos;
          }
          if (g_mn_forbid && g_mn_forbid->count((int)s)) block = false;
          if (block && !mn_off && !fusable && cfg.dtype == TN_CHALF && !st.sparse && tc_k && !cfg.no_gather &&
              (split_set.empty() || (int)s < p.split_from)) {
            st.mn = true;
            st.mn_ma = ma;
            st.mn_kl = split_kl;
            st.mn_mm = split_mm;
          }
        }
        if (!fusable && !st.mn) by_next_use(kept);
        std::vector<int> PL = kept;
        PL.insert(PL.end(), R.begin(), R.end());
        st.perm = true;
        for (int l : PL) st.perm_axes.push_back((int)(std::find(L.begin(), L.end(), l) - L.begin()));
      } else {
        R.assign(L.end() - R.size(), L.end());
        kept.assign(L.begin(), L.end() - R.size());
      }
      std::vector<int> newl;
      for (int l : B)
        if (std::find(R.begin(), R.end(), l) == R.end()) newl.push_back(l);
      std::vector<int> out;
      if ((policy == 0 || policy == 2) && !st.sparse) {
        if (s + 1 == step_nodes.size()) {
          // the last step writes the result directly in output order (local modes only)
          for (int l : L)  // split tail: the split modes stay the outermost block
            if (split_set.count(l)) out.push_back(l);
          for (int l : p.open)
            if (std::find(shard.begin(), shard.end(), l) == shard.end() && !split_set.count(l)) out.push_back(l);
        } else {
          // [rest by next use] ++ [kept ∩ R_next] ++ [new ∩ R_next]  (new innermost)
          const std::set<int>& Rn = Rsets[s + 1];
          std::vector<int> rest, kl, nlo, nhi;
          for (int l : kept) (Rn.count(l) ? kl : rest).push_back(l);
          for (int l : newl) (Rn.count(l) ? nlo : nhi).push_back(l);
          // the scatter epilogue stores contiguous runs along the innermost new modes: worth it
          // only when a thread's 16 consecutive outputs are contiguous (>= 4 new modes innermost)
          // or no permutation would be needed anyway
          if (policy == 2 || nlo.size() >= 4 || kl.empty() || nhi.empty()) {
            rest.insert(rest.end(), nhi.begin(), nhi.end());
            by_next_use(rest);
            out = rest;
            out.insert(out.end(), kl.begin(), kl.end());
            out.insert(out.end(), nlo.begin(), nlo.end());
          } else {
            // identity output (TMA store): kept ++ [new by next use, new ∩ R_next innermost]
            by_next_use(nhi);
            out = kept;
            out.insert(out.end(), nhi.begin(), nhi.end());
            out.insert(out.end(), nlo.begin(), nlo.end());
          }
        }
        // B's N order follows the output order of the new labels (outer -> inner)
        std::vector<int> nord;
        for (int l : out)
          if (std::find(newl.begin(), newl.end(), l) != newl.end()) nord.push_back(l);
        newl = nord;
      } else {
        by_next_use(newl);
        // kept modes in the output: M order.  TN_MN_ROWPERM=1 (opt-in): after an MN-major step (M order
        // = stored order) every kept mode above the 64-row tile goes by next use, as a pass would have
        // ordered them, and the epilogue places each tile at its permuted row (RowPerm).  Measured on
        // C3 (3 interleaved reps): 277 ms with it vs 270 ms without (the 6 tile modes stay in stored
        // order either way, so the later layouts still differ from the pass path's), hence off.
        std::vector<int> kout = kept;
        static const bool rowperm_on = getenv("TN_MN_ROWPERM") && atoi(getenv("TN_MN_ROWPERM")) == 1;
        if (st.mn && rowperm_on) {
          std::vector<int> hi(kept.begin(), kept.end() - 6);
          by_next_use(hi);
          kout = hi;
          kout.insert(kout.end(), kept.end() - 6, kept.end());
        }
        out = kout;
        out.insert(out.end(), newl.begin(), newl.end());
        // (not for a SIMT row-streaming step, K <= 16, N <= 32, K*N <= 128: its transposed stores are
        // 4-byte scatters; C3 step 14 at 4 ranks took 6.9 ms instead of ~1.7 ms)
        static const bool rows_tr = getenv("TN_ROWS_TRANSPOSE") != nullptr;  // A/B knob
        const bool rows_step = !rows_tr && R.size() <= 4 && newl.size() <= 5 && R.size() + newl.size() <= 7;
        if (policy == 3 && !st.sparse && s + 1 < step_nodes.size() && !rows_step &&
            (split_set.empty() || (int)s + 1 < p.split_from)) {
          // transposed store C[n][m] (new modes outermost, kept modes innermost in M order) when that
          // puts more of the next step's contracted modes innermost: the next step then reads its
          // operand as stored or through a 16-byte fused gather instead of a permutation pass.  The
          // tcgen05 scatter epilogue writes it with each warp's 32 rows contiguous (128-byte stores).
          const std::set<int>& Rn = Rsets[s + 1];
          auto inner_hits = [&](const std::vector<int>& o) {
            int h = 0;
            for (auto it = o.rbegin(); it != o.rend() && Rn.count(*it); ++it) ++h;
            return h;
          };
          std::vector<int> tr = newl;
          tr.insert(tr.end(), kout.begin(), kout.end());
          const int hid = inner_hits(out), htr = inner_hits(tr);
          bool want = htr > hid && (htr == (int)Rn.size() || htr >= 2) && kept.size() >= 5;
          if (kept.size() >= 5) {
            st.tr_choice = true;
            if (g_tr_flip && g_tr_flip->count((int)s)) want = !want;
          }
          if (want) out = tr;
        }
      }
      st.R = R;
      st.kept = kept;
      st.newl = newl;
      st.mlog = (int)kept.size();
      st.klog = (int)R.size();
      st.nlog = (int)newl.size();
      st.out_layout = out;
      // tcgen05 when the tile carries enough work; small K*N steps go to the SIMT row-streaming
      // kernel (K <= 16, N <= 32, K*N <= 128: streams at HBM speed, k_gemm_simt.cu rows_ok; ncu
      // showed 128x16 tcgen05 tiles at 16 % of DRAM peak, profiles/r01_ncu_summary.md)
      const bool rows_kernel = st.klog <= 4 && st.nlog <= 5 && st.klog + st.nlog <= 7;
      st.tensor_core = (cfg.dtype == TN_CHALF) && st.klog >= 2 && !rows_kernel &&
                       ((st.klog >= 3 && st.nlog >= 3) || st.klog >= 4 || st.klog + st.nlog > 11);
      {
        std::set<int> chk(st.out_layout.begin(), st.out_layout.end());
        chk.insert(shard.begin(), shard.end());
        std::set<int> want;
        for (int l : n.labels)
          if (!sparse_set.count(l)) want.insert(l);
        if (chk != want || chk.size() != st.out_layout.size() + shard.size())
          throw err(TN_E_INVALID, "internal: step output labels mismatch");
      }
      // output address map: bit j of m (kept[mlog-1-j]) and of n (newl[nlog-1-j])
      {
        const int r = (int)out.size();
        auto stride_of = [&](int l) {
          int q = (int)(std::find(out.begin(), out.end(), l) - out.begin());
          return (int64_t)1 << (r - 1 - q);
        };
        st.m_stride.resize(st.mlog);
        st.n_stride.resize(st.nlog);
        for (int j = 0; j < st.mlog; ++j) st.m_stride[j] = stride_of(kept[st.mlog - 1 - j]);
        for (int j = 0; j < st.nlog; ++j) st.n_stride[j] = stride_of(newl[st.nlog - 1 - j]);
        std::vector<int> ident = kept;
        ident.insert(ident.end(), newl.begin(), newl.end());
        st.out_identity = (ident == out);
        std::vector<int> trans = newl;
        trans.insert(trans.end(), kept.begin(), kept.end());
        st.out_transposed = !st.out_identity && trans == out;
      }
      if (st.klog > 16 || st.nlog > 16) throw err(TN_E_UNSUPPORTED, "stem operand with K or N > 2^16");
      smax = std::max<uint64_t>(smax, 1ull << (st.mlog + st.klog));
      smax = std::max<uint64_t>(smax, 1ull << (st.mlog + st.nlog));
      double M = std::ldexp(1.0, st.mlog), K = std::ldexp(1.0, st.klog), N = std::ldexp(1.0, st.nlog);
      p.stem_flops += 8.0 * M * K * N;
      p.stem_bytes_alg += eb * (M * K + M * N) + 8.0 * K * N;
      if (st.perm && !st.mn) {
        p.perm_bytes += 2.0 * eb * M * K;
        p.n_permutes++;
      }
      L = st.out_layout;
      prev = st.node;
      p.steps.push_back(std::move(st));
    }
    p.final_layout = L;
    p.final_shard = shard;
    if (!p.split_modes.empty()) {
      // every tail step must keep the split modes as the outermost block of its input, of its
      // permuted input and of its output, so chunk v is the contiguous slab v everywhere
      const int j = (int)p.split_modes.size();
      auto prefix_ok = [&](const std::vector<int>& lay) {
        if ((int)lay.size() < j) return false;
        std::set<int> pre(lay.begin(), lay.begin() + j);
        return pre == split_set;
      };
      uint64_t cmax = 0;
      for (size_t s = p.split_from; s < p.steps.size(); ++s) {
        StemStep& st = p.steps[s];
        std::vector<int> permuted;
        for (int a : st.perm_axes) permuted.push_back(st.in_layout[a]);
        // the first tail step's permutation runs on the whole stem before chunking
        const bool in_ok = ((int)s == p.split_from && st.perm) ? true : prefix_ok(st.in_layout);
        if (st.swap) {
          int last = (int)s;  // restart with the tail after the tail's last swap
          for (size_t q = s; q < p.steps.size(); ++q)
            if (p.steps[q].swap) last = (int)q + 1;
          throw err(TN_E_INFEASIBLE, "split-retry:" + std::to_string(last));
        }
        if (!in_ok || !prefix_ok(st.out_layout) || (st.perm && !prefix_ok(permuted)) || st.mlog < j)
          throw err(TN_E_INFEASIBLE, "split: the split modes do not stay outermost in the tail (step " +
                                         std::to_string(s) + ", from " + std::to_string(p.split_from) + ", in " +
                                         std::to_string(prefix_ok(st.in_layout)) + " out " +
                                         std::to_string(prefix_ok(st.out_layout)) + ")");
        st.split = 1;
        cmax = std::max<uint64_t>(cmax, 1ull << (st.in_layout.size() - j));
        cmax = std::max<uint64_t>(cmax, 1ull << (st.out_layout.size() - j));
      }
      p.split_chunk_max = cmax;
      // chunk v = value v of the split legs in the order of the first tail step's (permuted) input
      {
        const StemStep& f = p.steps[p.split_from];
        std::vector<int> lay0;
        if (f.perm)
          for (int a : f.perm_axes) lay0.push_back(f.in_layout[a]);
        else
          lay0 = f.in_layout;
        p.split_modes.assign(lay0.begin(), lay0.begin() + j);
      }
      p.final_perm = false;  // the host reorders the chunked result (each chunk has its own scale)
      // the free buffer holds two chunk regions plus the assembled result
      // the full-size tensors of the tail are never materialised: one buffer holds the tail's input
      // (the stem entering the split point) + one chunk region, the other one chunk region + the
      // result slots (runtime.cu split_contract)
      const uint64_t in_full = 1ull << p.steps[p.split_from].in_layout.size();
      uint64_t need = std::max<uint64_t>(cmax + (1ull << L.size()), align_up(in_full * eb, 1024) / eb + cmax);
      for (int s = 0; s <= p.split_from && s < (int)p.steps.size(); ++s) {
        const StemStep& st = p.steps[s];
        need = std::max<uint64_t>(need, 1ull << st.in_layout.size());
        if (s < p.split_from) need = std::max<uint64_t>(need, 1ull << st.out_layout.size());
      }
      smax = need;
    }
    // ---- fused permutations (gathered-A tcgen05 GEMM): a permutation before a tensor-core step is
    // folded into the GEMM's A load when the two innermost input modes are contracted (16-byte
    // pieces stay contiguous), the step is not chunked (split tail) and M >= 128.  K order = R in
    // input order, M order = kept as the permutation would have placed them, so B_P and the output
    // layout are unchanged.
    if (!cfg.no_gather && cfg.dtype == TN_CHALF) {
      for (auto& st : p.steps) {
        if (!st.perm || !st.tensor_core || st.split || st.sparse || st.mlog < 7 || st.klog < 3) continue;
        const std::vector<int>& IL = st.in_layout;
        const int r = (int)IL.size();
        std::set<int> Rs(st.R.begin(), st.R.end());
        if (r < 5) continue;
        auto src_stride = [&](int l) {
          return (int64_t)1 << (r - 1 - (int)(std::find(IL.begin(), IL.end(), l) - IL.begin()));
        };
        st.a_m_stride.resize(st.mlog);
        st.a_k_stride.resize(st.klog);
        for (int j = 0; j < st.mlog; ++j) st.a_m_stride[j] = src_stride(st.kept[st.mlog - 1 - j]);
        for (int j = 0; j < st.klog; ++j) st.a_k_stride[j] = src_stride(st.R[st.klog - 1 - j]);
        if (st.a_k_stride[0] != 1 || st.a_k_stride[1] != 2) {
          // 4-byte pieces (k_gemm_tc.cu mode 4): fuse only when the lanes read 128 contiguous bytes
          // 4-byte gather is opt-in: measured 2-4x slower than pass + TMA GEMM on the C3 steps (per-thread
        // cp.async.4 requests cap it near 1.2 TB/s aggregate), kept for layouts nothing else can read
        static const bool no_word = getenv("TN_WORD_GATHER") == nullptr;
          if (no_word) continue;
          std::vector<int64_t> bits(st.a_m_stride.begin(), st.a_m_stride.begin() + 7);
          for (int j = 0; j < std::min(5, st.klog); ++j) bits.push_back(st.a_k_stride[j]);
          std::sort(bits.begin(), bits.end());
          bool contig = true;
          for (int j = 0; j < 5; ++j) contig = contig && bits[j] == ((int64_t)1 << j);
          if (!contig) continue;
        }
        st.gather_a = true;
        st.perm = false;
        st.perm_axes.clear();
        p.perm_bytes -= 2.0 * eb * std::ldexp(1.0, st.mlog + st.klog);
        p.n_permutes--;
      }
    }
    if (shard.empty() && p.split_modes.empty() && p.sparse_from < 0 && L != p.open) {
      p.final_perm = true;
      for (int l : p.open) p.final_perm_axes.push_back((int)(std::find(L.begin(), L.end(), l) - L.begin()));
      p.perm_bytes += 2.0 * eb * std::ldexp(1.0, (int)L.size());
    }
  }
  smax = std::max<uint64_t>(smax, (payload_bytes + eb - 1) / eb);
  if (p.sparse_from >= 0) {
    // sparse tail: the stem entering it stays in one buffer (every chunk of subspaces re-reads it),
    // the tail ping-pongs between two regions of the other: size the buffers so that at least one
    // subspace at a time fits (runtime.cu sparse_need; larger batches are chunked)
    uint64_t tmax = 0;
    for (size_t s = p.sparse_from; s < p.steps.size(); ++s)
      tmax = std::max<uint64_t>(tmax, std::max<uint64_t>(1ull << p.steps[s].in_layout.size(),
                                                         1ull << p.steps[s].out_layout.size()));
    const uint64_t need = 2 * align_up(tmax * eb, 1024) + 8 * (p.steps.size() - p.sparse_from) + 4096;
    smax = std::max<uint64_t>(smax, (need + eb - 1) / eb);
  }
  p.stem_elems_max = smax;
  p.max_stem_log2 = 0;
  while ((1ull << p.max_stem_log2) < smax) p.max_stem_log2++;
  if (cfg.stem_capacity_bytes && smax * eb > cfg.stem_capacity_bytes)
    throw err(TN_E_INFEASIBLE, "largest stem tensor exceeds stem_capacity_bytes");

  // ---- flops
  p.total_flops = p.stem_flops;
  for (int id : p.common_order) p.total_flops += 8.0 * p.nodes[id].cost;

  // ---- workspace layout
  uint64_t off = 0;
  for (auto& lf : p.leaves) {
    lf.ws_off = off;
    off += align_up(8ull << lf.labels.size(), 256);
  }
  p.ws_leaves = off;
  p.h2d_bytes = off;
  for (int id : p.common_order) {
    p.nodes[id].ws_off = off;
    off += align_up(8ull << p.nodes[id].labels.size(), 256);
  }
  p.ws_common = off;
  static const bool fold_off = getenv("TN_NO_FOLD") != nullptr;  // A/B knob
  for (auto& st : p.steps) {
    uint64_t kn = 1ull << (st.klog + st.nlog);
    const uint64_t nb = 1ull << st.b_sparse.size();  // sparse tail: one block per sparse-leg value
    st.b_tmp_off = off;
    off += align_up(8 * kn, 1024) * nb;
    st.fold = 1;
    // (a transposed output only for f = 2 and N = 16: the folded tile is then one C^T box {256 m, 16 n})
    if (cfg.dtype == TN_CHALF && !fold_off && !st.gather_a && !st.mn && !st.split && !st.sparse &&
        st.klog >= 1 && st.klog <= 4 && (st.out_identity || (st.out_transposed && st.klog == 4 && st.nlog == 4))) {
      int fl = 0;
      while ((4 << (st.klog + fl)) < 128) ++fl;  // rows of 2K fp16 -> 128 bytes
      if (st.mlog - fl >= 8) {
        st.fold = 1 << fl;
        st.tensor_core = true;
        const uint64_t rows = std::max<uint64_t>((uint64_t)st.fold * 2 << st.nlog, 16);
        st.b_fold_bytes = align_up(rows * ((uint64_t)st.fold * 2 << st.klog) * 2, 1024);
      }
    }
    if (cfg.dtype == TN_CHALF && st.fold > 1) {
      // B' = blockdiag(B_P x fold), then the B_P scratch it is built from
      st.b_off = off;
      st.b_blk = st.b_fold_bytes;
      off += st.b_fold_bytes + align_up(std::max<uint64_t>(8 * kn, 64ull << st.klog), 1024);
    } else if (cfg.dtype == TN_CHALF) {
      st.b_off = off;
      // fp16 [max(2N, 16)][2K]: rows beyond 2N are zero (tcgen05 N >= 16)
      // sparse tail: blocks back to back (the batched GEMM's B map steps by exactly one block)
      st.b_blk = st.sparse ? std::max<uint64_t>(8 * kn, 64ull << st.klog)
                           : align_up(std::max<uint64_t>(8 * kn, 64ull << st.klog), 1024);
      off += align_up(st.b_blk * nb, 1024);
    } else {
      st.b_off = st.b_tmp_off;
      st.b_blk = align_up(8 * kn, 1024);
    }
  }
  p.ws_b = off;
  p.ws_slice = off;
  off += 256;
  p.ws_scratch = off;
  size_t S = p.steps.size();
  p.n_exp_slots = (int)(2 * S + 4);
  // max_slot[S+2], b_bound[S+2], b_max[S+2], exps[n_exp_slots], entry_max (runtime.cu scratch_of)
  off += align_up(4 * 4 * (S + 2) + 4 * p.n_exp_slots + 4 + 64, 256);
  if (!p.split_modes.empty()) {
    // per chunk: max slots [T+1] and step exponents [T] of the tail (each chunk has its own scale)
    const uint64_t T = p.steps.size() - p.split_from, c = 1ull << p.split_log2;
    // + the post-selected member of each subspace (uint64 per chunk)
    off += align_up(4 * c * (2 * T + 1) + 8 * c + 64, 256);
  }
  if (world > 1) {
    // sharded readout: every rank's result block (rank order) and, with a split tail, every rank's
    // per-chunk exponents are gathered here (the stem buffers may still hold the tail's input)
    p.ws_gather = off;
    off += align_up((uint64_t)eb << p.open.size(), 256);
    p.ws_gather_exp = off;
    if (!p.split_modes.empty())
      off += align_up(4ull * world * (1ull << p.split_log2) * (p.steps.size() - p.split_from), 256);
  }
  p.ws_total = off;
  return P.release();
}

static void jlist(std::ostringstream& o, const std::vector<int>& v) {
  o << "[";
  for (size_t i = 0; i < v.size(); ++i) o << (i ? "," : "") << v[i];
  o << "]";
}

std::string report_json(const Plan& p, const std::vector<float>& ms) {
  std::ostringstream o;
  o.precision(17);
  o << "{\"dtype\":\"" << (p.cfg.dtype == TN_CHALF ? "chalf" : "cfloat") << "\"";
  o << ",\"stem_entry\":" << p.stem_entry << ",\"n_common\":" << p.common_order.size();
  o << ",\"stem_flops\":" << p.stem_flops << ",\"total_flops\":" << p.total_flops;
  o << ",\"stem_bytes_alg\":" << p.stem_bytes_alg << ",\"perm_bytes\":" << p.perm_bytes;
  o << ",\"max_stem_log2\":" << p.max_stem_log2 << ",\"final_perm\":" << (p.final_perm ? 1 : 0);
  o << ",\"steps\":[";
  for (size_t i = 0; i < p.steps.size(); ++i) {
    const StemStep& s = p.steps[i];
    o << (i ? "," : "") << "{\"node\":" << s.node << ",\"branch\":" << s.branch << ",\"m\":" << s.mlog
      << ",\"k\":" << s.klog << ",\"n\":" << s.nlog << ",\"perm\":" << (s.perm ? 1 : 0)
      << ",\"tc\":" << (s.tensor_core ? 1 : 0) << ",\"ga\":" << (s.gather_a ? 1 : 0) << ",\"split\":" << s.split << ",\"swap\":" << (s.swap ? 1 : 0)
      << ",\"quant\":" << (s.quant ? 1 : 0) << ",\"sparse\":" << s.sparse
      << ",\"fuse_quant\":" << (s.fuse_quant ? 1 : 0)
      << ",\"out_kind\":" << (s.out_identity ? 0 : (s.out_transposed ? 1 : 2)) << ",\"mn\":" << (s.mn ? s.mn_ma : 0) << ",\"mn_split\":[" << s.mn_kl << "," << s.mn_mm << "]"
      << ",\"fold\":" << s.fold
      << ",\"gmode\":"
      << (s.gather_a && !s.a_m_stride.empty()
              ? gather_mode_of_strides(s.mlog, s.klog, s.a_m_stride.data(), s.a_k_stride.data())
              : -1)
      << ",\"kern\":\"" << (i < p.step_kern.size() ? p.step_kern[i] : std::string()) << "\""
      << ",\"pass\":" << (i < p.step_pass.size() ? p.step_pass[i] : (s.perm ? 1 : 0))
      << ",\"in\":";
    jlist(o, s.in_layout);
    o << ",\"R\":";
    jlist(o, s.R);
    o << ",\"out\":";
    jlist(o, s.out_layout);
    if (s.sparse) {
      o << ",\"b_sparse\":";
      jlist(o, s.b_sparse);
    }
    if (s.swap) {
      o << ",\"shard_before\":";
      jlist(o, s.shard_before);
      o << ",\"shard_after\":";
      jlist(o, s.shard_after);
      o << ",\"swap_out_pos\":";
      jlist(o, s.swap_out_pos);
      o << ",\"swap_in\":";
      jlist(o, s.swap_in);
      o << ",\"send_layout\":";
      jlist(o, s.send_layout);
    }
    o << "}";
  }
  o << "],\"common\":[";  // per common contraction: [out rank, unsliced rank of u, of v, reduced modes]
  for (size_t i = 0; i < p.common_order.size(); ++i) {
    const Node& n = p.nodes[p.common_order[i]];
    auto urank = [&](int id) {
      int r = 0;
      for (int l : p.nodes[id].labels)
        if (std::find(p.sliced.begin(), p.sliced.end(), l) == p.sliced.end()) ++r;
      return r;
    };
    const int ru = urank(n.u), rv = urank(n.v), ro = (int)n.labels.size();
    o << (i ? "," : "") << "[" << ro << "," << ru << "," << rv << "," << (ru + rv - ro) / 2 << "]";
  }
  o << "],\"entry_layout\":";
  jlist(o, p.stem_entry >= 0 ? p.nodes[p.stem_entry].labels : std::vector<int>());
  o << ",\"split_modes\":";
  jlist(o, p.split_modes);
  o << ",\"split_from\":" << p.split_from << ",\"recompute_from\":" << p.recompute_from
    << ",\"sparse_from\":" << p.sparse_from
    << ",\"sparse_chunks\":" << p.sparse_chunks << ",\"sparse_flops\":" << p.sparse_flops << ",\"sparse_legs\":";
  jlist(o, p.sparse_legs);
  o << ",\"shard0\":";
  jlist(o, p.shard0);
  o << ",\"final_layout\":";
  jlist(o, p.final_layout);
  o << ",\"launches\":" << p.launches << ",\"world\":" << p.world << ",\"n_swaps\":" << p.n_swaps
    << ",\"swap_bytes\":" << p.swap_bytes << ",\"n_fused_swaps\":" << p.n_fused_swaps << ",\"n_peer_swaps\":" << p.n_peer_swaps << ",\"n_composed_swaps\":" << p.n_composed_swaps << ",\"final_shard\":";
  jlist(o, p.final_shard);
  if (!ms.empty()) {  // [common_ms, (perm_ms, gemm_ms) per step..., final_ms]
    o << ",\"ms\":[";
    for (size_t i = 0; i < ms.size(); ++i) o << (i ? "," : "") << ms[i];
    o << "]";
  }
  o << "}";
  return o.str();
}

}  // namespace tn
