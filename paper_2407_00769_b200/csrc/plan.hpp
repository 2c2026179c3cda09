// Plan representation and host-side lowering.
// Host only: no CUDA types here, so the lowering can be unit-tested without a GPU.
#pragma once
#include <cstdint>
#include <string>
#include <vector>

#include "../../include/tn.h"

namespace tn {

struct TnError {
  int code;
  std::string msg;
};

// A strided view of a complex tensor with every mode of dimension 2.
struct Leaf {
  std::vector<int> labels;        // full (unsliced) label list, row-major order
  std::vector<double> data;       // interleaved complex128 (2 * 2^rank doubles)
  uint64_t ws_off = 0;            // byte offset of its complex64 copy in the workspace
};

enum NodeKind { NODE_LEAF = 0, NODE_COMMON = 1, NODE_STEM = 2 };

struct Node {
  int u = -1, v = -1;             // children (internal nodes)
  int kind = NODE_LEAF;
  std::vector<int> labels;        // labels after slicing; for leaves/common = device layout order
  uint64_t ws_off = 0;            // complex64 storage of common results (bytes into ws)
  double cost = 0;                // complex MACs of this contraction (sliced)
  double sub_cost = 0;            // subtree complex MACs
};

// One stem step: [optional permutation] + GEMM  C[kept, new] = A[kept, R] * B[R, new].
// k_gemm_tc.cu: the A-operand path of a gathered step (0 direct box, 2 core-matrix box, 3 raw box,
// 1 cp.async 16 B, 4 cp.async 4 B), for the lowering's cost model
int gather_mode_of_strides(int mlog, int klog, const int64_t* ms, const int64_t* ks);

struct StemStep {
  int node = -1;                  // tree node produced by this step
  int branch = -1;                // the non-stem operand (common node or leaf)
  std::vector<int> in_layout;     // stem layout before the step (outermost first)
  bool perm = false;              // standalone permutation pass needed
  std::vector<int> perm_axes;     // numpy-transpose axes: perm_layout[j] = in_layout[perm_axes[j]]
  std::vector<int> R, kept, newl; // contracted (K order), kept (M order), new (N order)
  int mlog = 0, klog = 0, nlog = 0;
  std::vector<int> out_layout;    // kept + newl
  uint64_t b_off = 0;             // ws offset: B operand (fp16 B_P for chalf, c64 [K][N] for cfloat)
  uint64_t b_tmp_off = 0;         // ws offset: gathered complex64 [K][N] (chalf path)
  bool tensor_core = false;       // tcgen05 GEMM (else SIMT)
  // permutation fused into the GEMM's A load: A[m, k] at sum bit_j(m) a_m_stride[j] +
  // sum bit_j(k) a_k_stride[j] of the UNPERMUTED in_layout (perm == false then)
  bool gather_a = false;
  std::vector<int64_t> a_m_stride, a_k_stride;
  // stored order [other kept | R | mn_ma kept modes] (mn_ma >= 7): the permutation is folded into an
  // MN-major A operand (k_gemm_tc2.cu launch_gemm_chalf_mn, B' via launch_pad_b_mn) when the launch
  // geometry allows (runtime mn_active); perm / perm_axes stay as the fallback
  bool mn = false;
  int mn_ma = 0;
  // split contraction block [other kept | R_hi | mn_mm kept | R_lo (mn_kl modes) | mn_ma kept]: one
  // kept run inside the contracted modes (a 5-d A map); 0 = one contiguous block
  int mn_kl = 0, mn_mm = 0;
  // row folding (plain A, row-major output, 2K x 2 B < 128 B): the tcgen05 GEMM runs on [M/f][f 2K] x
  // blockdiag(B_P x f) -> [M/f][f 2N], the same bytes read as rows of 128 B (the TMA engine's
  // per-row cost made 64-byte rows its limit); B' at b_off, B_P scratch at b_off + b_fold_bytes
  bool tr_choice = false;         // layout policy 3 weighed a transposed output here (search point)
  int fold = 1;
  uint64_t b_fold_bytes = 0;
  // output address of C[m, n] = sum_j bit_j(m) m_stride[j] + sum_j bit_j(n) n_stride[j] (elements)
  std::vector<int64_t> m_stride, n_stride;
  bool out_identity = true;       // out_layout == kept ++ newl (plain row-major [M][N])
  bool out_transposed = false;    // out_layout == newl ++ kept (C[n][m], layout policy 3)
  int split = 0;                  // 1 = split-type (chunked tail) step
  int sparse = 0;                 // 1 = sparse-state tail step (gather-batched GEMM, Fig. 5)
  std::vector<int> b_sparse;      // sparse legs of the branch (B_P block index bits, MSB first)
  uint64_t b_blk = 0;             // bytes of one B_P block
  // sharded stem (world > 1), Alg. 1: mode swap before this step when R ∩ shard != ∅
  bool swap = false;
  std::vector<int> shard_before, shard_after;  // shard labels, rank bit order (MSB first)
  std::vector<int> swap_out_pos;  // positions (in shard_before) of the contracted shard modes
  std::vector<int> swap_in;       // local labels that become shard modes (same positions)
  bool send_perm = false;         // local permutation putting swap_in outermost before sending
  bool quant = false;             // this swap's payload is group-quantised (else fp16)
  bool fuse_quant = false;        // quantised + send_perm keeps the innermost log2(g/2) modes: fused codec
  std::vector<int> send_perm_axes;
  std::vector<int> send_layout;   // local layout being sent (swap_in outermost)
};

struct Plan {
  tn_config cfg{};
  std::vector<Leaf> leaves;
  std::vector<Node> nodes;        // leaves first, then internal in SSA order
  std::vector<int> open;          // output legs in output order
  std::vector<int> sliced;        // bit j of slice id fixes sliced[j]
  std::vector<int> stem;          // leaf->root node ids
  int root = -1;
  int stem_entry = -1;            // node converted into the stem buffer (-1: no stem steps)
  std::vector<int> common_order;  // internal common nodes in execution (post) order
  std::vector<StemStep> steps;
  std::vector<int> final_layout;  // stem layout after the last step
  bool final_perm = false;        // final permutation into `open` order
  std::vector<int> final_perm_axes;
  int split_from = -1;            // first split-type step index (-1: none)
  std::vector<int> sparse_legs;   // open legs given per correlated subspace (sparse-state batch)
  int sparse_from = -1;           // first sparse-tail step (-1: none)
  int recompute_from = -1;        // recomputation on halves: the step producing the largest tensor
  uint64_t sparse_chunks = 0;     // subspace chunks of the last sparse-tail run
  double sparse_flops = 0;        // 8 x complex MACs of the last sparse-tail run (every chunk)
  int split_log2 = 0;             // chunks = 2^split_log2
  std::vector<int> split_modes;   // open legs fixed per chunk (outermost in every tail layout)
  uint64_t split_chunk_max = 0;   // largest per-chunk stem tensor of the tail (elements)
  int stem_cur = 0;               // buffer holding the stem after tn_stem_contract (split mode)
  uint64_t result_off = 0;        // element offset of the result inside its buffer
  std::vector<uint64_t> tail_slots;  // chunk id held by each result slot of the last tail run
  // workspace layout
  uint64_t ws_leaves = 0, ws_common = 0, ws_b = 0, ws_scratch = 0, ws_total = 0;
  uint64_t ws_gather = 0;         // world > 1: gathered result (eb << n_open bytes)
  uint64_t ws_gather_exp = 0;     // world > 1 with a split tail: gathered per-chunk exponents
  uint64_t ws_slice = 0;          // uint64 slice id, read by the kernels (one CUDA graph serves every slice)
  uint64_t stem_elems_max = 0;    // largest stem tensor (elements)
  int max_stem_log2 = 0;
  // scratch slots (offsets in bytes from ws_scratch)
  //   float max_slot[S+2] (slot i = max |real| of the stem entering step i), float b_bound[S+2],
  //   uint b_max[S+2], int exps[n_exp_slots], uint entry_max  (runtime.cu scratch_of)
  int n_exp_slots = 0;
  double stem_flops = 0, total_flops = 0, stem_bytes_alg = 0, perm_bytes = 0;
  int n_permutes = 0;
  uint64_t h2d_bytes = 0;
  // runtime state
  int result_buf = 0;             // which stem buffer holds the result
  bool result_in_ws = false;      // no stem steps: result is a common node in ws (c64)
  int timing = 0;
  // timing events (cudaEvent_t as void*): [0] start, [1] stem entry ready, then per step i
  // [2+2i] after the permutation, [3+2i] after the GEMM; [2+2S] after the final permutation.
  std::vector<void*> ev;
  bool ev_valid = false;
  uint64_t launches = 0;          // kernels launched by the last tn_stem_contract
  void* pinned = nullptr;         // pinned host copy of leaves (complex64), lazily allocated
  int world = 1, rank = 0;
  int shard_log2 = 0;             // log2(world): the stem is sharded on this many modes
  std::vector<int> shard0;        // initial shard labels (outermost of the entry layout)
  std::vector<int> final_shard;   // shard labels after the last step (the result's rank bits)
  int n_swaps = 0;
  double swap_bytes = 0;          // payload bytes each rank sends per slice (codec applied)
  int n_fused_swaps = 0;          // swaps of the last run done inside the previous GEMM's epilogue
  int n_peer_swaps = 0;           // other swaps of the last run moved by a peer-memory pass (no NCCL)
  int n_composed_swaps = 0;       // of those, passes that also did the next step's permutation
  std::vector<std::string> step_kern;  // per step: GEMM kernel family of the last (eager / captured) run
  std::vector<int> step_pass;          // per step: 1 when a permutation pass ran before its GEMM
  std::vector<void*> peer_stem;   // [2 r + j]: rank r's stem buffer j as this rank addresses it
  const void* peer_key[2] = {nullptr, nullptr};  // the local buffers peer_stem was set up for
  std::vector<void*> ipc_open;    // CUDA IPC mappings opened for peer_stem (closed on free)
  // level-batched common phase (runtime.cu run_common): device copies of every common contraction's
  // arguments, grouped by tree level, built for one workspace (key)
  void* common_dev = nullptr;
  const void* common_key = nullptr;
  std::vector<int> common_level_nodes;     // per level: node count
  std::vector<uint32_t> common_level_blocks;  // per level: blocks of the launch
  std::vector<uint64_t> common_level_args, common_level_start;  // byte offsets into common_dev
  tn_comm* comm = nullptr;
  // CUDA graph of the whole tn_stem_contract body (world == 1; sharded: the head, or all with TN_GRAPH_NCCL=1): captured once per buffer set on a
  // library stream, replayed on the caller's stream.  Opaque CUDA handles as void*.
  void* graph_exec = nullptr;
  bool nccl_warm = false;  // sharded: one eager call done (NCCL connections exist) before capture
  void* cap_stream = nullptr;
  const void* graph_key[4] = {nullptr, nullptr, nullptr, nullptr};
  uint64_t graph_stem_bytes = 0;
  uint64_t graph_launches = 0;
  int graph_stem_cur = 0, graph_result_buf = 0, graph_timing = 0;
  bool graph_off = false;         // tn_set_graph(p, 0)
};

// Parse JSON + validate + lower.  Throws TnError.
Plan* load_plan(const char* json, size_t len, const tn_config* cfg, int world = 1);
std::string report_json(const Plan& p, const std::vector<float>& ms);

inline uint64_t align_up(uint64_t x, uint64_t a) { return (x + a - 1) / a * a; }

}  // namespace tn
