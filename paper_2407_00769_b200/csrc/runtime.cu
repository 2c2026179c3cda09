// C-ABI implementation (include/tn.h): plan lifecycle and the per-slice executor.
//
// Executor for one subtask:
//   1. common phase: every non-stem contraction of the sliced network, complex64,
//      in the workspace arena; slicing = base offsets into the uploaded leaves;
//   2. stem operands: each branch is gathered to the dense [K][N] layout its step needs and padded
//      to B_P per Eq. 6 with an exact power-of-two scale (C-A8);
//   3. stem entry: the first large stem tensor is converted into stem buffer 0;
//   4. stem loop (Alg. 1 "performer computation of currEin"): per step an optional
//      permutation buf p -> buf 1-p, then the GEMM buf p -> buf 1-p (static double buffers).
//   No host synchronisation inside the loop: all scale exponents live on the device.
#include <cuda.h>
#include <dlfcn.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <condition_variable>
#include <cstring>
#include <mutex>
#include <vector>

#include "common.cuh"

using namespace tn;
namespace tn {
thread_local const char* g_last_kern = "";
}

static thread_local std::string g_err;

static int fail(int code, const std::string& m) {
  g_err = m;
  return code;
}

#define TN_TRY(...)                                    \
  try {                                                \
    __VA_ARGS__;                                       \
    return TN_OK;                                      \
  } catch (const TnError& e) {                         \
    return fail(e.code, e.msg);                        \
  } catch (const std::bad_alloc&) {                    \
    return fail(TN_E_CAPACITY, "host allocation failed"); \
  } catch (const std::exception& e) {                  \
    return fail(TN_E_INVALID, e.what());               \
  }

struct tn_plan {
  Plan* p;
};

// Loopback transport: `world` virtual ranks on ONE device, each driven by its own host thread
// (as real ranks are driven by their own processes).  A collective is a host rendezvous of the
// ranks plus stream-ordered device work: every rank publishes its buffers and an event, waits on its
// peers' events, moves the data with device-to-device copies (or a tiny max kernel) on its own
// stream, and waits until its peers have finished reading its buffers before it proceeds.  The
// same lowering, codec kernels and swap schedule run as with NCCL; only the byte mover differs.
struct LoopGroup {
  int world = 0, device = 0, refs = 0;
  std::mutex mu;
  std::condition_variable cv;
  int arrived = 0;
  uint64_t gen = 0;
  bool broken = false;
  std::vector<cudaEvent_t> ready, done;
  struct Post {
    int dst;
    const void* ptr;
    uint64_t bytes;
  };
  std::vector<std::vector<Post>> board;  // board[src]: sends posted by rank src, in order
  std::vector<const void*> ptr;          // per rank: the buffer of an all-reduce / all-gather
  std::vector<void*> stem_ptrs;          // per rank: its two stem buffers (fused mode swaps)
  void barrier() {
    std::unique_lock<std::mutex> lk(mu);
    if (broken) throw TnError{TN_E_NCCL, "loopback group broken by an earlier timeout"};
    const uint64_t g = gen;
    if (++arrived == world) {
      arrived = 0;
      ++gen;
      cv.notify_all();
      return;
    }
    // a rank that never arrives (error on its thread) must not hang the others forever
    if (!cv.wait_for(lk, std::chrono::seconds(600), [&] { return gen != g; })) {
      broken = true;
      cv.notify_all();
      throw TnError{TN_E_NCCL, "loopback rendezvous timed out (a virtual rank did not arrive)"};
    }
  }
};

struct tn_comm {
  void* nccl_comm = nullptr;
  int rank = 0, world = 1, device = 0;
  LoopGroup* loop = nullptr;   // loopback transport (virtual ranks on one device)
};

// ---- NCCL (dlopen'ed: the process's torch already carries libnccl.so.2) ----
namespace {
enum { NCCL_INT8 = 0, NCCL_FLOAT16 = 6, NCCL_FLOAT32 = 7, NCCL_MAX = 2 };
void* nccl_sym(const char* name) {
  static void* h = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
  });
  void* f = h ? dlsym(h, name) : nullptr;
  if (!f) throw TnError{TN_E_NCCL, std::string("NCCL symbol unavailable: ") + name};
  return f;
}
void nccl_check(int r, const char* what) {
  if (r != 0) throw TnError{TN_E_NCCL, std::string(what) + " failed (" + std::to_string(r) + ")"};
}
void nccl_group(bool start) {
  typedef int (*fn_t)();
  static fn_t gs = (fn_t)nccl_sym("ncclGroupStart"), ge = (fn_t)nccl_sym("ncclGroupEnd");
  nccl_check(start ? gs() : ge(), start ? "ncclGroupStart" : "ncclGroupEnd");
}
void nccl_send(const void* buf, size_t count, int type, int peer, void* comm, cudaStream_t s) {
  typedef int (*fn_t)(const void*, size_t, int, int, void*, cudaStream_t);
  static fn_t f = (fn_t)nccl_sym("ncclSend");
  nccl_check(f(buf, count, type, peer, comm, s), "ncclSend");
}
void nccl_recv(void* buf, size_t count, int type, int peer, void* comm, cudaStream_t s) {
  typedef int (*fn_t)(void*, size_t, int, int, void*, cudaStream_t);
  static fn_t f = (fn_t)nccl_sym("ncclRecv");
  nccl_check(f(buf, count, type, peer, comm, s), "ncclRecv");
}
void nccl_allreduce_max(float* buf, size_t count, void* comm, cudaStream_t s) {
  typedef int (*fn_t)(const void*, void*, size_t, int, int, void*, cudaStream_t);
  static fn_t f = (fn_t)nccl_sym("ncclAllReduce");
  nccl_check(f(buf, buf, count, NCCL_FLOAT32, NCCL_MAX, comm, s), "ncclAllReduce");
}
void nccl_allgather(const void* send, void* recv, size_t count, int type, void* comm, cudaStream_t s) {
  typedef int (*fn_t)(const void*, void*, size_t, int, void*, cudaStream_t);
  static fn_t f = (fn_t)nccl_sym("ncclAllGather");
  nccl_check(f(send, recv, count, type, comm, s), "ncclAllGather");
}
}  // namespace

namespace {

// ---- transport: the byte movers of the sharded stem (NCCL between processes, or loopback) ----
struct Xfer {
  int peer;
  void* ptr;
  uint64_t bytes;
};

// Calls on a plan with a communicator run on the communicator's device (a virtual rank's thread,
// or a process that drives several libraries, need not have selected it).
void select_device(const Plan& p) {
  if (p.comm) TN_CUDA(cudaSetDevice(p.comm->device));
}

void comm_check(const Plan& p) {
  if (!p.comm || (!p.comm->nccl_comm && !p.comm->loop))
    throw TnError{TN_E_NCCL, "sharded plan without a communicator"};
}

// Grouped point-to-point exchange: every (send, recv) pair with the same peer is matched in order.
void xfer_exchange(Plan& p, const std::vector<Xfer>& sends, const std::vector<Xfer>& recvs, cudaStream_t s) {
  comm_check(p);
  tn_comm* c = p.comm;
  if (!c->loop) {
    nccl_group(true);
    for (const Xfer& x : sends) nccl_send(x.ptr, x.bytes, NCCL_INT8, x.peer, c->nccl_comm, s);
    for (const Xfer& x : recvs) nccl_recv(x.ptr, x.bytes, NCCL_INT8, x.peer, c->nccl_comm, s);
    nccl_group(false);
    return;
  }
  LoopGroup& g = *c->loop;
  const int me = c->rank;
  {
    std::lock_guard<std::mutex> lk(g.mu);
    g.board[me].clear();
    for (const Xfer& x : sends) g.board[me].push_back({x.peer, x.ptr, x.bytes});
  }
  TN_CUDA(cudaEventRecord(g.ready[me], s));  // the payload is complete once this event fires
  g.barrier();
  std::vector<int> taken(g.world, 0);
  for (const Xfer& x : recvs) {
    const LoopGroup::Post* src = nullptr;
    int k = 0;
    for (const auto& post : g.board[x.peer])
      if (post.dst == me && k++ == taken[x.peer]) {
        src = &post;
        break;
      }
    if (!src || src->bytes != x.bytes) throw TnError{TN_E_NCCL, "loopback exchange: unmatched send/recv"};
    ++taken[x.peer];
    TN_CUDA(cudaStreamWaitEvent(s, g.ready[x.peer], 0));
    TN_CUDA(cudaMemcpyAsync(x.ptr, src->ptr, x.bytes, cudaMemcpyDeviceToDevice, s));
  }
  TN_CUDA(cudaEventRecord(g.done[me], s));
  g.barrier();
  // the peers' copies out of this rank's send buffers must finish before it writes them again
  for (const Xfer& x : sends) TN_CUDA(cudaStreamWaitEvent(s, g.done[x.peer], 0));
}

// 1-float max over ranks (every rank scales the next stem step by the same power of two, C-A28).
void xfer_allreduce_max(Plan& p, float* slot, cudaStream_t s) {
  comm_check(p);
  tn_comm* c = p.comm;
  if (!c->loop) {
    nccl_allreduce_max(slot, 1, c->nccl_comm, s);
    return;
  }
  LoopGroup& g = *c->loop;
  g.ptr[c->rank] = slot;
  TN_CUDA(cudaEventRecord(g.ready[c->rank], s));
  g.barrier();
  MaxSlots ms;
  ms.n = g.world;
  for (int r = 0; r < g.world; ++r) {
    ms.p[r] = static_cast<const float*>(g.ptr[r]);
    if (r != c->rank) TN_CUDA(cudaStreamWaitEvent(s, g.ready[r], 0));
  }
  launch_max_slots(slot, ms, s);
  TN_CUDA(cudaEventRecord(g.done[c->rank], s));
  g.barrier();
  for (int r = 0; r < g.world; ++r)
    if (r != c->rank) TN_CUDA(cudaStreamWaitEvent(s, g.done[r], 0));
}

// recv[r * bytes ..] = rank r's `send` (rank order).
void xfer_allgather(Plan& p, const void* send, void* recv, uint64_t bytes, cudaStream_t s) {
  comm_check(p);
  tn_comm* c = p.comm;
  if (!c->loop) {
    nccl_allgather(send, recv, bytes, NCCL_INT8, c->nccl_comm, s);
    return;
  }
  LoopGroup& g = *c->loop;
  g.ptr[c->rank] = send;
  TN_CUDA(cudaEventRecord(g.ready[c->rank], s));
  g.barrier();
  for (int r = 0; r < g.world; ++r) {
    if (r != c->rank) TN_CUDA(cudaStreamWaitEvent(s, g.ready[r], 0));
    TN_CUDA(cudaMemcpyAsync(static_cast<unsigned char*>(recv) + (uint64_t)r * bytes, g.ptr[r], bytes,
                            cudaMemcpyDeviceToDevice, s));
  }
  TN_CUDA(cudaEventRecord(g.done[c->rank], s));
  g.barrier();
  for (int r = 0; r < g.world; ++r)
    if (r != c->rank) TN_CUDA(cudaStreamWaitEvent(s, g.done[r], 0));
}

// ---- peer buffers for mode swaps fused into a GEMM epilogue (PeerTarget, common.cuh) ----
// Every rank's two stem buffers as device pointers this rank can store to: loopback ranks share
// the device (plain pointers); NCCL ranks map each other's buffers with CUDA IPC (handles of the
// allocations holding the caller's buffers, exchanged with an all-gather, opened once per buffer
// set).  Collective: every rank calls it with its buffers at the same point.
typedef CUresult (*addr_range_t)(CUdeviceptr*, size_t*, CUdeviceptr);

void close_peers(Plan& p) {
  for (void* q : p.ipc_open) cudaIpcCloseMemHandle(q);
  p.ipc_open.clear();
  p.peer_stem.clear();
  p.peer_key[0] = p.peer_key[1] = nullptr;
}

void ensure_peers(Plan& p, const tn_buffers* b, cudaStream_t s) {
  if (p.world <= 1 || !p.comm) return;
  if (p.peer_key[0] == b->d_stem[0] && p.peer_key[1] == b->d_stem[1]) return;  // set up (or refused) already
  close_peers(p);
  tn_comm* c = p.comm;
  std::vector<void*> ptrs(2 * p.world, nullptr);
  if (c->loop) {
    LoopGroup& g = *c->loop;
    {
      std::lock_guard<std::mutex> lk(g.mu);
      if (g.stem_ptrs.size() != 2u * g.world) g.stem_ptrs.assign(2 * g.world, nullptr);
      g.stem_ptrs[2 * c->rank] = b->d_stem[0];
      g.stem_ptrs[2 * c->rank + 1] = b->d_stem[1];
    }
    g.barrier();
    {
      std::lock_guard<std::mutex> lk(g.mu);
      ptrs = g.stem_ptrs;
    }
    g.barrier();  // nobody republishes before every rank has read
  } else {
    static addr_range_t range = nullptr;
    if (!range) {
      void* fn = nullptr;
      cudaDriverEntryPointQueryResult q;
      if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &fn, cudaEnableDefault, &q) != cudaSuccess ||
          q != cudaDriverEntryPointSuccess)
        throw TnError{TN_E_CUDA, "cuMemGetAddressRange unavailable"};
      range = (addr_range_t)fn;
    }
    // Every rank takes part in both collectives whatever fails locally, and all ranks agree on the
    // outcome: if any rank cannot export or map a buffer, nobody uses peer memory (the swaps then go
    // through the transport), instead of some ranks storing into peers that never mapped them.
    struct Rec {
      cudaIpcMemHandle_t h[2];
      uint64_t off[2];
      int ok;
      int pad;
    };
    Rec mine;
    memset(&mine, 0, sizeof(mine));
    mine.ok = 1;
    for (int j = 0; j < 2 && mine.ok; ++j) {
      CUdeviceptr base = 0;
      size_t sz = 0;
      if (range(&base, &sz, (CUdeviceptr)b->d_stem[j]) != CUDA_SUCCESS ||
          cudaIpcGetMemHandle(&mine.h[j], (void*)base) != cudaSuccess) {
        cudaGetLastError();
        mine.ok = 0;
        break;
      }
      mine.off[j] = (uint64_t)((CUdeviceptr)b->d_stem[j] - base);
    }
    unsigned char* d = nullptr;
    TN_CUDA(cudaMalloc(&d, sizeof(Rec) * (p.world + 1) + 256));
    std::vector<Rec> all(p.world);
    bool ok = true;
    try {
      TN_CUDA(cudaMemcpyAsync(d, &mine, sizeof(Rec), cudaMemcpyHostToDevice, s));
      xfer_allgather(p, d, d + sizeof(Rec), sizeof(Rec), s);
      TN_CUDA(cudaMemcpyAsync(all.data(), d + sizeof(Rec), sizeof(Rec) * p.world, cudaMemcpyDeviceToHost, s));
      TN_CUDA(cudaStreamSynchronize(s));
      for (const Rec& r : all) ok = ok && r.ok;
      std::vector<std::pair<cudaIpcMemHandle_t, void*>> opened;  // one mapping per allocation
      bool mapped = true;
      for (int r = 0; ok && mapped && r < p.world; ++r)
        for (int j = 0; mapped && j < 2; ++j) {
          if (r == p.rank) {
            ptrs[2 * r + j] = b->d_stem[j];
            continue;
          }
          void* base = nullptr;
          for (auto& o : opened)
            if (!memcmp(&o.first, &all[r].h[j], sizeof(cudaIpcMemHandle_t))) base = o.second;
          if (!base) {
            if (cudaIpcOpenMemHandle(&base, all[r].h[j], cudaIpcMemLazyEnablePeerAccess) != cudaSuccess) {
              cudaGetLastError();
              mapped = false;
              break;
            }
            opened.push_back({all[r].h[j], base});
            p.ipc_open.push_back(base);
          }
          ptrs[2 * r + j] = static_cast<unsigned char*>(base) + all[r].off[j];
        }
      if (ok) {
        // second agreement: every rank mapped every peer (max over ranks of "failed")
        float* flag = reinterpret_cast<float*>(d + sizeof(Rec) * (p.world + 1));
        const float failed = mapped ? 0.f : 1.f;
        TN_CUDA(cudaMemcpyAsync(flag, &failed, 4, cudaMemcpyHostToDevice, s));
        xfer_allreduce_max(p, flag, s);
        float any = 0.f;
        TN_CUDA(cudaMemcpyAsync(&any, flag, 4, cudaMemcpyDeviceToHost, s));
        TN_CUDA(cudaStreamSynchronize(s));
        ok = any == 0.f;
      }
    } catch (...) {
      cudaFree(d);
      throw;
    }
    TN_CUDA(cudaFree(d));
    if (!ok) {
      fprintf(stderr, "tn: peer-memory mode swaps unavailable (CUDA IPC); using the transport\n");
      close_peers(p);
      p.peer_key[0] = b->d_stem[0];  // do not retry for this buffer set
      p.peer_key[1] = b->d_stem[1];
      return;
    }
  }
  p.peer_stem = ptrs;
  p.peer_key[0] = b->d_stem[0];
  p.peer_key[1] = b->d_stem[1];
}

// Members of a mode swap (Alg. 1): this rank's member index (its bits at the swapped shard
// positions, position 0 = rank MSB) and the rank of member v.
struct SwapMembers {
  int S = 0, sx = 0, me = 0, rank = 0;
  std::vector<int> out_pos;
  SwapMembers(const Plan& p, const StemStep& st) : S((int)st.shard_before.size()), sx((int)st.swap_out_pos.size()),
                                                    rank(p.rank), out_pos(st.swap_out_pos) {
    for (int t = 0; t < sx; ++t) me = (me << 1) | ((rank >> (S - 1 - out_pos[t])) & 1);
  }
  int peer_of(int v) const {
    int r = rank;
    for (int t = 0; t < sx; ++t) {
      const int shift = S - 1 - out_pos[t], bit = (v >> (sx - 1 - t)) & 1;
      r = (r & ~(1 << shift)) | (bit << shift);
    }
    return r;
  }
};

bool fused_swap_enabled(const Plan& p) {
  static const char* e = getenv("TN_NO_FUSED_SWAP");  // A/B knob (same as cfg.no_fused_swap = 1)
  return p.world > 1 && !p.cfg.no_fused_swap && !(e && atoi(e) != 0);
}

// The mode swap before step i+1 done by step i's GEMM epilogue: each output element goes straight
// to the rank that owns it after the swap.  Same result as mode_swap (send permutation putting
// swap_in outermost, chunk v to member v, received at chunk `me`): the receiver's local index is the
// element's index with the swap_in bits removed, behind the outermost `me` chunk bits.  Only fp16
// swaps (a quantised one needs the codec) after a tensor-core step; the launcher decides whether
// its epilogue can (PeerTarget::honored), else the runtime falls back to mode_swap.
bool fused_swap_target(const Plan& p, size_t i, int cur, PeerTarget& pt) {
  if (i + 1 >= p.steps.size() || !fused_swap_enabled(p)) return false;
  if (getenv("TN_NO_EPILOGUE_SWAP")) return false;  // test knob (read per call): the peer-pass swap only
  const StemStep& st = p.steps[i];
  const StemStep& nx = p.steps[i + 1];
  if (!nx.swap || nx.quant || p.cfg.dtype != TN_CHALF || !st.tensor_core || st.split || st.sparse || st.fold > 1)
    return false;
  if (!(st.out_identity || st.out_transposed) || p.peer_stem.size() != 2u * p.world) return false;
  if (nx.send_layout.size() != st.out_layout.size()) return false;
  const SwapMembers sm(p, nx);
  if (sm.sx > 3) return false;
  memset(&pt, 0, sizeof(pt));
  pt.nsw = sm.sx;
  const int L = (int)st.out_layout.size();
  for (int t = 0; t < sm.sx; ++t) {
    const auto it = std::find(st.out_layout.begin(), st.out_layout.end(), nx.swap_in[t]);
    if (it == st.out_layout.end()) return false;
    const int64_t stride = (int64_t)1 << (L - 1 - (int)(it - st.out_layout.begin()));
    int is_n = -1, bit = -1;
    for (int j = 0; j < st.mlog; ++j)
      if (st.m_stride[j] == stride) is_n = 0, bit = j;
    for (int j = 0; j < st.nlog; ++j)
      if (st.n_stride[j] == stride) is_n = 1, bit = j;
    if (is_n < 0) return false;
    pt.is_n[t] = is_n;
    pt.bit[t] = bit;
    pt.vbit[t] = sm.sx - 1 - t;
  }
  const uint64_t chunk_bytes = (4ull << L) >> sm.sx;  // complex-half
  for (int v = 0; v < (1 << sm.sx); ++v)
    pt.base[v] = static_cast<unsigned char*>(p.peer_stem[2 * sm.peer_of(v) + (1 - cur)]) + (uint64_t)sm.me * chunk_bytes;
  return true;
}

struct Scratch {
  float* max_slot;    // [S+2]   max |real| of the stem entering step i (float bits via atomicMax)
  float* b_bound;     // [S+2]
  uint32_t* b_max;    // [S+2]
  float* redo_in;     // [S+2]   input max of the scale re-run of step i (-1: not needed)
  int* exps;          // [n_exp_slots]
  uint32_t* entry_max;
  uint64_t bytes;
};

Scratch scratch_of(const Plan& p, unsigned char* W) {
  Scratch s;
  size_t S = p.steps.size();
  unsigned char* base = W + p.ws_scratch;
  s.max_slot = reinterpret_cast<float*>(base);
  s.b_bound = s.max_slot + (S + 2);
  s.b_max = reinterpret_cast<uint32_t*>(s.b_bound + (S + 2));
  s.redo_in = reinterpret_cast<float*>(s.b_max + (S + 2));
  s.exps = reinterpret_cast<int*>(s.redo_in + (S + 2));
  s.entry_max = reinterpret_cast<uint32_t*>(s.exps + p.n_exp_slots);
  s.bytes = p.ws_total - p.ws_scratch;
  return s;
}

// strided complex64 view of a node for a given slice
struct View {
  const float2* base;
  SliceOff so{};                  // sliced-leaf offset, resolved on the device from the slice id
  std::vector<int> labels;
  std::vector<int64_t> strides;
  int64_t stride_of(int l) const {
    for (size_t i = 0; i < labels.size(); ++i)
      if (labels[i] == l) return strides[i];
    return -1;
  }
};

// A node's tensor as strides over its labels.  A sliced leaf's offset (slicing fixes the
// sliced labels) is resolved on the device from the slice id in the workspace (SliceOff).
View view_of(const Plan& p, int id, unsigned char* W) {
  View v;
  const Node& n = p.nodes[id];
  if (n.kind == NODE_LEAF) {
    const Leaf& lf = p.leaves[id];
    int r = (int)lf.labels.size();
    v.so.slice = reinterpret_cast<const uint64_t*>(W + p.ws_slice);
    for (int i = 0; i < r; ++i) {
      int l = lf.labels[i];
      int64_t st = 1ll << (r - 1 - i);
      auto it = std::find(p.sliced.begin(), p.sliced.end(), l);
      if (it != p.sliced.end()) {
        int j = (int)(it - p.sliced.begin());
        if (j < 64) {  // bits >= 64 of a slice id are 0 (C-A27)
          if (v.so.n >= 8) throw TnError{TN_E_UNSUPPORTED, "leaf with more than 8 sliced labels"};
          v.so.bit[v.so.n] = j;
          v.so.stride[v.so.n] = st;
          v.so.n++;
        }
      } else {
        v.labels.push_back(l);
        v.strides.push_back(st);
      }
    }
    v.base = reinterpret_cast<const float2*>(W + lf.ws_off);
  } else {
    int r = (int)n.labels.size();
    v.labels = n.labels;
    for (int i = 0; i < r; ++i) v.strides.push_back(1ll << (r - 1 - i));
    v.base = reinterpret_cast<const float2*>(W + n.ws_off);
  }
  return v;
}

ContractArgs common_args(const Plan& p, int id, unsigned char* W);

// The common phase level by level (one launch per tree level; TN_COMMON_SERIAL=1: one launch per
// contraction, the round-1 form).  The argument tables live in a library-owned device buffer built
// once per workspace, before any capture (prepare_common).
void prepare_common(Plan& p, unsigned char* W) {
  if (p.common_dev && p.common_key == W) return;
  if (p.common_dev) cudaFree(p.common_dev);
  p.common_dev = nullptr;
  p.common_level_nodes.clear();
  p.common_level_blocks.clear();
  p.common_level_args.clear();
  p.common_level_start.clear();
  std::vector<int> level(p.nodes.size(), 0);
  int maxl = -1;
  for (int id : p.common_order) {  // children before parents
    const Node& n = p.nodes[id];
    int l = 0;
    for (int c : {n.u, n.v})
      if (c >= 0 && p.nodes[c].kind == NODE_COMMON) l = std::max(l, level[c] + 1);
    level[id] = l;
    maxl = std::max(maxl, l);
  }
  std::vector<unsigned char> host;
  for (int l = 0; l <= maxl; ++l) {
    std::vector<ContractArgs> args;
    std::vector<uint32_t> start(1, 0);
    for (int id : p.common_order)
      if (level[id] == l) {
        args.push_back(common_args(p, id, W));
        const uint64_t n = 1ull << args.back().n_out;
        const uint64_t nb = std::min<uint64_t>((n + 255) / 256, 148 * 16);
        start.push_back(start.back() + (uint32_t)nb);
      }
    auto put = [&](const void* src, size_t bytes) {
      const uint64_t off = (host.size() + 255) / 256 * 256;
      host.resize(off + bytes);
      memcpy(host.data() + off, src, bytes);
      return off;
    };
    p.common_level_nodes.push_back((int)args.size());
    p.common_level_blocks.push_back(start.back());
    p.common_level_args.push_back(put(args.data(), args.size() * sizeof(ContractArgs)));
    p.common_level_start.push_back(put(start.data(), start.size() * sizeof(uint32_t)));
  }
  if (!host.empty()) {
    TN_CUDA(cudaMalloc(&p.common_dev, host.size()));
    TN_CUDA(cudaMemcpy(p.common_dev, host.data(), host.size(), cudaMemcpyHostToDevice));
  }
  p.common_key = W;
}

void run_common(const Plan& p, unsigned char* W, cudaStream_t s) {
  static const bool serial = getenv("TN_COMMON_SERIAL") != nullptr;  // A/B knob
  if (!serial && p.common_dev && p.common_key == W) {
    const unsigned char* d = static_cast<const unsigned char*>(p.common_dev);
    for (size_t l = 0; l < p.common_level_nodes.size(); ++l)
      launch_contract_c64_level(reinterpret_cast<const ContractArgs*>(d + p.common_level_args[l]),
                                reinterpret_cast<const uint32_t*>(d + p.common_level_start[l]),
                                p.common_level_nodes[l], p.common_level_blocks[l], s);
    return;
  }
  for (int id : p.common_order) launch_contract_c64(common_args(p, id, W), s);
}

ContractArgs common_args(const Plan& p, int id, unsigned char* W) {
  {
    const Node& n = p.nodes[id];
    View a = view_of(p, n.u, W), b = view_of(p, n.v, W);
    ContractArgs args;
    memset(&args, 0, sizeof(args));
    args.a = a.base;
    args.b = b.base;
    args.sa = a.so;
    args.sb = b.so;
    args.c = reinterpret_cast<float2*>(W + n.ws_off);
    args.n_out = (int)n.labels.size();
    if (args.n_out > kMaxModes) throw TnError{TN_E_UNSUPPORTED, "common contraction with too many modes"};
    for (int j = 0; j < args.n_out; ++j) {
      int l = n.labels[args.n_out - 1 - j];
      int64_t sa = a.stride_of(l), sb = b.stride_of(l);
      args.out_sa[j] = sa < 0 ? 0 : sa;
      args.out_sb[j] = sb < 0 ? 0 : sb;
    }
    int nr = 0;
    for (size_t i = 0; i < a.labels.size(); ++i) {
      int64_t sb = b.stride_of(a.labels[i]);
      if (sb >= 0) {
        if (nr >= kMaxModes) throw TnError{TN_E_UNSUPPORTED, "too many reduced modes"};
        args.red_sa[nr] = a.strides[i];
        args.red_sb[nr] = sb;
        ++nr;
      }
    }
    args.n_red = nr;
    return args;
  }
}

// Sparse-tail step: the branch is dense over its sparse legs; block b of its operand is
// the branch with those legs fixed to the bits of b (MSB = first leg), i.e. a slice of it.  All
// blocks share one power-of-two scale (the max over every block), so the batched GEMM has one
// exponent per step.
// The step's permutation folded into an MN-major A operand (StemStep::mn): decided the same way for
// the operand preparation (B') and the launch (no permutation pass, launch_gemm_chalf_mn).
// Output address map of a stem step (the whole step, or one chunk of a split tail: mshift > 0)
OutMap step_outmap(const StemStep& st, int mshift) {
  const int mlog = st.mlog - mshift;
  OutMap om;
  memset(&om, 0, sizeof(om));
  om.identity = st.out_identity ? 1 : 0;
  om.transposed = (st.out_transposed && mshift == 0) ? 1 : 0;
  om.mbits = mlog;
  om.nbits = st.nlog;
  for (int j = 0; j < mlog; ++j) om.ms[j] = st.m_stride[j];
  for (int j = 0; j < st.nlog; ++j) om.ns[j] = st.n_stride[j];
  return om;
}

bool mn_active(const Plan& p, const StemStep& st) {
  if (!st.mn || p.cfg.dtype != TN_CHALF || !st.tensor_core || st.split || st.sparse) return false;
  const OutMap om = step_outmap(st, 0);
  return mn_gemm_supported(1ull << st.mlog, 1u << st.klog, 1u << st.nlog, st.mn_ma, &om, st.mn_kl, st.mn_mm);
}

void prepare_b_sparse(const Plan& p, const StemStep& st, size_t i, unsigned char* W, const Scratch& sc, cudaStream_t s) {
  View v = view_of(p, st.branch, W);
  const int nsp = (int)st.b_sparse.size();
  const uint64_t nb = 1ull << nsp, kn = 1ull << (st.klog + st.nlog);
  const uint64_t tmp_blk = align_up(8 * kn, 1024);
  for (uint64_t bv = 0; bv < nb; ++bv) {
    GatherArgs g;
    memset(&g, 0, sizeof(g));
    int64_t off = 0;
    for (int t = 0; t < nsp; ++t)
      if ((bv >> (nsp - 1 - t)) & 1) off += v.stride_of(st.b_sparse[t]);
    g.src = v.base + off;
    g.ss = v.so;
    g.dst = reinterpret_cast<float2*>(W + st.b_tmp_off + bv * tmp_blk);
    g.klog = st.klog;
    g.nlog = st.nlog;
    for (int j = 0; j < st.klog; ++j) g.sk[j] = v.stride_of(st.R[st.klog - 1 - j]);
    for (int j = 0; j < st.nlog; ++j) g.sn[j] = v.stride_of(st.newl[st.nlog - 1 - j]);
    launch_gather_kn(g, s);
    const_cast<Plan&>(p).launches++;
    if (p.cfg.dtype == TN_CHALF) launch_max_abs_f32(reinterpret_cast<const float*>(g.dst), 2 * kn, &sc.b_max[i], s);
  }
  if (p.cfg.dtype != TN_CHALF) {
    // complex64 path: the blocks are consumed as [K][N] complex64 at b_off + bv * b_blk
    for (uint64_t bv = 0; bv < nb; ++bv) {
      if (st.b_off + bv * st.b_blk != st.b_tmp_off + bv * tmp_blk)
        TN_CUDA(cudaMemcpyAsync(W + st.b_off + bv * st.b_blk, W + st.b_tmp_off + bv * tmp_blk, 8 * kn,
                                cudaMemcpyDeviceToDevice, s));
      launch_colnorm_c64(reinterpret_cast<const float2*>(W + st.b_tmp_off + bv * tmp_blk), st.klog, st.nlog,
                         &sc.b_bound[i], s);
    }
    return;
  }
  for (uint64_t bv = 0; bv < nb; ++bv) {
    unsigned char* bp = W + st.b_off + bv * st.b_blk;
    if (st.nlog < 3) TN_CUDA(cudaMemsetAsync(bp, 0, 64ull << st.klog, s));
    launch_pad_b(reinterpret_cast<__half*>(bp), reinterpret_cast<const float2*>(W + st.b_tmp_off + bv * tmp_blk),
                 st.klog, st.nlog, &sc.b_max[i], &sc.b_bound[i], &sc.exps[1 + 2 * i], s);
    const_cast<Plan&>(p).launches++;
  }
}

void prepare_b(const Plan& p, unsigned char* W, const Scratch& sc, cudaStream_t s) {
  for (size_t i = 0; i < p.steps.size(); ++i) {
    const StemStep& st = p.steps[i];
    if (st.sparse) {
      prepare_b_sparse(p, st, i, W, sc, s);
      continue;
    }
    View v = view_of(p, st.branch, W);
    GatherArgs g;
    memset(&g, 0, sizeof(g));
    g.src = v.base;
    g.ss = v.so;
    g.dst = reinterpret_cast<float2*>(W + st.b_tmp_off);
    g.klog = st.klog;
    g.nlog = st.nlog;
    for (int j = 0; j < st.klog; ++j) g.sk[j] = v.stride_of(st.R[st.klog - 1 - j]);
    for (int j = 0; j < st.nlog; ++j) g.sn[j] = v.stride_of(st.newl[st.nlog - 1 - j]);
    launch_gather_kn(g, s);
    if (p.cfg.dtype != TN_CHALF) {
      launch_colnorm_c64(g.dst, st.klog, st.nlog, &sc.b_bound[i], s);
      const_cast<Plan&>(p).launches++;
    }
    if (p.cfg.dtype == TN_CHALF) {
      const_cast<Plan&>(p).launches += 2;
      uint64_t kn = 1ull << (st.klog + st.nlog);
      if (st.nlog < 3)  // zero the padding rows of B_P (tcgen05 needs N >= 16 real columns)
        TN_CUDA(cudaMemsetAsync(W + st.b_off, 0, 64ull << st.klog, s));
      launch_max_abs_f32(reinterpret_cast<const float*>(g.dst), 2 * kn, &sc.b_max[i], s);
      if (st.fold > 1) {
        __half* scratch = reinterpret_cast<__half*>(W + st.b_off + st.b_fold_bytes);
        if (st.nlog < 3) TN_CUDA(cudaMemsetAsync(scratch, 0, 64ull << st.klog, s));
        launch_pad_b(scratch, g.dst, st.klog, st.nlog, &sc.b_max[i], &sc.b_bound[i], &sc.exps[1 + 2 * i], s);
        launch_fold_b(reinterpret_cast<__half*>(W + st.b_off), scratch, st.klog, st.nlog, st.fold, s);
        const_cast<Plan&>(p).launches++;
      } else if (mn_active(p, st))
        launch_pad_b_mn(reinterpret_cast<__half*>(W + st.b_off), g.dst, st.klog, st.nlog, &sc.b_max[i],
                        &sc.b_bound[i], &sc.exps[1 + 2 * i], s);
      else
        launch_pad_b(reinterpret_cast<__half*>(W + st.b_off), g.dst, st.klog, st.nlog, &sc.b_max[i], &sc.b_bound[i],
                     &sc.exps[1 + 2 * i], s);
    }
  }
}

void check_buffers(const Plan& p, const tn_buffers* b) {
  if (!b) throw TnError{TN_E_INVALID, "buffers is NULL"};
  if (!b->d_ws || b->ws_bytes < p.ws_total)
    throw TnError{TN_E_CAPACITY, "workspace too small: need " + std::to_string(p.ws_total)};
  const int eb = p.cfg.dtype == TN_CHALF ? 4 : 8;
  if (!p.steps.empty() && (!b->d_stem[0] || !b->d_stem[1] || b->stem_bytes < p.stem_elems_max * eb))
    throw TnError{TN_E_CAPACITY, "stem buffers too small: need " + std::to_string(p.stem_elems_max * eb)};
}

// Sharded mode swap before step `st` (Alg. 1 "intra-node communication"; group
// quantisation Eq. 1).  The contracted shard modes (positions swap_out_pos of the shard
// set) trade places with the local modes swap_in: the sender's layout has swap_in outermost, so
// chunk v (the v-th block of those bits) belongs to the group member whose swapped-out bits are v.
// The receiver stores the chunk from member v at slot v, so after the exchange the swapped-out shard
// modes are the outermost local modes.  Only members that differ in the swapped bits talk (partial
// swap, reading C-A17).  int8: each chunk is quantised in groups of comm_group reals (groups never
// straddle chunks), sent as codes + fp32 scale/zero, and dequantised straight into complex-half.
// An fp16 / complex64 mode swap without the transport: the send permutation (or a plain chunk copy)
// writes every member's chunk straight into that member's receive buffer over NVLink peer memory
// (one pass, no NCCL payload); bar_slot = an already reduced max slot whose re-reduction is the
// barrier before (no rank still reads the buffer its peers write) and after (every chunk is in).
// TN_SWAP_NCCL=1 keeps the transport (A/B knob); quantised swaps always use it (the codec).
bool peer_swap_enabled(const Plan& p) {
  const char* e = getenv("TN_SWAP_NCCL");  // A/B and test knob (read per call)
  return fused_swap_enabled(p) && !(e && atoi(e) != 0) && p.peer_stem.size() == 2u * p.world;
}

// The peer-memory swap pass composed with step st's own permutation (st.perm, no MN-major read):
// ONE pass from the sender's layout straight into the receiver's permuted layout.  The sender sees
// the permuted layout with each swapped-out shard mode replaced by the swap_in mode at the same
// position t (V[j] = send_layout[perm_axes[j]]); that bit picks the member (bit sx-1-t of v) and is
// replaced by this rank's own member bit (bit sx-1-t of me), which is where the receiver keeps it.
// Saves the receiver's separate permutation pass (a full local read + write).  Returns false (no
// work done) when the routing bits would fall inside a 16-byte vector or TN_NO_SWAP_COMPOSE is set.
bool mode_swap_composed(Plan& p, const StemStep& st, const tn_buffers* b, int& cur, cudaStream_t s,
                        float* bar_slot) {
  const char* e = getenv("TN_NO_SWAP_COMPOSE");  // A/B knob (read per call)
  if ((e && atoi(e) != 0) || st.quant || !bar_slot || !peer_swap_enabled(p) || !st.perm || mn_active(p, st))
    return false;
  const int eb = p.cfg.dtype == TN_CHALF ? 4 : 8;
  const SwapMembers sm(p, st);
  const int n = (int)st.send_layout.size();
  if (sm.sx < 1 || sm.sx > 3 || (int)st.perm_axes.size() != n) return false;
  // the member bit splits the output into runs of 2^pos elements alternating between destinations:
  // short runs make NVLink stores inefficient (C3 at 2 GPUs: pos = 2, 16-byte runs, the composed
  // pass took 16.5 ms against 11.4 ms for swap pass + permutation pass), so compose only when runs
  // are >= 16 KB (TN_SWAP_COMPOSE_MIN_POS overrides, for tests; >= the 16-byte vector)
  const char* mp = getenv("TN_SWAP_COMPOSE_MIN_POS");
  const int min_pos = std::max(eb == 4 ? 2 : 1, mp ? atoi(mp) : (eb == 4 ? 12 : 11));
  PeerChunks pc;
  memset(&pc, 0, sizeof(pc));
  pc.nsw = sm.sx;
  std::vector<int> axes(n);
  for (int j = 0; j < n; ++j) {
    const int q = st.perm_axes[j];
    axes[j] = st.send_perm ? st.send_perm_axes[q] : q;
    if (q < sm.sx) {
      const int pos = n - 1 - j;
      if (pos < min_pos) return false;
      pc.pos[q] = pos;
      pc.vbit[q] = sm.sx - 1 - q;
      pc.mebit[q] = (sm.me >> (sm.sx - 1 - q)) & 1;
    }
  }
  for (int v = 0; v < (1 << sm.sx); ++v) pc.base[v] = p.peer_stem[2 * sm.peer_of(v) + (1 - cur)];
  if (getenv("TN_DEBUG_COMPOSE")) {
    fprintf(stderr, "compose n=%d sx=%d pos=%d axes(outermost first):", n, sm.sx, pc.pos[0]);
    for (int j = 0; j < n; ++j) fprintf(stderr, " %d", axes[j]);
    fprintf(stderr, "\n");
  }
  xfer_allreduce_max(p, bar_slot, s);
  launch_permute(nullptr, b->d_stem[cur], eb, n, axes.data(), s, &pc);
  ++p.launches;
  xfer_allreduce_max(p, bar_slot, s);
  cur = 1 - cur;
  ++p.n_peer_swaps;
  ++p.n_composed_swaps;
  return true;
}

void mode_swap(Plan& p, const StemStep& st, const tn_buffers* b, int& cur, cudaStream_t s, float* bar_slot) {
  comm_check(p);
  const int eb = p.cfg.dtype == TN_CHALF ? 4 : 8;
  if (!st.quant && bar_slot && peer_swap_enabled(p)) {
    const SwapMembers sm(p, st);
    const uint64_t n_local = 1ull << st.send_layout.size();
    PeerChunks pc;
    memset(&pc, 0, sizeof(pc));
    pc.chunk_bytes = (n_local >> sm.sx) * eb;
    for (int v = 0; v < (1 << sm.sx); ++v)
      pc.base[v] = static_cast<unsigned char*>(p.peer_stem[2 * sm.peer_of(v) + (1 - cur)]) + (uint64_t)sm.me * pc.chunk_bytes;
    std::vector<int> axes;
    if (st.send_perm) {
      axes = st.send_perm_axes;
    } else {
      for (size_t j = 0; j < st.send_layout.size(); ++j) axes.push_back((int)j);
    }
    xfer_allreduce_max(p, bar_slot, s);
    launch_permute(nullptr, b->d_stem[cur], eb, (int)st.send_layout.size(), axes.data(), s, &pc);
    ++p.launches;
    xfer_allreduce_max(p, bar_slot, s);
    cur = 1 - cur;
    ++p.n_peer_swaps;
    return;
  }
  // quantised swaps read the unpermuted stem group by group when the permutation keeps the
  // innermost log2(g/2) modes in place (k_quant.cu group_base): no separate permutation pass
  GroupPerm gp;
  const bool fused = st.fuse_quant &&
                     make_group_perm(gp, (int)st.send_layout.size(), st.send_perm_axes.data(), p.cfg.comm_group);
  if (st.send_perm && !fused) {
    launch_permute(b->d_stem[1 - cur], b->d_stem[cur], eb, (int)st.send_layout.size(), st.send_perm_axes.data(), s);
    ++p.launches;
    cur = 1 - cur;
  }
  const int sx = (int)st.swap_out_pos.size();
  const int S = (int)st.shard_before.size();
  const uint64_t n_local = 1ull << st.send_layout.size();
  const uint64_t chunk = n_local >> sx;  // complex elements per chunk
  // member index of this rank: its bits at the swapped shard positions (position 0 = rank MSB)
  auto bit_of = [&](int r, int pos) { return (r >> (S - 1 - pos)) & 1; };
  int me = 0;
  for (int t = 0; t < sx; ++t) me = (me << 1) | bit_of(p.rank, st.swap_out_pos[t]);
  auto peer_of = [&](int v) {
    int r = p.rank;
    for (int t = 0; t < sx; ++t) {
      int pos = st.swap_out_pos[t], bit = (v >> (sx - 1 - t)) & 1;
      int shift = S - 1 - pos;
      r = (r & ~(1 << shift)) | (bit << shift);
    }
    return r;
  };
  unsigned char* X = static_cast<unsigned char*>(b->d_stem[cur]);
  unsigned char* Y = static_cast<unsigned char*>(b->d_stem[1 - cur]);
  std::vector<Xfer> sends, recvs;
  const bool quant = st.quant;  // lowering: int8/int4 codec, complex-half, late enough in the path
  if (quant) {
    const bool tensor = p.cfg.comm_codec == TN_COMM_INT8_TENSOR;  // Table 1 preset: one group per chunk
    const uint64_t reals = 2 * n_local, creals = 2 * chunk;
    const uint64_t g = tensor ? creals : (uint64_t)p.cfg.comm_group;
    const bool int4 = p.cfg.comm_codec == TN_COMM_INT4;
    if (creals % g) throw TnError{TN_E_INFEASIBLE, "swap chunk is not a multiple of the quantisation group"};
    const uint64_t ng = reals / g, cng = creals / g;
    const uint64_t cbytes = int4 ? creals / 2 : creals;  // code bytes per chunk
    const uint64_t codes_bytes = align_up(int4 ? reals / 2 : reals, 256);
    // codes + scales + zeros live in one stem buffer (the lowering sizes the buffers for it)
    if (codes_bytes + 3 * align_up(8 * ng, 256) > b->stem_bytes)
      throw TnError{TN_E_CAPACITY, "quantised swap payload exceeds the stem buffer"};
    auto codes = [&](unsigned char* base) { return reinterpret_cast<int8_t*>(base); };
    auto scales = [&](unsigned char* base) { return reinterpret_cast<float*>(base + codes_bytes); };
    auto zeros = [&](unsigned char* base) { return reinterpret_cast<float*>(base + codes_bytes + align_up(4 * ng, 256)); };
    if (tensor)
      launch_quant_int8_exp_half(codes(Y), scales(Y), zeros(Y), reinterpret_cast<const __half*>(X), reals, g, 0.2,
                                 reinterpret_cast<uint32_t*>(Y + codes_bytes + 2 * align_up(4 * ng, 256)), s);
    else if (int4)
      launch_quant_int4_half(reinterpret_cast<uint8_t*>(codes(Y)), scales(Y), zeros(Y), reinterpret_cast<const __half*>(X),
                             reals, (int)g, s, fused ? &gp : nullptr);
    else
      launch_quant_int8_half(codes(Y), scales(Y), zeros(Y), reinterpret_cast<const __half*>(X), reals, (int)g, s,
                             fused ? &gp : nullptr);
    for (int v = 0; v < (1 << sx); ++v) {
      if (v == me) continue;
      int peer = peer_of(v);
      sends.push_back({peer, codes(Y) + v * cbytes, cbytes});
      sends.push_back({peer, scales(Y) + v * cng, 4 * cng});
      sends.push_back({peer, zeros(Y) + v * cng, 4 * cng});
      recvs.push_back({peer, codes(X) + v * cbytes, cbytes});
      recvs.push_back({peer, scales(X) + v * cng, 4 * cng});
      recvs.push_back({peer, zeros(X) + v * cng, 4 * cng});
    }
    xfer_exchange(p, sends, recvs, s);
    TN_CUDA(cudaMemcpyAsync(codes(X) + me * cbytes, codes(Y) + me * cbytes, cbytes, cudaMemcpyDeviceToDevice, s));
    TN_CUDA(cudaMemcpyAsync(scales(X) + me * cng, scales(Y) + me * cng, 4 * cng, cudaMemcpyDeviceToDevice, s));
    TN_CUDA(cudaMemcpyAsync(zeros(X) + me * cng, zeros(Y) + me * cng, 4 * cng, cudaMemcpyDeviceToDevice, s));
    if (tensor)
      launch_dequant_int8_exp_half(reinterpret_cast<__half*>(Y), codes(X), scales(X), zeros(X), reals, g, 0.2, s);
    else if (int4)
      launch_dequant_int4_half(reinterpret_cast<__half*>(Y), reinterpret_cast<const uint8_t*>(codes(X)), scales(X),
                               zeros(X), reals, (int)g, s);
    else
      launch_dequant_int8_half(reinterpret_cast<__half*>(Y), codes(X), scales(X), zeros(X), reals, (int)g, s);
    p.launches += 2;
  } else {
    const uint64_t cb = chunk * eb;  // bytes per chunk
    for (int v = 0; v < (1 << sx); ++v) {
      if (v == me) continue;
      int peer = peer_of(v);
      sends.push_back({peer, X + (uint64_t)v * cb, cb});
      recvs.push_back({peer, Y + (uint64_t)v * cb, cb});
    }
    xfer_exchange(p, sends, recvs, s);
    TN_CUDA(cudaMemcpyAsync(Y + (uint64_t)me * cb, X + (uint64_t)me * cb, cb, cudaMemcpyDeviceToDevice, s));
  }
  cur = 1 - cur;
}

void rec_event(Plan& p, size_t k, cudaStream_t s) {
  if (!p.timing) return;
  // under stream capture an External record becomes an event-record node (every replay records it)
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  TN_CUDA(cudaStreamIsCapturing(s, &cs));
  if (cs == cudaStreamCaptureStatusActive)
    TN_CUDA(cudaEventRecordWithFlags((cudaEvent_t)p.ev[k], s, cudaEventRecordExternal));
  else
    TN_CUDA(cudaEventRecord((cudaEvent_t)p.ev[k], s));
}

// One stem GEMM (Eq. 6 on tcgen05, SIMT for small K*N, complex64 SIMT for the fp32 path) from
// `src` to `dst`; mshift > 0 runs it on one chunk of the split tail (the top mshift m bits fixed).
int redo_bits() {
  // 18: below that the lost headroom costs nothing.  The output is stored in fp16 with its realised
  // max at 2^(14-d) (d = bits lost) and the next step rescales from that max; only values under
  // fp16's normal floor 2^-14 (subnormal spacing 2^-24) lose relative precision, i.e. values below
  // max * 2^(d-28).  At d < 18 their absolute error is <= 2^-20 of the max, 2^-18 of the rms of a
  // Porter-Thomas-like tensor (max ~ 4.6 rms): < 1 % of fp16's own 2^-11 rounding (reading C-A28).
  // (10 re-ran C3 step 31, m16 k16 n5, whose random-phase sum over 2^16 terms sits ~2^8 under the
  // 1-norm bound: +5 ms per subtask for nothing.)
  static const int b = getenv("TN_REDO_BITS") ? atoi(getenv("TN_REDO_BITS")) : 18;
  return b;
}

void run_gemm_once(Plan& p, const StemStep& st, size_t i, const void* src, void* dst, int mshift, const float* in_max,
                   uint32_t* out_max, int* exp_slot, unsigned char* W, const Scratch& sc, cudaStream_t s,
                   PeerTarget* peer = nullptr);

// One stem GEMM plus its scale re-run (complex-half: redo_check + the same launch, which exits at once
// unless the realised output max lost more than TN_REDO_BITS (default 18) bits of fp16 headroom).
// collective (sharded main path): every rank must scale by the same power of two, so the realised max is
// all-reduced before the re-run decision, which every rank then takes alike (per-rank split-tail
// chains pass false).
void run_gemm(Plan& p, const StemStep& st, size_t i, const void* src, void* dst, int mshift, const float* in_max,
              uint32_t* out_max, int* exp_slot, unsigned char* W, const Scratch& sc, cudaStream_t s,
              bool collective = false, PeerTarget* peer = nullptr) {
  run_gemm_once(p, st, i, src, dst, mshift, in_max, out_max, exp_slot, W, sc, s, peer);
  const bool coll = collective && p.world > 1;  // both dtypes scale by powers of two (C-A8)
  // (a fused swap: this all-reduce is also the barrier after which every rank's peer stores are in)
  if (coll) xfer_allreduce_max(p, reinterpret_cast<float*>(out_max), s);
  if (p.cfg.dtype != TN_CHALF || !in_max || redo_bits() <= 0) return;
  launch_redo_check(out_max, in_max, &sc.redo_in[i], redo_bits(), s);  // also sets the re-run's max
  run_gemm_once(p, st, i, src, dst, mshift, &sc.redo_in[i], nullptr, exp_slot, W, sc, s, peer);
  ++p.launches;
  // a re-run rewrites the peers' boxes: barrier again (an all-reduce of the already reduced max)
  if (coll && peer && peer->honored) xfer_allreduce_max(p, reinterpret_cast<float*>(out_max), s);
}

void run_gemm_once(Plan& p, const StemStep& st, size_t i, const void* src, void* dst, int mshift, const float* in_max,
                   uint32_t* out_max, int* exp_slot, unsigned char* W, const Scratch& sc, cudaStream_t s,
                   PeerTarget* peer) {
  const int mlog = st.mlog - mshift;
  const uint64_t M = 1ull << mlog;
  const uint32_t K = 1u << st.klog, N = 1u << st.nlog;
  OutMap om = step_outmap(st, mshift);
  if (peer) peer->honored = 0;
  om.peer = mshift == 0 ? peer : nullptr;
  if (p.cfg.dtype == TN_CHALF) {
    AGather ag;
    if (st.gather_a) {  // the step's permutation, fused into the A load (mshift == 0: not a split step)
      memset(&ag, 0, sizeof(ag));
      ag.mlog = st.mlog;
      ag.klog = st.klog;
      for (int j = 0; j < st.mlog; ++j) ag.ms[j] = st.a_m_stride[j];
      for (int j = 0; j < st.klog; ++j) ag.ks[j] = st.a_k_stride[j];
    }
    if (mshift == 0 && st.fold > 1) {
      // row folding: [M/f][f 2K] x blockdiag(B_P) -> [M/f][f 2N], the same row-major bytes
      OutMap fo = identity_map(M / st.fold, (uint32_t)st.fold * N);
      fo.peer = nullptr;
      fo.fold_t = st.out_transposed ? st.fold : 0;  // (f = 2, N = 16: epilogue mode 6)
      launch_gemm_chalf_tc(reinterpret_cast<__half*>(dst), reinterpret_cast<const __half*>(src),
                           reinterpret_cast<const __half*>(W + st.b_off), M / st.fold, st.fold * 2 * K,
                           st.fold * 2 * N, in_max, &sc.b_bound[i], out_max, exp_slot, &fo, s, nullptr);
    } else if (mshift == 0 && mn_active(p, st))
      launch_gemm_chalf_mn(reinterpret_cast<__half*>(dst), reinterpret_cast<const __half*>(src),
                           reinterpret_cast<const __half*>(W + st.b_off), M, K, N, st.mn_ma, in_max, &sc.b_bound[i],
                           out_max, exp_slot, &om, s, st.mn_kl, st.mn_mm);
    else if (st.tensor_core)
      launch_gemm_chalf_tc(reinterpret_cast<__half*>(dst), reinterpret_cast<const __half*>(src),
                           reinterpret_cast<const __half*>(W + st.b_off), M, 2 * K, 2 * N, in_max, &sc.b_bound[i],
                           out_max, exp_slot, &om, s, st.gather_a ? &ag : nullptr);
    else
      launch_gemm_chalf_simt(reinterpret_cast<__half2*>(dst), reinterpret_cast<const __half2*>(src),
                             reinterpret_cast<const __half*>(W + st.b_off), M, K, N, in_max, &sc.b_bound[i], out_max,
                             exp_slot, &om, s);
  } else {
    launch_gemm_c64(reinterpret_cast<float2*>(dst), reinterpret_cast<const float2*>(src),
                    reinterpret_cast<const float2*>(W + st.b_off), M, K, N, &om, s, in_max, &sc.b_bound[i], out_max,
                    exp_slot);
  }
  ++p.launches;
}

// The subtask body: every launch after the slice id is in the workspace.  Nothing here depends on
// the slice id on the host, so one capture of it serves every slice (stem_contract).
// head = everything before the first collective (scratch reset, common phase, operand prep, the
// rank-local stem entry conversion); tail = the rest.  Sharded plans capture only the head.
void stem_body(Plan& p, const tn_buffers* b, cudaStream_t s, bool head = true, bool tail = true) {
  unsigned char* W = static_cast<unsigned char*>(b->d_ws);
  Scratch sc = scratch_of(p, W);
  if (head) {
    rec_event(p, 0, s);
    TN_CUDA(cudaMemsetAsync(W + p.ws_scratch, 0, sc.bytes, s));
    run_common(p, W, s);
    static const bool serial = getenv("TN_COMMON_SERIAL") != nullptr;
    p.launches += (!serial && p.common_dev && p.common_key == W) ? p.common_level_nodes.size() : p.common_order.size();
  }
  p.result_in_ws = p.steps.empty();
  if (p.steps.empty()) return;
  const int eb = p.cfg.dtype == TN_CHALF ? 4 : 8;
  if (head) {
  prepare_b(p, W, sc, s);
  p.launches += p.steps.size() + 2;  // gathers + entry conversion (max + convert)
  // stem entry -> buffer 0
  {
    const Node& e = p.nodes[p.stem_entry];
    uint64_t n = 1ull << e.labels.size();
    const uint64_t n_local = n >> p.shard_log2;  // this rank's shard: shard modes are outermost
    const float2* src;
    if (e.kind == NODE_LEAF) {
      View v = view_of(p, p.stem_entry, W);
      GatherArgs g;
      memset(&g, 0, sizeof(g));
      g.src = v.base;
      g.ss = v.so;
      g.dst = reinterpret_cast<float2*>(b->d_stem[1]);  // scratch use of the other buffer
      g.klog = 0;
      g.nlog = (int)v.labels.size();
      for (int j = 0; j < g.nlog; ++j) g.sn[j] = v.strides[g.nlog - 1 - j];
      if (n * 8 > b->stem_bytes) throw TnError{TN_E_CAPACITY, "stem entry leaf exceeds stem buffer"};
      launch_gather_kn(g, s);
      src = g.dst;
    } else {
      src = reinterpret_cast<const float2*>(W + e.ws_off);
    }
    if (p.cfg.dtype == TN_CHALF) {
      if (e.kind == NODE_LEAF) {
        // convert in place is impossible across buffers of different element size: go through ws
        throw TnError{TN_E_UNSUPPORTED, "complex-half stem entry at a leaf: raise stem_min_log2"};
      }
      // the exponent comes from the whole entry tensor (identical on every rank)
      launch_max_abs_f32(reinterpret_cast<const float*>(src), 2 * n, sc.entry_max, s);
      launch_c64_to_chalf(reinterpret_cast<__half2*>(b->d_stem[0]), src + (uint64_t)p.rank * n_local, n_local,
                          sc.entry_max, &sc.exps[0], reinterpret_cast<uint32_t*>(&sc.max_slot[0]), s);
    } else {
      launch_max_abs_f32(reinterpret_cast<const float*>(src), 2 * n, sc.entry_max, s);
      launch_c64_scale(reinterpret_cast<float2*>(b->d_stem[0]), src + (uint64_t)p.rank * n_local, n_local,
                       sc.entry_max, &sc.exps[0], reinterpret_cast<uint32_t*>(&sc.max_slot[0]), s);
    }
  }
  }
  if (!tail) return;
  // every rank scales the first step by the same power of two
  if (p.world > 1) xfer_allreduce_max(p, &sc.max_slot[0], s);
  int cur = 0;
  rec_event(p, 1, s);
  const size_t n_main = !p.split_modes.empty() ? (size_t)p.split_from
                                               : (p.sparse_from >= 0 ? (size_t)p.sparse_from : p.steps.size());
  bool swapped = false;  // the swap before step i was done by step i-1's epilogue
  p.n_fused_swaps = 0;
  p.n_peer_swaps = 0;
  p.n_composed_swaps = 0;
  for (size_t i = 0; i < n_main; ++i) {
    const StemStep& st = p.steps[i];
    bool composed = false;  // the swap pass also did this step's permutation
    if (st.swap && !swapped) {
      composed = mode_swap_composed(p, st, b, cur, s, &sc.max_slot[i]);
      if (!composed) mode_swap(p, st, b, cur, s, &sc.max_slot[i]);
    }
    swapped = false;
    if (p.step_kern.size() != p.steps.size()) {
      p.step_kern.assign(p.steps.size(), "");
      p.step_pass.assign(p.steps.size(), 0);
    }
    p.step_pass[i] = st.perm && !mn_active(p, st);
    if (st.perm && !mn_active(p, st) && !composed) {
      launch_permute(b->d_stem[1 - cur], b->d_stem[cur], eb, (int)st.in_layout.size(), st.perm_axes.data(), s);
      ++p.launches;
      cur = 1 - cur;
    }
    // the swap before step i+1 inside this GEMM's epilogue (fp16, NVLink peer stores): first a
    // barrier (an all-reduce of the already reduced input max) after which no rank still reads the
    // buffer its peers are about to write
    PeerTarget pt;
    const bool fuse = i + 1 < n_main && fused_swap_target(p, i, cur, pt);
    if (fuse) xfer_allreduce_max(p, &sc.max_slot[i], s);
    rec_event(p, 2 + 2 * i, s);
    // (sharded: the max all-reduces inside make every rank scale the next step identically)
    g_last_kern = "";
    run_gemm(p, st, i, b->d_stem[cur], b->d_stem[1 - cur], 0, &sc.max_slot[i],
             reinterpret_cast<uint32_t*>(&sc.max_slot[i + 1]), &sc.exps[2 + 2 * i], W, sc, s, true,
             fuse ? &pt : nullptr);
    p.step_kern[i] = g_last_kern;
    cur = 1 - cur;
    if (fuse && pt.honored) {
      swapped = true;
      ++p.n_fused_swaps;
    }
    rec_event(p, 3 + 2 * i, s);
  }
  if (!p.split_modes.empty()) {
    // entering the split tail: its first permutation (split modes outermost) runs on the whole stem
    const StemStep& st = p.steps[p.split_from];
    if (st.perm) {
      launch_permute(b->d_stem[1 - cur], b->d_stem[cur], eb, (int)st.in_layout.size(), st.perm_axes.data(), s);
      ++p.launches;
      cur = 1 - cur;
    }
    p.stem_cur = cur;
    return;  // the chunked tail runs in tn_split_contract
  }
  p.stem_cur = cur;
  if (p.sparse_from >= 0) return;  // the sparse-state tail runs in tn_sample_amplitudes (needs the prefixes)
  if (p.final_perm) {
    launch_permute(b->d_stem[1 - cur], b->d_stem[cur], eb, (int)p.final_layout.size(), p.final_perm_axes.data(), s);
    ++p.launches;
    cur = 1 - cur;
  }
  rec_event(p, 2 + 2 * p.steps.size(), s);
  p.ev_valid = p.timing != 0;
  p.result_buf = cur;
  p.result_off = 0;
}

bool graph_wanted(const Plan& p) {
  static const bool env_off = getenv("TN_NO_GRAPH") != nullptr;
  return !env_off && !p.graph_off;
}

// Sharded plans keep only the collective-free head in the graph; TN_GRAPH_NCCL=1 (experiment knob)
// captures the whole subtask, NCCL swaps and max all-reduces included (stream-capturable once
// NCCL's connections exist, so the first call runs eagerly).  Measured slower on C3 (2 GPUs: 59.2
// vs 55.6 ms/subtask; 4 GPUs: 41.6 vs 34.0), hence off.
bool graph_whole(const Plan& p) {
  static const char* e = getenv("TN_GRAPH_NCCL");
  static const bool on = e != nullptr && atoi(e) != 0;
  return p.world == 1 || on;
}

// Capture stem_body on the library stream and instantiate it (once per buffer set).
void capture_stem(Plan& p, const tn_buffers* b) {
  if (!p.cap_stream) {
    cudaStream_t cs;
    TN_CUDA(cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking));
    p.cap_stream = (void*)cs;
  }
  if (p.graph_exec) {
    cudaGraphExecDestroy((cudaGraphExec_t)p.graph_exec);
    p.graph_exec = nullptr;
  }
  cudaStream_t cs = (cudaStream_t)p.cap_stream;
  p.launches = 0;
  TN_CUDA(cudaStreamBeginCapture(cs, cudaStreamCaptureModeThreadLocal));
  try {
    stem_body(p, b, cs, true, graph_whole(p));  // else (sharded): the collective-free head only
  } catch (...) {
    cudaGraph_t junk = nullptr;
    cudaStreamEndCapture(cs, &junk);
    if (junk) cudaGraphDestroy(junk);
    throw;
  }
  cudaGraph_t g = nullptr;
  TN_CUDA(cudaStreamEndCapture(cs, &g));
  cudaGraphExec_t ex = nullptr;
  cudaError_t e = cudaGraphInstantiate(&ex, g, 0);
  cudaGraphDestroy(g);
  TN_CUDA(e);
  p.graph_exec = (void*)ex;
  p.graph_key[0] = b->d_ws;
  p.graph_key[1] = b->d_stem[0];
  p.graph_key[2] = b->d_stem[1];
  p.graph_stem_bytes = b->stem_bytes;
  p.graph_timing = p.timing;
  p.graph_launches = p.launches;
  p.graph_stem_cur = p.stem_cur;
  p.graph_result_buf = p.result_buf;
}

// One sliced subtask (P:318 slicing; P:8-22 the stem path).  The slice id goes to the device first
// (one tiny kernel), then the body runs eagerly or as a replay of its CUDA graph: the common phase
// alone is hundreds of small launches whose CPU cost would otherwise not shrink with more GPUs.
void stem_contract(Plan& p, const tn_buffers* b, uint64_t slice_id, cudaStream_t s) {
  select_device(p);
  check_buffers(p, b);
  p.tail_slots.clear();  // a new stem: any earlier tail result is stale
  if (p.world > 1 && !p.comm) throw TnError{TN_E_INVALID, "plan lowered for several ranks without a communicator"};
  if (p.sliced.size() < 64 && slice_id >= (1ull << p.sliced.size()))
    throw TnError{TN_E_INVALID, "slice_id >= 2^|sliced|"};
  unsigned char* W = static_cast<unsigned char*>(b->d_ws);
  p.ev_valid = false;
  if (p.timing && p.ev.empty()) {
    p.ev.resize(3 + 2 * p.steps.size());
    for (auto& e : p.ev) {
      cudaEvent_t ce;
      TN_CUDA(cudaEventCreate(&ce));
      e = (void*)ce;
    }
  }
  launch_set_u64(reinterpret_cast<uint64_t*>(W + p.ws_slice), slice_id, s);
  if (fused_swap_enabled(p) && p.n_swaps > 0) ensure_peers(p, b, s);  // outside any capture
  prepare_common(p, W);
  if (graph_wanted(p)) {
    const bool same = p.graph_exec && p.graph_key[0] == b->d_ws && p.graph_key[1] == b->d_stem[0] &&
                      p.graph_key[2] == b->d_stem[1] && p.graph_stem_bytes == b->stem_bytes && p.graph_timing == p.timing;
    if (!same && p.world > 1 && graph_whole(p) && !p.nccl_warm) {
      // first sharded call: eager, so NCCL sets up its peer connections outside any capture
      p.launches = 0;
      stem_body(p, b, s);
      p.launches += 1;
      p.nccl_warm = true;
      return;
    }
    if (!same) capture_stem(p, b);
    TN_CUDA(cudaGraphLaunch((cudaGraphExec_t)p.graph_exec, s));
    p.launches = p.graph_launches + 1;
    if (p.world > 1 && !graph_whole(p)) {  // the tail (swaps, GEMMs) eagerly on the caller's stream
      stem_body(p, b, s, false, true);
      return;
    }
    p.stem_cur = p.graph_stem_cur;
    p.result_buf = p.graph_result_buf;
    p.result_off = 0;
    p.result_in_ws = p.steps.empty();
    p.ev_valid = p.timing != 0 && p.split_modes.empty() && p.sparse_from < 0;  // the graph records the same events
    return;
  }
  p.launches = 0;
  stem_body(p, b, s);
  p.launches += 1;
}

// Split-type tail ("dividing the stem tensor into smaller chunks", P:22 chunks inside the
// double buffers, P:526 chunk count from capacity).  The split modes are the outermost modes of
// every tail layout, so chunk v is the contiguous slab v of each tail tensor: chunk v's input is
// read in place from the stem buffer, its intermediates ping-pong between two chunk regions at the
// start of the other buffer, and its result lands in slot v of a result region behind them.  Each
// chunk keeps its own max/exponent chain (the first tail step starts from the global bound).
// ids == nullptr: every chunk, result slot v = chunk v.  Otherwise only the listed chunks (the
// sparse-state batch of P:525-537: only the requested prefixes are contracted), slot i = ids[i].
void split_contract(Plan& p, const tn_buffers* b, cudaStream_t s, const std::vector<uint64_t>* ids = nullptr) {
  if (p.split_modes.empty()) return;
  select_device(p);
  check_buffers(p, b);
  unsigned char* W = static_cast<unsigned char*>(b->d_ws);
  Scratch sc = scratch_of(p, W);
  const int eb = p.cfg.dtype == TN_CHALF ? 4 : 8;
  const int j = (int)p.split_modes.size();
  const uint64_t chunks = 1ull << j, T = p.steps.size() - p.split_from, cmax = p.split_chunk_max;
  const uint64_t nsel = ids ? ids->size() : chunks;
  if (nsel > chunks) throw TnError{TN_E_INVALID, "more prefixes than chunks"};
  if (ids)
    for (uint64_t v : *ids)
      if (v >= chunks) throw TnError{TN_E_INVALID, "prefix out of range"};
  p.tail_slots.assign(nsel, 0);
  for (uint64_t i = 0; i < nsel; ++i) p.tail_slots[i] = ids ? (*ids)[i] : i;
  const uint64_t chunk_in = 1ull << (p.steps[p.split_from].in_layout.size() - j);
  const uint64_t chunk_out = 1ull << (p.final_layout.size() - j);
  // the chunk intermediates ping-pong between region RA at the start of the free buffer and region RB
  // behind the tail's input in the stem buffer (which every chunk reads in place); the result slots
  // follow RA.  Each buffer then holds at most one chunk-sized intermediate, so halving the tail
  // (recomputation) halves the peak bytes per buffer.
  const uint64_t in_bytes = align_up(chunks * chunk_in * eb, 1024);
  if ((cmax + chunks * chunk_out) * eb > b->stem_bytes || in_bytes + cmax * eb > b->stem_bytes)
    throw TnError{TN_E_CAPACITY, "split tail: chunk regions do not fit the stem buffers"};
  unsigned char* X = static_cast<unsigned char*>(b->d_stem[p.stem_cur]);
  unsigned char* Y = static_cast<unsigned char*>(b->d_stem[1 - p.stem_cur]);
  unsigned char* RA = Y;
  unsigned char* RB = X + in_bytes;
  unsigned char* RES = Y + cmax * eb;
  float* cmaxs = reinterpret_cast<float*>(sc.entry_max + 1);   // [chunks][T+1]
  int* cexps = reinterpret_cast<int*>(cmaxs + chunks * (T + 1));  // [chunks][T]
  // timing: the whole chunked tail is attributed to the final interval of the report
  for (uint64_t t = 0; t < T; ++t) {
    rec_event(p, 2 + 2 * (p.split_from + t), s);
    rec_event(p, 3 + 2 * (p.split_from + t), s);
  }
  // fresh per-slot scale chains (the tail may run again for a sparse-state batch)
  TN_CUDA(cudaMemsetAsync(cmaxs, 0, 4 * chunks * (2 * T + 1), s));
  for (uint64_t sl = 0; sl < nsel; ++sl) {
    const uint64_t v = p.tail_slots[sl];  // chunk id; `sl` indexes the result slot and scratch
    unsigned char* current = X + v * chunk_in * eb;
    for (uint64_t t = 0; t < T; ++t) {
      const size_t i = p.split_from + t;
      const StemStep& st = p.steps[i];
      if (st.perm && t > 0) {  // (the first tail step's permutation ran on the whole stem)
        unsigned char* dst = (current == RA) ? RB : RA;
        std::vector<int> axes;
        for (size_t a = j; a < st.perm_axes.size(); ++a) axes.push_back(st.perm_axes[a] - j);
        launch_permute(dst, current, eb, (int)st.in_layout.size() - j, axes.data(), s);
        ++p.launches;
        current = dst;
      }
      unsigned char* dst = (t + 1 == T) ? RES + sl * chunk_out * eb : ((current == RA) ? RB : RA);
      const float* in_max = t == 0 ? &sc.max_slot[i] : &cmaxs[sl * (T + 1) + t];
      run_gemm(p, st, i, current, dst, j, in_max, reinterpret_cast<uint32_t*>(&cmaxs[sl * (T + 1) + t + 1]),
               &cexps[sl * T + t], W, sc, s);
      current = dst;
    }
  }
  rec_event(p, 2 + 2 * p.steps.size(), s);
  p.ev_valid = p.timing != 0;
  p.result_buf = 1 - p.stem_cur;
  p.result_off = cmax;
}

// ---- sparse-state tail (Fig. 5) ----
// Per tail step t: the distinct values (keys) that the sparse legs held after the step take among
// the requested subspaces; output entry c = key c; A entry index_a[c] = c's key restricted to the legs
// held before the step; B block index_b[c] = c's bits on the branch's sparse legs.
struct SparseStep {
  std::vector<uint64_t> keys;     // sorted prefix values masked to the legs held after the step
  std::vector<int32_t> ia, ib;
  uint64_t n_in = 1;              // entries of the step's input
};

std::vector<SparseStep> sparse_schedule(const Plan& p, const std::vector<uint64_t>& pre) {
  const int L = (int)p.sparse_legs.size();
  auto leg_bit = [&](int label) {
    const int t = (int)(std::find(p.sparse_legs.begin(), p.sparse_legs.end(), label) - p.sparse_legs.begin());
    return L - 1 - t;  // prefix bit of sparse leg t (MSB first)
  };
  std::vector<SparseStep> out;
  uint64_t mask = 0;
  std::vector<uint64_t> prev_keys{0};
  for (size_t i = p.sparse_from; i < p.steps.size(); ++i) {
    const StemStep& st = p.steps[i];
    for (int l : st.b_sparse) mask |= 1ull << leg_bit(l);
    SparseStep ss;
    ss.n_in = prev_keys.size();
    for (uint64_t v : pre) ss.keys.push_back(v & mask);
    std::sort(ss.keys.begin(), ss.keys.end());
    ss.keys.erase(std::unique(ss.keys.begin(), ss.keys.end()), ss.keys.end());
    const uint64_t prev_mask = mask & ~[&] {
      uint64_t m = 0;
      for (int l : st.b_sparse) m |= 1ull << leg_bit(l);
      return m;
    }();
    for (uint64_t c : ss.keys) {
      const uint64_t a = c & prev_mask;
      ss.ia.push_back((int32_t)(std::lower_bound(prev_keys.begin(), prev_keys.end(), a) - prev_keys.begin()));
      int32_t bidx = 0;
      for (int l : st.b_sparse) bidx = (bidx << 1) | (int32_t)((c >> leg_bit(l)) & 1);
      ss.ib.push_back(bidx);
    }
    prev_keys = ss.keys;
    out.push_back(std::move(ss));
  }
  return out;
}

uint64_t pow2_at_least(uint64_t n) {
  uint64_t r = 1;
  while (r < n) r <<= 1;
  return r;
}

// Bytes of the free stem buffer one chunk of subspaces needs: two ping-pong regions (each the largest
// tail tensor, permutation passes run on a power-of-two batch) + the index arrays + the top-1 slots.
uint64_t sparse_need(const Plan& p, const std::vector<SparseStep>& sch, uint64_t& region, uint64_t& idx_off) {
  const int eb = p.cfg.dtype == TN_CHALF ? 4 : 8;
  uint64_t r = 0, nidx = 0;
  for (size_t t = 0; t < sch.size(); ++t) {
    const StemStep& st = p.steps[p.sparse_from + t];
    const uint64_t n_in = st.perm ? pow2_at_least(sch[t].n_in) : sch[t].n_in;
    r = std::max(r, n_in << st.in_layout.size());
    r = std::max(r, (uint64_t)sch[t].keys.size() << st.out_layout.size());
    nidx += 2 * sch[t].keys.size();
  }
  region = align_up(r * eb, 1024);
  idx_off = 2 * region;
  return idx_off + align_up(4 * nidx, 256) + 8 * (sch.empty() ? 1 : sch.back().keys.size()) + 256;
}

// Runs the sparse-state tail for the subspaces `pre` (in chunks of subspaces when the free stem
// buffer cannot hold the whole batch: "the number of chunks is determined by the current
// remaining capacity") and reads their amplitudes + post-selected members.
void sparse_tail(Plan& p, const tn_buffers* b, const uint64_t* prefixes, size_t n_sub, double* h_amps, int k,
                 uint64_t* top_idx, cudaStream_t s) {
  select_device(p);
  check_buffers(p, b);
  const int L = (int)p.sparse_legs.size();
  for (size_t i = 0; i < n_sub; ++i)
    if (L < 64 && (prefixes[i] >> L) != 0) throw TnError{TN_E_INVALID, "prefix has bits beyond the sparse legs"};
  unsigned char* W = static_cast<unsigned char*>(b->d_ws);
  Scratch sc = scratch_of(p, W);
  const int eb = p.cfg.dtype == TN_CHALF ? 4 : 8;
  const size_t t0 = (size_t)p.sparse_from, T = p.steps.size() - t0;
  unsigned char* X = static_cast<unsigned char*>(b->d_stem[p.stem_cur]);
  unsigned char* Y = static_cast<unsigned char*>(b->d_stem[1 - p.stem_cur]);
  // distinct subspaces, sorted: the chunks cut this list
  std::vector<uint64_t> uniq(prefixes, prefixes + n_sub);
  std::sort(uniq.begin(), uniq.end());
  uniq.erase(std::unique(uniq.begin(), uniq.end()), uniq.end());
  int jc = 0;
  for (;; ++jc) {
    const uint64_t c = 1ull << jc, per = (uniq.size() + c - 1) / c;
    bool fits = true;
    for (uint64_t q = 0; q < c && fits; ++q) {
      const uint64_t lo = q * per, hi = std::min<uint64_t>(uniq.size(), lo + per);
      if (lo >= hi) continue;
      uint64_t region, idx;
      std::vector<uint64_t> part(uniq.begin() + lo, uniq.begin() + hi);
      fits = sparse_need(p, sparse_schedule(p, part), region, idx) <= b->stem_bytes;
    }
    if (fits) break;
    if (c >= uniq.size()) throw TnError{TN_E_CAPACITY, "sparse tail: one subspace does not fit the free stem buffer"};
  }
  p.sparse_chunks = 1ull << jc;
  p.sparse_flops = 0;
  // members: the open legs without the sparse legs, `open` order; stored in the final dense layout
  std::vector<int> mord;
  for (int l : p.open)
    if (std::find(p.sparse_legs.begin(), p.sparse_legs.end(), l) == p.sparse_legs.end()) mord.push_back(l);
  const std::vector<int>& lay = p.final_layout;
  const int r = (int)lay.size();
  if ((int)mord.size() != r) throw TnError{TN_E_INVALID, "internal: sparse result layout does not cover the members"};
  const uint64_t members = 1ull << r;
  std::vector<int> bitpos(r);
  for (int t = 0; t < r; ++t) bitpos[t] = r - 1 - (int)(std::find(lay.begin(), lay.end(), mord[t]) - lay.begin());
  MemberMap mm;
  mm.r = r;
  for (int t = 0; t < r; ++t) mm.src_bit[t] = (int8_t)bitpos[t];
  const uint64_t c = 1ull << jc, per = (uniq.size() + c - 1) / c;
  std::vector<double> amp_of(2 * members * uniq.size());
  std::vector<uint64_t> top_of(uniq.size());
  for (uint64_t q = 0; q < c; ++q) {
    const uint64_t lo = q * per, hi = std::min<uint64_t>(uniq.size(), lo + per);
    if (lo >= hi) continue;
    std::vector<uint64_t> part(uniq.begin() + lo, uniq.begin() + hi);
    const std::vector<SparseStep> sch = sparse_schedule(p, part);
    uint64_t region, idx_off;
    sparse_need(p, sch, region, idx_off);
    unsigned char* RA = Y;
    unsigned char* RB = Y + region;
    // index arrays: staged on the host, one copy (the stream orders it before the GEMMs)
    std::vector<int32_t> hidx;
    std::vector<uint64_t> ia_off(T), ib_off(T);
    for (size_t t = 0; t < T; ++t) {
      ia_off[t] = hidx.size();
      hidx.insert(hidx.end(), sch[t].ia.begin(), sch[t].ia.end());
      ib_off[t] = hidx.size();
      hidx.insert(hidx.end(), sch[t].ib.begin(), sch[t].ib.end());
    }
    int32_t* didx = reinterpret_cast<int32_t*>(Y + idx_off);
    TN_CUDA(cudaMemcpyAsync(didx, hidx.data(), 4 * hidx.size(), cudaMemcpyHostToDevice, s));
    // fresh tail scale chain for this chunk (the stem entering the tail keeps its max slot)
    // (every tail GEMM rewrites its exponent slot 2 + 2i; the B_P slots 1 + 2i stay from the head)
    TN_CUDA(cudaMemsetAsync(&sc.max_slot[t0 + 1], 0, 4 * T, s));
    const unsigned char* cur = X;
    for (size_t t = 0; t < T; ++t) {
      const size_t i = t0 + t;
      const StemStep& st = p.steps[i];
      const uint64_t n_in = sch[t].n_in, n_out = sch[t].keys.size();
      unsigned char* other = (cur == RA) ? RB : RA;
      if (st.perm) {  // the same permutation of every entry: batch bits outermost, untouched
        const int nb = (int)std::log2((double)pow2_at_least(n_in));
        std::vector<int> axes;
        for (int a = 0; a < nb; ++a) axes.push_back(a);
        for (int a : st.perm_axes) axes.push_back(a + nb);
        launch_permute(other, cur, eb, nb + (int)st.in_layout.size(), axes.data(), s);
        ++p.launches;
        cur = other;
        other = (cur == RA) ? RB : RA;
      }
      const uint64_t M = 1ull << st.mlog;
      const uint32_t K = 1u << st.klog, N = 1u << st.nlog;
      p.sparse_flops += 8.0 * (double)n_out * (double)M * K * N;
      const float* in_max = &sc.max_slot[i];
      uint32_t* out_max = reinterpret_cast<uint32_t*>(&sc.max_slot[i + 1]);
      int* exp_slot = &sc.exps[2 + 2 * i];
      const bool batched = p.cfg.dtype == TN_CHALF && st.tensor_core && M % 128 == 0 && N >= 8 && K >= 4;
      // scale re-run (run_gemm): the whole batched step again when the realised max lost too many bits
      for (int pass = 0; pass < (p.cfg.dtype == TN_CHALF && redo_bits() > 0 ? 2 : 1); ++pass) {
      if (pass == 1) {
        launch_redo_check(out_max, &sc.max_slot[i], &sc.redo_in[i], redo_bits(), s);
        in_max = &sc.redo_in[i];
        out_max = nullptr;  // redo_check already holds the re-run's max
      }
      if (batched) {
        BatchSpec bs;
        bs.ia = didx + ia_off[t];
        bs.ib = didx + ib_off[t];
        bs.n_out = n_out;
        bs.n_a = n_in;
        bs.n_b = 1ull << st.b_sparse.size();
        launch_gemm_chalf_tc_batched(reinterpret_cast<__half*>(other), reinterpret_cast<const __half*>(cur),
                                     reinterpret_cast<const __half*>(W + st.b_off), M, 2 * K, 2 * N, in_max,
                                     &sc.b_bound[i], out_max, exp_slot, bs, s);
        ++p.launches;
      } else if (p.cfg.dtype == TN_CHALF) {
        // small steps (K < 4, N < 8, < 128 rows per entry): one batched SIMT launch
        launch_gemm_chalf_batched_simt(reinterpret_cast<__half2*>(other), reinterpret_cast<const __half2*>(cur),
                                       reinterpret_cast<const __half*>(W + st.b_off), M, K, N, n_out,
                                       didx + ia_off[t], didx + ib_off[t], st.b_blk / 2, in_max, &sc.b_bound[i],
                                       out_max, exp_slot, s);
        ++p.launches;
      } else {
        // complex64: one GEMM per entry (identical scale inputs, so every entry writes the same exponent)
        OutMap om = identity_map(M, N);
        for (uint64_t e = 0; e < n_out; ++e) {
          const unsigned char* a = cur + (uint64_t)sch[t].ia[e] * (M * K) * eb;
          const unsigned char* bb = W + st.b_off + (uint64_t)sch[t].ib[e] * st.b_blk;
          unsigned char* cc = other + e * (M * N) * eb;
          if (p.cfg.dtype == TN_CHALF) {
            if (st.tensor_core)
              launch_gemm_chalf_tc(reinterpret_cast<__half*>(cc), reinterpret_cast<const __half*>(a),
                                   reinterpret_cast<const __half*>(bb), M, 2 * K, 2 * N, in_max, &sc.b_bound[i], out_max,
                                   exp_slot, &om, s);
            else
              launch_gemm_chalf_simt(reinterpret_cast<__half2*>(cc), reinterpret_cast<const __half2*>(a),
                                     reinterpret_cast<const __half*>(bb), M, K, N, in_max, &sc.b_bound[i], out_max,
                                     exp_slot, &om, s);
          } else {
            launch_gemm_c64(reinterpret_cast<float2*>(cc), reinterpret_cast<const float2*>(a),
                            reinterpret_cast<const float2*>(bb), M, K, N, &om, s, in_max, &sc.b_bound[i], out_max,
                            exp_slot);
          }
          ++p.launches;
        }
      }
      }
      cur = other;
    }
    // read this chunk: amplitudes, exponents, post-selection
    const uint64_t n_last = sch.back().keys.size();
    uint64_t* d_top = reinterpret_cast<uint64_t*>(Y + align_up(idx_off + 4 * hidx.size(), 256));
    const bool dev_top = p.cfg.dtype == TN_CHALF && top_idx && k == 1;
    if (dev_top) launch_top1_chalf(reinterpret_cast<const __half2*>(cur), n_last, members, mm, d_top, s);
    std::vector<int> ex(p.n_exp_slots);
    TN_CUDA(cudaMemcpyAsync(ex.data(), sc.exps, 4 * ex.size(), cudaMemcpyDeviceToHost, s));
    std::vector<uint64_t> top(n_last);
    if (dev_top) TN_CUDA(cudaMemcpyAsync(top.data(), d_top, 8 * n_last, cudaMemcpyDeviceToHost, s));
    std::vector<double> vals(2 * n_last * members);
    if (p.cfg.dtype == TN_CHALF) {
      std::vector<__half> buf(vals.size());
      TN_CUDA(cudaMemcpyAsync(buf.data(), cur, 2 * buf.size(), cudaMemcpyDeviceToHost, s));
      TN_CUDA(cudaStreamSynchronize(s));
      for (size_t e = 0; e < buf.size(); ++e) vals[e] = (double)__half2float(buf[e]);
    } else {
      std::vector<float> buf(vals.size());
      TN_CUDA(cudaMemcpyAsync(buf.data(), cur, 4 * buf.size(), cudaMemcpyDeviceToHost, s));
      TN_CUDA(cudaStreamSynchronize(s));
      for (size_t e = 0; e < buf.size(); ++e) vals[e] = buf[e];
    }
    int E = 0;
    for (int e : ex) E += e;
    for (uint64_t u = lo; u < hi; ++u) {
      const uint64_t e = (uint64_t)(std::lower_bound(sch.back().keys.begin(), sch.back().keys.end(), uniq[u]) -
                                    sch.back().keys.begin());
      double* out = &amp_of[2 * members * u];
      for (uint64_t o = 0; o < members; ++o) {
        uint64_t g = 0;
        for (int t = 0; t < r; ++t)
          if ((o >> (r - 1 - t)) & 1) g |= 1ull << bitpos[t];
        out[2 * o] = std::ldexp(vals[2 * (e * members + g)], -E);
        out[2 * o + 1] = std::ldexp(vals[2 * (e * members + g) + 1], -E);
      }
      top_of[u] = dev_top ? top[e] : 0;
    }
  }
  for (size_t i = 0; i < n_sub; ++i) {
    const uint64_t u = (uint64_t)(std::lower_bound(uniq.begin(), uniq.end(), prefixes[i]) - uniq.begin());
    memcpy(h_amps + 2 * members * i, &amp_of[2 * members * u], 16 * members);
    if (top_idx && k > 0) {
      if (k == 1 && p.cfg.dtype == TN_CHALF) {
        top_idx[i] = top_of[u];
      } else {
        const double* a = h_amps + 2 * members * i;
        std::vector<uint64_t> idx(members);
        for (uint64_t m = 0; m < members; ++m) idx[m] = m;
        auto prob = [&](uint64_t m) {
          const double pr = a[2 * m] * a[2 * m] + a[2 * m + 1] * a[2 * m + 1];
          return pr == pr ? pr : -1.0;
        };
        std::stable_sort(idx.begin(), idx.end(), [&](uint64_t x, uint64_t y) { return prob(x) > prob(y); });
        for (int q = 0; q < k && (uint64_t)q < members; ++q) top_idx[i * k + q] = idx[q];
      }
    }
  }
}

// Result readout (a.8 + a.9), synchronous.  The result block of every rank (sharded: gathered in
// rank order into the workspace) is read to the host, each amplitude is unscaled exactly by its
// accumulated power-of-two exponent (global steps + its split chunk's own chain, C-A8), and the
// amplitudes are reordered from the storage layout into member order.
//   ids == nullptr (dense): all 2^n_open amplitudes in `open` order (every chunk of a split tail).
//   ids (sparse-state batch, Fig. 5): the requested correlated subspaces are prefix values
//   of the split legs; only those chunks of the tail are contracted; n_sub blocks of 2^(n_open - j)
//   members (open legs without the split legs, `open` order).
// top_idx: k most probable members per block, ties -> the smaller member index (C-A23): k = 1 on
// the device for a single-rank complex-half batch, else on the host.
void read_result(Plan& p, const tn_buffers* b, cudaStream_t s, const std::vector<uint64_t>* ids, double* h_amps,
                 int k, uint64_t* top_idx) {
  unsigned char* W = static_cast<unsigned char*>(b->d_ws);
  const int eb = p.cfg.dtype == TN_CHALF ? 4 : 8;
  const bool split = !p.split_modes.empty();
  if (ids && !split)
    throw TnError{TN_E_UNSUPPORTED, "sparse-state batch needs a split plan (cfg.split_log2 = prefix legs)"};
  if (split) {
    if (ids) {
      split_contract(p, b, s, ids);
    } else {  // dense readout needs every chunk in its own slot (a sparse batch may have run last)
      bool all = p.tail_slots.size() == (1ull << p.split_modes.size());
      for (size_t i = 0; all && i < p.tail_slots.size(); ++i) all = p.tail_slots[i] == i;
      if (!all) split_contract(p, b, s);
    }
  }
  const int j = (int)p.split_modes.size(), R = (int)p.world;
  const uint64_t chunks = 1ull << j, T = split ? p.steps.size() - p.split_from : 0;
  const uint64_t nsel = ids ? ids->size() : 1;  // result blocks (slots) per rank
  // storage layout of one block: split tail -> the final layout without the split legs
  std::vector<int> lay(p.final_layout.begin() + (ids ? j : 0), p.final_layout.end());
  if (p.final_perm) lay = p.open;  // (one rank, no split) the last pass wrote `open` order
  if (!ids && split) {  // slot v = chunk v: split legs (chunk order) outermost
    lay.assign(p.split_modes.begin(), p.split_modes.end());
    lay.insert(lay.end(), p.final_layout.begin() + j, p.final_layout.end());
  }
  const uint64_t local = 1ull << lay.size();  // elements per block and rank
  const unsigned char* res = static_cast<const unsigned char*>(b->d_stem[p.result_buf]) + p.result_off * eb;
  Scratch sc = scratch_of(p, W);
  const int* cexp = reinterpret_cast<const int*>(reinterpret_cast<const float*>(sc.entry_max + 1) + chunks * (T + 1));
  const uint64_t ncexp = ids ? nsel * T : chunks * T;  // per-slot exponents (slot-major)
  // members: global layout = rank bits (final_shard) ++ lay; member order = `open` minus split legs
  std::vector<int> glay = p.final_shard;
  glay.insert(glay.end(), lay.begin(), lay.end());
  std::vector<int> mord;
  for (int l : p.open)
    if (!ids || std::find(p.split_modes.begin(), p.split_modes.end(), l) == p.split_modes.end()) mord.push_back(l);
  const int r = (int)glay.size();
  if ((int)mord.size() != r) throw TnError{TN_E_INVALID, "internal: result layout does not cover the output legs"};
  std::vector<int> bitpos(r);  // member bit (r-1-t) <- layout bit bitpos[t]
  for (int t = 0; t < r; ++t)
    bitpos[t] = r - 1 - (int)(std::find(glay.begin(), glay.end(), mord[t]) - glay.begin());
  std::vector<uint64_t> top_dev;
  const bool dev_top = ids && top_idx && k == 1 && p.cfg.dtype == TN_CHALF && R == 1;
  if (dev_top) {
    // behind the per-chunk scale chains in the split scratch (the stem must stay intact: a later
    // dense readout re-runs the tail from it)
    uintptr_t top_addr = reinterpret_cast<uintptr_t>(reinterpret_cast<const float*>(sc.entry_max + 1) +
                                                     chunks * (2 * T + 1));
    uint64_t* d_top = reinterpret_cast<uint64_t*>((top_addr + 7) & ~(uintptr_t)7);
    MemberMap mm;
    mm.r = r;
    for (int t = 0; t < r; ++t) mm.src_bit[t] = (int8_t)bitpos[t];
    launch_top1_chalf(reinterpret_cast<const __half2*>(res), nsel, local, mm, d_top, s);
    top_dev.resize(nsel);
    TN_CUDA(cudaMemcpyAsync(top_dev.data(), d_top, 8 * nsel, cudaMemcpyDeviceToHost, s));
  }
  if (R > 1) {
    if (nsel * local * R * eb > (uint64_t)eb << p.open.size()) throw TnError{TN_E_CAPACITY, "gather region too small"};
    xfer_allgather(p, res, W + p.ws_gather, nsel * local * eb, s);
    res = W + p.ws_gather;
    if (split) {
      xfer_allgather(p, cexp, W + p.ws_gather_exp, 4 * ncexp, s);
      cexp = reinterpret_cast<const int*>(W + p.ws_gather_exp);
    }
  }
  std::vector<int> ex(p.n_exp_slots), ce(R * ncexp);
  TN_CUDA(cudaMemcpyAsync(ex.data(), sc.exps, 4 * ex.size(), cudaMemcpyDeviceToHost, s));
  if (split) TN_CUDA(cudaMemcpyAsync(ce.data(), cexp, 4 * ce.size(), cudaMemcpyDeviceToHost, s));
  const uint64_t total = R * nsel * local;
  std::vector<double> vals(2 * total);
  if (p.cfg.dtype == TN_CHALF) {
    std::vector<__half> buf(2 * total);
    TN_CUDA(cudaMemcpyAsync(buf.data(), res, 4 * total, cudaMemcpyDeviceToHost, s));
    TN_CUDA(cudaStreamSynchronize(s));
    for (size_t i = 0; i < buf.size(); ++i) vals[i] = (double)__half2float(buf[i]);
  } else {
    std::vector<float> buf(2 * total);
    TN_CUDA(cudaMemcpyAsync(buf.data(), res, 8 * total, cudaMemcpyDeviceToHost, s));
    TN_CUDA(cudaStreamSynchronize(s));
    for (size_t i = 0; i < buf.size(); ++i) vals[i] = buf[i];
  }
  int E = 0;
  for (int e : ex) E += e;
  // exponent of (rank q, slot sl): dense split -> slot = chunk = top j bits of `lay`
  auto chain = [&](int q, uint64_t sl) {
    int e = E;
    for (uint64_t t = 0; t < T; ++t) e += ce[(uint64_t)q * ncexp + sl * T + t];
    return e;
  };
  const uint64_t members = 1ull << r;
  const int lbits = (int)lay.size();
  for (uint64_t sl = 0; sl < nsel; ++sl) {
    double* out = h_amps + 2 * sl * members;
    for (uint64_t o = 0; o < members; ++o) {
      uint64_t g = 0;  // index in the global layout (rank bits, then the block layout)
      for (int t = 0; t < r; ++t)
        if ((o >> (r - 1 - t)) & 1) g |= 1ull << bitpos[t];
      const int q = (int)(g >> lbits);
      const uint64_t li = g & (local - 1);
      const int e = !split ? E : chain(q, ids ? sl : (li >> (lbits - j)));
      const uint64_t src = ((uint64_t)q * nsel + sl) * local + li;
      out[2 * o] = std::ldexp(vals[2 * src], -e);
      out[2 * o + 1] = std::ldexp(vals[2 * src + 1], -e);
    }
    if (top_idx && k > 0) {
      if (!top_dev.empty()) {
        top_idx[sl] = top_dev[sl];
      } else {
        std::vector<uint64_t> idx(members);
        for (uint64_t i = 0; i < members; ++i) idx[i] = i;
        auto prob = [&](uint64_t i) {
          const double pr = out[2 * i] * out[2 * i] + out[2 * i + 1] * out[2 * i + 1];
          return pr == pr ? pr : -1.0;
        };
        std::stable_sort(idx.begin(), idx.end(), [&](uint64_t x, uint64_t y) { return prob(x) > prob(y); });
        for (int q = 0; q < k && (uint64_t)q < members; ++q) top_idx[sl * k + q] = idx[q];
      }
    }
  }
}

}  // namespace

extern "C" {

const char* tn_last_error(void) { return g_err.c_str(); }
int tn_version(void) { return 1; }

int tn_set_device(int device) {
  TN_TRY(TN_CUDA(cudaSetDevice(device)));
}

int tn_plan_load(const char* json, size_t len, const tn_config* cfg, tn_comm* comm, tn_plan** out) {
  if (!json || !out) return fail(TN_E_INVALID, "NULL argument");
  *out = nullptr;
  TN_TRY({
    // virtual_world > 1 without a communicator: lower for that many ranks (host-only inspection
    // of the sharded schedule; such a plan cannot be executed)
    const int vworld = (!comm && cfg && cfg->virtual_world > 1) ? cfg->virtual_world : 1;
    Plan* p = load_plan(json, len, cfg, comm ? comm->world : vworld);
    if (comm) {
      p->comm = comm;
      p->rank = comm->rank;
    }
    *out = new tn_plan{p};
  });
}

int tn_plan_info_get(const tn_plan* h, tn_plan_info* info) {
  if (!h || !info) return fail(TN_E_INVALID, "NULL argument");
  const Plan& p = *h->p;
  memset(info, 0, sizeof(*info));
  info->ws_bytes = p.ws_total;
  info->stem_bytes = p.steps.empty() ? 0 : p.stem_elems_max * (p.cfg.dtype == TN_CHALF ? 4 : 8);
  info->n_slices_log2 = p.sliced.size();
  info->n_stem_steps = p.steps.size();
  info->n_permutes = p.n_permutes + (p.final_perm ? 1 : 0);
  info->n_common = p.common_order.size();
  info->stem_flops = p.stem_flops;
  info->total_flops = p.total_flops;
  info->stem_bytes_alg = p.stem_bytes_alg;
  info->perm_bytes = p.perm_bytes;
  info->n_open = p.open.size();
  info->max_stem_log2 = p.max_stem_log2;
  info->h2d_bytes = p.h2d_bytes;
  info->split_chunks = 1ull << p.split_log2;
  info->n_launches = p.launches;
  info->n_sparse_legs = p.sparse_legs.size();
  return TN_OK;
}

void tn_plan_free(tn_plan* h) {
  if (!h) return;
  if (h->p->pinned) cudaFreeHost(h->p->pinned);
  close_peers(*h->p);
  if (h->p->common_dev) cudaFree(h->p->common_dev);
  if (h->p->graph_exec) cudaGraphExecDestroy((cudaGraphExec_t)h->p->graph_exec);
  if (h->p->cap_stream) cudaStreamDestroy((cudaStream_t)h->p->cap_stream);
  for (void* e : h->p->ev) cudaEventDestroy((cudaEvent_t)e);
  delete h->p;
  delete h;
}

int tn_plan_upload(tn_plan* h, const tn_buffers* b, void* stream) {
  if (!h || !b || !b->d_ws) return fail(TN_E_INVALID, "NULL argument");
  TN_TRY({
    Plan& p = *h->p;
    select_device(p);
    if (b->ws_bytes < p.ws_total) throw TnError{TN_E_CAPACITY, "workspace too small"};
    if (!p.pinned) {
      TN_CUDA(cudaMallocHost(&p.pinned, p.ws_leaves));
      memset(p.pinned, 0, p.ws_leaves);
      for (auto& lf : p.leaves) {
        float* dst = reinterpret_cast<float*>(static_cast<unsigned char*>(p.pinned) + lf.ws_off);
        for (size_t i = 0; i < lf.data.size(); ++i) dst[i] = (float)lf.data[i];
      }
    }
    TN_CUDA(cudaMemcpyAsync(b->d_ws, p.pinned, p.ws_leaves, cudaMemcpyHostToDevice, (cudaStream_t)stream));
  });
}

int tn_stem_contract(tn_plan* h, const tn_buffers* b, uint64_t slice_id, void* stream) {
  if (!h) return fail(TN_E_INVALID, "NULL plan");
  TN_TRY(stem_contract(*h->p, b, slice_id, (cudaStream_t)stream));
}

int tn_split_contract(tn_plan* h, const tn_buffers* b, void* stream) {
  if (!h || !b) return fail(TN_E_INVALID, "NULL argument");
  TN_TRY(split_contract(*h->p, b, (cudaStream_t)stream));  // no-op without a split tail
}

int tn_sample_amplitudes(tn_plan* h, const tn_buffers* b, const uint64_t* prefixes, size_t n_sub, double* h_amps,
                         int k, uint64_t* top_idx, void* stream) {
  if (!h || !b || !h_amps) return fail(TN_E_INVALID, "NULL argument");
  if ((prefixes == nullptr) != (n_sub == 0)) return fail(TN_E_INVALID, "prefixes and n_sub must come together");
  if (k < 0) return fail(TN_E_INVALID, "k < 0");
  TN_TRY({
    Plan& p = *h->p;
    select_device(p);
    cudaStream_t s = (cudaStream_t)stream;
    if (p.sparse_from >= 0) {
      if (!prefixes) throw TnError{TN_E_INVALID, "a sparse-state plan needs the subspace prefixes"};
      sparse_tail(p, b, prefixes, n_sub, h_amps, k, top_idx, s);
      return TN_OK;
    }
    if (prefixes) {
      // prefix bits follow the split legs in `open` order (plan order), whatever order the lowering
      // gave the chunks (split_modes: layout-, policy- and world-dependent): prefix -> chunk id
      const int j = (int)p.split_modes.size();
      std::vector<int> canon;
      for (int l : p.open)
        if (std::find(p.split_modes.begin(), p.split_modes.end(), l) != p.split_modes.end()) canon.push_back(l);
      std::vector<uint64_t> ids(n_sub);
      for (size_t i = 0; i < n_sub; ++i) {
        if (j < 64 && (prefixes[i] >> j) != 0) throw TnError{TN_E_INVALID, "prefix out of range"};
        uint64_t v = 0;
        for (int t = 0; t < j; ++t) {
          const int c = (int)(std::find(canon.begin(), canon.end(), p.split_modes[t]) - canon.begin());
          v = (v << 1) | ((prefixes[i] >> (j - 1 - c)) & 1);
        }
        ids[i] = v;
      }
      read_result(p, b, s, &ids, h_amps, k, top_idx);
      return TN_OK;
    }
    if (!p.result_in_ws) {
      check_buffers(p, b);
      read_result(p, b, s, nullptr, h_amps, k, top_idx);
      return TN_OK;
    }
    // no stem steps: the root is a common-type node in the workspace (complex64, one rank)
    const uint64_t n = 1ull << p.open.size();
    unsigned char* W = static_cast<unsigned char*>(b->d_ws);
    const Node& rt = p.nodes[p.root];
    if (rt.kind == NODE_LEAF) throw TnError{TN_E_UNSUPPORTED, "single-tensor network"};
    std::vector<float> buf(2 * n);
    TN_CUDA(cudaMemcpyAsync(buf.data(), W + rt.ws_off, 8 * n, cudaMemcpyDeviceToHost, s));
    TN_CUDA(cudaStreamSynchronize(s));
    const std::vector<int>& layout = rt.labels;
    const int r = (int)p.open.size();
    std::vector<int> pos(r);
    for (int i = 0; i < r; ++i) pos[i] = (int)(std::find(layout.begin(), layout.end(), p.open[i]) - layout.begin());
    for (uint64_t o = 0; o < n; ++o) {
      uint64_t src = 0;
      for (int i = 0; i < r; ++i)
        if ((o >> (r - 1 - i)) & 1) src |= 1ull << (r - 1 - pos[i]);
      h_amps[2 * o] = buf[2 * src];
      h_amps[2 * o + 1] = buf[2 * src + 1];
    }
    if (top_idx && k > 0) {
      std::vector<uint64_t> idx(n);
      for (uint64_t i = 0; i < n; ++i) idx[i] = i;
      auto prob = [&](uint64_t i) { return h_amps[2 * i] * h_amps[2 * i] + h_amps[2 * i + 1] * h_amps[2 * i + 1]; };
      std::stable_sort(idx.begin(), idx.end(), [&](uint64_t a, uint64_t c) { return prob(a) > prob(c); });
      for (int q = 0; q < k && (uint64_t)q < n; ++q) top_idx[q] = idx[q];
    }
  });
}

int tn_report_json(const tn_plan* h, char* buf, size_t cap, size_t* needed) {
  if (!h) return fail(TN_E_INVALID, "NULL plan");
  TN_TRY({
    const Plan& p = *h->p;
    std::vector<float> ms;
    if (p.ev_valid) {
      TN_CUDA(cudaEventSynchronize((cudaEvent_t)p.ev.back()));
      ms.resize(p.ev.size() - 1);
      for (size_t i = 0; i + 1 < p.ev.size(); ++i)
        TN_CUDA(cudaEventElapsedTime(&ms[i], (cudaEvent_t)p.ev[i], (cudaEvent_t)p.ev[i + 1]));
    }
    std::string s = report_json(p, ms);
    if (needed) *needed = s.size() + 1;
    if (buf && cap) {
      size_t n = std::min(cap - 1, s.size());
      memcpy(buf, s.data(), n);
      buf[n] = 0;
      if (cap < s.size() + 1) throw TnError{TN_E_CAPACITY, "report buffer too small"};
    }
  });
}

int tn_set_timing(tn_plan* h, int enable) {
  if (!h) return fail(TN_E_INVALID, "NULL plan");
  h->p->timing = enable;
  return TN_OK;
}

int tn_set_graph(tn_plan* h, int enable) {
  if (!h) return fail(TN_E_INVALID, "NULL plan");
  h->p->graph_off = !enable;
  return TN_OK;
}

int tn_permute(void* d_dst, const void* d_src, int elem_bytes, int n, const int* perm, void* stream) {
  if (!d_dst || !d_src || (!perm && n > 0)) return fail(TN_E_INVALID, "NULL argument");
  TN_TRY(launch_permute(d_dst, d_src, elem_bytes, n, perm, (cudaStream_t)stream));
}

int tn_gemm_chalf(void* d_c, const void* d_a, const void* d_bp, uint64_t M, uint32_t K, uint32_t N,
                  const float* d_in_max, const float* d_b_bound, uint32_t* d_out_max, int* d_exp, void* stream) {
  if (!d_c || !d_a || !d_bp) return fail(TN_E_INVALID, "NULL argument");
  if (!K || !N || (K & (K - 1)) || (N & (N - 1))) return fail(TN_E_INVALID, "K and N must be powers of two");
  TN_TRY({
    const float* im = (d_in_max && d_b_bound) ? d_in_max : nullptr;
    const float* bb = (d_in_max && d_b_bound) ? d_b_bound : nullptr;
    if (K >= 4)
      launch_gemm_chalf_tc((__half*)d_c, (const __half*)d_a, (const __half*)d_bp, M, 2 * K, 2 * N, im, bb, d_out_max,
                           d_exp, nullptr, (cudaStream_t)stream);
    else
      launch_gemm_chalf_simt((__half2*)d_c, (const __half2*)d_a, (const __half*)d_bp, M, K, N, im, bb, d_out_max,
                             d_exp, nullptr, (cudaStream_t)stream);
  });
}

int tn_gemm_chalf_gather(void* d_c, const void* d_a, const void* d_bp, int mlog, int klog, uint32_t N,
                         const int64_t* m_stride, const int64_t* k_stride, const float* d_in_max,
                         const float* d_b_bound, uint32_t* d_out_max, int* d_exp, void* stream) {
  if (!d_c || !d_a || !d_bp || !m_stride || !k_stride) return fail(TN_E_INVALID, "NULL argument");
  if (mlog < 7 || mlog >= kMaxModes || klog < 3 || klog > 16 || !N || (N & (N - 1)))
    return fail(TN_E_INVALID, "gathered GEMM: need mlog in [7, 48), klog in [3, 16], N a power of two");
  TN_TRY({
    AGather ag;
    memset(&ag, 0, sizeof(ag));
    ag.mlog = mlog;
    ag.klog = klog;
    for (int j = 0; j < mlog; ++j) ag.ms[j] = m_stride[j];
    for (int j = 0; j < klog; ++j) ag.ks[j] = k_stride[j];
    const float* im = (d_in_max && d_b_bound) ? d_in_max : nullptr;
    const float* bb = (d_in_max && d_b_bound) ? d_b_bound : nullptr;
    launch_gemm_chalf_tc((__half*)d_c, (const __half*)d_a, (const __half*)d_bp, 1ull << mlog, 2u << klog, 2 * N, im,
                         bb, d_out_max, d_exp, nullptr, (cudaStream_t)stream, &ag);
  });
}

int tn_gemm_chalf_batched(void* d_c, const void* d_a, const void* d_bp, uint64_t M, uint32_t K, uint32_t N,
                          uint64_t n_out, const int32_t* d_index_a, const int32_t* d_index_b, uint64_t n_a,
                          uint64_t n_b, const float* d_in_max, const float* d_b_bound, uint32_t* d_out_max,
                          int* d_exp, void* stream) {
  if (!d_c || !d_a || !d_bp || !d_index_a || !d_index_b) return fail(TN_E_INVALID, "NULL argument");
  TN_TRY({
    BatchSpec bs;
    bs.ia = d_index_a;
    bs.ib = d_index_b;
    bs.n_out = n_out;
    bs.n_a = n_a;
    bs.n_b = n_b;
    const float* im = (d_in_max && d_b_bound) ? d_in_max : nullptr;
    const float* bb = (d_in_max && d_b_bound) ? d_b_bound : nullptr;
    launch_gemm_chalf_tc_batched((__half*)d_c, (const __half*)d_a, (const __half*)d_bp, M, 2 * K, 2 * N, im, bb,
                                 d_out_max, d_exp, bs, (cudaStream_t)stream);
  });
}

int tn_gemm_chalf_padded(void* d_c, const void* d_a, const void* d_bp, uint64_t M, uint32_t K, uint32_t N,
                         uint64_t n_a, const int32_t* d_table, int m_r, uint64_t n_b, const float* d_in_max,
                         const float* d_b_bound, uint32_t* d_out_max, int* d_exp, void* stream) {
  if (!d_c || !d_a || !d_bp || !d_table) return fail(TN_E_INVALID, "NULL argument");
  if (m_r <= 0) return fail(TN_E_INVALID, "m_r must be positive");
  TN_TRY({
    BatchSpec bs;
    bs.pad_r = m_r;
    bs.table = d_table;
    bs.n_out = n_a;
    bs.n_a = n_a;
    bs.n_b = n_b;
    const float* im = (d_in_max && d_b_bound) ? d_in_max : nullptr;
    const float* bb = (d_in_max && d_b_bound) ? d_b_bound : nullptr;
    launch_gemm_chalf_tc_batched((__half*)d_c, (const __half*)d_a, (const __half*)d_bp, M, 2 * K, 2 * N, im, bb,
                                 d_out_max, d_exp, bs, (cudaStream_t)stream);
  });
}

int tn_gemm_cfloat(void* d_c, const void* d_a, const void* d_b, uint64_t M, uint32_t K, uint32_t N, void* stream) {
  if (!d_c || !d_a || !d_b) return fail(TN_E_INVALID, "NULL argument");
  TN_TRY(launch_gemm_c64((float2*)d_c, (const float2*)d_a, (const float2*)d_b, M, K, N, nullptr, (cudaStream_t)stream));
}

int tn_gemm_chalf_mn(void* d_c, const void* d_a, const void* d_bpm, uint64_t M, uint32_t K, uint32_t N, int ma,
                     const float* d_in_max, const float* d_b_bound, uint32_t* d_out_max, int* d_exp, void* stream) {
  if (!d_c || !d_a || !d_bpm) return fail(TN_E_INVALID, "NULL argument");
  if (!mn_gemm_supported(M, K, N, ma, nullptr)) return fail(TN_E_INVALID, "MN-major GEMM: unsupported geometry");
  TN_TRY({
    const float* im = (d_in_max && d_b_bound) ? d_in_max : nullptr;
    const float* bb = (d_in_max && d_b_bound) ? d_b_bound : nullptr;
    launch_gemm_chalf_mn((__half*)d_c, (const __half*)d_a, (const __half*)d_bpm, M, K, N, ma, im, bb, d_out_max,
                         d_exp, nullptr, (cudaStream_t)stream);
  });
}

int tn_pad_b_mn(void* d_bpm, const void* d_b, uint32_t K, uint32_t N, float* d_b_bound, int* d_exp, void* d_scratch,
                void* stream) {
  if (!d_bpm || !d_b || !d_scratch) return fail(TN_E_INVALID, "NULL argument");
  if (!K || !N || (K & (K - 1)) || (N & (N - 1))) return fail(TN_E_INVALID, "K and N must be powers of two");
  TN_TRY({
    cudaStream_t s = (cudaStream_t)stream;
    int klog = 0, nlog = 0;
    while ((1u << klog) < K) ++klog;
    while ((1u << nlog) < N) ++nlog;
    uint32_t* mx = static_cast<uint32_t*>(d_scratch);
    TN_CUDA(cudaMemsetAsync(mx, 0, 4, s));
    if (d_b_bound) TN_CUDA(cudaMemsetAsync(d_b_bound, 0, 4, s));
    launch_max_abs_f32((const float*)d_b, 2ull * K * N, mx, s);
    launch_pad_b_mn((__half*)d_bpm, (const float2*)d_b, klog, nlog, d_exp ? mx : nullptr, d_b_bound, d_exp, s);
  });
}

int tn_pad_b(void* d_bp, const void* d_b, uint32_t K, uint32_t N, float* d_b_bound, int* d_exp, void* d_scratch,
             void* stream) {
  if (!d_bp || !d_b || !d_scratch) return fail(TN_E_INVALID, "NULL argument");
  if (!K || !N || (K & (K - 1)) || (N & (N - 1))) return fail(TN_E_INVALID, "K and N must be powers of two");
  TN_TRY({
    cudaStream_t s = (cudaStream_t)stream;
    int klog = 0, nlog = 0;
    while ((1u << klog) < K) ++klog;
    while ((1u << nlog) < N) ++nlog;
    uint32_t* mx = static_cast<uint32_t*>(d_scratch);
    TN_CUDA(cudaMemsetAsync(mx, 0, 4, s));
    if (d_b_bound) TN_CUDA(cudaMemsetAsync(d_b_bound, 0, 4, s));
    launch_max_abs_f32((const float*)d_b, 2ull * K * N, mx, s);
    launch_pad_b((__half*)d_bp, (const float2*)d_b, klog, nlog, d_exp ? mx : nullptr, d_b_bound, d_exp, s);
  });
}

int tn_quant_int8(int8_t* d_codes, float* d_scales, float* d_zeros, const float* d_x, uint64_t n, int g, void* stream) {
  if (!d_codes || !d_scales || !d_zeros || !d_x) return fail(TN_E_INVALID, "NULL argument");
  TN_TRY(launch_quant_int8(d_codes, d_scales, d_zeros, d_x, n, g, (cudaStream_t)stream));
}

int tn_dequant_int8(float* d_y, const int8_t* d_codes, const float* d_scales, const float* d_zeros, uint64_t n, int g,
                    void* stream) {
  if (!d_y || !d_codes || !d_scales || !d_zeros) return fail(TN_E_INVALID, "NULL argument");
  TN_TRY(launch_dequant_int8(d_y, d_codes, d_scales, d_zeros, n, g, (cudaStream_t)stream));
}

int tn_quant_int8_f16(int8_t* d_codes, float* d_scales, float* d_zeros, const void* d_x, uint64_t n, int g,
                      void* stream) {
  if (!d_codes || !d_scales || !d_zeros || !d_x) return fail(TN_E_INVALID, "NULL argument");
  TN_TRY(launch_quant_int8_half(d_codes, d_scales, d_zeros, (const __half*)d_x, n, g, (cudaStream_t)stream));
}

int tn_permute_quant_f16(void* d_codes, float* d_scales, float* d_zeros, const void* d_x, int n, const int* perm,
                         int g, int codec, void* stream) {
  if (!d_codes || !d_scales || !d_zeros || !d_x || !perm) return fail(TN_E_INVALID, "NULL argument");
  if (codec != TN_COMM_INT8 && codec != TN_COMM_INT4) return fail(TN_E_INVALID, "codec must be int8 or int4");
  TN_TRY({
    GroupPerm gp;
    if (n < 0 || n > 46) throw TnError{TN_E_INVALID, "permute_quant: rank out of range"};
    std::vector<int> seen(n, 0);
    for (int j = 0; j < n; ++j)
      if (perm[j] < 0 || perm[j] >= n || seen[perm[j]]++) throw TnError{TN_E_INVALID, "permute_quant: not a permutation"};
    if (!make_group_perm(gp, n, perm, g))
      throw TnError{TN_E_INVALID, "permute_quant: g must be a power of two whose innermost log2(g/2) axes stay in place"};
    const uint64_t reals = 2ull << n;
    if (codec == TN_COMM_INT8)
      launch_quant_int8_half((int8_t*)d_codes, d_scales, d_zeros, (const __half*)d_x, reals, g, (cudaStream_t)stream, &gp);
    else
      launch_quant_int4_half((uint8_t*)d_codes, d_scales, d_zeros, (const __half*)d_x, reals, g, (cudaStream_t)stream, &gp);
  });
}

int tn_quant_int8_exp_f16(int8_t* d_codes, float* d_scales, float* d_zeros, const void* d_x, uint64_t n, uint64_t g,
                          double e, void* d_tmp, void* stream) {
  if (!d_codes || !d_scales || !d_zeros || !d_x || !d_tmp) return fail(TN_E_INVALID, "NULL argument");
  TN_TRY(launch_quant_int8_exp_half(d_codes, d_scales, d_zeros, (const __half*)d_x, n, g, e, (uint32_t*)d_tmp,
                                    (cudaStream_t)stream));
}

int tn_dequant_int8_exp_f16(void* d_y, const int8_t* d_codes, const float* d_scales, const float* d_zeros, uint64_t n,
                            uint64_t g, double e, void* stream) {
  if (!d_y || !d_codes || !d_scales || !d_zeros) return fail(TN_E_INVALID, "NULL argument");
  TN_TRY(launch_dequant_int8_exp_half((__half*)d_y, d_codes, d_scales, d_zeros, n, g, e, (cudaStream_t)stream));
}

int tn_quant_int4_f16(uint8_t* d_packed, float* d_scales, float* d_zeros, const void* d_x, uint64_t n, int g,
                      void* stream) {
  if (!d_packed || !d_scales || !d_zeros || !d_x) return fail(TN_E_INVALID, "NULL argument");
  TN_TRY(launch_quant_int4_half(d_packed, d_scales, d_zeros, (const __half*)d_x, n, g, (cudaStream_t)stream));
}

int tn_dequant_int4_f16(void* d_y, const uint8_t* d_packed, const float* d_scales, const float* d_zeros, uint64_t n,
                        int g, void* stream) {
  if (!d_y || !d_packed || !d_scales || !d_zeros) return fail(TN_E_INVALID, "NULL argument");
  TN_TRY(launch_dequant_int4_half((__half*)d_y, d_packed, d_scales, d_zeros, n, g, (cudaStream_t)stream));
}

int tn_dequant_int8_f16(void* d_y, const int8_t* d_codes, const float* d_scales, const float* d_zeros, uint64_t n,
                        int g, void* stream) {
  if (!d_y || !d_codes || !d_scales || !d_zeros) return fail(TN_E_INVALID, "NULL argument");
  TN_TRY(launch_dequant_int8_half((__half*)d_y, d_codes, d_scales, d_zeros, n, g, (cudaStream_t)stream));
}

// ---- NCCL (dlopen'ed: the process's torch already carries libnccl.so.2) ----
typedef struct {
  char internal[128];
} nccl_uid_t;
typedef int (*nccl_get_uid_fn)(nccl_uid_t*);
typedef int (*nccl_init_rank_fn)(void**, int, nccl_uid_t, int);
typedef int (*nccl_destroy_fn)(void*);

int tn_comm_unique_id(uint8_t out[128]) {
  if (!out) return fail(TN_E_INVALID, "NULL argument");
  TN_TRY({
    auto fn = (nccl_get_uid_fn)nccl_sym("ncclGetUniqueId");
    nccl_uid_t id;
    if (fn(&id) != 0) throw TnError{TN_E_NCCL, "ncclGetUniqueId failed"};
    memcpy(out, id.internal, 128);
  });
}

int tn_comm_init(const uint8_t uid[128], int rank, int world, int device, tn_comm** out) {
  if (!uid || !out) return fail(TN_E_INVALID, "NULL argument");
  if (world != 1 && world != 2 && world != 4 && world != 8) return fail(TN_E_UNSUPPORTED, "world must be 1,2,4,8");
  if (rank < 0 || rank >= world) return fail(TN_E_INVALID, "rank out of range");
  TN_TRY({
    TN_CUDA(cudaSetDevice(device));
    tn_comm* c = new tn_comm();
    c->rank = rank;
    c->world = world;
    c->device = device;
    if (world > 1) {
      nccl_init_rank_fn fn = nullptr;
      try {
        fn = (nccl_init_rank_fn)nccl_sym("ncclCommInitRank");
      } catch (...) {
        delete c;
        throw;
      }
      nccl_uid_t id;
      memcpy(id.internal, uid, 128);
      if (fn(&c->nccl_comm, world, id, rank) != 0) {
        delete c;
        throw TnError{TN_E_NCCL, "ncclCommInitRank failed"};
      }
    }
    *out = c;
  });
}

int tn_comm_init_loopback(int world, int device, tn_comm** out) {
  if (!out) return fail(TN_E_INVALID, "NULL argument");
  if (world != 1 && world != 2 && world != 4 && world != 8) return fail(TN_E_UNSUPPORTED, "world must be 1,2,4,8");
  TN_TRY({
    TN_CUDA(cudaSetDevice(device));
    LoopGroup* g = new LoopGroup();
    g->world = world;
    g->device = device;
    g->board.resize(world);
    g->ptr.assign(world, nullptr);
    g->ready.assign(world, nullptr);
    g->done.assign(world, nullptr);
    for (int r = 0; r < world; ++r) {
      TN_CUDA(cudaEventCreateWithFlags(&g->ready[r], cudaEventDisableTiming));
      TN_CUDA(cudaEventCreateWithFlags(&g->done[r], cudaEventDisableTiming));
    }
    for (int r = 0; r < world; ++r) {
      tn_comm* c = new tn_comm();
      c->rank = r;
      c->world = world;
      c->device = device;
      c->loop = g;
      g->refs++;
      out[r] = c;
    }
  });
}

void tn_comm_free(tn_comm* c) {
  if (!c) return;
  if (c->loop) {
    LoopGroup* g = c->loop;
    bool last = false;
    {
      std::lock_guard<std::mutex> lk(g->mu);
      last = --g->refs == 0;
    }
    if (last) {
      for (cudaEvent_t e : g->ready) cudaEventDestroy(e);
      for (cudaEvent_t e : g->done) cudaEventDestroy(e);
      delete g;
    }
    delete c;
    return;
  }
  if (c->nccl_comm) {
    try {
      auto fn = (nccl_destroy_fn)nccl_sym("ncclCommDestroy");
      fn(c->nccl_comm);
    } catch (...) {
    }
  }
  delete c;
}

}  // extern "C"
