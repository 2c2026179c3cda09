// Stem mode permutation ("Tensor contraction involves dimension
// reordering and matrix multiplication").  Y = X.transpose(perm) for a rank-n tensor whose modes
// all have dimension 2, so an element index is an n-bit word and the permutation is a bit
// permutation of the index.
//
// B200 design: HBM-bound (algorithmic bytes = 2 * elem_bytes * 2^n per pass).
//  * leading modes that stay innermost in the same order are folded into a wider element
//    (up to 16 bytes), so pure block moves become 16-byte copies;
//  * each CTA moves tiles of 2^u elements (32 KB) spanning the innermost INPUT bits and the
//    innermost OUTPUT bits (extended alternately until the tile reaches 32 KB, so overlapping
//    inner modes never shrink the tile), staged through shared memory: HBM reads are 16-byte
//    vectors along the input's innermost bits, HBM writes 16-byte vectors along the output's;
//  * stem-sized tensors (permute_pipe_kernel): per-thread offsets in registers, a 3-deep cp.async
//    ring of XOR-swizzled tiles, grid = 148 x 2 persistent CTAs (measured best of 16/32/64 KB
//    tiles x 1-8 CTAs/SM on C3: 32 KB x 2);  tiny tensors: permute_kernel (smem index tables).
#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "common.cuh"

namespace tn {

struct PermArgs2 {
  int n;          // bits of the (folded) index
  int u;          // tile bits
  int vb;         // log2(vector elements): 16-byte vectors
  int64_t tile_in[16];   // input stride of tile bit j (read order: input bits 0..a-1 first)
  int64_t tile_out[16];  // output stride of tile bit j
  int wr_map[16];        // write-order bit k -> read-order tile bit
  int64_t outer_in[64];
  int64_t outer_out[64];
};

// Output routed to the swap members (mode swap through NVLink peer memory, runtime.cu mode_swap):
// output element O (in T units) goes to base[O >> shift] + (O & (2^shift - 1)).
// Bit routing (nsw > 0, the swap pass composed with the next step's permutation): member v's bit
// vbit[t] is O's bit pos[t], which is replaced by mebit[t] (this rank's own member bit).
struct PeerRoute {
  int on, shift, nsw;
  int pos[3], vbit[3], mebit[3];
  unsigned char* base[8];
};

template <typename T>
__device__ __forceinline__ T* route_out(T* dst, const PeerRoute& pr, int64_t o) {
  if (!pr.on) return dst + o;
  if (pr.nsw) {
    int v = 0;
    for (int t = 0; t < pr.nsw; ++t) {
      v |= (int)((o >> pr.pos[t]) & 1) << pr.vbit[t];
      o = (o & ~(1ll << pr.pos[t])) | ((int64_t)pr.mebit[t] << pr.pos[t]);
    }
    return reinterpret_cast<T*>(pr.base[v]) + o;
  }
  return reinterpret_cast<T*>(pr.base[o >> pr.shift]) + (o & ((1ll << pr.shift) - 1));
}

template <typename T>
__global__ void __launch_bounds__(256) permute_kernel(T* __restrict__ dst, const T* __restrict__ src,
                                                      const PermArgs2 args, uint64_t n_tiles,
                                                      const __grid_constant__ PeerRoute pr) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int u = args.u, vb = args.vb;
  const int tsz = 1 << u, nvec = tsz >> vb, V = 1 << vb;
  int64_t* in_tbl = reinterpret_cast<int64_t*>(smem_raw);           // [nvec] input offset of read vector
  int64_t* out_tbl = in_tbl + nvec;                                  // [nvec] output offset of write vector
  uint16_t* wr_tbl = reinterpret_cast<uint16_t*>(out_tbl + nvec);   // [tsz] tile index of write element
  T* tile = reinterpret_cast<T*>(smem_raw + (size_t)nvec * 16 + (((size_t)tsz * 2 + 15) & ~(size_t)15));
  for (int v = threadIdx.x; v < nvec; v += blockDim.x) {
    const int e = v << vb;
    int64_t io = 0;
    for (int j = vb; j < u; ++j)
      if ((e >> j) & 1) io += args.tile_in[j];
    in_tbl[v] = io;
    int64_t oo = 0;
    for (int j = vb; j < u; ++j)
      if ((e >> j) & 1) oo += args.tile_out[args.wr_map[j]];
    out_tbl[v] = oo;
  }
  for (int w = threadIdx.x; w < tsz; w += blockDim.x) {
    int r = 0;
    for (int j = 0; j < u; ++j)
      if ((w >> j) & 1) r |= 1 << args.wr_map[j];
    wr_tbl[w] = (uint16_t)r;
  }
  __syncthreads();
  const int n_outer = args.n - u;
  for (uint64_t t = blockIdx.x; t < n_tiles; t += gridDim.x) {
    int64_t bi = 0, bo = 0;
    for (int j = 0; j < n_outer; ++j)
      if ((t >> j) & 1) {
        bi += args.outer_in[j];
        bo += args.outer_out[j];
      }
    const T* s = src + bi;
    if (V == 1) {
#pragma unroll 4
      for (int v = threadIdx.x; v < nvec; v += blockDim.x) tile[v] = __ldg(s + in_tbl[v]);
    } else {
#pragma unroll 4
      for (int v = threadIdx.x; v < nvec; v += blockDim.x)
        reinterpret_cast<uint4*>(tile)[v] = __ldg(reinterpret_cast<const uint4*>(s + in_tbl[v]));
    }
    __syncthreads();
    if (V == 1) {
#pragma unroll 4
      for (int v = threadIdx.x; v < nvec; v += blockDim.x) *route_out(dst, pr, bo + out_tbl[v]) = tile[wr_tbl[v]];
    } else {
#pragma unroll 2
      for (int v = threadIdx.x; v < nvec; v += blockDim.x) {
        const uint16_t* wt = wr_tbl + (v << vb);
        uint4 x;
        T* xp = reinterpret_cast<T*>(&x);
        for (int j = 0; j < V; ++j) xp[j] = tile[wt[j]];
        *reinterpret_cast<uint4*>(route_out(dst, pr, bo + out_tbl[v])) = x;
      }
    }
    __syncthreads();
  }
}

// Pipelined variant for full 16-byte vectors (the stem-sized case): the tile structure is the same
// for every tile, so each thread keeps its NV read offsets, write offsets and gather indices in
// registers (no smem tables), and tiles stream through a ring of kPermStages shared-memory buffers
// filled by cp.async (LDGSTS, 16 B): kPermStages-1 tiles of reads are in flight while one is written.
constexpr int kPermStages = 3;

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"((uint32_t)__cvta_generic_to_shared(smem)),
               "l"(gmem)
               : "memory");
}

// 16-byte slots of a tile are XOR-swizzled (slot bits 0-2 ^= the XOR of bit triples 3-5, 6-8, 9-11)
// so the write-side gathers, which step through the tile at power-of-two strides, spread over the
// banks whichever tile bits vary across a warp.  Bits >= 3 are unchanged: a bijection.
__device__ __forceinline__ int perm_swz(int v) { return v ^ (((v >> 3) ^ (v >> 6) ^ (v >> 9)) & 7); }

template <typename T, int NV>
__global__ void __launch_bounds__(256) permute_pipe_kernel(T* __restrict__ dst, const T* __restrict__ src,
                                                           const PermArgs2 args, uint64_t n_tiles,
                                                           const __grid_constant__ PeerRoute pr) {
  extern __shared__ __align__(16) uint4 ring[];
  constexpr int V = 16 / sizeof(T);
  const int u = args.u, vb = args.vb;
  const int nvec = (1 << u) >> vb;
  int64_t in_off[NV], out_off[NV];
  uint16_t gi[NV][V];
#pragma unroll
  for (int i = 0; i < NV; ++i) {
    const int v = threadIdx.x + 256 * i;
    const int e = v << vb;
    int64_t io = 0, oo = 0;
    for (int j = vb; j < u; ++j)
      if ((e >> j) & 1) {
        io += args.tile_in[j];
        oo += args.tile_out[args.wr_map[j]];
      }
    in_off[i] = io;
    out_off[i] = oo;
#pragma unroll
    for (int q = 0; q < V; ++q) {
      const int w = e + q;
      int r = 0;
      for (int j = 0; j < u; ++j)
        if ((w >> j) & 1) r |= 1 << args.wr_map[j];
      gi[i][q] = (uint16_t)((perm_swz(r >> vb) << vb) | (r & ((1 << vb) - 1)));
    }
  }
  const int n_outer = args.n - u;
  auto base_of = [&](uint64_t t, int64_t& bi, int64_t& bo) {
    bi = 0;
    bo = 0;
    for (int j = 0; j < n_outer; ++j)
      if ((t >> j) & 1) {
        bi += args.outer_in[j];
        bo += args.outer_out[j];
      }
  };
  auto issue = [&](uint64_t t, int slot) {
    int64_t bi, bo;
    base_of(t, bi, bo);
    uint4* buf = ring + (size_t)slot * nvec;
#pragma unroll
    for (int i = 0; i < NV; ++i) {
      const int v = threadIdx.x + 256 * i;
      if (v < nvec) cp_async16(buf + perm_swz(v), src + bi + in_off[i]);
    }
  };
#pragma unroll
  for (int st = 0; st < kPermStages - 1; ++st) {
    const uint64_t t = blockIdx.x + (uint64_t)st * gridDim.x;
    if (t < n_tiles) issue(t, st);
    asm volatile("cp.async.commit_group;" ::: "memory");
  }
  int slot = 0;
  for (uint64_t t = blockIdx.x; t < n_tiles; t += gridDim.x) {
    const uint64_t t2 = t + (uint64_t)(kPermStages - 1) * gridDim.x;
    if (t2 < n_tiles) issue(t2, (slot + kPermStages - 1) % kPermStages);
    asm volatile("cp.async.commit_group;" ::: "memory");
    asm volatile("cp.async.wait_group %0;" ::"n"(kPermStages - 1) : "memory");
    __syncthreads();
    int64_t bi, bo;
    base_of(t, bi, bo);
    const T* tile = reinterpret_cast<const T*>(ring + (size_t)slot * nvec);
#pragma unroll
    for (int i = 0; i < NV; ++i) {
      const int v = threadIdx.x + 256 * i;
      if (v < nvec) {
        uint4 x;
        T* xp = reinterpret_cast<T*>(&x);
#pragma unroll
        for (int q = 0; q < V; ++q) xp[q] = tile[gi[i][q]];
        *reinterpret_cast<uint4*>(route_out(dst, pr, bo + out_off[i])) = x;
      }
    }
    __syncthreads();
    slot = (slot + 1) % kPermStages;
  }
  asm volatile("cp.async.wait_group 0;" ::: "memory");
}

template <typename T>
static void launch_pipe(void* dst, const void* src, const PermArgs2& args, uint64_t n_tiles, int nvec, cudaStream_t s,
                        const PeerRoute& pr) {
  const size_t smem = (size_t)kPermStages * nvec * 16;
  static bool attr = false;
  if (!attr) {
    TN_CUDA(cudaFuncSetAttribute(permute_pipe_kernel<T, 16>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
    TN_CUDA(cudaFuncSetAttribute(permute_pipe_kernel<T, 8>, cudaFuncAttributeMaxDynamicSharedMemorySize, 112 * 1024));
    TN_CUDA(cudaFuncSetAttribute(permute_pipe_kernel<T, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024));
    TN_CUDA(cudaFuncSetAttribute(permute_pipe_kernel<T, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024));
    TN_CUDA(cudaFuncSetAttribute(permute_pipe_kernel<T, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024));
    attr = true;
  }
  static const int ctas = getenv("TN_PERM_CTAS") ? atoi(getenv("TN_PERM_CTAS")) : 2;  // tuning knob
  const int blocks = (int)std::min<uint64_t>(n_tiles, 148ull * ctas);
  if (nvec > 2048)
    permute_pipe_kernel<T, 16><<<blocks, 256, smem, s>>>((T*)dst, (const T*)src, args, n_tiles, pr);
  else if (nvec > 1024)
    permute_pipe_kernel<T, 8><<<blocks, 256, smem, s>>>((T*)dst, (const T*)src, args, n_tiles, pr);
  else if (nvec > 512)
    permute_pipe_kernel<T, 4><<<blocks, 256, smem, s>>>((T*)dst, (const T*)src, args, n_tiles, pr);
  else if (nvec > 256)
    permute_pipe_kernel<T, 2><<<blocks, 256, smem, s>>>((T*)dst, (const T*)src, args, n_tiles, pr);
  else
    permute_pipe_kernel<T, 1><<<blocks, 256, smem, s>>>((T*)dst, (const T*)src, args, n_tiles, pr);
}

// PeerRoute for element type T from the byte-level routing (chunk_bytes per member, base[v] already
// at this rank's chunk in member v's buffer)
template <typename T>
static PeerRoute route_for(const PeerChunks* pc, int elem_bytes, int vb) {
  PeerRoute r;
  memset(&r, 0, sizeof(r));
  if (!pc) return r;
  r.on = 1;
  if (pc->nsw > 0) {
    int f = 0;  // element bits folded into T
    while ((elem_bytes << f) < (int)sizeof(T)) ++f;
    r.nsw = pc->nsw;
    for (int t = 0; t < pc->nsw; ++t) {
      r.pos[t] = pc->pos[t] - f;
      if (r.pos[t] < vb) throw TnError{TN_E_INVALID, "permute: a routing bit lies inside a 16-byte vector"};
      r.vbit[t] = pc->vbit[t];
      r.mebit[t] = pc->mebit[t];
    }
    for (int v = 0; v < 8; ++v) r.base[v] = static_cast<unsigned char*>(pc->base[v]);
    return r;
  }
  uint64_t c = pc->chunk_bytes / sizeof(T);
  while ((1ull << r.shift) < c) ++r.shift;
  for (int v = 0; v < 8; ++v) r.base[v] = static_cast<unsigned char*>(pc->base[v]);
  return r;
}

void launch_permute(void* dst, const void* src, int elem_bytes, int n, const int* perm, cudaStream_t s,
                    const PeerChunks* pc) {
  if (n < 0 || n > 46) throw TnError{TN_E_INVALID, "permute: rank out of range"};
  if (elem_bytes != 4 && elem_bytes != 8 && elem_bytes != 16)
    throw TnError{TN_E_INVALID, "permute: elem_bytes must be 4, 8 or 16"};
  // q -> p: destination bit position q comes from source bit position p(q)
  std::vector<int> p_of_q(n);
  std::vector<int> seen(n, 0);
  bool ident = true;
  for (int j = 0; j < n; ++j) {
    if (perm[j] < 0 || perm[j] >= n || seen[perm[j]]++) throw TnError{TN_E_INVALID, "permute: not a permutation"};
    if (perm[j] != j) ident = false;
    p_of_q[n - 1 - j] = n - 1 - perm[j];
  }
  const uint64_t total = 1ull << n;
  if (pc && (pc->chunk_bytes & (pc->chunk_bytes - 1)))
    throw TnError{TN_E_INVALID, "permute: member chunks must be powers of two"};
  if (ident && !(pc && pc->nsw > 0)) {
    if (!pc) {
      TN_CUDA(cudaMemcpyAsync(dst, src, total * elem_bytes, cudaMemcpyDeviceToDevice, s));
    } else {
      const uint64_t nc = total * elem_bytes / pc->chunk_bytes;
      for (uint64_t v = 0; v < nc; ++v)
        TN_CUDA(cudaMemcpyAsync(pc->base[v], static_cast<const unsigned char*>(src) + v * pc->chunk_bytes,
                                pc->chunk_bytes, cudaMemcpyDeviceToDevice, s));
    }
    return;
  }
  // fold leading bits that stay in place into a wider element (up to 16 bytes)
  int eb = elem_bytes, nn = n;
  std::vector<int> P = p_of_q;
  while (nn > 0 && P[0] == 0 && eb < 16) {
    eb *= 2;
    std::vector<int> P2(nn - 1);
    for (int q = 1; q < nn; ++q) P2[q - 1] = P[q] - 1;
    P = P2;
    --nn;
  }
  std::vector<int> Q(nn);
  for (int q = 0; q < nn; ++q) Q[P[q]] = q;
  const int vb_full = eb == 4 ? 2 : (eb == 8 ? 1 : 0);  // 16-byte vectors
  const int vb = (nn >= vb_full) ? vb_full : 0;  // tiny tensors: scalar elements
  // tile: input bits 0..a-1 and output bits 0..b-1, extended until 16 KB (or the whole tensor)
  static const int ux = getenv("TN_PERM_UX") ? atoi(getenv("TN_PERM_UX")) : 1;  // tuning knob: tile bits
  const int u_target = std::min(nn, (eb == 4 ? 12 : (eb == 8 ? 11 : 10)) + ux);
  std::vector<char> in_tile(nn, 0);
  std::vector<int> tile_bits;
  int a = 0, b = 0;
  auto add = [&](int x) {
    if (!in_tile[x]) {
      in_tile[x] = 1;
      tile_bits.push_back(x);
    }
  };
  // read order must start with input bits 0..vb-1 and contain output bits 0..vb-1
  for (; a < vb; ++a) add(a);
  for (; b < vb; ++b) add(P[b]);
  while ((int)tile_bits.size() < u_target) {
    if (a < nn && (a <= b || b >= nn)) {
      add(a++);
    } else if (b < nn) {
      add(P[b++]);
    } else {
      break;
    }
  }
  // reorder tile bits: input bits 0..a-1 first in input order (contiguous reads), then the rest
  std::vector<int> rd;
  for (int x = 0; x < nn; ++x)
    if (in_tile[x] && x < a) rd.push_back(x);
  for (int x : tile_bits)
    if (x >= a) rd.push_back(x);
  // the first vb read bits are input bits 0..vb-1 (a >= vb); the first vb write bits are output
  // bits 0..vb-1
  PermArgs2 args;
  memset(&args, 0, sizeof(args));
  args.n = nn;
  args.u = (int)rd.size();
  args.vb = vb;
  if (args.u > 16) throw TnError{TN_E_INVALID, "permute: tile too large"};
  for (int j = 0; j < args.u; ++j) {
    args.tile_in[j] = 1ll << rd[j];
    args.tile_out[j] = 1ll << Q[rd[j]];
  }
  std::vector<int> wr;
  std::vector<char> used(args.u, 0);
  for (int q = 0; q < b; ++q) {
    int idx = (int)(std::find(rd.begin(), rd.end(), P[q]) - rd.begin());
    wr.push_back(idx);
    used[idx] = 1;
  }
  for (int j = 0; j < args.u; ++j)
    if (!used[j]) wr.push_back(j);
  for (int j = 0; j < args.u; ++j) args.wr_map[j] = wr[j];
  int no = 0;
  for (int x = 0; x < nn; ++x)
    if (!in_tile[x]) {
      args.outer_in[no] = 1ll << x;
      args.outer_out[no] = 1ll << Q[x];
      ++no;
    }
  const uint64_t n_tiles = 1ull << (nn - args.u);
  const int tsz = 1 << args.u, nvec = tsz >> vb;
  static const bool legacy = getenv("TN_PERM_LEGACY") != nullptr;  // A/B knob for the old kernel
  if (vb == vb_full && nvec <= 4096 && !legacy) {
    switch (eb) {
      case 4: launch_pipe<uint32_t>(dst, src, args, n_tiles, nvec, s, route_for<uint32_t>(pc, elem_bytes, vb)); break;
      case 8: launch_pipe<uint2>(dst, src, args, n_tiles, nvec, s, route_for<uint2>(pc, elem_bytes, vb)); break;
      default: launch_pipe<uint4>(dst, src, args, n_tiles, nvec, s, route_for<uint4>(pc, elem_bytes, vb)); break;
    }
    TN_CUDA(cudaGetLastError());
    return;
  }
  size_t smem = (size_t)nvec * 16 + (((size_t)tsz * 2 + 15) & ~(size_t)15) + (size_t)tsz * eb;
  int blocks = (int)std::min<uint64_t>(n_tiles, 148ull * 8);
  static bool attr_set[3] = {false, false, false};
  switch (eb) {
    case 4:
      if (!attr_set[0]) {
        TN_CUDA(cudaFuncSetAttribute(permute_kernel<uint32_t>, cudaFuncAttributeMaxDynamicSharedMemorySize, 96 * 1024));
        attr_set[0] = true;
      }
      permute_kernel<uint32_t><<<blocks, 256, smem, s>>>((uint32_t*)dst, (const uint32_t*)src, args, n_tiles,
                                                         route_for<uint32_t>(pc, elem_bytes, vb));
      break;
    case 8:
      if (!attr_set[1]) {
        TN_CUDA(cudaFuncSetAttribute(permute_kernel<uint2>, cudaFuncAttributeMaxDynamicSharedMemorySize, 96 * 1024));
        attr_set[1] = true;
      }
      permute_kernel<uint2><<<blocks, 256, smem, s>>>((uint2*)dst, (const uint2*)src, args, n_tiles,
                                                      route_for<uint2>(pc, elem_bytes, vb));
      break;
    default:
      if (!attr_set[2]) {
        TN_CUDA(cudaFuncSetAttribute(permute_kernel<uint4>, cudaFuncAttributeMaxDynamicSharedMemorySize, 96 * 1024));
        attr_set[2] = true;
      }
      permute_kernel<uint4><<<blocks, 256, smem, s>>>((uint4*)dst, (const uint4*)src, args, n_tiles,
                                                      route_for<uint4>(pc, elem_bytes, vb));
      break;
  }
  TN_CUDA(cudaGetLastError());
}

}  // namespace tn
