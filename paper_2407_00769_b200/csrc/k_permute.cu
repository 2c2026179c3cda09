// Stem mode permutation ("Tensor contraction involves dimension
// reordering and matrix multiplication").  Y = X.transpose(perm) for a rank-n tensor whose modes
// all have dimension 2, so an element index is an n-bit word and the permutation is a bit
// permutation of the index.
//
// B200 design: HBM-bound (algorithmic bytes = 2 * elem_bytes * 2^n per pass).
//  * leading modes that stay innermost in the same order are folded into a wider element
//    (up to 16 bytes), so pure block moves become 16-byte copies;
//  * each CTA moves tiles of 2^u elements (16 KB) spanning the innermost INPUT bits and the
//    innermost OUTPUT bits (extended alternately until the tile reaches 16 KB, so overlapping
//    inner modes never shrink the tile), staged through shared memory: HBM reads are 16-byte
//    vectors along the input's innermost bits, HBM writes 16-byte vectors along the output's;
//  * tile index tables are built once per CTA; grid-stride over tiles, grid = 148 x CTAs/SM.
#include <algorithm>
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

template <typename T>
__global__ void __launch_bounds__(256) permute_kernel(T* __restrict__ dst, const T* __restrict__ src,
                                                      const PermArgs2 args, uint64_t n_tiles) {
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
    T* d = dst + bo;
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
      for (int v = threadIdx.x; v < nvec; v += blockDim.x) d[out_tbl[v]] = tile[wr_tbl[v]];
    } else {
#pragma unroll 2
      for (int v = threadIdx.x; v < nvec; v += blockDim.x) {
        const uint16_t* wt = wr_tbl + (v << vb);
        uint4 x;
        T* xp = reinterpret_cast<T*>(&x);
        for (int j = 0; j < V; ++j) xp[j] = tile[wt[j]];
        *reinterpret_cast<uint4*>(d + out_tbl[v]) = x;
      }
    }
    __syncthreads();
  }
}

void launch_permute(void* dst, const void* src, int elem_bytes, int n, const int* perm, cudaStream_t s) {
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
  if (ident) {
    TN_CUDA(cudaMemcpyAsync(dst, src, total * elem_bytes, cudaMemcpyDeviceToDevice, s));
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
  const int u_target = std::min(nn, (eb == 4 ? 12 : (eb == 8 ? 11 : 10)));
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
  size_t smem = (size_t)nvec * 16 + (((size_t)tsz * 2 + 15) & ~(size_t)15) + (size_t)tsz * eb;
  int blocks = (int)std::min<uint64_t>(n_tiles, 148ull * 8);
  static bool attr_set[3] = {false, false, false};
  switch (eb) {
    case 4:
      if (!attr_set[0]) {
        TN_CUDA(cudaFuncSetAttribute(permute_kernel<uint32_t>, cudaFuncAttributeMaxDynamicSharedMemorySize, 96 * 1024));
        attr_set[0] = true;
      }
      permute_kernel<uint32_t><<<blocks, 256, smem, s>>>((uint32_t*)dst, (const uint32_t*)src, args, n_tiles);
      break;
    case 8:
      if (!attr_set[1]) {
        TN_CUDA(cudaFuncSetAttribute(permute_kernel<uint2>, cudaFuncAttributeMaxDynamicSharedMemorySize, 96 * 1024));
        attr_set[1] = true;
      }
      permute_kernel<uint2><<<blocks, 256, smem, s>>>((uint2*)dst, (const uint2*)src, args, n_tiles);
      break;
    default:
      if (!attr_set[2]) {
        TN_CUDA(cudaFuncSetAttribute(permute_kernel<uint4>, cudaFuncAttributeMaxDynamicSharedMemorySize, 96 * 1024));
        attr_set[2] = true;
      }
      permute_kernel<uint4><<<blocks, 256, smem, s>>>((uint4*)dst, (const uint4*)src, args, n_tiles);
      break;
  }
  TN_CUDA(cudaGetLastError());
}

}  // namespace tn
