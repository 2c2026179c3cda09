// Stem mode permutation ("Tensor contraction involves dimension
// reordering and matrix multiplication").  Y = X.transpose(perm) for a rank-n tensor whose modes
// all have dimension 2, so an element index is an n-bit word and the permutation is a bit
// permutation of the index.
//
// B200 design: HBM-bound (algorithmic bytes = 2 * elem_bytes * 2^n per pass).  Each CTA moves
// tiles of 2^u elements (u <= 10) spanning the 5 innermost INPUT bits and the 5 innermost OUTPUT
// bits, staged through shared memory so both the HBM read and the HBM write are coalesced; the
// index tables of a tile are built once per CTA in shared memory (grid-stride over tiles, grid
// sized in multiples of the 148 SMs).
#include <algorithm>
#include <cstring>
#include <vector>

#include "common.cuh"

namespace tn {

template <typename T>
__global__ void __launch_bounds__(256) permute_kernel(T* __restrict__ dst, const T* __restrict__ src,
                                                      const PermArgs args, uint64_t n_tiles) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int u = args.u;
  const int tsz = 1 << u;
  int64_t* in_tbl = reinterpret_cast<int64_t*>(smem_raw);
  int64_t* out_tbl = in_tbl + tsz;
  uint16_t* wr_tbl = reinterpret_cast<uint16_t*>(out_tbl + tsz);
  T* tile = reinterpret_cast<T*>(smem_raw + (size_t)tsz * 16 + (((size_t)tsz * 2 + 15) & ~(size_t)15));
  for (int e = threadIdx.x; e < tsz; e += blockDim.x) {
    int64_t io = 0;
    for (int j = 0; j < u; ++j)
      if (e >> j & 1) io += args.tile_in[j];
    in_tbl[e] = io;
    int r = 0;
    int64_t oo = 0;
    for (int j = 0; j < u; ++j)
      if (e >> j & 1) {
        r |= 1 << args.wr_map[j];
        oo += args.tile_out[args.wr_map[j]];
      }
    wr_tbl[e] = (uint16_t)r;
    out_tbl[e] = oo;
  }
  __syncthreads();
  const int n_outer = args.n - u;
  for (uint64_t t = blockIdx.x; t < n_tiles; t += gridDim.x) {
    int64_t bi = 0, bo = 0;
    for (int j = 0; j < n_outer; ++j)
      if (t >> j & 1) {
        bi += args.outer_in[j];
        bo += args.outer_out[j];
      }
    const T* s = src + bi;
    T* d = dst + bo;
#pragma unroll 4
    for (int e = threadIdx.x; e < tsz; e += blockDim.x) tile[e] = __ldg(s + in_tbl[e]);
    __syncthreads();
#pragma unroll 4
    for (int w = threadIdx.x; w < tsz; w += blockDim.x) d[out_tbl[w]] = tile[wr_tbl[w]];
    __syncthreads();
  }
}

void launch_permute(void* dst, const void* src, int elem_bytes, int n, const int* perm, cudaStream_t s) {
  if (n < 0 || n > 46) throw TnError{TN_E_INVALID, "permute: rank out of range"};
  if (elem_bytes != 4 && elem_bytes != 8 && elem_bytes != 16)
    throw TnError{TN_E_INVALID, "permute: elem_bytes must be 4, 8 or 16"};
  // q -> p: destination bit position q comes from source bit position p(q)
  std::vector<int> p_of_q(n), q_of_p(n);
  std::vector<int> seen(n, 0);
  bool ident = true;
  for (int j = 0; j < n; ++j) {
    if (perm[j] < 0 || perm[j] >= n || seen[perm[j]]++) throw TnError{TN_E_INVALID, "permute: not a permutation"};
    if (perm[j] != j) ident = false;
    int q = n - 1 - j, p = n - 1 - perm[j];
    p_of_q[q] = p;
    q_of_p[p] = q;
  }
  const uint64_t total = 1ull << n;
  if (ident) {
    TN_CUDA(cudaMemcpyAsync(dst, src, total * elem_bytes, cudaMemcpyDeviceToDevice, s));
    return;
  }
  // leading run: destination low bits that already come from the same source low bits move as
  // contiguous chunks; fold them into a wider element (up to 16 bytes) when possible.
  int run = 0;
  while (run < n && p_of_q[run] == run) ++run;
  int eb = elem_bytes, nn = n;
  std::vector<int> P = p_of_q;
  while (run > 0 && eb < 16) {  // merge bit 0 into the element
    eb *= 2;
    --run;
    std::vector<int> P2(nn - 1);
    for (int q = 1; q < nn; ++q) P2[q - 1] = P[q] - 1;
    P = P2;
    --nn;
  }
  std::vector<int> Q(nn);
  for (int q = 0; q < nn; ++q) Q[P[q]] = q;
  const int a = std::min(5, nn), b = std::min(5, nn);
  std::vector<int> tile_bits;  // source bit positions, read order
  std::vector<char> in_tile(nn, 0);
  for (int x = 0; x < a; ++x) {
    tile_bits.push_back(x);
    in_tile[x] = 1;
  }
  for (int q = 0; q < b; ++q)
    if (!in_tile[P[q]]) {
      tile_bits.push_back(P[q]);
      in_tile[P[q]] = 1;
    }
  PermArgs args;
  memset(&args, 0, sizeof(args));
  args.n = nn;
  args.u = (int)tile_bits.size();
  for (int j = 0; j < args.u; ++j) {
    args.tile_in[j] = 1ll << tile_bits[j];
    args.tile_out[j] = 1ll << Q[tile_bits[j]];
  }
  // write order: destination bits 0..b-1 first, then the remaining tile bits
  std::vector<int> wr;
  std::vector<char> used(args.u, 0);
  for (int q = 0; q < b; ++q) {
    int idx = (int)(std::find(tile_bits.begin(), tile_bits.end(), P[q]) - tile_bits.begin());
    wr.push_back(idx);
    used[idx] = 1;
  }
  for (int j = 0; j < args.u; ++j)
    if (!used[j]) wr.push_back(j);
  // wr_map[k] : write-order bit k -> read-order tile bit; the kernel needs read bit -> write bit
  for (int k = 0; k < args.u; ++k) args.wr_map[k] = 0;
  // kernel iterates write index w with bit j meaning write-order bit j; it needs for each
  // write-order bit j the read-order position: r |= 1 << wr_map[j]
  for (int j = 0; j < args.u; ++j) args.wr_map[j] = wr[j];
  int no = 0;
  for (int x = 0; x < nn; ++x)
    if (!in_tile[x]) {
      args.outer_in[no] = 1ll << x;
      args.outer_out[no] = 1ll << Q[x];
      ++no;
    }
  args.o = b;
  const uint64_t n_tiles = 1ull << (nn - args.u);
  const int tsz = 1 << args.u;
  size_t smem = (size_t)tsz * 16 + (((size_t)tsz * 2 + 15) & ~(size_t)15) + (size_t)tsz * eb;
  int blocks = (int)std::min<uint64_t>(n_tiles, 148ull * 8);
  switch (eb) {
    case 4:
      permute_kernel<uint32_t><<<blocks, 256, smem, s>>>((uint32_t*)dst, (const uint32_t*)src, args, n_tiles);
      break;
    case 8:
      permute_kernel<uint2><<<blocks, 256, smem, s>>>((uint2*)dst, (const uint2*)src, args, n_tiles);
      break;
    default:
      permute_kernel<uint4><<<blocks, 256, smem, s>>>((uint4*)dst, (const uint4*)src, args, n_tiles);
      break;
  }
  TN_CUDA(cudaGetLastError());
}

}  // namespace tn
