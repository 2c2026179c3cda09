// Feasibility probe: can a TMA bulk-tensor store (cp.async.bulk.tensor.2d.global.shared::cta) target
// a peer GPU's memory (P2P over NVLink, UVA address)?  GPU 0 stores a 128x64 fp16 tile into a
// buffer on GPU 1; the host checks it.  Also times a large peer-store stream (TMA vs st.global.v4).
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <vector>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); return 1; } } while (0)

typedef CUresult (*encode_t)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                             const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                             CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

__global__ void tma_store_kernel(const __grid_constant__ CUtensorMap map, int rows_total, int iters) {
  __shared__ __align__(128) uint16_t tile[128 * 64];
  for (int i = threadIdx.x; i < 128 * 64; i += blockDim.x) tile[i] = (uint16_t)(i + blockIdx.x);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int it = 0; it < iters; ++it) {
      int row = ((blockIdx.x + it * gridDim.x) * 128) % rows_total;
      asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];" ::"l"(&map), "r"(0), "r"(row),
                   "r"((uint32_t)__cvta_generic_to_shared(tile)) : "memory");
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
      asm volatile("cp.async.bulk.wait_group.read 4;" ::: "memory");
    }
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  }
}

__global__ void st_kernel(uint4* dst, size_t n16, int iters) {
  for (int it = 0; it < iters; ++it)
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n16; i += (size_t)gridDim.x * blockDim.x)
      dst[i] = make_uint4((uint32_t)i, 1, 2, 3);
}

int main() {
  int n = 0;
  CK(cudaGetDeviceCount(&n));
  if (n < 2) { printf("needs 2 GPUs\n"); return 0; }
  int can = 0;
  CK(cudaDeviceCanAccessPeer(&can, 0, 1));
  printf("can access peer 0->1: %d\n", can);
  CK(cudaSetDevice(1));
  const int rows = 1 << 18;  // 256 Ki rows x 64 fp16 = 32 MiB
  uint16_t* d1 = nullptr;
  CK(cudaMalloc(&d1, (size_t)rows * 64 * 2));
  CK(cudaMemset(d1, 0, (size_t)rows * 64 * 2));
  CK(cudaSetDevice(0));
  CK(cudaDeviceEnablePeerAccess(1, 0));
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q));
  encode_t enc = (encode_t)fn;
  CUtensorMap map;
  cuuint64_t dims[2] = {64, (cuuint64_t)rows};
  cuuint64_t strides[1] = {128};
  cuuint32_t box[2] = {64, 128};
  cuuint32_t es[2] = {1, 1};
  CUresult r = enc(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, d1, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  printf("encode on peer buffer: %d\n", (int)r);
  tma_store_kernel<<<1, 128>>>(map, rows, 1);
  CK(cudaGetLastError());
  CK(cudaDeviceSynchronize());
  std::vector<uint16_t> h(128 * 64);
  CK(cudaMemcpy(h.data(), d1, h.size() * 2, cudaMemcpyDefault));
  int bad = 0;
  for (int i = 0; i < 128 * 64; ++i) bad += h[i] != (uint16_t)i;
  printf("TMA peer store check: %s (%d bad)\n", bad ? "FAIL" : "ok", bad);
  // bandwidth: 148 CTAs storing 16 KB tiles round-robin over 32 MiB, repeated
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  const int iters = 2048;
  tma_store_kernel<<<148, 128>>>(map, rows, 16);
  CK(cudaEventRecord(e0));
  tma_store_kernel<<<148, 128>>>(map, rows, iters);
  CK(cudaEventRecord(e1));
  CK(cudaEventSynchronize(e1));
  float ms = 0;
  CK(cudaEventElapsedTime(&ms, e0, e1));
  double bytes = 148.0 * iters * 16384;
  printf("TMA peer store: %.1f GB in %.2f ms = %.0f GB/s\n", bytes / 1e9, ms, bytes / ms / 1e6);
  CK(cudaEventRecord(e0));
  st_kernel<<<148 * 4, 512>>>((uint4*)d1, (size_t)rows * 64 * 2 / 16, 64);
  CK(cudaEventRecord(e1));
  CK(cudaEventSynchronize(e1));
  CK(cudaEventElapsedTime(&ms, e0, e1));
  bytes = 64.0 * rows * 128;
  printf("st.global.v4 peer store: %.1f GB in %.2f ms = %.0f GB/s\n", bytes / 1e9, ms, bytes / ms / 1e6);
  // local for comparison
  uint16_t* d0 = nullptr;
  CK(cudaMalloc(&d0, (size_t)rows * 64 * 2));
  CUtensorMap map0;
  enc(&map0, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, d0, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
      CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  CK(cudaEventRecord(e0));
  tma_store_kernel<<<148, 128>>>(map0, rows, iters);
  CK(cudaEventRecord(e1));
  CK(cudaEventSynchronize(e1));
  CK(cudaEventElapsedTime(&ms, e0, e1));
  bytes = 148.0 * iters * 16384;
  printf("TMA local store (L2-resident 32 MiB): %.0f GB/s\n", bytes / ms / 1e6);
  return 0;
}
