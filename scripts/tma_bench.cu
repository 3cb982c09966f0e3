// Micro-benchmark: how fast can one CTA per SM gather 64 KB "key tiles" made of scattered
// small blocks into shared memory?  Compares 2-D TMA boxes of 2 KB, 1-D bulk copies of 2 KB
// and 8 KB, and contiguous 16 KB TMA boxes.  nvcc -gencode arch=compute_100a,code=sm_100a.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>
#include <vector>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t c) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(c));
}
__device__ __forceinline__ void expect_tx(uint64_t* b, uint32_t n) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(n) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t par) {
  asm volatile(
      "{\n.reg .pred P1;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n@P1 bra D_%=;\nbra "
      "W_%=;\nD_%=:\n}" ::"r"(smem_u32(b)),
      "r"(par)
      : "memory");
}
__device__ __forceinline__ void tma2d(void* dst, const CUtensorMap* m, uint64_t* b, int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(
          smem_u32(dst)),
      "l"((uint64_t)m), "r"(smem_u32(b)), "r"(c0), "r"(c1)
      : "memory");
}
__device__ __forceinline__ void bulk1d(void* dst, const void* src, uint32_t bytes, uint64_t* b) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"((uint64_t)src), "r"(bytes), "r"(smem_u32(b))
               : "memory");
}

// mode 0: 32 x TMA 2D (64 x 16) = 2 KB; mode 1: 32 x bulk 2 KB; mode 2: 8 x bulk 8 KB; mode 3: 4 x TMA (64 x 128)
__global__ void __launch_bounds__(32) gather_kernel(const __grid_constant__ CUtensorMap m16,
                                                    const __grid_constant__ CUtensorMap m128, const char* base,
                                                    const int* rows, int ntiles, int mode, long long* cycles) {
  extern __shared__ __align__(1024) char sm[];
  __shared__ uint64_t bar[2];
  if (threadIdx.x == 0) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  if (threadIdx.x != 0) return;
  long long t0 = clock64();
  const int* r = rows + (size_t)blockIdx.x * ntiles * 32;
  for (int t = 0; t < ntiles; ++t) {
    const int s = t & 1;
    if (t >= 2) mbar_wait(&bar[s], ((t - 2) >> 1) & 1);
    char* dst = sm + s * 65536;
    expect_tx(&bar[s], 65536);
    if (mode == 0) {
      for (int q = 0; q < 32; ++q) tma2d(dst + q * 2048, &m16, &bar[s], (q & 1) * 64, r[t * 32 + q]);
    } else if (mode == 1) {
      for (int q = 0; q < 32; ++q) bulk1d(dst + q * 2048, base + (size_t)r[t * 32 + q] * 256, 2048, &bar[s]);
    } else if (mode == 2) {
      for (int q = 0; q < 8; ++q) bulk1d(dst + q * 8192, base + (size_t)r[t * 32 + q] * 256, 8192, &bar[s]);
    } else if (mode == 4) {
      for (int q = 0; q < 16; ++q) bulk1d(dst + q * 4096, base + (size_t)r[t * 32 + q] * 256, 4096, &bar[s]);
    } else {
      for (int q = 0; q < 4; ++q) tma2d(dst + q * 16384, &m128, &bar[s], (q & 1) * 64, (r[t * 32] / 128) * 128);
    }
  }
  mbar_wait(&bar[(ntiles - 1) & 1], ((ntiles - 1) >> 1) & 1);
  mbar_wait(&bar[(ntiles - 2) & 1], ((ntiles - 2) >> 1) & 1);
  cycles[blockIdx.x] = clock64() - t0;
}

int main() {
  const size_t bytes = 1ull << 30;  // 1 GiB, rows of 256 B (128 bf16)
  const int nrows = bytes / 256;
  char* buf;
  cudaMalloc(&buf, bytes);
  cudaMemset(buf, 1, bytes);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int ntiles = 64;
  std::vector<int> h((size_t)sms * ntiles * 32);
  srand(1);
  for (auto& x : h) x = (rand() % (nrows / 16 - 2)) * 16;
  int* rows;
  cudaMalloc(&rows, h.size() * 4);
  cudaMemcpy(rows, h.data(), h.size() * 4, cudaMemcpyHostToDevice);
  long long* cyc;
  cudaMalloc(&cyc, sms * 8);
  PFN_cuTensorMapEncodeTiled_v12000 enc;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q);
  CUtensorMap m16, m128;
  cuuint64_t dims[2] = {128, (cuuint64_t)nrows};
  cuuint64_t str[1] = {256};
  cuuint32_t b16[2] = {64, 16}, b128[2] = {64, 128}, es[2] = {1, 1};
  enc(&m16, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, buf, dims, str, b16, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
      CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  enc(&m128, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, buf, dims, str, b128, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
      CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  cudaFuncSetAttribute(gather_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 2 * 65536);
  const char* names[5] = {"tma2d 32x2KB", "bulk 32x2KB", "bulk 8x8KB", "tma2d 4x16KB contiguous", "bulk 16x4KB"};
  for (int mode = 0; mode < 5; ++mode) {
    for (int rep = 0; rep < 3; ++rep) {
      cudaEvent_t e0, e1;
      cudaEventCreate(&e0);
      cudaEventCreate(&e1);
      cudaEventRecord(e0);
      gather_kernel<<<sms, 32, 2 * 65536>>>(m16, m128, buf, rows, ntiles, mode, cyc);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      if (rep == 2)
        printf("%-26s %8.2f us total, %6.3f us/tile/SM, %7.1f GB/s\n", names[mode], ms * 1e3,
               ms * 1e3 / ntiles, (double)sms * ntiles * 65536 / (ms * 1e-3) / 1e9);
    }
  }
  cudaError_t e = cudaGetLastError();
  printf("status %s\n", cudaGetErrorString(e));
  return 0;
}
