// Micro-benchmark: fixed cost of launching a persistent 576-thread / ~225 KB smem / 512-column
// TMEM kernel (the score kernel's launch shape) after a small-smem kernel, vs its CTA lifetime.
//   variants: big smem + TMEM, big smem only, small smem; each after a tiny "other" kernel that
//   uses the default carveout or the max-smem carveout hint.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2601_13631_b200/csrc \
//      scripts/launch_bench.cu -o scripts/launch_bench
#include <cuda_runtime.h>
#include <cstdio>

#include "tc_ptx.cuh"

using namespace ckv;

__device__ unsigned long long g_t[2][160];

__device__ __forceinline__ unsigned long long gtime() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

template <bool TMEM>
__global__ void __launch_bounds__(576, 1) big_kernel(int spin_ns) {
  extern __shared__ uint8_t raw[];
  __shared__ uint32_t slot;
  const unsigned long long t0 = gtime();
  if (TMEM && (threadIdx.x >> 5) == 1) ptx::tmem_alloc<512>(&slot);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  raw[threadIdx.x] = 1;
  while (gtime() - t0 < (unsigned long long)spin_ns) {
  }
  ptx::tc_fence_before();
  __syncthreads();
  if (TMEM && (threadIdx.x >> 5) == 1) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc<512>(slot);
  }
  if (threadIdx.x == 0) {
    g_t[0][blockIdx.x] = t0;
    g_t[1][blockIdx.x] = gtime();
  }
}

__global__ void small_kernel(float* x) {
  __shared__ float s[256];
  s[threadIdx.x] = x[threadIdx.x];
  __syncthreads();
  x[threadIdx.x] = s[255 - threadIdx.x] + 1.f;
}

int main() {
  float* x;
  cudaMalloc(&x, 1 << 20);
  cudaMemset(x, 0, 1 << 20);
  const int smem_big = 225 * 1024;
  cudaFuncSetAttribute(big_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_big);
  cudaFuncSetAttribute(big_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_big);
  cudaStream_t st;
  cudaStreamCreate(&st);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int spin = 20000;  // 20 us of CTA lifetime
  for (int carve = 0; carve < 2; ++carve) {
    if (carve) {
      cudaFuncSetAttribute(small_kernel, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
      cudaFuncSetAttribute(big_kernel<true>, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
      cudaFuncSetAttribute(big_kernel<false>, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    }
    for (int var = 0; var < 4; ++var) {
      // var 0: big+TMEM alone; 1: small then big+TMEM; 2: small then big (no TMEM); 3: small then small-smem big
      float best = 1e9, sum = 0;
      unsigned long long life = 0;
      const int reps = 20;
      for (int r = 0; r < reps + 3; ++r) {
        cudaStreamSynchronize(st);
        if (var >= 1) small_kernel<<<148, 256, 0, st>>>(x);
        cudaEventRecord(e0, st);
        if (var <= 1) big_kernel<true><<<148, 576, smem_big, st>>>(spin);
        if (var == 2) big_kernel<false><<<148, 576, smem_big, st>>>(spin);
        if (var == 3) big_kernel<false><<<148, 576, 1024, st>>>(spin);
        cudaEventRecord(e1, st);
        cudaStreamSynchronize(st);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        if (r >= 3) {
          sum += ms;
          best = ms < best ? ms : best;
          unsigned long long h[2][160];
          cudaMemcpyFromSymbol(h, g_t, sizeof h);
          unsigned long long s0 = ~0ull, e = 0;
          for (int b = 0; b < 148; ++b) {
            s0 = h[0][b] < s0 ? h[0][b] : s0;
            e = h[1][b] > e ? h[1][b] : e;
          }
          life += e - s0;
        }
      }
      printf("carveout_hint=%d variant=%d event_us mean %.2f min %.2f  cta_span_us %.2f\n", carve, var,
             sum / reps * 1e3, best * 1e3, life / (double)reps * 1e-3);
    }
  }
  // back-to-back pairs (small, big) x 50 in one timed region, with and without the carveout hint
  for (int carve = 0; carve < 2; ++carve) {
    const int hint = carve ? 100 : -1;
    cudaFuncSetAttribute(small_kernel, cudaFuncAttributePreferredSharedMemoryCarveout, hint);
    cudaFuncSetAttribute(big_kernel<true>, cudaFuncAttributePreferredSharedMemoryCarveout, hint);
    for (int rep = 0; rep < 2; ++rep) {
      cudaStreamSynchronize(st);
      cudaEventRecord(e0, st);
      for (int i = 0; i < 50; ++i) {
        small_kernel<<<148, 256, 0, st>>>(x);
        big_kernel<true><<<148, 576, smem_big, st>>>(spin);
      }
      cudaEventRecord(e1, st);
      cudaStreamSynchronize(st);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      if (rep) printf("pairs carveout_hint=%d: %.2f us per (small, big) pair (big CTA lifetime %d us)\n", hint,
                      ms * 1e3 / 50, spin / 1000);
    }
  }
  printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
