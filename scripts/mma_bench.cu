// Micro-benchmark: tcgen05.mma kind::f16 throughput per SM, SS mode, cta_group::1.
// A unit = 8 MMAs (K = 128) of M=128 x N into one of two TMEM accumulators.
//   mode 0: all units back to back, one commit at the end
//   mode 1: commit per unit; the issuer waits for unit u-2 before reusing its accumulator
//   mode 2: as mode 1 but 16 epilogue warps wait acc_full and arrive acc_empty (score-kernel shape)
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2601_13631_b200/csrc
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>

#include "tc_ptx.cuh"

using namespace ckv;

template <int N, bool TS = false>
__global__ void __launch_bounds__(576, 1) mma_kernel(int units, int mode, long long* cyc) {
  extern __shared__ uint8_t raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
  uint8_t* A = sm;                 // 128 x 128 bf16 = 32 KB (two 64-col halves)
  uint8_t* B = sm + 32768;         // N x 128 bf16
  uint64_t* bars = reinterpret_cast<uint64_t*>(sm + 32768 + N * 256);
  uint64_t* acc_full = bars;       // [2]
  uint64_t* acc_empty = bars + 2;  // [2]
  uint64_t* done = bars + 4;
  uint32_t* slot = reinterpret_cast<uint32_t*>(bars + 6);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < (32768 + N * 256) / 16; i += blockDim.x)
    reinterpret_cast<uint4*>(sm)[i] = make_uint4(0, 0, 0, 0);
  if (threadIdx.x == 0) {
    for (int i = 0; i < 2; ++i) {
      ptx::mbar_init(&acc_full[i], 1);
      ptx::mbar_init(&acc_empty[i], 16);
    }
    ptx::mbar_init(done, 1);
    ptx::fence_mbar_init();
  }
  if (warp == 1) ptx::tmem_alloc<512>(slot);
  ptx::fence_proxy_async_smem();
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = *slot;
  if (warp == 1 && lane == 0) {
    constexpr uint32_t idesc = ptx::idesc_bf16_f32(128, N);
    const long long t0 = clock64();
    for (int u = 0; u < units; ++u) {
      const int ab = u & 1;
      if (mode == 1 && u >= 2) ptx::mbar_wait(&acc_full[ab], ((u - 2) >> 1) & 1);
      if (mode == 2) ptx::mbar_wait(&acc_empty[ab], ((u >> 1) & 1) ^ 1);
      ptx::tc_fence_after();
      if (mode == 3) {  // 128 / N independent N-wide accumulators, K-step outer (interleaved)
#pragma unroll
        for (int k = 0; k < 8; ++k)
#pragma unroll
          for (int c = 0; c < 128 / N; ++c)
            ptx::mma_bf16_ts(tmem + ab * 128 + c * N, tmem + 384 + k * 8,
                             ptx::umma_desc_sw128(ptx::smem_u32(B) + (k >> 2) * (N * 128) + (k & 3) * 32), idesc, k > 0);
        continue;
      }
      if (mode == 4) {  // same, chunk outer (dependent accumulations back to back)
#pragma unroll
        for (int c = 0; c < 128 / N; ++c)
#pragma unroll
          for (int k = 0; k < 8; ++k)
            ptx::mma_bf16_ts(tmem + ab * 128 + c * N, tmem + 384 + k * 8,
                             ptx::umma_desc_sw128(ptx::smem_u32(B) + (k >> 2) * (N * 128) + (k & 3) * 32), idesc, k > 0);
        continue;
      }
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const uint32_t oa = (k >> 2) * 16384 + (k & 3) * 32;
        const uint32_t ob = (k >> 2) * (N * 128) + (k & 3) * 32;
        if constexpr (TS)
          ptx::mma_bf16_ts(tmem + ab * 128, tmem + 384 + k * 8, ptx::umma_desc_sw128(ptx::smem_u32(B) + ob), idesc,
                           k > 0);
        else
          ptx::mma_bf16(tmem + ab * 256, ptx::umma_desc_sw128(ptx::smem_u32(A) + oa),
                        ptx::umma_desc_sw128(ptx::smem_u32(B) + ob), idesc, k > 0);
      }
      if (mode >= 1) ptx::mma_commit(&acc_full[ab]);
    }
    ptx::mma_commit(done);
    ptx::mbar_wait(done, 0);
    const long long t1 = clock64();
    cyc[blockIdx.x] = t1 - t0;
  } else if (warp >= 2 && mode == 2) {
    for (int u = 0; u < units; ++u) {
      const int ab = u & 1;
      ptx::mbar_wait(&acc_full[ab], (u >> 1) & 1);
      ptx::tc_fence_after();
      __syncwarp();
      if (lane == 0) ptx::mbar_arrive(&acc_empty[ab]);
    }
  }
  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 1) ptx::tmem_dealloc<512>(tmem);
}

template <int N, bool TS = false>
void run(int units, int mode) {
  const size_t smem = 1024 + 32768 + N * 256 + 128;
  cudaFuncSetAttribute(mma_kernel<N, TS>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  long long* cyc;
  cudaMalloc(&cyc, 148 * sizeof(long long));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  mma_kernel<N, TS><<<148, 576, smem>>>(units, mode, cyc);
  cudaEventRecord(e0);
  mma_kernel<N, TS><<<148, 576, smem>>>(units, mode, cyc);
  cudaEventRecord(e1);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) {
    printf("error %s\n", cudaGetErrorString(e));
    exit(1);
  }
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  long long h[148];
  cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
  double avg = 0;
  for (int i = 0; i < 148; ++i) avg += h[i] / 148.0;
  const double flops = 2.0 * 128 * (mode >= 3 ? 128 : N) * 128 * (double)units * 148;
  printf("%s N=%d mode=%d units=%d: %.1f cyc/unit (floor %d), kernel %.2f us, %.0f TFLOP/s\n", TS ? "TS" : "SS", N,
         mode, units,
         avg / units, 8 * 128 * N / 256, ms * 1e3, flops / (ms * 1e-3) / 1e12);
  cudaFree(cyc);
}

int main() {
  run<256>(256, 0);
  run<128>(256, 0);
  run<16>(256, 0);
  run<128, true>(256, 0);
  run<64, true>(256, 0);
  run<32, true>(256, 0);
  run<16, true>(256, 0);
  run<8, true>(256, 0);
  run<16, true>(256, 3);
  run<16, true>(256, 4);
  run<8, true>(256, 3);
  run<32, true>(256, 3);
  return 0;
}
