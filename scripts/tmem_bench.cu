// Micro-benchmark: TMEM read (tcgen05.ld 32x32b.x32) throughput per SM and its interaction
// with MUFU ex2, with 16 warps (4 per TMEM lane quadrant) like the score epilogue.
//   mode 0: LDTM + wait only      mode 1: LDTM + 32 ex2 + sum      mode 2: 32 ex2 + sum only
//   mode 3: as 1, max-subtracted (the score epilogue's arithmetic)
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2601_13631_b200/csrc
#include <cuda_runtime.h>
#include <cstdio>

#include "common.cuh"
#include "tc_ptx.cuh"

using namespace ckv;

template <int N, int G>
__device__ __forceinline__ void tsum(float* a) {
  if constexpr (G > 1) {
    tsum<N, G / 2>(a);
#pragma unroll
    for (int i = 0; i < N / G; ++i) a[i] = a[2 * i] + a[2 * i + 1];
  }
}

template <int MODE>
__global__ void __launch_bounds__(512, 1) tmem_kernel(int iters, float* out, long long* cyc) {
  __shared__ uint32_t slot;
  const int warp = threadIdx.x >> 5;
  if (warp == 0) ptx::tmem_alloc<512>(&slot);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = slot;
  const int quad = warp & 3, part = warp >> 2;  // 4 warps per quadrant, 64 columns each of 256
  float acc = 0.f;
  float v[32];
#pragma unroll
  for (int i = 0; i < 32; ++i) v[i] = -0.01f * i;
  __syncthreads();
  const long long t0 = clock64();
  if (MODE >= 4) {  // score epilogue: 64 columns, one max, C = 16 chunk sums, lg2 per chunk (+ stores)
    for (int it = 0; it < iters; ++it) {
      float w[64];
      ptx::tmem_ld32p(tmem + (it & 1) * 256 + part * 64 + ((uint32_t)(quad * 32) << 16), w);
      ptx::tmem_ld32p(tmem + (it & 1) * 256 + part * 64 + 32 + ((uint32_t)(quad * 32) << 16), w + 32);
      float m = w[0];
#pragma unroll
      for (int i = 1; i < 64; ++i) m = fmaxf(m, w[i]);
      const float ms = m * 0.127f;
#pragma unroll
      for (int i = 0; i < 64; ++i) w[i] = fast_exp2(fmaf(w[i], 0.127f, -ms) - 1.f);
      tsum<64, 16>(w);
      float tot = 0.f;
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const float l = ms + fast_log2(w[i]);
        tot += w[i];
        if (MODE == 5) out[(size_t)148 * 512 * (1 + (it & 63) * 4 + i) + blockIdx.x * 512 + threadIdx.x] = l;
        else acc += l;
      }
      acc += fast_log2(tot);
    }
  } else
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int g = 0; g < 2; ++g) {
      const uint32_t col = (it & 1) * 256 + part * 64 + g * 32;
      if (MODE != 2) ptx::tmem_ld32p(tmem + col + ((uint32_t)(quad * 32) << 16), v);
      if (MODE == 0) {
        acc += v[0];
      } else {
        float m = 0.f;
        if (MODE == 3) {
#pragma unroll
          for (int i = 0; i < 32; ++i) m = fmaxf(m, v[i]);
        }
        float s = 0.f;
#pragma unroll
        for (int i = 0; i < 32; ++i) s += fast_exp2(fmaf(v[i], 0.127f, -m) - 1.f);
        acc += s;
        if (MODE == 2) v[it & 31] += s * 1e-9f;
      }
    }
  }
  __syncthreads();
  const long long t1 = clock64();
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 0) ptx::tmem_dealloc<512>(tmem);
}

template <int MODE>
void run(const char* name) {
  float* out;
  long long* cyc;
  cudaMalloc(&out, (size_t)148 * 512 * 4 * 260);
  cudaMalloc(&cyc, 148 * 8);
  const int iters = 512;
  tmem_kernel<MODE><<<148, 512>>>(iters, out, cyc);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) {
    printf("error %s\n", cudaGetErrorString(e));
    return;
  }
  long long h[148];
  cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
  double avg = 0;
  for (int i = 0; i < 148; ++i) avg += h[i] / 148.0;
  // one "unit" = 128 lanes x 256 columns (what one score work unit reads)
  printf("%s: %.0f cycles per 128x256 unit (MUFU floor 2048)\n", name, avg / iters);
}

int main() {
  run<0>("ldtm only");
  run<1>("ldtm + ex2 + sum");
  run<2>("ex2 + sum (no ldtm)");
  run<3>("ldtm + max + ex2 + sum");
  run<4>("score epilogue (64 cols, C=16, lg2), no stores");
  run<5>("score epilogue + coalesced lam stores");
  return 0;
}
