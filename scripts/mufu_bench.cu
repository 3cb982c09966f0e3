// Micro-benchmark: MUFU.EX2 and FFMA throughput per SM (one CTA of 512 threads per SM,
// 8 independent chains per thread).  nvcc -gencode arch=compute_100a,code=sm_100a -O3
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>

__device__ __forceinline__ float ex2(float x) {
  float y;
  asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

__device__ __forceinline__ uint32_t ex2h2(uint32_t x) {
  uint32_t y;
  asm volatile("ex2.approx.f16x2 %0, %1;" : "=r"(y) : "r"(x));
  return y;
}

template <int MODE>
__global__ void __launch_bounds__(512, 1) k(int iters, float* out, long long* cyc) {
  float v[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) v[i] = -1e-3f * (threadIdx.x + i);
  __syncthreads();
  const long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (MODE == 0) v[i] = ex2(v[i]) - 1.0f;  // MUFU + FADD
      if (MODE == 1) v[i] = fmaf(v[i], 0.999f, -1e-7f);
      if (MODE == 2) v[i] = ex2(v[i]);         // MUFU only (value converges to a fixed point)
      if (MODE == 3) v[i] = __uint_as_float(ex2h2(__float_as_uint(v[i])));  // 2 exps per lane-op
      if (MODE == 4 && (i & 1) == 0) {  // FFMA2: 2 fp32 FMAs per lane-op (counted as 2 ops)
        float2 r = __ffma2_rn(make_float2(v[i], v[i + 1]), make_float2(0.999f, 0.999f), make_float2(-1e-7f, -1e-7f));
        v[i] = r.x;
        v[i + 1] = r.y;
      }
    }
  }
  __syncthreads();
  const long long t1 = clock64();
  float s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += v[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

template <int MODE>
void run(const char* name) {
  float* out;
  long long* cyc;
  cudaMalloc(&out, 148 * 512 * 4);
  cudaMalloc(&cyc, 148 * 8);
  const int iters = 4096;
  k<MODE><<<148, 512>>>(iters, out, cyc);
  cudaDeviceSynchronize();
  long long h[148];
  cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
  double avg = 0;
  for (int i = 0; i < 148; ++i) avg += h[i] / 148.0;
  const double ops = 512.0 * 8 * iters;
  printf("%s: %.2f ops/clk/SM\n", name, ops / avg);
}

int main() {
  run<0>("ex2+fadd");
  run<2>("ex2");
  run<1>("ffma");
  run<3>("ex2.f16x2 (lane-ops)");
  run<4>("ffma2 (fp32 FMAs)");
  return 0;
}
