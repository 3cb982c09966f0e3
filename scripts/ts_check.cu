// Correctness probe for the per-chunk attention MMA scheme: S = Q K^T with Q (A operand) in TMEM
// and one N = c MMA per chunk record, then O = P V with V read straight from the chunk records
// (MN-major, 128-byte swizzle, LBO = half distance, SBO = 8-key group distance).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2601_13631_b200/csrc
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "tc_ptx.cuh"

using namespace ckv;

__global__ void __launch_bounds__(128) ts_kernel(int C, const uint4* recs_g, const uint4* p_img, const uint32_t* q,
                                                 float* s_out, float* o_out) {
  extern __shared__ uint8_t raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
  uint8_t* recs = sm;            // 64 KB: 128 / C records of 512 C bytes
  uint8_t* pbuf = sm + 65536;    // 32 KB: [half][128 rows][64] swizzled
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  const int t = threadIdx.x, warp = t >> 5;
  for (int i = t; i < 4096; i += 128) reinterpret_cast<uint4*>(recs)[i] = recs_g[i];
  for (int i = t; i < 2048; i += 128) reinterpret_cast<uint4*>(pbuf)[i] = p_img[i];
  ptx::fence_proxy_async_smem();
  if (t == 0) {
    ptx::mbar_init(&bar, 1);
    ptx::fence_mbar_init();
  }
  if (warp == 0) ptx::tmem_alloc<512>(&slot);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = slot;
  const uint32_t lane_off = (uint32_t)(warp * 32) << 16;
  {  // Q row t -> TMEM columns 384 .. 447 (two bf16 per column)
    float v[32];
    for (int h = 0; h < 2; ++h) {
      for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(q[t * 64 + h * 32 + i]);
      ptx::tmem_st32(tmem + 384 + h * 32 + lane_off, v);
    }
  }
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  if (t == 0) {
    const int nch = 128 / C;
    const uint32_t idesc_s = ptx::idesc_bf16_f32(128, C);
    for (int ch = 0; ch < nch; ++ch)
      for (int k = 0; k < 8; ++k) {
        const uint32_t ka = ptx::smem_u32(recs + ch * 512 * C + (k >> 2) * (C * 128) + (k & 3) * 32);
        ptx::mma_bf16_ts(tmem + ch * C, tmem + 384 + k * 8, ptx::umma_desc_sw128(ka), idesc_s, k > 0);
      }
    const uint32_t idesc_o = ptx::idesc_bf16_f32(128, 128, true);
    for (int k = 0; k < 8; ++k) {
      uint32_t va, lbo, sbo;
      if (C >= 16) {
        const int ch = (k * 16) / C, row0 = (k * 16) % C;
        va = ptx::smem_u32(recs + ch * 512 * C + 2 * C * 128 + row0 * 128);
        lbo = C * 128;
        sbo = 1024;
      } else {  // C == 8: one K step spans chunks 2k, 2k + 1
        va = ptx::smem_u32(recs + (2 * k) * 4096 + 2 * 1024);
        lbo = 1024;
        sbo = 4096;
      }
      const uint32_t pa = ptx::smem_u32(pbuf + (k >> 2) * 16384 + (k & 3) * 32);
      ptx::mma_bf16(tmem + 256, ptx::umma_desc_sw128(pa), ptx::umma_desc_sw128_mn(va, lbo, sbo), idesc_o, k > 0);
    }
    ptx::mma_commit(&bar);
  }
  ptx::mbar_wait(&bar, 0);
  ptx::tc_fence_after();
  float v[32];
  for (int g = 0; g < 4; ++g) {
    ptx::tmem_ld32(tmem + g * 32 + lane_off, v);
    for (int i = 0; i < 32; ++i) s_out[t * 128 + g * 32 + i] = v[i];
    ptx::tmem_ld32(tmem + 256 + g * 32 + lane_off, v);
    for (int i = 0; i < 32; ++i) o_out[t * 128 + g * 32 + i] = v[i];
  }
  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 0) ptx::tmem_dealloc<512>(tmem);
}

static float bf(float x) { return __bfloat162float(__float2bfloat16(x)); }
static uint16_t bits(float x) {
  __nv_bfloat16 b = __float2bfloat16(x);
  return *reinterpret_cast<uint16_t*>(&b);
}

int run(int C) {
  std::vector<float> Q(128 * 128), K(128 * 128), V(128 * 128), P(128 * 128);
  srand(7 + C);
  auto rnd = [] { return bf((rand() / (float)RAND_MAX - 0.5f) * 2.f); };
  for (auto* a : {&Q, &K, &V, &P})
    for (auto& x : *a) x = rnd();
  // chunk records: [K h0][K h1][V h0][V h1], rows of 64 bf16 with 16-byte units XOR (row & 7)
  std::vector<uint16_t> rec(128 * 128 * 2);
  for (int j = 0; j < 128; ++j)
    for (int x = 0; x < 128; ++x)
      for (int kv = 0; kv < 2; ++kv) {
        const int ch = j / C, p = j % C, half = x >> 6, xi = x & 63, u = (xi >> 3) ^ (p & 7);
        const size_t off = (size_t)ch * 256 * C + ((kv * 2 + half) * C + p) * 64 + u * 8 + (xi & 7);
        rec[off] = bits(kv ? V[j * 128 + x] : K[j * 128 + x]);
      }
  std::vector<uint16_t> pimg(128 * 128);
  for (int i = 0; i < 128; ++i)
    for (int j = 0; j < 128; ++j) {
      const int half = j >> 6, ji = j & 63, u = (ji >> 3) ^ (i & 7);
      pimg[(half * 128 + i) * 64 + u * 8 + (ji & 7)] = bits(P[i * 128 + j]);
    }
  std::vector<uint32_t> qw(128 * 64);
  for (int i = 0; i < 128; ++i)
    for (int c = 0; c < 64; ++c)
      qw[i * 64 + c] = (uint32_t)bits(Q[i * 128 + 2 * c]) | ((uint32_t)bits(Q[i * 128 + 2 * c + 1]) << 16);
  uint4 *drec, *dp;
  uint32_t* dq;
  float *ds, *dout;
  cudaMalloc(&drec, rec.size() * 2);
  cudaMalloc(&dp, pimg.size() * 2);
  cudaMalloc(&dq, qw.size() * 4);
  cudaMalloc(&ds, 128 * 128 * 4);
  cudaMalloc(&dout, 128 * 128 * 4);
  cudaMemcpy(drec, rec.data(), rec.size() * 2, cudaMemcpyHostToDevice);
  cudaMemcpy(dp, pimg.data(), pimg.size() * 2, cudaMemcpyHostToDevice);
  cudaMemcpy(dq, qw.data(), qw.size() * 4, cudaMemcpyHostToDevice);
  const int smem = 65536 + 32768 + 1024;
  cudaFuncSetAttribute(ts_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  ts_kernel<<<1, 128, smem>>>(C, drec, dp, dq, ds, dout);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) {
    printf("C=%d: CUDA error %s\n", C, cudaGetErrorString(e));
    return 1;
  }
  std::vector<float> S(128 * 128), O(128 * 128);
  cudaMemcpy(S.data(), ds, S.size() * 4, cudaMemcpyDeviceToHost);
  cudaMemcpy(O.data(), dout, O.size() * 4, cudaMemcpyDeviceToHost);
  double es = 0, eo = 0;
  for (int i = 0; i < 128; ++i)
    for (int j = 0; j < 128; ++j) {
      double s = 0, o = 0;
      for (int x = 0; x < 128; ++x) {
        s += (double)Q[i * 128 + x] * K[j * 128 + x];
        o += (double)P[i * 128 + x] * V[x * 128 + j];
      }
      es = fmax(es, fabs(s - S[i * 128 + j]));
      eo = fmax(eo, fabs(o - O[i * 128 + j]));
    }
  printf("C=%d: max|S err| %.3g  max|O err| %.3g  %s\n", C, es, eo, (es < 1e-2 && eo < 1e-2) ? "OK" : "MISMATCH");
  return 0;
}

int main() {
  run(16);
  run(32);
  run(8);
  return 0;
}
