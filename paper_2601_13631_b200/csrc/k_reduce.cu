// A2 score-reduce.
//   Lambda2[h, r] = log2 of the softmax normaliser of suffix row r of head h over the
//   prefix keys (Q1: prefix-only; FULLROW adds the causal suffix keys), combined over
//   key splits and, on W GPUs, over shards in rank order;
//   A_j = sum_h sum_r 2^(lam2[h, r, j] - Lambda2[h, r])  (Eq. 1 with a_i the column sum
//   of the row softmax over the query axis, Q2, Q4).
// Reductions use a fixed order (no float atomics): run-to-run deterministic.
#include "common.cuh"

namespace ckv {
namespace {

__device__ __forceinline__ void lse2_acc(float& M, float& S, float v) {
  if (v == -INFINITY) return;
  if (v > M) {
    S = S * fast_exp2(M - v) + 1.f;
    M = v;
  } else {
    S += fast_exp2(v - M);
  }
}

// Block = 8 warps x 32 rows: lane <-> row, warp w reduces splits w, w+8, ... (fixed order),
// then warp 0 merges the 8 partials in order and adds the FULLROW suffix term.
template <typename T>
__global__ void __launch_bounds__(256) row_lse_kernel(LayerGeom g, const float* __restrict__ lampart, int nsplit,
                                                      const T* __restrict__ q, const T* __restrict__ ks, int fullrow,
                                                      const float* __restrict__ lam_all, int W,
                                                      float* __restrict__ Lam2, float* __restrict__ lam_local_out) {
  __shared__ float sM[8][32], sS[8][32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int idx = blockIdx.x * 32 + lane;  // = kvh * R + row = h * ns + r
  const bool ok = idx < g.Hkv * g.R;
  const int kvh = ok ? idx / g.R : 0, row = ok ? idx % g.R : 0;
  float M = -INFINITY, S = 0.f;
  if (ok) {
    if (lam_all == nullptr) {
      const float* src = lampart + (size_t)kvh * nsplit * g.R + row;
      for (int sp = warp; sp < nsplit; sp += 8) lse2_acc(M, S, src[(size_t)sp * g.R]);
    } else {
      const int n = g.Hkv * g.R;
      for (int w = warp; w < W; w += 8) lse2_acc(M, S, lam_all[(size_t)w * n + idx]);
    }
  }
  sM[warp][lane] = M;
  sS[warp][lane] = S;
  __syncthreads();
  if (warp != 0 || !ok) return;
  M = -INFINITY;
  S = 0.f;
  for (int w = 0; w < 8; ++w) {
    const float m = sM[w][lane], s = sS[w][lane];
    if (s > 0.f) lse2_acc(M, S, m + fast_log2(s));
  }
  if (lam_all == nullptr && lam_local_out) lam_local_out[idx] = (S > 0.f) ? M + fast_log2(S) : -INFINITY;
  if (fullrow) {
    // causal suffix keys t <= r of the same KV head (Q1 FULLROW, Q9)
    const int gq = row / g.ns, r = row % g.ns, h = kvh * g.G + gq;
    const float scale = kLog2e * rsqrtf((float)g.d);
    const T* qr = q + ((size_t)r * g.Hq + h) * g.d;
    for (int t = 0; t <= r; ++t) {
      const T* kt = ks + ((size_t)t * g.Hkv + kvh) * g.d;
      float acc = 0.f;
      for (int x = 0; x < g.d; ++x) acc = fmaf(to_f(qr[x]), to_f(kt[x]), acc);
      lse2_acc(M, S, acc * scale);
    }
  }
  Lam2[idx] = (S > 0.f) ? M + fast_log2(S) : -INFINITY;
}

// One warp per chunk j: lanes stride over (kvh, row), then a fixed xor-tree reduce.
__global__ void chunk_sum_kernel(LayerGeom g, const float* __restrict__ lam2, const float* __restrict__ Lam2,
                                 float* __restrict__ A) {
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (warp >= g.m_loc) return;
  float acc = 0.f;
  for (int kvh = 0; kvh < g.Hkv; ++kvh) {
    const float* src = lam2 + ((size_t)kvh * g.m_loc + warp) * g.R;
    const float* L = Lam2 + (size_t)kvh * g.R;
    for (int row = lane; row < g.R; row += 32) acc += fast_exp2(src[row] - L[row]);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if (lane == 0) A[warp] = acc;
}

}  // namespace

template <typename T>
cudaError_t launch_row_lse(const LayerGeom& g, const float* lampart, int nsplit, const T* q, const T* k_suf,
                           int fullrow, const float* lam_all, int W, float* Lam2, float* lam_local_out,
                           cudaStream_t st) {
  const int n = g.Hkv * g.R;
  row_lse_kernel<T><<<(n + 31) / 32, 256, 0, st>>>(g, lampart, nsplit, q, k_suf, fullrow, lam_all, W, Lam2,
                                                     lam_local_out);
  return cudaGetLastError();
}
template cudaError_t launch_row_lse<float>(const LayerGeom&, const float*, int, const float*, const float*, int,
                                           const float*, int, float*, float*, cudaStream_t);
template cudaError_t launch_row_lse<__nv_bfloat16>(const LayerGeom&, const float*, int, const __nv_bfloat16*,
                                                   const __nv_bfloat16*, int, const float*, int, float*, float*,
                                                   cudaStream_t);

cudaError_t launch_chunk_sum(const LayerGeom& g, const float* lam2, const float* Lam2, float* A, cudaStream_t st) {
  const int threads = 256, warps_per_block = threads / 32;
  const int blocks = (g.m_loc + warps_per_block - 1) / warps_per_block;
  chunk_sum_kernel<<<blocks, threads, 0, st>>>(g, lam2, Lam2, A);
  return cudaGetLastError();
}

}  // namespace ckv
