// A2 score-reduce.
//   Lambda2[h, r] = log2 of the softmax normaliser of suffix row r of head h over the
//   prefix keys (Q1: prefix-only; FULLROW adds the causal suffix keys), combined over
//   key splits and, on W GPUs, over shards in rank order;
//   A_j = sum_h sum_r 2^(lam2[h, r, j] - Lambda2[h, r])  (Eq. 1 with a_i the column sum
//   of the row softmax over the query axis, Q2, Q4).
// Reductions use a fixed order (no float atomics): run-to-run deterministic.
#include <cstdlib>

#include "common.cuh"
#include "plan.cuh"

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
// merge a partial (m, s) = m + log2(s) into (M, S)
__device__ __forceinline__ void lse2_merge(float& M, float& S, float m, float s) {
  if (s <= 0.f) return;
  if (S <= 0.f) {
    M = m;
    S = s;
  } else if (m > M) {
    S = S * fast_exp2(M - m) + s;
    M = m;
  } else {
    S += s * fast_exp2(m - M);
  }
}

constexpr int kRowsPerBlock = 32;
constexpr int kSplitWarps = 32;  // 1024 threads: lane = row, warp = split group

// Block = 32 warps over 32 flattened rows (idx = kvh * R + row = h * ns + r): lane l owns row
// idx0 + l, warp w the splits w, w + 32, ... (each warp load is one coalesced 128-byte row
// segment; sixteen loads in flight per thread); the 32 split-group partials are merged in a fixed
// order by warp 0.
template <typename T>
__global__ void __launch_bounds__(1024) row_lse_kernel(LayerGeom g, const float* __restrict__ lampart, int nsplit,
                                                       const T* __restrict__ q, const T* __restrict__ ks, int fullrow,
                                                       const float* __restrict__ lam_all, int W,
                                                       float* __restrict__ Lam2, float* __restrict__ lam_local_out,
                                                       int transposed) {
  pdl_wait();
  pdl_trigger();
  __shared__ float sM[kSplitWarps][kRowsPerBlock + 1], sS[kSplitWarps][kRowsPerBlock + 1];
  const int nrows = g.Hkv * g.R;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int idx = min(blockIdx.x * kRowsPerBlock + lane, nrows - 1);
  const float* base;
  int stride, nparts;
  if (lam_all == nullptr) {
    const int kvh = idx / g.R, row = idx - kvh * g.R;
    base = lampart + (size_t)kvh * nsplit * g.R + row;
    stride = g.R;
    nparts = nsplit;
  } else {
    base = lam_all + idx;
    stride = nrows;
    nparts = W;
  }
  // up to 16 loads in flight per thread (the whole split range of c3_7b in one round); two-pass
  // LSE per round (max, then independent exponentials) so no exp2 chain is serial
  float M = -INFINITY, S = 0.f;
  for (int sp0 = w; sp0 < nparts; sp0 += 16 * kSplitWarps) {
    float v[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      const int sp = sp0 + i * kSplitWarps;
      v[i] = sp < nparts ? base[(size_t)sp * stride] : -INFINITY;
    }
    float m = v[0];
#pragma unroll
    for (int i = 1; i < 16; ++i) m = fmaxf(m, v[i]);
    if (m == -INFINITY) continue;
    float t[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
    for (int i = 0; i < 16; ++i) t[i & 3] += fast_exp2(v[i] - m);
    lse2_merge(M, S, m, (t[0] + t[1]) + (t[2] + t[3]));
  }
  sM[w][lane] = M;
  sS[w][lane] = S;
  __syncthreads();
  if (!fullrow && transposed) {
    // transposed merge: warp w merges row w's 32 split-group partials across its lanes (max, then
    // rescaled sum, both by butterfly reductions -- a fixed order, so run-to-run deterministic)
    const int row_w = blockIdx.x * kRowsPerBlock + w;
    if (row_w >= nrows) return;
    const float si = sS[lane][w], mi = si > 0.f ? sM[lane][w] : -INFINITY;
    float Mt = mi;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) Mt = fmaxf(Mt, __shfl_xor_sync(0xffffffffu, Mt, o));
    float St = (Mt != -INFINITY && si > 0.f) ? si * fast_exp2(mi - Mt) : 0.f;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) St += __shfl_xor_sync(0xffffffffu, St, o);
    if (lane == 0) {
      const float lse = (St > 0.f) ? Mt + fast_log2(St) : -INFINITY;
      if (lam_all == nullptr && lam_local_out) lam_local_out[row_w] = lse;
      Lam2[row_w] = lse;
    }
    return;
  }
  if (w != 0) return;
  const int row_idx = blockIdx.x * kRowsPerBlock + lane;
  if (row_idx >= nrows) return;
  // merge the 32 split-warp partials of this row: max first, then independent rescales (fixed order)
  float Mt = -INFINITY;
#pragma unroll 8
  for (int i = 0; i < kSplitWarps; ++i) Mt = fmaxf(Mt, sS[i][lane] > 0.f ? sM[i][lane] : -INFINITY);
  float St = 0.f;
  if (Mt != -INFINITY) {
    float t[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll 8
    for (int i = 0; i < kSplitWarps; ++i) {
      const float si = sS[i][lane];
      if (si > 0.f) t[i & 3] += si * fast_exp2(sM[i][lane] - Mt);
    }
    St = (t[0] + t[1]) + (t[2] + t[3]);
  }
  if (lam_all == nullptr && lam_local_out) lam_local_out[row_idx] = (St > 0.f) ? Mt + fast_log2(St) : -INFINITY;
  if (fullrow) {
    // causal suffix keys t <= r of the same KV head (Q1 FULLROW, Q9)
    const int kvh = row_idx / g.R, row = row_idx % g.R;
    const int gq = row / g.ns, r = row % g.ns, h = kvh * g.G + gq;
    const float scale = kLog2e * rsqrtf((float)g.d);
    const T* qr = q + ((size_t)r * g.Hq + h) * g.d;
    for (int t = 0; t <= r; ++t) {
      const T* kt = ks + ((size_t)t * g.Hkv + kvh) * g.d;
      float acc = 0.f;
      for (int x = 0; x < g.d; ++x) acc = fmaf(to_f(qr[x]), to_f(kt[x]), acc);
      lse2_acc(Mt, St, acc * scale);
    }
  }
  Lam2[row_idx] = (St > 0.f) ? Mt + fast_log2(St) : -INFINITY;
}

// One warp per (kv head, chunk j): lanes take 4 consecutive rows at a time (float4 when
// R % 4 == 0), 4 independent partial sums, then a fixed xor-tree reduce.  Writes the per-KV-head
// partial Apart[kvh][j]; the top-k adds the Hkv partials in a fixed order.
__device__ __forceinline__ void chunk_sum_warp(const LayerGeom& g, const float* __restrict__ lam2,
                                               const float* __restrict__ Lam2, float* __restrict__ Apart, int warp,
                                               int lane) {
  const int kvh = warp / g.m_loc, j = warp % g.m_loc;
  float acc[4] = {0.f, 0.f, 0.f, 0.f};
  const float* src = lam2 + ((size_t)kvh * g.m_loc + j) * g.R;
  const float* L = Lam2 + (size_t)kvh * g.R;
  if ((g.R & 3) == 0) {
#pragma unroll 4
    for (int row = lane * 4; row < g.R; row += 128) {
      const float4 a = *reinterpret_cast<const float4*>(src + row);
      const float4 b = *reinterpret_cast<const float4*>(L + row);
      acc[0] += fast_exp2(a.x - b.x);
      acc[1] += fast_exp2(a.y - b.y);
      acc[2] += fast_exp2(a.z - b.z);
      acc[3] += fast_exp2(a.w - b.w);
    }
  } else {
    for (int row = lane; row < g.R; row += 32) acc[row & 3] += fast_exp2(src[row] - L[row]);
  }
  float s = (acc[0] + acc[1]) + (acc[2] + acc[3]);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if (lane == 0) Apart[warp] = s;
}

// lam2 comes from the score kernel, which is older than this kernel's stream predecessor (the row
// normaliser) and so has completed when this kernel starts (programmatic launch: at most two
// kernels of a stream overlap, common.cuh): its loads are issued BEFORE pdl_wait() and overlap the
// row normaliser; only Lam2 needs the wait.  (R % 4 == 0, R <= 1024: 8 x 16 B per lane in flight.)
__global__ void chunk_sum_kernel(LayerGeom g, const float* __restrict__ lam2, const float* __restrict__ Lam2,
                                 float* __restrict__ Apart) {
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  const bool live = warp < g.m_loc * g.Hkv;
  if (live && (g.R & 3) == 0 && g.R <= 1024) {
    const int kvh = warp / g.m_loc, j = warp % g.m_loc;
    const float* src = lam2 + ((size_t)kvh * g.m_loc + j) * g.R;
    float4 a[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int row = lane * 4 + 128 * i;
      if (row < g.R) a[i] = __ldcg(reinterpret_cast<const float4*>(src + row));
    }
    pdl_wait();
    pdl_trigger();
    const float* L = Lam2 + (size_t)kvh * g.R;
    float acc[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int row = lane * 4 + 128 * i;
      if (row < g.R) {
        const float4 b = *reinterpret_cast<const float4*>(L + row);
        acc[0] += fast_exp2(a[i].x - b.x);
        acc[1] += fast_exp2(a[i].y - b.y);
        acc[2] += fast_exp2(a[i].z - b.z);
        acc[3] += fast_exp2(a[i].w - b.w);
      }
    }
    float sum = (acc[0] + acc[1]) + (acc[2] + acc[3]);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
    if (lane == 0) Apart[warp] = sum;
    return;
  }
  pdl_wait();
  pdl_trigger();
  if (!live) return;
  chunk_sum_warp(g, lam2, Lam2, Apart, warp, lane);
}

const int kReg = register_kernels({(const void*)row_lse_kernel<float>, (const void*)row_lse_kernel<__nv_bfloat16>,
                                   (const void*)chunk_sum_kernel});

}  // namespace

template <typename T>
cudaError_t launch_row_lse(const LayerGeom& g, const float* lampart, int nsplit, const T* q, const T* k_suf,
                           int fullrow, const float* lam_all, int W, float* Lam2, float* lam_local_out,
                           cudaStream_t st) {
  const int n = g.Hkv * g.R;
  static int tr = -1;  // A/B knob: CKV_LSE_SERIAL=1 keeps the one-warp serial merge
  if (tr < 0) tr = (tuning_env("CKV_LSE_SERIAL") && tuning_env("CKV_LSE_SERIAL")[0] == '1') ? 0 : 1;
  if (cudaError_t e_ = launch_kernel(row_lse_kernel<T>, (n + kRowsPerBlock - 1) / kRowsPerBlock, 32 * kSplitWarps, 0, st,
                                     g, lampart, nsplit, q, k_suf, fullrow, lam_all, W, Lam2, lam_local_out, tr))
    return e_;
  return cudaGetLastError();
}
template cudaError_t launch_row_lse<float>(const LayerGeom&, const float*, int, const float*, const float*, int,
                                           const float*, int, float*, float*, cudaStream_t);
template cudaError_t launch_row_lse<__nv_bfloat16>(const LayerGeom&, const float*, int, const __nv_bfloat16*,
                                                   const __nv_bfloat16*, int, const float*, int, float*, float*,
                                                   cudaStream_t);

cudaError_t launch_chunk_sum(const LayerGeom& g, const float* lam2, const float* Lam2, float* Apart,
                             cudaStream_t st) {
  const int threads = 256, warps_per_block = threads / 32;
  const int blocks = (g.m_loc * g.Hkv + warps_per_block - 1) / warps_per_block;
  if (cudaError_t e_ = launch_kernel(chunk_sum_kernel, blocks, threads, 0, st, g, lam2, Lam2, Apart)) return e_;
  return cudaGetLastError();
}

}  // namespace ckv
