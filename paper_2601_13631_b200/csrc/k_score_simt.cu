// A1 score-partial, SIMT (FFMA) variant: used in fp32 mode (no tf32)
// and as the bf16 fallback for shapes outside the tcgen05 kernel.
//
// Computes, for one KV head, every logit l = q.k / sqrt(d) of the G*n_s suffix rows
// against the shard's prefix keys (PAPER.md:99, 429 with Q3's 1/sqrt(d)), and for each
// (row, chunk) the base-2 log-sum-exp   lam2 = log2 sum_{i in chunk j} 2^(l_i * log2 e)
// (chunk j = tokens [j c, min((j+1)c, n)), Eq. 1 / Q5-Q6), plus a per-(row, split)
// partial of the row normaliser.  A2 finishes A_j = sum_rows 2^(lam2 - Lambda2).
#include "common.cuh"

namespace ckv {
namespace {

constexpr int RB = 64;   // rows per CTA
constexpr int KB = 64;   // keys per sub-tile
constexpr int NT = 256;  // threads

template <typename T>
__global__ void __launch_bounds__(NT) score_simt_kernel(LayerGeom g, const T* __restrict__ q,
                                                        const T* __restrict__ probe, float* __restrict__ lam2,
                                                        float* __restrict__ lampart, int nsplit) {
  pdl_wait();
  pdl_trigger();
  extern __shared__ float sm[];
  const int d = g.d;
  float* Qt = sm;                 // [d][RB]
  float* Kt = Qt + d * RB;        // [d][KB]
  float* S = Kt + d * KB;         // [RB][KB + 1]
  const int kvh = blockIdx.z, split = blockIdx.y, row0 = blockIdx.x * RB;
  const int tid = threadIdx.x;
  const int cps = (g.m_loc + nsplit - 1) / nsplit;
  const int cj0 = split * cps, cj1 = min(g.m_loc, cj0 + cps);
  const int key0 = cj0 * g.c, key1 = min(g.n_loc, cj1 * g.c);
  const float scale = kLog2e * rsqrtf((float)d);

  // Q tile, transposed to [d][RB]; row rho = gq * ns + r -> head kvh * G + gq
  for (int e = tid; e < RB * d; e += NT) {
    int rr = e / d, x = e % d, rho = row0 + rr;
    float val = 0.f;
    if (rho < g.R) {
      int gq = rho / g.ns, r = rho % g.ns;
      val = to_f(q[((size_t)r * g.Hq + kvh * g.G + gq) * d + x]);
    }
    Qt[x * RB + rr] = val;
  }
  // per-row walk state (threads 0..RB-1)
  int cur = -1;
  float mx = -INFINITY, s = 0.f;
  float pm = -INFINITY, ps = 0.f;  // row partial LSE over flushed chunks
  const int my_row = row0 + tid;
  const T* kbase = probe + (size_t)kvh * g.n_pad * d;
  const int ty = tid / 16, tx = tid % 16;

  for (int kb = key0; kb < key1; kb += KB) {
    __syncthreads();
    for (int e = tid; e < KB * d; e += NT) {
      int kk = e / d, x = e % d, i = kb + kk;
      Kt[x * KB + kk] = (i < key1) ? to_f(kbase[(size_t)i * d + x]) : 0.f;
    }
    __syncthreads();
    float acc[4][4] = {};
    for (int x = 0; x < d; ++x) {
      float4 a = *reinterpret_cast<const float4*>(&Qt[x * RB + ty * 4]);
      float4 b = *reinterpret_cast<const float4*>(&Kt[x * KB + tx * 4]);
      float av[4] = {a.x, a.y, a.z, a.w}, bv[4] = {b.x, b.y, b.z, b.w};
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(av[i], bv[j], acc[i][j]);
    }
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) S[(ty * 4 + i) * (KB + 1) + tx * 4 + j] = acc[i][j];
    __syncthreads();
    if (KB % g.c == 0) {
      // chunks align to the 64-key sub-tiles (c | 64; kb is a multiple of c): every thread takes
      // whole (row, chunk) items -- max, exponentials and sum of the chunk's c logits -- and the
      // row threads fold the sub-tile's chunk values into the split's row partial
      float* Lc = Kt;  // [KB / c][RB] chunk values of this sub-tile (K tile no longer needed)
      const int cpt = KB / g.c;
      for (int it = tid; it < RB * cpt; it += NT) {
        const int rr = it % RB, cc = it / RB, kk0 = cc * g.c;
        const int kend = min(g.c, key1 - kb - kk0);
        float l2 = -INFINITY;
        if (kend > 0 && row0 + rr < g.R) {
          const float* srow = S + rr * (KB + 1) + kk0;
          float m = srow[0];
          for (int t = 1; t < kend; ++t) m = fmaxf(m, srow[t]);
          m *= scale;
          float sum = 0.f;
          for (int t = 0; t < kend; ++t) sum += fast_exp2(fmaf(srow[t], scale, -m));
          l2 = m + fast_log2(sum);
          lam2[((size_t)kvh * g.m_loc + (kb + kk0) / g.c) * g.R + row0 + rr] = l2;
        }
        Lc[cc * RB + rr] = l2;
      }
      __syncthreads();
      if (tid < RB && my_row < g.R) {
        for (int cc = 0; cc < cpt; ++cc) {
          const float l2 = Lc[cc * RB + tid];
          if (l2 == -INFINITY) continue;
          const float nm = fmaxf(pm, l2);
          ps = ps * fast_exp2(pm - nm) + fast_exp2(l2 - nm);
          pm = nm;
        }
      }
      continue;
    }
    if (tid < RB && my_row < g.R) {
      const int kend = min(KB, key1 - kb);
      for (int kk = 0; kk < kend; ++kk) {
        const int i = kb + kk;
        const int ch = i / g.c;
        const float x = S[tid * (KB + 1) + kk] * scale;
        if (ch != cur) {
          if (cur >= 0) {
            float l2 = mx + fast_log2(s);
            lam2[((size_t)kvh * g.m_loc + cur) * g.R + my_row] = l2;
            float nm = fmaxf(pm, l2);
            ps = ps * fast_exp2(pm - nm) + fast_exp2(l2 - nm);
            pm = nm;
          }
          cur = ch;
          mx = x;
          s = 1.f;
        } else if (x > mx) {
          s = s * fast_exp2(mx - x) + 1.f;
          mx = x;
        } else {
          s += fast_exp2(x - mx);
        }
      }
    }
  }
  if (tid < RB && my_row < g.R) {
    if (cur >= 0) {
      float l2 = mx + fast_log2(s);
      lam2[((size_t)kvh * g.m_loc + cur) * g.R + my_row] = l2;
      float nm = fmaxf(pm, l2);
      ps = ps * fast_exp2(pm - nm) + fast_exp2(l2 - nm);
      pm = nm;
    }
    lampart[((size_t)kvh * nsplit + split) * g.R + my_row] = (ps > 0.f) ? pm + fast_log2(ps) : -INFINITY;
  }
}

const int kReg = register_kernels({(const void*)score_simt_kernel<float>, (const void*)score_simt_kernel<__nv_bfloat16>});

}  // namespace

template <typename T>
cudaError_t launch_score_simt(const LayerGeom& g, const T* q, const T* probe_layer, float* lam2, float* lampart,
                              int nsplit, cudaStream_t st) {
  if (g.d % 4 != 0 || g.d > 128) return cudaErrorNotSupported;
  size_t smem = sizeof(float) * ((size_t)g.d * RB + (size_t)g.d * KB + (size_t)RB * (KB + 1));
  auto kfn = score_simt_kernel<T>;
  static int attr_done = 0;  // per template instance; set before any graph capture
  if (!attr_done) {
    cudaError_t e = cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, 48 * 1024 * 4);
    if (e != cudaSuccess) return e;
    attr_done = 1;
  }
  dim3 grid((g.R + RB - 1) / RB, nsplit, g.Hkv);
  if (cudaError_t e_ = launch_kernel(kfn, grid, NT, smem, st, g, q, probe_layer, lam2, lampart, nsplit)) return e_;
  return cudaGetLastError();
}

template cudaError_t launch_score_simt<float>(const LayerGeom&, const float*, const float*, float*, float*, int,
                                              cudaStream_t);
template cudaError_t launch_score_simt<__nv_bfloat16>(const LayerGeom&, const __nv_bfloat16*,
                                                      const __nv_bfloat16*, float*, float*, int, cudaStream_t);

}  // namespace ckv
