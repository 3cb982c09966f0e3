// A7 split-K exact attention (SIMT variant) and A8 LSE combine / cross-shard merge.
//
// Every suffix row attends, exactly, over the kept prefix chunks (all visible; padding
// of a partial last chunk masked, Q6) plus the causal suffix keys t <= r (Q9):
//   O = sum_k softmax_k(q.k / sqrt(d)) v_k      (Def. 1 at PAPER.md:159).
// Rows are GQA-packed per KV head (rho = g * n_s + r).  The key list is split across
// CTAs; each split writes a normalised partial O and its base-2 LSE, merged by
//   O = sum_s 2^(lse_s - M) O_s / sum_s 2^(lse_s - M).
#include "common.cuh"

namespace ckv {
namespace {

constexpr int RB = 64;
constexpr int KB = 64;
constexpr int NT = 256;

template <typename T>
__global__ void __launch_bounds__(NT) attn_simt_kernel(LayerGeom g, const T* __restrict__ q, const T* __restrict__ ks,
                                                       const T* __restrict__ vs, const T* __restrict__ pool,
                                                       int64_t rec_elems, const int32_t* __restrict__ kept_slots,
                                                       const int32_t* __restrict__ kept_ids,
                                                       const int32_t* __restrict__ n_kept_dev, int k_cap,
                                                       int include_suffix, int nsplit, float* __restrict__ o_part,
                                                       float* __restrict__ lse_part) {
  pdl_wait();
  pdl_trigger();
  extern __shared__ float sm[];
  const int d = g.d;
  float* Qt = sm;               // [d][RB]
  float* Kt = Qt + d * RB;      // [d][KB]
  float* Vs = Kt + d * KB;      // [KB][d]
  float* S = Vs + KB * d;       // [RB][KB+1]
  float* row_m = S + RB * (KB + 1);
  float* row_l = row_m + RB;
  float* row_a = row_l + RB;
  int* kmeta = reinterpret_cast<int*>(row_a + RB);  // [KB]: -2 invalid, -1 prefix, >=0 suffix token

  const int kvh = blockIdx.z, sp = blockIdx.y, row0 = blockIdx.x * RB, tid = threadIdx.x;
  const int n_kept = *n_kept_dev;
  const int cps = (k_cap + nsplit - 1) / nsplit;
  const int t0 = min(n_kept, sp * cps), t1 = min(n_kept, t0 + cps);
  const int npre = (t1 - t0) * g.c;
  const int nkeys = npre + ((include_suffix && sp == nsplit - 1) ? g.ns : 0);
  const float scale = kLog2e * rsqrtf((float)d);

  for (int e = tid; e < RB * d; e += NT) {
    int rr = e / d, x = e % d, rho = row0 + rr;
    float val = 0.f;
    if (rho < g.R) {
      int gq = rho / g.ns, r = rho % g.ns;
      val = to_f(q[((size_t)r * g.Hq + kvh * g.G + gq) * d + x]);
    }
    Qt[x * RB + rr] = val;
  }
  if (tid < RB) {
    row_m[tid] = -INFINITY;
    row_l[tid] = 0.f;
  }
  const int ty = tid / 16, tx = tid % 16;
  const int DPT = d / 16;
  float acc[4][8];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 8; ++j) acc[i][j] = 0.f;

  for (int kb = 0; kb < nkeys; kb += KB) {
    __syncthreads();
    if (tid < KB) {
      const int p = kb + tid;
      int meta = -2;
      if (p < npre) {
        const int t = t0 + p / g.c, off = p % g.c;
        if ((int64_t)kept_ids[t] * g.c + off < g.n_loc) meta = -1;
      } else if (p < nkeys) {
        meta = p - npre;
      }
      kmeta[tid] = meta;
    }
    for (int e = tid; e < KB * d; e += NT) {
      const int kk = e / d, x = e % d, p = kb + kk;
      float kv = 0.f, vv = 0.f;
      if (p < npre) {
        const int t = t0 + p / g.c, off = p % g.c;
        const T* rec = pool + (int64_t)kept_slots[t] * rec_elems;
        kv = to_f(rec[rec_elem(g.rec_swz, 0, kvh, off, x, g.Hkv, g.c, d)]);
        vv = to_f(rec[rec_elem(g.rec_swz, 1, kvh, off, x, g.Hkv, g.c, d)]);
      } else if (p < nkeys) {
        const int ts = p - npre;
        kv = to_f(ks[((int64_t)ts * g.Hkv + kvh) * d + x]);
        vv = to_f(vs[((int64_t)ts * g.Hkv + kvh) * d + x]);
      }
      Kt[x * KB + kk] = kv;
      Vs[kk * d + x] = vv;
    }
    __syncthreads();
    {
      float sacc[4][4] = {};
      for (int x = 0; x < d; ++x) {
        float4 a = *reinterpret_cast<const float4*>(&Qt[x * RB + ty * 4]);
        float4 b = *reinterpret_cast<const float4*>(&Kt[x * KB + tx * 4]);
        float av[4] = {a.x, a.y, a.z, a.w}, bv[4] = {b.x, b.y, b.z, b.w};
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int j = 0; j < 4; ++j) sacc[i][j] = fmaf(av[i], bv[j], sacc[i][j]);
      }
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int rho = row0 + ty * 4 + i;
        const int r = rho % g.ns;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const int meta = kmeta[tx * 4 + j];
          const bool ok = (meta == -1) || (meta >= 0 && meta <= r);
          S[(ty * 4 + i) * (KB + 1) + tx * 4 + j] = ok ? sacc[i][j] * scale : -INFINITY;
        }
      }
    }
    __syncthreads();
    {  // online softmax: 4 threads per row, 16 keys each
      const int rr = tid >> 2, part = tid & 3;
      float* srow = S + rr * (KB + 1) + part * 16;
      float mx = -INFINITY;
#pragma unroll
      for (int i = 0; i < 16; ++i) mx = fmaxf(mx, srow[i]);
      mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 1));
      mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 2));
      const float m_old = row_m[rr];
      const float m_new = fmaxf(m_old, mx);
      float sum = 0.f;
      if (m_new == -INFINITY) {
#pragma unroll
        for (int i = 0; i < 16; ++i) srow[i] = 0.f;
      } else {
#pragma unroll
        for (int i = 0; i < 16; ++i) {
          const float p = fast_exp2(srow[i] - m_new);
          srow[i] = p;
          sum += p;
        }
      }
      sum += __shfl_xor_sync(0xffffffffu, sum, 1);
      sum += __shfl_xor_sync(0xffffffffu, sum, 2);
      __syncwarp();
      if (part == 0) {
        const float alpha = (m_old == -INFINITY) ? 0.f : fast_exp2(m_old - m_new);
        row_a[rr] = alpha;
        row_l[rr] = row_l[rr] * alpha + sum;
        row_m[rr] = m_new;
      }
    }
    __syncthreads();
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const float a = row_a[ty * 4 + i];
#pragma unroll
      for (int j = 0; j < 8; ++j) acc[i][j] *= a;
    }
    for (int kk = 0; kk < KB; ++kk) {
      float pv[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) pv[i] = S[(ty * 4 + i) * (KB + 1) + kk];
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        if (j < DPT) {
          const float v = Vs[kk * d + tx * DPT + j];
#pragma unroll
          for (int i = 0; i < 4; ++i) acc[i][j] = fmaf(pv[i], v, acc[i][j]);
        }
      }
    }
  }
  __syncthreads();
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int rr = ty * 4 + i, rho = row0 + rr;
    if (rho >= g.R) continue;
    const float l = row_l[rr];
    const float inv = (l > 0.f) ? 1.f / l : 0.f;
    float* dst = o_part + (((int64_t)sp * g.Hkv + kvh) * g.R + rho) * d;
#pragma unroll
    for (int j = 0; j < 8; ++j)
      if (j < DPT) dst[tx * DPT + j] = acc[i][j] * inv;
    if (tx == 0) lse_part[((int64_t)sp * g.Hkv + kvh) * g.R + rho] = (l > 0.f) ? row_m[rr] + fast_log2(l) : -INFINITY;
  }
}

// Merge of split partials, one warp per row (input row (kvh, rho = g*ns + r), output row
// (r, h)): the split weights 2^(lse_s - M) are computed once per lane-split and broadcast;
// each lane owns d/32 contiguous output columns (float4 loads when d % 128 == 0).
template <typename T>
__global__ void attn_combine_kernel(LayerGeom g, const float* __restrict__ o_part, const float* __restrict__ lse_part,
                                    int nsplit, T* __restrict__ out, float* __restrict__ o_f32,
                                    float* __restrict__ lse_nat, XPartDst xd) {
  pdl_wait();
  pdl_trigger();
  const int row = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;  // kvh * R + rho
  const int lane = threadIdx.x & 31;
  const int64_t nrow = (int64_t)g.Hkv * g.R;
  if (row >= nrow) return;
  const int kvh = row / g.R, rho = row % g.R;
  const int gq = rho / g.ns, r = rho % g.ns, h = kvh * g.G + gq;
  // d = 128, <= 8 splits: the partial O loads are issued first, so their L2 round trip overlaps
  // the LSE loads and the weight reduction (empty splits' partials are loaded but never used)
  const bool d128 = g.d == 128 && nsplit <= 8;
  float4 v[8];
  if (d128) {
#pragma unroll
    for (int sp = 0; sp < 8; ++sp)
      if (sp < nsplit) v[sp] = __ldcg(reinterpret_cast<const float4*>(o_part + (sp * nrow + row) * g.d + lane * 4));
  }
  // lane s < nsplit holds split s's lse (nsplit <= 64: two rounds)
  float l0 = (lane < nsplit) ? lse_part[lane * nrow + row] : -INFINITY;
  float l1 = (lane + 32 < nsplit) ? lse_part[(lane + 32) * nrow + row] : -INFINITY;
  float M = fmaxf(l0, l1);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) M = fmaxf(M, __shfl_xor_sync(0xffffffffu, M, o));
  const float w0 = (l0 == -INFINITY) ? 0.f : fast_exp2(l0 - M);
  const float w1 = (l1 == -INFINITY) ? 0.f : fast_exp2(l1 - M);
  float den = w0 + w1;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) den += __shfl_xor_sync(0xffffffffu, den, o);
  const int64_t obase = ((int64_t)r * g.Hq + h) * g.d;
  const float inv = den > 0.f ? 1.f / den : 0.f;
  // fp32 row destination: the caller's o_f32, or (fused exchange) slot `self` of the window of the
  // rank that merges this row's slice (reduce-scatter over output rows, xchg.cuh)
  if (xd.xp.W > 0) {
    const int row_out = r * g.Hq + h, s = row_out / xd.rps, lr = row_out - s * xd.rps;
    char* wb = xd.xp.base[s];
    o_f32 = reinterpret_cast<float*>(wb + xd.part_o) + ((size_t)xd.xp.self * xd.rps_max + lr) * g.d - obase;
    lse_nat = reinterpret_cast<float*>(wb + xd.part_lse) + (size_t)xd.xp.self * xd.rps_max + lr - row_out;
  }
  if ((g.d & 127) == 0 && nsplit <= 8) {
    // all split loads issued before the weighted sum (independent 16-byte loads in flight)
    for (int x = lane * 4; x < g.d; x += 128) {
      if (!d128) {
#pragma unroll
        for (int sp = 0; sp < 8; ++sp)
          if (sp < nsplit) v[sp] = __ldcg(reinterpret_cast<const float4*>(o_part + (sp * nrow + row) * g.d + x));
      }
      float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
      for (int sp = 0; sp < 8; ++sp) {
        if (sp >= nsplit) break;
        const float w = __shfl_sync(0xffffffffu, w0, sp);
        if (w == 0.f) continue;  // empty split (its partial is not written)
        acc.x += w * v[sp].x;
        acc.y += w * v[sp].y;
        acc.z += w * v[sp].z;
        acc.w += w * v[sp].w;
      }
      const float o4[4] = {acc.x * inv, acc.y * inv, acc.z * inv, acc.w * inv};
      if (out) {
        if constexpr (sizeof(T) == 2) {
          __nv_bfloat162 b0 = __floats2bfloat162_rn(o4[0], o4[1]), b1 = __floats2bfloat162_rn(o4[2], o4[3]);
          uint2 u;
          u.x = *reinterpret_cast<uint32_t*>(&b0);
          u.y = *reinterpret_cast<uint32_t*>(&b1);
          *reinterpret_cast<uint2*>(out + obase + x) = u;
        } else {
#pragma unroll
          for (int i = 0; i < 4; ++i) out[obase + x + i] = from_f<T>(o4[i]);
        }
      }
      if (o_f32) *reinterpret_cast<float4*>(o_f32 + obase + x) = make_float4(o4[0], o4[1], o4[2], o4[3]);
    }
  } else if ((g.d & 127) == 0) {
    for (int x = lane * 4; x < g.d; x += 128) {
      float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
      for (int sp = 0; sp < nsplit; ++sp) {
        const float w = __shfl_sync(0xffffffffu, sp < 32 ? w0 : w1, sp & 31);
        if (w == 0.f) continue;
        const float4 v = *reinterpret_cast<const float4*>(o_part + (sp * nrow + row) * g.d + x);
        acc.x += w * v.x;
        acc.y += w * v.y;
        acc.z += w * v.z;
        acc.w += w * v.w;
      }
      const float o4[4] = {acc.x * inv, acc.y * inv, acc.z * inv, acc.w * inv};
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        if (out) out[obase + x + i] = from_f<T>(o4[i]);
        if (o_f32) o_f32[obase + x + i] = o4[i];
      }
    }
  } else {
    for (int x = lane; x < g.d; x += 32) {
      float num = 0.f;
      for (int sp = 0; sp < nsplit; ++sp) {
        const float w = __shfl_sync(0xffffffffu, sp < 32 ? w0 : w1, sp & 31);
        if (w != 0.f) num += w * o_part[(sp * nrow + row) * g.d + x];
      }
      if (out) out[obase + x] = from_f<T>(num * inv);
      if (o_f32) o_f32[obase + x] = num * inv;
    }
  }
  if (lse_nat && lane == 0) lse_nat[(int64_t)r * g.Hq + h] = den > 0.f ? (M + log2f(den)) * kLn2 : -INFINITY;
}

__global__ void lse_merge_prepare_kernel(int rows, int d, const float* __restrict__ o, const float* __restrict__ lse,
                                         const float* __restrict__ lse_max, float* __restrict__ buf) {
  pdl_wait();
  pdl_trigger();
  const int i = blockIdx.x;
  if (i >= rows) return;
  const float l = lse[i], M = lse_max[i];
  const float w = (l == -INFINITY) ? 0.f : __expf(l - M);
  for (int x = threadIdx.x; x < d; x += blockDim.x) buf[(int64_t)i * (d + 1) + x] = o[(int64_t)i * d + x] * w;
  if (threadIdx.x == 0) buf[(int64_t)i * (d + 1) + d] = w;
}

template <typename T>
__global__ void lse_merge_finish_kernel(int rows, int d, const float* __restrict__ buf, T* __restrict__ out) {
  pdl_wait();
  pdl_trigger();
  const int i = blockIdx.x;
  if (i >= rows) return;
  const float den = buf[(int64_t)i * (d + 1) + d];
  for (int x = threadIdx.x; x < d; x += blockDim.x)
    out[(int64_t)i * d + x] = from_f<T>(den > 0.f ? buf[(int64_t)i * (d + 1) + x] / den : 0.f);
}

const int kReg = register_kernels({(const void*)attn_simt_kernel<float>, (const void*)attn_simt_kernel<__nv_bfloat16>,
                                   (const void*)attn_combine_kernel<float>, (const void*)attn_combine_kernel<__nv_bfloat16>,
                                   (const void*)lse_merge_prepare_kernel, (const void*)lse_merge_finish_kernel<float>,
                                   (const void*)lse_merge_finish_kernel<__nv_bfloat16>});

}  // namespace

template <typename T>
cudaError_t launch_attn_simt(const LayerGeom& g, const T* q, const T* k_suf, const T* v_suf, const T* pool_layer,
                             int64_t rec_elems, const int32_t* kept_slots, const int32_t* kept_ids,
                             const int32_t* n_kept_dev, int k_cap, int include_suffix, int nsplit, float* o_part,
                             float* lse_part, cudaStream_t st) {
  if (g.d % 16 != 0 || g.d > 128) return cudaErrorNotSupported;
  size_t smem = sizeof(float) * ((size_t)g.d * RB + (size_t)g.d * KB + (size_t)KB * g.d + RB * (KB + 1) + 3 * RB) +
                sizeof(int) * KB;
  auto kfn = attn_simt_kernel<T>;
  static int attr_done = 0;  // per template instance; set before any graph capture
  if (!attr_done) {
    cudaError_t e = cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, 48 * 1024 * 4);
    if (e != cudaSuccess) return e;
    attr_done = 1;
  }
  dim3 grid((g.R + RB - 1) / RB, nsplit, g.Hkv);
  if (cudaError_t e_ = launch_kernel(kfn, grid, NT, smem, st, g, q, k_suf, v_suf, pool_layer, rec_elems, kept_slots, kept_ids, n_kept_dev, k_cap,
                              include_suffix, nsplit, o_part, lse_part)) return e_;
  return cudaGetLastError();
}

template <typename T>
cudaError_t launch_attn_combine(const LayerGeom& g, const float* o_part, const float* lse_part, int nsplit, T* out,
                                float* o_f32, float* lse_nat, cudaStream_t st, const XPartDst* xd) {
  XPartDst x{};
  if (xd) x = *xd;
  if (cudaError_t e_ = launch_kernel(attn_combine_kernel<T>, (g.Hkv * g.R + 7) / 8, 256, 0, st, g, o_part, lse_part,
                                     nsplit, out, o_f32, lse_nat, x))
    return e_;
  return cudaGetLastError();
}

cudaError_t launch_lse_merge_prepare(int rows, int d, const float* o, const float* lse, const float* lse_max,
                                     float* buf, cudaStream_t st) {
  if (cudaError_t e_ = launch_kernel(lse_merge_prepare_kernel, rows, 128, 0, st, rows, d, o, lse, lse_max, buf)) return e_;
  return cudaGetLastError();
}

template <typename T>
cudaError_t launch_lse_merge_finish(int rows, int d, const float* buf, T* out, cudaStream_t st) {
  if (cudaError_t e_ = launch_kernel(lse_merge_finish_kernel<T>, rows, 128, 0, st, rows, d, buf, out)) return e_;
  return cudaGetLastError();
}

#define CKV_INST(T)                                                                                                 \
  template cudaError_t launch_attn_simt<T>(const LayerGeom&, const T*, const T*, const T*, const T*, int64_t,       \
                                           const int32_t*, const int32_t*, const int32_t*, int, int, int, float*,   \
                                           float*, cudaStream_t);                                                   \
  template cudaError_t launch_attn_combine<T>(const LayerGeom&, const float*, const float*, int, T*, float*, float*, \
                                              cudaStream_t, const XPartDst*);                                                        \
  template cudaError_t launch_lse_merge_finish<T>(int, int, const float*, T*, cudaStream_t);
CKV_INST(float)
CKV_INST(__nv_bfloat16)
#undef CKV_INST

}  // namespace ckv
