// A4 cache plan, A5 whole-chunk gather, A9 cache-score update, and the store-prefix
// layout kernels.
//
// HBM chunk cache (§4.4, 424-455): per (layer, chunk) the cumulative importance
// I_j and access count F_j live in a table that survives eviction; the
// cache score is S_j = I_j * F_j (Eq. 2).  Selected chunks are checked
// against the cache before loading; misses take free slots first, then the
// slots of the lowest-(S, j) residents that are neither requested nor pinned by an
// in-flight prefetch ("Both heaps will evict low-scored ContiguousChunks").
// Every transfer moves one whole chunk record (unit of storage = unit of transfer =
// unit of eviction), so read amplification is 1.
#include "common.cuh"
#include <cstdlib>

#include "plan.cuh"

namespace ckv {
namespace {

constexpr int NT = 1024;

__global__ void __launch_bounds__(NT) cache_plan_kernel(CacheLayer cl, const int32_t* __restrict__ ids,
                                                        const int32_t* __restrict__ n_ids_dev, int n_ids_host,
                                                        int prefetch, int quota, int epoch, int64_t rec_bytes,
                                                        int32_t* __restrict__ scratch, PlanOut out) {
  pdl_wait();
  pdl_trigger();
  __shared__ PlanSmem ps;
  extern __shared__ uint64_t plan_skeys[];
  const int n_ids = n_ids_dev ? *n_ids_dev : n_ids_host;
  const bool smem_keys = cl.P > NT * kPlanKPT && cl.P <= kPlanSmemKeysMax;
  cache_plan_body<NT>(cl, ids, n_ids, prefetch, quota, epoch, rec_bytes, scratch, out, ps,
                      smem_keys ? plan_skeys : nullptr);
}

// Two plans in one launch (CTA 0: job a, CTA 1: job b) on disjoint per-layer pools: this layer's
// demand plan and the next layer's speculative plan, so the speculation needs no single-CTA
// planner on the side stream (which could not share an SM with the next layer's persistent score
// kernel and so ran only after it).
__global__ void __launch_bounds__(NT) cache_plan2_kernel(PlanJob a, PlanJob b) {
  pdl_wait();
  pdl_trigger();
  __shared__ PlanSmem ps;
  extern __shared__ uint64_t plan_skeys[];
  const PlanJob& j = blockIdx.x == 0 ? a : b;
  const int n_ids = j.n_ids_dev ? *j.n_ids_dev : j.n_ids_host;
  const bool smem_keys = j.cl.P > NT * kPlanKPT && j.cl.P <= kPlanSmemKeysMax;
  cache_plan_body<NT>(j.cl, j.ids, n_ids, j.prefetch, j.quota, j.epoch, j.rec_bytes, j.scratch, j.out, ps,
                      smem_keys ? plan_skeys : nullptr);
}

// A3 + the two plans above in one launch: the top-k is single-CTA work, so both CTAs compute it
// (same keys, same result) instead of a separate one-CTA launch whose completion the plans would
// wait for -- one kernel boundary less on the layer's serial chain.
// Shared-memory layout of the table copies: ids [k], A, slot_of, I, F [m], owner, pf_epoch [P] (4-byte words).
inline size_t tables_smem_bytes(int k, int m, int P) { return 4 * ((size_t)k + 4 * (size_t)m + 2 * (size_t)P); }

template <int KPT>
__global__ void __launch_bounds__(NT) topk_plan2_kernel(TopkJob t, PlanJob a, PlanJob b, int use_tables) {
  __shared__ PlanSmem ps;
  extern __shared__ uint64_t plan_skeys[];
  const bool c0 = blockIdx.x == 0;
  const PlanJob& j = c0 ? a : b;
  PlanTables tc;
  float* As = nullptr;
  int32_t* ids_s = nullptr;
  if (use_tables) {  // this CTA's layer tables -> shared memory, asynchronously, while the top-k runs
    int32_t* w = reinterpret_cast<int32_t*>(plan_skeys);
    ids_s = w;
    As = reinterpret_cast<float*>(w + t.k);
    int32_t* sl = w + t.k + t.m;
    float* sI = reinterpret_cast<float*>(sl + t.m);
    int32_t* sF = sl + 2 * t.m;
    int32_t* so = sl + 3 * t.m;
    int32_t* sp = so + j.cl.P;
    for (int i = threadIdx.x; i < t.m; i += NT) {
      cp_async4(sl + i, j.cl.slot_of + i);
      cp_async4(sI + i, j.cl.I + i);
      cp_async4(sF + i, j.cl.F + i);
    }
    for (int i = threadIdx.x; i < j.cl.P; i += NT) {
      cp_async4(so + i, j.cl.owner + i);
      cp_async4(sp + i, j.cl.pf_epoch + i);
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
    // (issued before pdl_wait: the tables' last writers -- the previous request's plans and the
    // speculative plan of this layer, CTA 1 of the previous layer's launch -- are older than this
    // kernel's stream predecessor, the chunk sums, so they have completed)
    tc.ids = ids_s;
    tc.A = As;
    tc.slot_of = sl;
    tc.I = sI;
    tc.F = sF;
    tc.owner = so;
    tc.pf_epoch = sp;
  }
  pdl_wait();
  pdl_trigger();
  dtl_mark(1);
  topk_body<NT, KPT>(c0 ? t.A : nullptr, t.Apart, t.nparts, t.m, t.k, 0, 1, c0 ? t.ids : t.ids_b, c0 ? t.cand : t.cand_b,
                     t.k, c0 ? t.n_out : t.n_b, ps.ss, As, ids_s);
  if (use_tables) asm volatile("cp.async.wait_all;" ::: "memory");
  __syncthreads();  // this CTA's ids / n / keys (and CTA 0's A, read by the fused A9) are written
  dtl_mark(2);
  const int n_ids = use_tables ? min(t.k, t.m) : (j.n_ids_dev ? *j.n_ids_dev : j.n_ids_host);
  const bool smem_keys = !use_tables && j.cl.P > NT * kPlanKPT && j.cl.P <= kPlanSmemKeysMax;
  cache_plan_body<NT>(j.cl, j.ids, n_ids, j.prefetch, j.quota, j.epoch, j.rec_bytes, j.scratch, j.out, ps,
                      smem_keys ? plan_skeys : nullptr, tc);
  __syncthreads();
  dtl_mark(3);
}

// Whole-record copy host store -> HBM slot: work items are 4 KiB segments of records so a
// few misses still keep many 16-B loads in flight over the host link.  Small CTAs (4 warps,
// <= 64 registers): one fits on an SM beside a persistent score / attention CTA (576 threads x
// 96 registers), so a side-stream prefetch never holds an SM the next layer's persistent
// kernels need (a blocked SM would delay their whole statically partitioned launch).
constexpr int GATHER_SEG = 4096;
constexpr int GATHER_THREADS = 128;
constexpr int GATHER_BLOCKS = 128;

__global__ void __launch_bounds__(GATHER_THREADS, 8) gather_kernel(const int32_t* __restrict__ list,
                                                                const int32_t* __restrict__ n_load,
                                                                const char* __restrict__ host_layer,
                                                                char* __restrict__ pool_layer, int64_t rec_bytes) {
  pdl_wait();
  pdl_trigger();
  const int n = *n_load;
  if (n == 0) return;
  const int nseg = (int)((rec_bytes + GATHER_SEG - 1) / GATHER_SEG);
  const int total = n * nseg;
  const int lane = threadIdx.x & 31;
  const int warp = (blockIdx.x * GATHER_THREADS + threadIdx.x) >> 5;
  const int nwarps = (gridDim.x * GATHER_THREADS) >> 5;
  for (int it = warp; it < total; it += nwarps) {
    const int e = it / nseg, sg = it % nseg;
    const int j = list[2 * e], s = list[2 * e + 1];
    const int64_t off = (int64_t)sg * GATHER_SEG;
    const int cnt = (int)(min((int64_t)GATHER_SEG, rec_bytes - off) / 16);
    const int4* src = reinterpret_cast<const int4*>(host_layer + (int64_t)j * rec_bytes + off);
    int4* dst = reinterpret_cast<int4*>(pool_layer + (int64_t)s * rec_bytes + off);
    int4 v[GATHER_SEG / 16 / 32];
#pragma unroll
    for (int u = 0; u < GATHER_SEG / 16 / 32; ++u) {
      const int i = lane + 32 * u;
      if (i < cnt) v[u] = __ldg(src + i);
    }
#pragma unroll
    for (int u = 0; u < GATHER_SEG / 16 / 32; ++u) {
      const int i = lane + 32 * u;
      if (i < cnt) dst[i] = v[u];
    }
  }
}

__global__ void cache_update_kernel(CacheLayer cl, const int32_t* __restrict__ ids, const int32_t* n_ids_dev,
                                    const float* __restrict__ A, int tick) {
  pdl_wait();
  pdl_trigger();
  const int n = *n_ids_dev;
  for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < n; t += gridDim.x * blockDim.x) {
    const int j = ids[t];
    cl.I[j] += A[j];  // I_j = I_j + A_j
    cl.F[j] += 1;     // F_j: access count
    cl.T[j] = tick;   // last use (LRU ablation policy)
  }
}

template <typename T>
__global__ void pack_probe_kernel(const T* __restrict__ k, int64_t t0, int cyc_W, int cyc_g, int c, int n_loc,
                                  int n_pad, int Hkv, int d, T* __restrict__ probe) {
  pdl_wait();
  pdl_trigger();
  // probe[kvh][i][x] = k[t0 + i][kvh][x]
  const int64_t total = (int64_t)Hkv * n_loc * d;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int x = (int)(e % d);
    const int64_t r = e / d;
    const int i = (int)(r % n_loc), kvh = (int)(r / n_loc);
    probe[((int64_t)kvh * n_pad + i) * d + x] = k[(shard_token(i, t0, cyc_W, cyc_g, c) * Hkv + kvh) * d + x];
  }
}

template <typename T>
__global__ void pack_records_kernel(const T* __restrict__ k, const T* __restrict__ v, int64_t t0, int cyc_W,
                                    int cyc_g, int n_loc,
                                    int m_loc, int c, int Hkv, int d, int swz, T* __restrict__ rec) {
  pdl_wait();
  pdl_trigger();
  // one record per chunk j (layout: rec_elem), zero padding past n_loc
  const int nkv = swz == 2 ? 1 : 2;  // V-only records hold V alone
  const int64_t per = (int64_t)nkv * Hkv * c * d;
  const int64_t total = (int64_t)m_loc * per;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int j = (int)(e / per);
    int64_t r = e % per;
    const int x = (int)(r % d); r /= d;
    const int p = (int)(r % c); r /= c;
    const int kvh = (int)(r % Hkv);
    const int kv = swz == 2 ? 1 : (int)(r / Hkv);
    const int64_t i = (int64_t)j * c + p;
    T val = from_f<T>(0.f);
    if (i < n_loc) val = (kv == 0 ? k : v)[(shard_token(i, t0, cyc_W, cyc_g, c) * Hkv + kvh) * d + x];
    rec[(int64_t)j * per + rec_elem(swz, kv, kvh, p, x, Hkv, c, d)] = val;
  }
}

__global__ void epoch_inc_kernel(int32_t* e) {
  pdl_wait();
  pdl_trigger(); *e += 1; }

const int kReg2 = register_kernels({(const void*)topk_plan2_kernel<1>, (const void*)topk_plan2_kernel<2>,
                                    (const void*)topk_plan2_kernel<4>, (const void*)topk_plan2_kernel<8>});
const int kReg = register_kernels({(const void*)cache_plan_kernel, (const void*)cache_plan2_kernel, (const void*)gather_kernel,
                                   (const void*)cache_update_kernel, (const void*)pack_probe_kernel<float>,
                                   (const void*)pack_probe_kernel<__nv_bfloat16>, (const void*)pack_records_kernel<float>,
                                   (const void*)pack_records_kernel<__nv_bfloat16>, (const void*)epoch_inc_kernel});

}  // namespace

cudaError_t launch_epoch_inc(int32_t* epoch_dev, cudaStream_t st) {
  if (cudaError_t e_ = launch_kernel(epoch_inc_kernel, 1, 1, 0, st, epoch_dev)) return e_;
  return cudaGetLastError();
}

cudaError_t launch_cache_plan(const CacheLayer& cl, const int32_t* ids, const int32_t* n_ids_dev, int n_ids_host,
                              int prefetch, int quota, int epoch, int64_t rec_bytes, uint64_t*,
                              int32_t* scratch32, PlanOut out, cudaStream_t st) {
  size_t smem = 0;
  if (cl.P > NT * kPlanKPT && cl.P <= kPlanSmemKeysMax) {
    static bool attr = false;
    if (!attr) {
      if (cudaError_t e = cudaFuncSetAttribute(cache_plan_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                               (int)(kPlanSmemKeysMax * sizeof(uint64_t))))
        return e;
      attr = true;
    }
    smem = (size_t)cl.P * sizeof(uint64_t);
  }
  if (cudaError_t e_ = launch_kernel(cache_plan_kernel, 1, NT, smem, st, cl, ids, n_ids_dev, n_ids_host, prefetch, quota,
                                     epoch, rec_bytes, scratch32, out)) return e_;
  return cudaGetLastError();
}

cudaError_t launch_cache_plan2(const PlanJob& a, const PlanJob& b, cudaStream_t st) {
  size_t smem = 0;
  const int P = a.cl.P > b.cl.P ? a.cl.P : b.cl.P;
  if (P > NT * kPlanKPT && P <= kPlanSmemKeysMax) {
    static bool attr = false;
    if (!attr) {
      if (cudaError_t e = cudaFuncSetAttribute(cache_plan2_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                               (int)(kPlanSmemKeysMax * sizeof(uint64_t))))
        return e;
      attr = true;
    }
    smem = (size_t)P * sizeof(uint64_t);
  }
  if (cudaError_t e_ = launch_kernel(cache_plan2_kernel, 2, NT, smem, st, a, b)) return e_;
  return cudaGetLastError();
}

cudaError_t launch_topk_plan2(const TopkJob& t, const PlanJob& a, const PlanJob& b, cudaStream_t st) {
  size_t smem = 0;
  const int P = a.cl.P > b.cl.P ? a.cl.P : b.cl.P;
  const bool big = P > NT * kPlanKPT && P <= kPlanSmemKeysMax;
  if (big) smem = (size_t)P * sizeof(uint64_t);
  // table copies in shared memory: per-layer pools only (the demand and the speculative plan each
  // see one layer's [m_loc] tables) with register-resident victim keys (P <= NT * kPlanKPT)
  static const bool tables_on = !(tuning_env("CKV_PLAN_TABLES") && tuning_env("CKV_PLAN_TABLES")[0] == '0');
  const size_t tb = tables_smem_bytes(t.k, t.m, P);
  const int use_tables =
      (tables_on && !big && a.cl.m_loc == t.m && b.cl.m_loc == t.m && tb <= 200 * 1024) ? 1 : 0;
  if (use_tables) smem = tb;
  static bool attr = false;
  if (!attr) {
    for (auto kern : {topk_plan2_kernel<1>, topk_plan2_kernel<2>, topk_plan2_kernel<4>, topk_plan2_kernel<8>})
      if (cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024))
        return e;
    attr = true;
  }
  auto go = [&](void (*kern)(TopkJob, PlanJob, PlanJob, int)) -> cudaError_t {
    if (cudaError_t e_ = launch_kernel(kern, 2, NT, smem, st, t, a, b, use_tables)) return e_;
    return cudaGetLastError();
  };
  if (t.m <= NT) return go(topk_plan2_kernel<1>);
  if (t.m <= 2 * NT) return go(topk_plan2_kernel<2>);
  if (t.m <= 4 * NT) return go(topk_plan2_kernel<4>);
  if (t.m <= 8 * NT) return go(topk_plan2_kernel<8>);
  return cudaErrorNotSupported;
}

cudaError_t launch_gather(const int32_t* gather_list, const int32_t* n_load, const char* host_layer_dev,
                          char* pool_layer, int64_t rec_bytes, cudaStream_t st) {
  static int blocks = 0;
  if (!blocks) {  // tuning knob (CKV_GATHER_BLOCKS), default GATHER_BLOCKS
    const char* e = tuning_env("CKV_GATHER_BLOCKS");
    blocks = (e && atoi(e) > 0) ? atoi(e) : GATHER_BLOCKS;
  }
  if (cudaError_t e_ = launch_kernel(gather_kernel, blocks, GATHER_THREADS, 0, st, gather_list, n_load, host_layer_dev,
                                     pool_layer, rec_bytes)) return e_;
  return cudaGetLastError();
}

cudaError_t launch_cache_update(const CacheLayer& cl, const int32_t* ids, const int32_t* n_ids_dev, const float* A,
                                int tick, cudaStream_t st) {
  if (cudaError_t e_ = launch_kernel(cache_update_kernel, 8, 256, 0, st, cl, ids, n_ids_dev, A, tick)) return e_;
  return cudaGetLastError();
}

template <typename T>
cudaError_t launch_pack_probe(const T* k, int64_t t0, int cyc_W, int cyc_g, int c, int n_loc, int n_pad, int Hkv, int d,
                              T* probe_layer, cudaStream_t st) {
  if (cudaError_t e_ = launch_kernel(pack_probe_kernel<T>, 1184, 256, 0, st, k, t0, cyc_W, cyc_g, c, n_loc, n_pad, Hkv, d,
                                     probe_layer)) return e_;
  return cudaGetLastError();
}
template <typename T>
cudaError_t launch_pack_records(const T* k, const T* v, int64_t t0, int cyc_W, int cyc_g, int n_loc, int m_loc, int c,
                                int Hkv, int d, int swz, T* staging, cudaStream_t st) {
  if (cudaError_t e_ = launch_kernel(pack_records_kernel<T>, 1184, 256, 0, st, k, v, t0, cyc_W, cyc_g, n_loc, m_loc, c, Hkv,
                                     d, swz, staging)) return e_;
  return cudaGetLastError();
}
template cudaError_t launch_pack_probe<float>(const float*, int64_t, int, int, int, int, int, int, int, float*,
                                              cudaStream_t);
template cudaError_t launch_pack_probe<__nv_bfloat16>(const __nv_bfloat16*, int64_t, int, int, int, int, int, int, int,
                                                      __nv_bfloat16*, cudaStream_t);
template cudaError_t launch_pack_records<float>(const float*, const float*, int64_t, int, int, int, int, int, int, int,
                                                int, float*, cudaStream_t);
template cudaError_t launch_pack_records<__nv_bfloat16>(const __nv_bfloat16*, const __nv_bfloat16*, int64_t, int, int,
                                                        int, int, int, int, int, int, __nv_bfloat16*, cudaStream_t);

}  // namespace ckv
