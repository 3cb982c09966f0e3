// Shared device helpers and launcher declarations of libckv (sm_100a).
// Product code only: nothing here is shared with oracle/.
#pragma once
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <stdint.h>

#include <initializer_list>

#include "xchg.cuh"

namespace ckv {

// ---- programmatic dependent launch (PDL) ----
// Every kernel of libckv is launched with programmatic stream serialization (launch_kernel), so
// it may be scheduled while its stream predecessor is still running.  Each kernel calls
// pdl_wait() before its first access to memory another kernel of the stream writes or reads
// (griddepcontrol.wait: the predecessor grid has completed and its writes are visible), and
// pdl_trigger() only AFTER its own pdl_wait(): its successor is then scheduled no earlier than
// the completion of its predecessor, so at most two kernels of a stream overlap and every
// kernel older than the predecessor has completed.  (Triggering before the wait let three-
// kernel chains -- plan, gather, attention -- read stale data: measured on B200.)  Only
// constant inputs (q, k_suf, v_suf, the probe keys), TMEM / shared-memory setup, tensor-map
// prefetches and data whose last writer is older than the stream predecessor (chunk sums: the
// score kernel's lam2; the fused select: the cache tables) may precede pdl_wait().
#ifdef CKV_TUNING
// Device timeline (tuning build, CKV_DTL=1): CTA 0 / thread 0 of every kernel records the time its
// pdl_wait() returned (= its predecessor completed) with its grid / block size; the per-TU
// pointers are set by ckv_create (dtl_setters), ckv_destroy prints the records in time order.
static __device__ unsigned long long* g_dtl = nullptr;
static __device__ unsigned int* g_dtl_n = nullptr;
using DtlSetter = cudaError_t (*)(unsigned long long*, unsigned int*);
int register_dtl(DtlSetter f);
static cudaError_t dtl_set_tu(unsigned long long* b, unsigned int* n) {
  cudaError_t e = cudaMemcpyToSymbol(g_dtl, &b, sizeof b);
  if (e != cudaSuccess) return e;
  return cudaMemcpyToSymbol(g_dtl_n, &n, sizeof n);
}
static const int kDtlReg = register_dtl(dtl_set_tu);
#endif
__device__ __forceinline__ void pdl_wait() {
  asm volatile("griddepcontrol.wait;" ::: "memory");
#ifdef CKV_TUNING
  if (g_dtl && threadIdx.x == 0 && blockIdx.x == 0) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    const unsigned i = atomicAdd(g_dtl_n, 1u) & 8191u;
    g_dtl[2 * i] = t;
    g_dtl[2 * i + 1] = gridDim.x | ((unsigned long long)blockDim.x << 32);
  }
#endif
}
// tuning build: a device-timeline mark (tag, CTA) by thread 0 of the calling CTA (CKV_DTL=1)
__device__ __forceinline__ void dtl_mark(int tag) {
#ifdef CKV_TUNING
  if (g_dtl && threadIdx.x == 0) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    const unsigned i = atomicAdd(g_dtl_n, 1u) & 8191u;
    g_dtl[2 * i] = t;
    g_dtl[2 * i + 1] = 0xF0000000u | ((unsigned)tag << 8) | (blockIdx.x & 0xFF);
  }
#else
  (void)tag;
#endif
}
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
bool pdl_enabled();  // tuning build: CKV_PDL=0 disables the launch attribute (A/B measurements)
// A kernel that follows a cross-stream event wait is launched without the attribute (the
// programmatic relaxation must not weaken the event dependency); api.cu marks such streams.
void pdl_mark_event_wait(cudaStream_t st);
bool pdl_take_event_wait(cudaStream_t st);  // true (and cleared) if st was marked
void timeline_mark(const void* kern, cudaStream_t st);
void dtl_name(const void* kern, dim3 grid, dim3 block);  // tuning build: names for the device timeline
// Every kernel of the library is registered at load time (static initialisers, no CUDA call) and
// loaded by ckv_create (cudaFuncGetAttributes): with CUDA's lazy module loading, the first launch
// of a kernel can block the host until the device is idle, which deadlocks a host thread that
// drives several ranks whose streams wait on each other (fused exchange, xchg.cuh).
int register_kernels(std::initializer_list<const void*> ks);
cudaError_t preload_kernels();  // tuning build: CKV_TIMELINE=1 event after each launch
// Environment knobs exist only in the tuning build (-DCKV_TUNING, `build.py --tuning` ->
// libckv_tuning.so, used by scripts/ for A/B measurements).  The product library reads no
// environment variable: tuning_env() returns nullptr there, so every knob takes its default.
inline const char* tuning_env(const char* name) {
#ifdef CKV_TUNING
  return getenv(name);
#else
  (void)name;
  return nullptr;
#endif
}

template <typename... KArgs, typename... Args>
inline cudaError_t launch_kernel(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                                 Args&&... args) {
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  const bool after_wait = pdl_take_event_wait(st);
  attr[0].val.programmaticStreamSerializationAllowed =
      (pdl_enabled() && !after_wait) ? 1 : 0;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  const cudaError_t e = cudaLaunchKernelEx(&cfg, kern, static_cast<Args&&>(args)...);
  timeline_mark(reinterpret_cast<const void*>(kern), st);
  dtl_name(reinterpret_cast<const void*>(kern), grid, block);
  return e;
}

constexpr float kLog2e = 1.4426950408889634f;
constexpr float kLn2 = 0.6931471805599453f;

__device__ __forceinline__ float to_f(float x) { return x; }
__device__ __forceinline__ float to_f(__nv_bfloat16 x) { return __bfloat162float(x); }
template <typename T> __device__ __forceinline__ T from_f(float x);
template <> __device__ __forceinline__ float from_f<float>(float x) { return x; }
template <> __device__ __forceinline__ __nv_bfloat16 from_f<__nv_bfloat16>(float x) {
  return __float2bfloat16_rn(x);
}

__device__ __forceinline__ float fast_exp2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
// 2^x on the FMA/ALU pipes (x <= 0): round-to-nearest split x = i + f with the 1.5*2^23 trick,
// degree-5 Taylor of 2^f on [-0.5, 0.5] (rel. error < 3e-6), exponent added in the integer
// domain.  Used for part of the exponentials so the MUFU (ex2) pipe is not the only bound.
__device__ __forceinline__ float exp2_poly(float x) {
  x = fmaxf(x, -125.f);
  const float r = x + 12582912.f;
  const float f = x - (r - 12582912.f);
  float p = fmaf(f, 1.3333558e-3f, 9.6181291e-3f);
  p = fmaf(p, f, 5.5504109e-2f);
  p = fmaf(p, f, 2.4022651e-1f);
  p = fmaf(p, f, 6.9314718e-1f);
  p = fmaf(p, f, 1.0f);
  return __int_as_float(__float_as_int(p) + ((__float_as_int(r) - 0x4B400000) << 23));
}

// One warp's 64 key columns of one row tile (this thread: one suffix row): a single max over
// the 64 scores is the reference for every exponential (no running rescale), so the MUFU pipe
// sees one ex2 per score plus one lg2 per chunk piece and one for the quarter normaliser.

__device__ __forceinline__ float fast_log2(float x) {
  float y;
  asm("lg2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// Geometry of one layer's work as seen by the kernels (local shard view).
struct LayerGeom {
  int Hq, Hkv, G, d, c;
  int ns;          // suffix rows n_s of this call
  int R;           // rows per KV head = G * ns (row rho = g * ns + r)
  int m_loc;       // local chunks
  int n_loc;       // local prefix tokens
  int n_pad;       // probe-key row stride per KV head
  int rec_swz;     // chunk-record layout: 0 plain, 1 swizzled, 2 V-only swizzled (see rec_elem)
};

// Element offset inside one chunk record (one HBM slot / one host-store record).
//  plain    [K|V][Hkv][c][d]
//  swizzled (bf16, d = 128): [Hkv][K|V][half][c][64] with each 128-byte row's 16-byte units
//           XOR-swizzled by (row & 7) -- the exact shared-memory image the tcgen05 attention
//           consumes, so one (chunk, kv head) K+V block is a single contiguous bulk copy.
//  V-only   (swz 2, CKV_FLAG_V_ONLY_STORE): [Hkv][half][c][64] swizzled, V only (kv == 1); the
//           kept chunks' K comes from the HBM probe array
__host__ __device__ __forceinline__ int64_t rec_elem(int swz, int kv, int kvh, int p, int x, int Hkv, int c, int d) {
  if (!swz) return (((int64_t)kv * Hkv + kvh) * c + p) * d + x;
  const int half = x >> 6, xi = x & 63;
  const int u = (xi >> 3) ^ (p & 7);
  if (swz == 2) return (((int64_t)kvh * 2 + half) * c + p) * 64 + u * 8 + (xi & 7);
  return ((((int64_t)kvh * 2 + kv) * 2 + half) * c + p) * 64 + u * 8 + (xi & 7);
}

// ---- launchers (defined in the k_*.cu files) ----
// A1 SIMT: lam2[kvh][m_loc][R] = log2 sum_{i in chunk} 2^(l_i log2e), lampart[kvh][split][R]
template <typename T>
cudaError_t launch_score_simt(const LayerGeom& g, const T* q, const T* probe_layer, float* lam2,
                              float* lampart, int nsplit, cudaStream_t st);
// A1 tcgen05 (bf16 only, d == 128); returns cudaErrorNotSupported if the shape is outside it
// A6 speculative gather run by the score kernel's gather warp: (chunk, slot) pairs, count on device
struct SpecGather {
  const int32_t* list = nullptr;
  const int32_t* n_load = nullptr;
  const char* host_layer = nullptr;
  char* pool_layer = nullptr;
  int64_t rec_bytes = 0;
};
cudaError_t launch_score_tc(const LayerGeom& g, const __nv_bfloat16* q, const __nv_bfloat16* probe_layer,
                            float* lam2, float* lampart, int nsplit, void* qpack_ws, const SpecGather& spec,
                            cudaStream_t st);
int score_tc_nsplit(const LayerGeom& g);   // 0 if the shape is outside the tcgen05 kernel
size_t score_tc_qpack_elems(int Hkv, int R_max);
int score_tc_packs_q(const LayerGeom& g);  // 1 if the launch includes the Q pack kernel (n_s % 128 != 0)
// A2: Lambda2[kvh][R] = LSE2 over splits (+ causal suffix if fullrow) ; also writes row LSE for shards
template <typename T>
cudaError_t launch_row_lse(const LayerGeom& g, const float* lampart, int nsplit, const T* q, const T* k_suf,
                           int fullrow, const float* lam_all, int W, float* Lam2, float* lam_local_out,
                           cudaStream_t st);
cudaError_t launch_chunk_sum(const LayerGeom& g, const float* lam2, const float* Lam2, float* Apart,
                             cudaStream_t st);  // Apart [Hkv][m_loc]
// A3
// A [m] is written first as sum_h Apart[h][j] when Apart != nullptr (else A is the input)
cudaError_t launch_topk_scores(float* A, const float* Apart, int nparts, int m, int k, int id_offset, int id_mul, int32_t* ids,
                               uint64_t* cand_out, int n_cand_out, int32_t* n_out, cudaStream_t st);
cudaError_t launch_topk_merge(const uint64_t* cand_all, int n_cand, int k, int m_glob, int j0, int j1, int cyc_W,
                              int32_t* flag_scratch, int32_t* ids_glob, int32_t* ids_local,
                              int32_t* n_local, cudaStream_t st);
cudaError_t launch_block_cover(const int32_t* ids, int n_ids, int u, int B, int64_t n, int32_t* blocks,
                               int32_t* n_blocks, cudaStream_t st);
// Global prefix token of local token i: contiguous shards t0 + i; cyclic shards (cyc_W > 0) own
// chunks j = t*cyc_W + cyc_g, packed chunk by chunk.
__device__ __forceinline__ int64_t shard_token(int64_t i, int64_t t0, int cyc_W, int cyc_g, int c) {
  return cyc_W > 0 ? ((i / c) * cyc_W + cyc_g) * c + i % c : t0 + i;
}
// A4 / A5 / A9
// Owners are encoded as table indices e = layer * m_loc + j into the [L][m_loc] tables, so victims
// of any layer resolve with the *0 base pointers (the global heap of CKV_FLAG_GLOBAL_HEAP, where
// one pool of L * P slots serves every layer; per-layer pools see only their own layer's e).
struct CacheLayer {
  int32_t* slot_of;   // [m_loc] this layer's view
  int32_t* owner;     // [P] (the whole pool in global-heap mode)
  int32_t* pf_epoch;  // [P]
  float* I;           // [m_loc]
  int32_t* F;         // [m_loc]
  int32_t* T;         // [m_loc] request tick of the last selection (LRU policy)
  int32_t* slot_of0;  // [L * m_loc] layer-0 bases of the tables
  float* I0;
  int32_t* F0;
  int32_t* T0;
  int lbase;          // layer * m_loc
  int m_loc, P;
  int policy;         // ckv_cache_policy: eviction score S (0: I*F, 1: F, 2: last-use tick)
};
struct PlanOut {
  int32_t* gather_list;  // [2 * cap]: (chunk, slot)
  int32_t* n_load;       // [1]
  int32_t* kept_slots;   // [k] or null (prefetch mode)
  int32_t* victims;      // [cap] or null
  int32_t* counts;       // [4]: hits, loads, victims, spec_used  (or null)
  int64_t* stats;        // device counters or null
  const float* upd_A;    // if set (demand plans): fused A9 update I += A, F += 1 after planning
  const int32_t* epoch_dev;  // if set: request epoch read from device memory (graph-safe)
  int32_t* ids_out = nullptr;  // if set: copy of the planned ids (the caller's selected_ids)
  int mark_miss = 0;  // kept_slots of a miss = -(slot + 2): the consumer (compact_kv) loads it from the
                      // host store itself and fills the slot (no separate gather launch)
  const int32_t* gate_misses = nullptr;  // prefetch plans: demand misses of the previous layer ...
  int gate_max = -1;                     // ... at or below which nothing is speculated (adaptive)
  const uint64_t* rank_keys = nullptr;  // prefetch plans: per position of ids, the (score bits << 32 | ~id)
                                        // key of the identifying layer; over quota, the highest-scored
                                        // misses are loaded (else the first in chunk order)
};
cudaError_t launch_cache_plan(const CacheLayer& cl, const int32_t* ids, const int32_t* n_ids_dev, int n_ids_host,
                              int prefetch, int quota, int epoch, int64_t rec_bytes, uint64_t* scratch64,
                              int32_t* scratch32, PlanOut out, cudaStream_t st);
struct PlanJob {  // one cache_plan_body invocation (launch_cache_plan2)
  CacheLayer cl;
  const int32_t* ids;
  const int32_t* n_ids_dev;
  int n_ids_host, prefetch, quota, epoch;
  int64_t rec_bytes;
  int32_t* scratch;
  PlanOut out;
};
cudaError_t launch_cache_plan2(const PlanJob& a, const PlanJob& b, cudaStream_t st);
// A3 top-k of the local chunk scores fused with the two plans of launch_cache_plan2: both CTAs run
// the same top-k (deterministic); CTA 0 writes A, ids, n_ids, rank keys (cand) and plans job a on
// them; CTA 1 writes its copy to ids_b / cand_b / n_b and plans job b on those (job b's ids,
// n_ids_dev and out.rank_keys must point there).  m <= 8192, else cudaErrorNotSupported.
struct TopkJob {
  float* A;
  const float* Apart;
  int nparts, m, k;
  int32_t* ids;
  uint64_t* cand;
  int32_t* n_out;
  int32_t* ids_b;
  uint64_t* cand_b;
  int32_t* n_b;
};
cudaError_t launch_topk_plan2(const TopkJob& t, const PlanJob& a, const PlanJob& b, cudaStream_t st);
cudaError_t launch_epoch_inc(int32_t* epoch_dev, cudaStream_t st);
cudaError_t launch_gather(const int32_t* gather_list, const int32_t* n_load, const char* host_layer_dev,
                          char* pool_layer, int64_t rec_bytes, cudaStream_t st);
cudaError_t launch_cache_update(const CacheLayer& cl, const int32_t* ids, const int32_t* n_ids_dev,
                                const float* A, int tick, cudaStream_t st);
// store
template <typename T>
cudaError_t launch_pack_probe(const T* k, int64_t t0, int cyc_W, int cyc_g, int c, int n_loc, int n_pad, int Hkv, int d, T* probe_layer,
                              cudaStream_t st);
template <typename T>
cudaError_t launch_pack_records(const T* k, const T* v, int64_t t0, int cyc_W, int cyc_g, int n_loc, int m_loc, int c, int Hkv,
                                int d, int swz, T* staging, cudaStream_t st);
// A7 / A8
template <typename T>
cudaError_t launch_attn_simt(const LayerGeom& g, const T* q, const T* k_suf, const T* v_suf,
                             const T* pool_layer, int64_t rec_elems, const int32_t* kept_slots,
                             const int32_t* kept_ids, const int32_t* n_kept_dev, int k_cap,
                             int include_suffix, int nsplit, float* o_part, float* lse_part,
                             cudaStream_t st);
bool attn_tc_supported(const LayerGeom& g);
int attn_tc_nsplit(const LayerGeom& g, int k_cap, int include_suffix);
// tcgen05 attention = dense K/V compaction + attention kernel; dense_ws holds
// attn_tc_dense_bytes(g, k_cap, max_ns) bytes, zero-initialised once (padding keys stay finite)
size_t attn_tc_dense_bytes(const LayerGeom& g, int k_cap, int max_ns);
cudaError_t launch_attn_tc(const LayerGeom& g, const __nv_bfloat16* q, const __nv_bfloat16* k_suf,
                           const __nv_bfloat16* v_suf, const __nv_bfloat16* pool_layer, const int32_t* kept_slots,
                           const int32_t* kept_ids, const int32_t* n_kept_dev, int k_cap, int include_suffix,
                           int nsplit, float* o_part, float* lse_part, void* dense_ws, const char* host_layer,
                           const __nv_bfloat16* probe_layer, cudaEvent_t after_compact, const float* lam_ref,
                           cudaStream_t st);
template <typename T>
cudaError_t launch_attn_combine(const LayerGeom& g, const float* o_part, const float* lse_part, int nsplit,
                                T* out, float* o_f32, float* lse_nat, cudaStream_t st, const XPartDst* xd = nullptr);
// fused exchange (k_xchg.cu, xchg.cuh)
cudaError_t launch_xchg_put(const XPeers& xp, const void* src, size_t bytes, size_t dst_off, size_t flag_off,
                            cudaStream_t st);
template <typename T>
cudaError_t launch_xchg_merge(const XPeers& xp, const XLayout& xl, int N, int rps, int d, cudaStream_t st);
cudaError_t xchg_wait(cudaStream_t st, void* flag_dev, uint32_t target);
cudaError_t launch_lse_merge_prepare(int rows, int d, const float* o, const float* lse, const float* lse_max,
                                     float* buf, cudaStream_t st);
template <typename T>
cudaError_t launch_lse_merge_finish(int rows, int d, const float* buf, T* out, cudaStream_t st);

}  // namespace ckv
