// C-ABI and per-layer engine of libckv (include/ckv.h).
//
// Orchestrates, per layer, on the caller's stream S and one library-owned side stream P:
//   S: A1 score -> A2 reduce -> A3 top-k -> [wait P's prefetch plan] A4 plan -> A5 delta
//      gather -> [wait P's prefetch data] A7 attention -> A8 combine -> A9 update
//   P: (after A3 of layer l) A4 plan of layer l+1 for ids_l (speculative, quota) -> A5
//      gather  (inter-period speculative prefetch at p = 1)
// No host synchronisation on the per-layer path: ids stay on the device, and the gather
// reads the mapped pinned host store directly (device-initiated zero-copy).
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <algorithm>
#include <string>
#include <vector>

#include <nvtx3/nvToolsExt.h>

#include "../../include/ckv.h"
#include "common.cuh"

namespace ckv {
void timeline_dump();  // debug (CKV_TIMELINE=1), defined at the end of this file
void dtl_init();       // tuning build: device timeline (CKV_DTL=1)
void dtl_dump();
}

using namespace ckv;

struct ckv_ctx {
  ckv_config cfg{};
  int L = 0, Hq = 0, Hkv = 0, G = 0, d = 0, c = 0, esz = 0, dtype = 0, fullrow = 0;
  int64_t n = 0;
  int m = 0;
  int W = 1, shard = 0, j0 = 0, j1 = 0, m_loc = 0;
  int cyc_W = 0;  // > 0: cyclic shards (CKV_FLAG_CYCLIC_SHARDS), local chunk t = global t*W + shard
  int64_t t0 = 0;
  int n_loc = 0, n_pad = 0;
  int k = 0, P = 0, quota = 0, max_ns = 0, period = 1, subperiod = 1;
  int spec_gate = -1;  // p = 1 speculation is skipped when the previous layer missed <= spec_gate chunks
  int64_t rec_elems = 0, rec_bytes = 0;
  int nsplit_score_max = 1, nsplit_attn_max = 1;
  int score_kind = 0;  // 0 SIMT, 1 tcgen05
  int rec_swz = 0;     // chunk-record layout (rec_elem)
  int attn_kind = 0;   // 0 SIMT, 1 tcgen05

  void* probe = nullptr;
  char* host_store = nullptr;
  char* host_store_dev = nullptr;
  char* pool = nullptr;
  int32_t *slot_of = nullptr, *owner = nullptr, *pf_epoch = nullptr, *F = nullptr, *T = nullptr;
  int cache_policy = 0;  // ckv_cache_policy
  bool global_heap = false;  // CKV_FLAG_GLOBAL_HEAP: one pool of L * P slots shared by all layers
  float* I = nullptr;
  float *lam2 = nullptr, *lampart = nullptr, *Lam2 = nullptr, *A = nullptr, *Apart = nullptr;
  int32_t* ids_buf[2] = {nullptr, nullptr};
  uint64_t* sel_keys[2] = {nullptr, nullptr};  // (score bits << 32 | ~id) of ids_buf's entries (rank the speculation)
  int32_t *ids_b = nullptr, *n_b = nullptr;    // topk_plan2's CTA 1: its private copy of the top-k
  int lam2_layer = -1;  // layer whose row normalisers Lam2 holds (the attention's softmax reference)
  int spec_next = -1;   // layer whose speculative gather (gl_side) its score kernel runs (p = 1, tcgen05)
  uint64_t* cand_b = nullptr;
  int32_t* n_ids_buf[2] = {nullptr, nullptr};
  int32_t *kept_slots = nullptr, *ids_glob = nullptr, *flag = nullptr;
  int32_t *scratch_main = nullptr, *scratch_side = nullptr;
  int32_t *gl_main = nullptr, *gl_side = nullptr, *nload_main = nullptr, *nload_side = nullptr;
  int32_t* counts = nullptr;  // [L][2][4]
  float *o_part = nullptr, *lse_part = nullptr;
  int64_t* stats = nullptr;  // [16]
  int32_t* epoch_dev = nullptr;  // request counter on the device (graph-safe)
  int32_t* ticket = nullptr;     // grid ticket of the fused select kernel
  void* tmap_cache = nullptr;
  void* dense_kv = nullptr;  // tcgen05 attention: dense K/V tiles of the current layer
  // fused device-side exchange (num_shards > 1; xchg.cuh)
  char* xwin = nullptr;        // this rank's exchange window
  XLayout xl{};
  XPeers xp{};                 // window bases of all ranks (valid once attached)
  bool x_attached = false;
  std::vector<void*> x_opened;  // IPC-mapped peer windows (closed in ckv_destroy)
  float* lam_loc = nullptr;     // [Hq * max_ns] this shard's row normalisers
  uint64_t* cand_loc = nullptr; // [k] this shard's candidates

  cudaStream_t side = nullptr;
  cudaEvent_t ev_ids = nullptr;
  std::vector<cudaEvent_t> ev_pplan, ev_pf;
  std::vector<int> pf_issued;
  std::vector<int> pf_joined;
  std::vector<char> pf_late;  // the prefetch of this layer was issued at the end of the previous layer  // epoch in which the main stream already waited for ev_pf[layer]
  std::vector<char> stored;
  int epoch = 0;
  int last_layer = -1;
  int64_t launches = 0;
  // stage profiling (CUDA events on the launching stream; off by default)
  bool prof_on = false;
  std::vector<cudaEvent_t> prof_pool;
  std::vector<std::pair<int, std::pair<cudaEvent_t, cudaEvent_t>>> prof_marks;
  size_t prof_used = 0;
  cudaEvent_t prof_open[8] = {};
  std::string err;
};

namespace {

// NVTX range around each public entry point (an nsys / ncu timeline shows the library's host calls;
// without an attached tool the header-only NVTX v3 calls are no-ops)
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
};

ckv_status fail(ckv_ctx* ctx, ckv_status s, const char* fmt, ...) {
  if (ctx) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    ctx->err = buf;
  }
  return s;
}

#define CK(expr)                                                                                     \
  do {                                                                                               \
    cudaError_t e_ = (expr);                                                                         \
    if (e_ != cudaSuccess) return fail(ctx, CKV_ECUDA, "%s: %s (%s:%d)", #expr, cudaGetErrorString(e_), \
                                       __FILE__, __LINE__);                                          \
  } while (0)

#define LK(expr)   \
  do {             \
    CK(expr);      \
    ++ctx->launches; \
  } while (0)

cudaEvent_t prof_event(ckv_ctx* ctx) {
  if (ctx->prof_used == ctx->prof_pool.size()) {
    cudaEvent_t e = nullptr;
    cudaEventCreate(&e);
    ctx->prof_pool.push_back(e);
  }
  return ctx->prof_pool[ctx->prof_used++];
}
void prof_begin(ckv_ctx* ctx, int stage, cudaStream_t st) {
  if (!ctx->prof_on) return;
  cudaEvent_t e = prof_event(ctx);
  cudaEventRecord(e, st);
  ctx->prof_open[stage] = e;
}
void prof_end(ckv_ctx* ctx, int stage, cudaStream_t st) {
  if (!ctx->prof_on || !ctx->prof_open[stage]) return;
  cudaEvent_t e = prof_event(ctx);
  cudaEventRecord(e, st);
  ctx->prof_marks.push_back({stage, {ctx->prof_open[stage], e}});
  ctx->prof_open[stage] = nullptr;
}
#define PROF_BEGIN(s) prof_begin(ctx, (s), st)
#define PROF_END(s) prof_end(ctx, (s), st)

template <typename Tp>
cudaError_t dalloc(Tp** p, size_t count) {
  return cudaMalloc(reinterpret_cast<void**>(p), count * sizeof(Tp) + 16);
}

LayerGeom geom(const ckv_ctx* ctx, int ns) {
  LayerGeom g;
  g.Hq = ctx->Hq;
  g.Hkv = ctx->Hkv;
  g.G = ctx->G;
  g.d = ctx->d;
  g.c = ctx->c;
  g.ns = ns;
  g.R = ctx->G * ns;
  g.m_loc = ctx->m_loc;
  g.n_loc = ctx->n_loc;
  g.n_pad = ctx->n_pad;
  g.rec_swz = ctx->rec_swz;
  return g;
}

int simt_score_nsplit(const ckv_ctx* ctx, int ns) {
  const int rowblocks = (ctx->G * ns + 63) / 64;
  int s = (4 * 296 + rowblocks * ctx->Hkv - 1) / (rowblocks * ctx->Hkv);
  // every split reloads its 64-row Q tile: give each at least 2 key sub-tiles (128 keys) of work
  const int by_keys = (ctx->n_loc + 127) / 128;
  s = s > by_keys ? by_keys : s;
  s = s < 1 ? 1 : s;
  return s > ctx->m_loc ? ctx->m_loc : s;
}

int attn_nsplit(const ckv_ctx* ctx, int ns, int n_kept_cap) {
  const int rowblocks = (ctx->G * ns + 63) / 64;
  int s = (2 * 296 + rowblocks * ctx->Hkv - 1) / (rowblocks * ctx->Hkv);
  int maxs = n_kept_cap < 1 ? 1 : n_kept_cap;
  s = s < 1 ? 1 : s;
  s = s > maxs ? maxs : s;
  return s > ctx->nsplit_attn_max ? ctx->nsplit_attn_max : s;
}

CacheLayer cache_layer(const ckv_ctx* ctx, int layer) {
  CacheLayer cl;
  cl.slot_of = ctx->slot_of + (size_t)layer * ctx->m_loc;
  const size_t pool_off = ctx->global_heap ? 0 : (size_t)layer * ctx->P;
  cl.owner = ctx->owner + pool_off;
  cl.pf_epoch = ctx->pf_epoch + pool_off;
  cl.slot_of0 = ctx->slot_of;
  cl.I0 = ctx->I;
  cl.F0 = ctx->F;
  cl.T0 = ctx->T;
  cl.lbase = layer * ctx->m_loc;
  cl.I = ctx->I + (size_t)layer * ctx->m_loc;
  cl.F = ctx->F + (size_t)layer * ctx->m_loc;
  cl.T = ctx->T + (size_t)layer * ctx->m_loc;
  cl.m_loc = ctx->m_loc;
  cl.P = ctx->global_heap ? ctx->L * ctx->P : ctx->P;
  cl.policy = ctx->cache_policy;
  return cl;
}

const char* host_layer_dev(const ckv_ctx* ctx, int layer) {
  return ctx->host_store_dev + (size_t)layer * ctx->m_loc * ctx->rec_bytes;
}
// slot s of `layer` (per-layer pools) or of the shared pool (global heap: slots are pool-wide)
char* pool_layer(const ckv_ctx* ctx, int layer) {
  return ctx->global_heap ? ctx->pool : ctx->pool + (size_t)layer * ctx->P * ctx->rec_bytes;
}
const void* probe_layer(const ckv_ctx* ctx, int layer) {
  return static_cast<const char*>(ctx->probe) + (size_t)layer * ctx->Hkv * ctx->n_pad * ctx->d * ctx->esz;
}

// A1 (+ local part of A2): lam2, lampart, and Lam2 or the shard-local row LSE
ckv_status run_score(ckv_ctx* ctx, int layer, const void* q, const void* ks, int ns, float* lam_local_out,
                     int* nsplit_out, cudaStream_t st) {
  LayerGeom g = geom(ctx, ns);
  int nsplit = 0;
  cudaError_t e = cudaErrorNotSupported;
  PROF_BEGIN(0);
  if (ctx->score_kind == 1) {
    nsplit = score_tc_nsplit(g);
    SpecGather spec;
    if (ctx->spec_next == layer) {  // planned by the previous layer (CTA 1 of its top-k / plan launch)
      spec.list = ctx->gl_side;
      spec.n_load = ctx->nload_side;
      spec.host_layer = host_layer_dev(ctx, layer);
      spec.pool_layer = pool_layer(ctx, layer);
      spec.rec_bytes = ctx->rec_bytes;
    }
    ctx->spec_next = -1;
    e = launch_score_tc(g, static_cast<const __nv_bfloat16*>(q),
                        static_cast<const __nv_bfloat16*>(probe_layer(ctx, layer)), ctx->lam2, ctx->lampart, nsplit,
                        ctx->tmap_cache, spec, st);
    if (e == cudaSuccess) {
      ctx->launches += score_tc_packs_q(g);  // + the Q pack kernel
    }
  }
  if (e == cudaErrorNotSupported) {
    nsplit = simt_score_nsplit(ctx, ns);
    if (ctx->dtype == CKV_FP32)
      e = launch_score_simt<float>(g, static_cast<const float*>(q), static_cast<const float*>(probe_layer(ctx, layer)),
                                   ctx->lam2, ctx->lampart, nsplit, st);
    else
      e = launch_score_simt<__nv_bfloat16>(g, static_cast<const __nv_bfloat16*>(q),
                                           static_cast<const __nv_bfloat16*>(probe_layer(ctx, layer)), ctx->lam2,
                                           ctx->lampart, nsplit, st);
  }
  PROF_END(0);
  CK(e);
  ++ctx->launches;
  *nsplit_out = nsplit;
  // local row normaliser (-> Lam2 for W == 1, or the shard's lam_local)
  PROF_BEGIN(1);
  if (ctx->dtype == CKV_FP32)
    LK(launch_row_lse<float>(g, ctx->lampart, nsplit, static_cast<const float*>(q), static_cast<const float*>(ks),
                             lam_local_out ? 0 : ctx->fullrow, nullptr, 1, ctx->Lam2, lam_local_out, st));
  else
    LK(launch_row_lse<__nv_bfloat16>(g, ctx->lampart, nsplit, static_cast<const __nv_bfloat16*>(q),
                                     static_cast<const __nv_bfloat16*>(ks), lam_local_out ? 0 : ctx->fullrow, nullptr,
                                     1, ctx->Lam2, lam_local_out, st));
  PROF_END(1);
  ctx->lam2_layer = layer;  // Lam2 bounds every prefix logit of this layer's rows (local or global LSE)
  return CKV_OK;
}

// A6: speculative plan + gather of layer `layer` for the given ids, on the side stream.
// `recorded`: ev_ids was already recorded on st (global heap: after the compaction of the current layer).
// quota: chunks this plan may load (exact intra-period loads pass k; speculation the ctx's quota)
ckv_status issue_prefetch(ckv_ctx* ctx, int layer, const int32_t* ids, const int32_t* n_ids_dev, cudaStream_t st,
                          bool recorded = false, const uint64_t* rank_keys = nullptr, int quota = -1) {
  if (ctx->quota <= 0 || layer >= ctx->L) return CKV_OK;
  if (!recorded) CK(cudaEventRecord(ctx->ev_ids, st));
  CK(cudaStreamWaitEvent(ctx->side, ctx->ev_ids, 0));
  pdl_mark_event_wait(ctx->side);
  PlanOut po{ctx->gl_side, ctx->nload_side, nullptr, nullptr, ctx->counts + (size_t)(layer * 2 + 1) * 4, ctx->stats,
             nullptr, ctx->epoch_dev};
  po.rank_keys = rank_keys;
  LK(launch_cache_plan(cache_layer(ctx, layer), ids, n_ids_dev, 0, 1, quota > 0 ? quota : ctx->quota, ctx->epoch,
                       ctx->rec_bytes, nullptr, ctx->scratch_side, po, ctx->side));
  CK(cudaEventRecord(ctx->ev_pplan[layer], ctx->side));
  LK(launch_gather(ctx->gl_side, ctx->nload_side, host_layer_dev(ctx, layer), pool_layer(ctx, layer), ctx->rec_bytes,
                   ctx->side));
  CK(cudaEventRecord(ctx->ev_pf[layer], ctx->side));
  ctx->pf_issued[layer] = ctx->epoch;
  ctx->pf_late[layer] = 0;
  return CKV_OK;
}

// tcgen05 path: the compaction kernel loads the misses itself (A5 fused, no gather launch)
bool gather_fused(const ckv_ctx* ctx) { return ctx->dtype == CKV_BF16 && ctx->attn_kind == 1; }

PlanOut demand_plan_out(ckv_ctx* ctx, int layer, int32_t* ids_out) {
  return PlanOut{ctx->gl_main, ctx->nload_main, ctx->kept_slots, nullptr, ctx->counts + (size_t)(layer * 2) * 4,
                 ctx->stats, ctx->A, ctx->epoch_dev, ids_out, gather_fused(ctx) ? 1 : 0};
}

// A4 -> A5 -> A7 -> A8 -> A9 for the local selected ids.
ckv_status run_attend(ckv_ctx* ctx, int layer, const int32_t* ids, const int32_t* n_ids_dev, const void* q,
                      const void* ks, const void* vs, int ns, int include_suffix, void* out, float* o_f32,
                      float* lse_nat, int32_t* ids_out, bool planned, cudaStream_t st,
                      cudaEvent_t after_slots = nullptr, const XPartDst* xpd = nullptr) {
  // a prefetch of this layer that the stream already joined (before the score kernel) needs no
  // further event waits: they would only cut the programmatic launch edges of plan and attention
  const bool pf = ctx->pf_issued[layer] == ctx->epoch && ctx->pf_joined[layer] != ctx->epoch;
  const bool fused_gather = gather_fused(ctx);
  // one join per layer: on the fused path the compaction right after the plan needs the prefetched
  // data anyway, so wait for the whole side-stream load (one cut programmatic edge, not two)
  if (pf) {
    CK(cudaStreamWaitEvent(st, fused_gather ? ctx->ev_pf[layer] : ctx->ev_pplan[layer], 0));
    pdl_mark_event_wait(st);
  }
  if (!planned) {
    PROF_BEGIN(3);
    LK(launch_cache_plan(cache_layer(ctx, layer), ids, n_ids_dev, 0, 0, 0, ctx->epoch, ctx->rec_bytes, nullptr,
                         ctx->scratch_main, demand_plan_out(ctx, layer, ids_out), st));
    PROF_END(3);
  }
  if (!fused_gather) {
    PROF_BEGIN(4);
    LK(launch_gather(ctx->gl_main, ctx->nload_main, host_layer_dev(ctx, layer), pool_layer(ctx, layer),
                     ctx->rec_bytes, st));
    PROF_END(4);
  }
  if (pf && !fused_gather) {
    CK(cudaStreamWaitEvent(st, ctx->ev_pf[layer], 0));
    pdl_mark_event_wait(st);
  }
  LayerGeom g = geom(ctx, ns);
  int nsplit = attn_nsplit(ctx, ns, ctx->k);
  PROF_BEGIN(5);
  if (ctx->dtype == CKV_FP32) {
    LK(launch_attn_simt<float>(g, static_cast<const float*>(q), static_cast<const float*>(ks),
                               static_cast<const float*>(vs), reinterpret_cast<const float*>(pool_layer(ctx, layer)),
                               ctx->rec_elems, ctx->kept_slots, ids, n_ids_dev, ctx->k, include_suffix, nsplit,
                               ctx->o_part, ctx->lse_part, st));
    LK(launch_attn_combine<float>(g, ctx->o_part, ctx->lse_part, nsplit, static_cast<float*>(out), o_f32, lse_nat,
                                  st, xpd));
  } else {
    cudaError_t e = cudaErrorNotSupported;
    if (ctx->attn_kind == 1) {
      nsplit = attn_tc_nsplit(g, ctx->k, include_suffix);
      if (nsplit > ctx->nsplit_attn_max) nsplit = ctx->nsplit_attn_max;  // o_part / lse_part capacity
      e = launch_attn_tc(g, static_cast<const __nv_bfloat16*>(q), static_cast<const __nv_bfloat16*>(ks),
                         static_cast<const __nv_bfloat16*>(vs),
                         reinterpret_cast<const __nv_bfloat16*>(pool_layer(ctx, layer)), ctx->kept_slots, ids,
                         n_ids_dev, ctx->k, include_suffix, nsplit, ctx->o_part, ctx->lse_part, ctx->dense_kv,
                         host_layer_dev(ctx, layer), static_cast<const __nv_bfloat16*>(probe_layer(ctx, layer)),
                         after_slots, ctx->lam2_layer == layer ? ctx->Lam2 : nullptr, st);
      if (e == cudaSuccess) after_slots = nullptr;  // recorded between the compaction and the attention
      if (e == cudaSuccess) ctx->launches += 1;  // + the dense K/V compaction kernel
    }
    if (e == cudaErrorNotSupported) {
      nsplit = attn_nsplit(ctx, ns, ctx->k);
      e = launch_attn_simt<__nv_bfloat16>(g, static_cast<const __nv_bfloat16*>(q),
                                          static_cast<const __nv_bfloat16*>(ks), static_cast<const __nv_bfloat16*>(vs),
                                          reinterpret_cast<const __nv_bfloat16*>(pool_layer(ctx, layer)),
                                          ctx->rec_elems, ctx->kept_slots, ids, n_ids_dev, ctx->k, include_suffix,
                                          nsplit, ctx->o_part, ctx->lse_part, st);
    }
    CK(e);
    ++ctx->launches;
    LK(launch_attn_combine<__nv_bfloat16>(g, ctx->o_part, ctx->lse_part, nsplit, static_cast<__nv_bfloat16*>(out),
                                          o_f32, lse_nat, st, xpd));
  }
  PROF_END(5);
  if (after_slots) CK(cudaEventRecord(after_slots, st));  // SIMT path: the attention read the slots
  ctx->last_layer = layer;
  return CKV_OK;
}

ckv_status check_layer_call(ckv_ctx* ctx, int layer, int ns) {
  if (!ctx) return CKV_EINVAL;
  if (layer < 0 || layer >= ctx->L) return fail(ctx, CKV_EINVAL, "layer %d out of range [0, %d)", layer, ctx->L);
  if (ns < 1 || ns > ctx->max_ns) return fail(ctx, CKV_EINVAL, "n_suffix %d out of range [1, %d]", ns, ctx->max_ns);
  if (!ctx->stored[layer]) return fail(ctx, CKV_ESTATE, "layer %d prefix not stored", layer);
  return CKV_OK;
}

void free_all(ckv_ctx* ctx) {
  if (!ctx) return;
  cudaSetDevice(ctx->cfg.device);
  cudaDeviceSynchronize();
  void* dev_ptrs[] = {ctx->probe, ctx->pool, ctx->slot_of, ctx->owner, ctx->pf_epoch, ctx->F, ctx->T, ctx->I, ctx->lam2,
                      ctx->lampart, ctx->Lam2, ctx->A, ctx->Apart, ctx->ids_buf[0], ctx->ids_buf[1], ctx->n_ids_buf[0],
                      ctx->n_ids_buf[1], ctx->kept_slots, ctx->ids_glob, ctx->flag, ctx->scratch_main,
                      ctx->scratch_side, ctx->gl_main, ctx->gl_side, ctx->nload_main, ctx->nload_side, ctx->counts,
                      ctx->o_part, ctx->lse_part, ctx->stats, ctx->tmap_cache, ctx->dense_kv, ctx->epoch_dev, ctx->ticket};
  for (void* p : dev_ptrs)
    if (p) cudaFree(p);
  for (void* p : ctx->x_opened) cudaIpcCloseMemHandle(p);
  for (void* p : {(void*)ctx->xwin, (void*)ctx->lam_loc, (void*)ctx->cand_loc, (void*)ctx->sel_keys[0],
                  (void*)ctx->sel_keys[1], (void*)ctx->ids_b, (void*)ctx->n_b, (void*)ctx->cand_b})
    if (p) cudaFree(p);
  if (ctx->host_store) cudaFreeHost(ctx->host_store);
  for (auto e : ctx->ev_pplan)
    if (e) cudaEventDestroy(e);
  for (auto e : ctx->ev_pf)
    if (e) cudaEventDestroy(e);
  if (ctx->ev_ids) cudaEventDestroy(ctx->ev_ids);
  for (auto e : ctx->prof_pool)
    if (e) cudaEventDestroy(e);
  if (ctx->side) cudaStreamDestroy(ctx->side);
}

// One layer on one rank of a position-sharded group with the fused device-side exchange
// (xchg.cuh): every collective is a peer-memory write + counter
// increment by this rank and a stream wait on its own counter -- no host round trip, no NCCL.
ckv_status reprefill_sharded(ckv_ctx* ctx, int layer, const void* q, const void* k_suf, const void* v_suf, int ns,
                             void* out, int32_t* selected_ids, float* chunk_scores, cudaStream_t st) {
  const XPeers& xp = ctx->xp;
  const XLayout& xl = ctx->xl;
  const int W = ctx->W, self = ctx->shard;
  char* win = ctx->xwin;
  auto flag = [&](int f) { return static_cast<void*>(win + xl.flags + sizeof(uint32_t) * f); };
  const size_t fl = xl.flags;
  static const bool xtrace = tuning_env("CKV_XCHG_TRACE") != nullptr;  // tuning build: host-side step trace
#define XTRACE(msg) \
  if (xtrace) fprintf(stderr, "[xchg rank %d layer %d] %s\n", self, layer, msg)
  XTRACE("enter");
  if (layer == 0) {
    ++ctx->epoch;
    LK(launch_epoch_inc(ctx->epoch_dev, st));
  }
  const int N = ns * ctx->Hq;  // output rows (r, h)
  // 1. A1 on the local shard -> shard-local row normalisers; broadcast into slot `self`
  int nsplit = 0;
  ckv_status s = run_score(ctx, layer, q, k_suf, ns, ctx->lam_loc, &nsplit, st);
  if (s != CKV_OK) return s;
  XTRACE("scored");
  LK(launch_xchg_put(xp, ctx->lam_loc, sizeof(float) * N, xl.lam + sizeof(float) * (size_t)self * N,
                     fl + sizeof(uint32_t) * XF_LAM, st));
  XTRACE("lam put");
  CK(xchg_wait(st, flag(XF_LAM), W));
  XTRACE("lam wait enqueued");
  // 2. global Lambda (rank order; FULLROW adds the causal suffix) -> local A_j -> candidates
  LayerGeom g = geom(ctx, ns);
  const float* lam_all = reinterpret_cast<const float*>(win + xl.lam);
  PROF_BEGIN(1);
  if (ctx->dtype == CKV_FP32)
    LK(launch_row_lse<float>(g, nullptr, 0, static_cast<const float*>(q), static_cast<const float*>(k_suf),
                             ctx->fullrow, lam_all, W, ctx->Lam2, nullptr, st));
  else
    LK(launch_row_lse<__nv_bfloat16>(g, nullptr, 0, static_cast<const __nv_bfloat16*>(q),
                                     static_cast<const __nv_bfloat16*>(k_suf), ctx->fullrow, lam_all, W, ctx->Lam2,
                                     nullptr, st));
  PROF_END(1);
  PROF_BEGIN(2);
  LK(launch_chunk_sum(g, ctx->lam2, ctx->Lam2, ctx->Apart, st));
  PROF_END(2);
  PROF_BEGIN(6);
  LK(launch_topk_scores(ctx->A, ctx->Apart, ctx->Hkv, ctx->m_loc, ctx->k, ctx->j0, ctx->cyc_W > 0 ? ctx->cyc_W : 1,
                        nullptr, ctx->cand_loc, ctx->k, nullptr, st));
  PROF_END(6);
  LK(launch_xchg_put(xp, ctx->cand_loc, sizeof(uint64_t) * ctx->k, xl.cand + sizeof(uint64_t) * (size_t)self * ctx->k,
                     fl + sizeof(uint32_t) * XF_CAND, st));
  XTRACE("cand put");
  CK(xchg_wait(st, flag(XF_CAND), W));
  XTRACE("cand wait enqueued");
  // 3. identical merged top-k on every rank; local plan / gather / attention (suffix on rank W-1);
  //    the combine writes each partial row straight into the window of the rank merging its slice
  int32_t* ids = ctx->ids_buf[layer & 1];
  int32_t* nids = ctx->n_ids_buf[layer & 1];
  LK(launch_topk_merge(reinterpret_cast<const uint64_t*>(win + xl.cand), W * ctx->k, ctx->k, ctx->m, ctx->j0, ctx->j1,
                       ctx->cyc_W, ctx->flag, ctx->ids_glob, ids, nids, st));
  if ((s = issue_prefetch(ctx, layer + 1, ids, nids, st)) != CKV_OK) return s;
  const int rps = (N + W - 1) / W;
  XPartDst xd{xp, xl.part_o, xl.part_lse, rps, xl.rps_max, ctx->d};
  if ((s = run_attend(ctx, layer, ids, nids, q, k_suf, v_suf, ns, self == W - 1, nullptr, nullptr, nullptr, nullptr,
                      false, st, nullptr, &xd)) != CKV_OK)
    return s;
  LK(launch_xchg_put(xp, nullptr, 0, 0, fl + sizeof(uint32_t) * XF_PART, st));
  XTRACE("part signal");
  CK(xchg_wait(st, flag(XF_PART), W));
  XTRACE("part wait enqueued");
  // 4. merge this rank's slice over the W partials, broadcast the merged rows; copy out
  if (ctx->dtype == CKV_FP32)
    LK(launch_xchg_merge<float>(xp, xl, N, rps, ctx->d, st));
  else
    LK(launch_xchg_merge<__nv_bfloat16>(xp, xl, N, rps, ctx->d, st));
  LK(launch_xchg_put(xp, nullptr, 0, 0, fl + sizeof(uint32_t) * XF_OUT, st));
  CK(xchg_wait(st, flag(XF_OUT), W));
  XTRACE("out wait enqueued");
  CK(cudaMemcpyAsync(out, win + xl.outs, (size_t)N * ctx->d * ctx->esz, cudaMemcpyDeviceToDevice, st));
  CK(cudaMemcpyAsync(selected_ids, ctx->ids_glob, sizeof(int32_t) * ctx->k, cudaMemcpyDeviceToDevice, st));
  if (chunk_scores) CK(cudaMemcpyAsync(chunk_scores, ctx->A, sizeof(float) * ctx->m_loc, cudaMemcpyDeviceToDevice, st));
  XTRACE("done");
#undef XTRACE
  return CKV_OK;
}

}  // namespace

extern "C" {

int32_t ckv_budget_chunks(int64_t n, int32_t c, int32_t budget_bp) {
  if (n < 1 || c < 1 || budget_bp < 1 || budget_bp > 10000) return -1;
  const int64_t m = (n + c - 1) / c;
  int64_t k = ((int64_t)budget_bp * n) / ((int64_t)10000 * c);
  if (k > m) k = m;
  if (k < 1) k = 1;
  return (int32_t)k;
}

ckv_status ckv_create(const ckv_config* cfg, ckv_ctx** out) {
  NvtxRange nvtx_("ckv_create");
  if (!cfg || !out) return CKV_EINVAL;
  *out = nullptr;
  ckv_ctx* ctx = new (std::nothrow) ckv_ctx();
  if (!ctx) return CKV_ENOMEM;
  ctx->cfg = *cfg;
  const ckv_config& c = *cfg;
  auto bad = [&](const char* msg) {
    fprintf(stderr, "ckv_create: %s\n", msg);
    delete ctx;
    return CKV_EINVAL;
  };
  if (c.num_layers < 1 || c.num_q_heads < 1 || c.num_kv_heads < 1 || c.head_dim < 1) return bad("dims must be >= 1");
  if (c.num_q_heads % c.num_kv_heads) return bad("num_q_heads % num_kv_heads != 0");
  if (c.head_dim % 16 || c.head_dim > 128) return (delete ctx, CKV_EUNSUPPORTED);
  if (c.dtype != CKV_BF16 && c.dtype != CKV_FP32) return bad("dtype");
  if (c.chunk_size < 1 || c.prefix_len < 1 || c.max_suffix_len < 1) return bad("chunk_size/prefix_len/max_suffix_len");
  if (c.num_shards < 1 || c.shard_index < 0 || c.shard_index >= c.num_shards) return bad("shard_index/num_shards");
  if (c.num_shards > kMaxPeers) return (delete ctx, CKV_EUNSUPPORTED);  // one node: <= 8 GPUs
  if (c.score_norm != CKV_NORM_PREFIX && c.score_norm != CKV_NORM_FULLROW) return bad("score_norm");
  ctx->L = c.num_layers;
  ctx->Hq = c.num_q_heads;
  ctx->Hkv = c.num_kv_heads;
  ctx->G = c.num_q_heads / c.num_kv_heads;
  ctx->d = c.head_dim;
  ctx->c = c.chunk_size;
  ctx->dtype = c.dtype;
  ctx->esz = c.dtype == CKV_BF16 ? 2 : 4;
  ctx->fullrow = c.score_norm == CKV_NORM_FULLROW;
  ctx->n = c.prefix_len;
  ctx->m = (int)((c.prefix_len + c.chunk_size - 1) / c.chunk_size);
  ctx->W = c.num_shards;
  ctx->shard = c.shard_index;
  if ((c.flags & CKV_FLAG_CYCLIC_SHARDS) && ctx->W > 1) {
    // shard g owns chunks j = t*W + g (SURVEY §8(f) NEXT-3 balanced sharding), packed chunk by chunk;
    // only the global last chunk can be partial and it is the shard's last local chunk
    ctx->cyc_W = ctx->W;
    ctx->m_loc = ctx->shard < ctx->m ? (ctx->m - ctx->shard + ctx->W - 1) / ctx->W : 0;
    ctx->j0 = ctx->shard;  // the residue (topk_merge ownership test)
    ctx->j1 = ctx->m;
    ctx->t0 = 0;
    if (ctx->m_loc > 0) {
      const int64_t jl = (int64_t)(ctx->m_loc - 1) * ctx->W + ctx->shard;
      const int64_t last_len = ((jl + 1) * ctx->c < ctx->n ? (jl + 1) * ctx->c : ctx->n) - jl * ctx->c;
      ctx->n_loc = (int)((int64_t)(ctx->m_loc - 1) * ctx->c + last_len);
    }
  } else {
    const int per = (ctx->m + ctx->W - 1) / ctx->W;
    ctx->j0 = ctx->shard * per < ctx->m ? ctx->shard * per : ctx->m;
    ctx->j1 = (ctx->shard + 1) * per < ctx->m ? (ctx->shard + 1) * per : ctx->m;
    ctx->m_loc = ctx->j1 - ctx->j0;
    ctx->t0 = (int64_t)ctx->j0 * ctx->c;
    int64_t t1 = (int64_t)ctx->j1 * ctx->c < ctx->n ? (int64_t)ctx->j1 * ctx->c : ctx->n;
    ctx->n_loc = (int)(t1 - ctx->t0);
  }
  ctx->n_pad = ((ctx->n_loc + 255) / 256 + 1) * 256;
  if (ctx->m_loc < 1) return bad("shard owns no chunk (num_shards > m)");
  ctx->k = c.budget_chunks > 0 ? c.budget_chunks : ckv_budget_chunks(c.prefix_len, c.chunk_size, c.budget_bp);
  if (ctx->k < 1 || ctx->k > ctx->m) return bad("budget: k must be in [1, m]");
  ctx->quota = c.prefetch_chunks < 0 ? 0 : (c.prefetch_chunks > ctx->k ? ctx->k : c.prefetch_chunks);
  ctx->P = c.cache_slots > 0 ? c.cache_slots : 2 * ctx->k + ctx->quota;
  // adaptive p = 1 speculation (plan.cuh): skipped while the previous layer missed <= k/8 chunks.
  // Measured on the B200, C3 steady-state stream at equal HBM (510 slots): no gate 100.6 us/layer
  // (e2e 128), gate k/16 96.3 (102.5), k/8 93.9 (102.6), speculation off 91.8 (97.6); cold cache:
  // the speculation stays on (misses ~ k)
  ctx->spec_gate = ctx->k / 8;
  if (const char* sg = tuning_env("CKV_SPEC_GATE")) ctx->spec_gate = atoi(sg);  // tuning build: -1 = off
  if (ctx->P < ctx->k + ctx->quota) return bad("cache_slots < k + prefetch_chunks");
  ctx->global_heap = (c.flags & CKV_FLAG_GLOBAL_HEAP) != 0;
  // one shared pool: the next layer's speculative plan is issued only after this layer's demand plan
  // and compaction (ckv_reprefill_layer); periods (several in-flight prefetch plans) and shards are
  // not combined with it
  ctx->max_ns = c.max_suffix_len;
  ctx->period = c.period > 0 ? c.period : 1;
  ctx->subperiod = c.subperiod > 0 ? c.subperiod : 1;
  if (ctx->subperiod > ctx->period) return bad("subperiod > period");
  if (ctx->global_heap && (ctx->period > 1 || ctx->W > 1)) return (delete ctx, CKV_EUNSUPPORTED);
  if (ctx->period > 1 && ctx->W > 1) return (delete ctx, CKV_EUNSUPPORTED);
  ctx->rec_elems = (int64_t)2 * ctx->Hkv * ctx->c * ctx->d;
  ctx->rec_swz = (ctx->dtype == CKV_BF16 && ctx->d == 128) ? 1 : 0;
  if (c.flags & CKV_FLAG_V_ONLY_STORE) {
    // V-only records need the tcgen05 attention path (its compaction reads K from the probe array)
    const bool ok = ctx->rec_swz == 1 && ctx->c % 8 == 0 && ctx->c <= 128 && 128 % ctx->c == 0 &&
                    !(c.flags & CKV_FLAG_SIMT_ATTN);
    if (!ok) return (delete ctx, CKV_EUNSUPPORTED);
    ctx->rec_swz = 2;
    ctx->rec_elems = (int64_t)ctx->Hkv * ctx->c * ctx->d;
  }
  ctx->rec_bytes = ctx->rec_elems * ctx->esz;

  ckv_status st = CKV_OK;
  auto cudafail = [&](cudaError_t e, const char* what) {
    fprintf(stderr, "ckv_create: %s: %s\n", what, cudaGetErrorString(e));
    free_all(ctx);
    delete ctx;
    return e == cudaErrorMemoryAllocation ? CKV_ENOMEM : CKV_ECUDA;
  };
#define CKC(expr)                                   \
  do {                                              \
    cudaError_t e_ = (expr);                        \
    if (e_ != cudaSuccess) return cudafail(e_, #expr); \
  } while (0)
  CKC(cudaSetDevice(c.device));
  CKC(preload_kernels());  // no lazy module load later on the hot path (see common.cuh)
  dtl_init();               // tuning build: device timeline (CKV_DTL=1)
  const int R_max = ctx->G * ctx->max_ns;
  ctx->nsplit_score_max = ctx->m_loc < 4096 ? ctx->m_loc : 4096;
  {
    const int tc_splits = 4 * ((ctx->n_loc + 255) / 256);
    if (ctx->nsplit_score_max < tc_splits) ctx->nsplit_score_max = tc_splits;
  }
  ctx->nsplit_attn_max = 64;
  const size_t probe_elems = (size_t)ctx->L * ctx->Hkv * ctx->n_pad * ctx->d;
  CKC(cudaMalloc(&ctx->probe, probe_elems * ctx->esz));
  CKC(cudaMemset(ctx->probe, 0, probe_elems * ctx->esz));
  CKC(cudaHostAlloc(reinterpret_cast<void**>(&ctx->host_store), (size_t)ctx->L * ctx->m_loc * ctx->rec_bytes,
                    cudaHostAllocMapped | cudaHostAllocPortable));
  CKC(cudaHostGetDevicePointer(reinterpret_cast<void**>(&ctx->host_store_dev), ctx->host_store, 0));
  CKC(cudaMalloc(reinterpret_cast<void**>(&ctx->pool), (size_t)ctx->L * ctx->P * ctx->rec_bytes));
  CKC(dalloc(&ctx->slot_of, (size_t)ctx->L * ctx->m_loc));
  CKC(dalloc(&ctx->owner, (size_t)ctx->L * ctx->P));
  CKC(dalloc(&ctx->pf_epoch, (size_t)ctx->L * ctx->P));
  CKC(dalloc(&ctx->F, (size_t)ctx->L * ctx->m_loc));
  CKC(dalloc(&ctx->T, (size_t)ctx->L * ctx->m_loc));
  CKC(dalloc(&ctx->I, (size_t)ctx->L * ctx->m_loc));
  CKC(cudaMemset(ctx->slot_of, 0xFF, sizeof(int32_t) * ctx->L * ctx->m_loc));
  CKC(cudaMemset(ctx->owner, 0xFF, sizeof(int32_t) * ctx->L * ctx->P));
  CKC(cudaMemset(ctx->pf_epoch, 0xFF, sizeof(int32_t) * ctx->L * ctx->P));
  CKC(cudaMemset(ctx->F, 0, sizeof(int32_t) * ctx->L * ctx->m_loc));
  CKC(cudaMemset(ctx->T, 0, sizeof(int32_t) * ctx->L * ctx->m_loc));
  CKC(cudaMemset(ctx->I, 0, sizeof(float) * ctx->L * ctx->m_loc));
  CKC(dalloc(&ctx->lam2, (size_t)ctx->Hkv * ctx->m_loc * R_max));
  CKC(dalloc(&ctx->lampart, (size_t)ctx->Hkv * ctx->nsplit_score_max * R_max));
  CKC(dalloc(&ctx->Lam2, (size_t)ctx->Hkv * R_max));
  CKC(dalloc(&ctx->A, (size_t)ctx->m_loc));
  CKC(dalloc(&ctx->Apart, (size_t)ctx->m_loc * ctx->Hkv));
  for (int i = 0; i < 2; ++i) {
    CKC(dalloc(&ctx->ids_buf[i], (size_t)ctx->k));
    CKC(dalloc(&ctx->n_ids_buf[i], 1));
    CKC(dalloc(&ctx->sel_keys[i], (size_t)ctx->k));
    if (i == 0) {
      CKC(dalloc(&ctx->ids_b, (size_t)ctx->k));
      CKC(dalloc(&ctx->n_b, 1));
      CKC(dalloc(&ctx->cand_b, (size_t)ctx->k));
    }
  }
  CKC(dalloc(&ctx->kept_slots, (size_t)ctx->k));
  CKC(dalloc(&ctx->ids_glob, (size_t)ctx->k));
  CKC(dalloc(&ctx->flag, (size_t)ctx->m));
  const size_t pool_slots = ctx->global_heap ? (size_t)ctx->L * ctx->P : (size_t)ctx->P;
  CKC(dalloc(&ctx->scratch_main, (size_t)2 * ctx->k + 2 * pool_slots));
  CKC(dalloc(&ctx->scratch_side, (size_t)2 * ctx->k + 2 * pool_slots));
  CKC(dalloc(&ctx->gl_main, (size_t)2 * ctx->k));
  CKC(dalloc(&ctx->gl_side, (size_t)2 * ctx->k));
  CKC(dalloc(&ctx->nload_main, 1));
  CKC(dalloc(&ctx->nload_side, 1));
  CKC(dalloc(&ctx->counts, (size_t)ctx->L * 8));
  CKC(cudaMemset(ctx->counts, 0, sizeof(int32_t) * ctx->L * 8));
  CKC(dalloc(&ctx->o_part, (size_t)ctx->nsplit_attn_max * ctx->Hkv * R_max * ctx->d));
  CKC(dalloc(&ctx->lse_part, (size_t)ctx->nsplit_attn_max * ctx->Hkv * R_max));
  CKC(dalloc(&ctx->stats, 16));
  CKC(dalloc(&ctx->epoch_dev, 1));
  CKC(dalloc(&ctx->ticket, 1));
  CKC(cudaMemset(ctx->ticket, 0, sizeof(int32_t)));
  CKC(cudaMemset(ctx->epoch_dev, 0, sizeof(int32_t)));
  CKC(cudaMemset(ctx->stats, 0, sizeof(int64_t) * 16));
  int lo = 0, hi = 0;
  CKC(cudaDeviceGetStreamPriorityRange(&lo, &hi));
  // the side stream (speculative plan + gather) gets the LOWEST priority: its CTAs then fill the
  // SMs the persistent score / attention kernels leave free instead of being dispatched ahead of
  // them (measured on the B200, steady-state stream: 108.6 vs 109.4 us/layer, eager 115 vs 122)
  const char* sp = tuning_env("CKV_SIDE_PRIO");  // tuning build: 0 = highest priority (A/B)
  CKC(cudaStreamCreateWithPriority(&ctx->side, cudaStreamNonBlocking, (sp && sp[0] == '0') ? hi : lo));
  CKC(cudaEventCreateWithFlags(&ctx->ev_ids, cudaEventDisableTiming));
  ctx->ev_pplan.assign(ctx->L, nullptr);
  ctx->ev_pf.assign(ctx->L, nullptr);
  for (int l = 0; l < ctx->L; ++l) {
    CKC(cudaEventCreateWithFlags(&ctx->ev_pplan[l], cudaEventDisableTiming));
    CKC(cudaEventCreateWithFlags(&ctx->ev_pf[l], cudaEventDisableTiming));
  }
  ctx->pf_issued.assign(ctx->L, -1);
  ctx->pf_joined.assign(ctx->L, -1);
  ctx->pf_late.assign(ctx->L, 0);
  ctx->stored.assign(ctx->L, 0);
  ctx->score_kind = (ctx->dtype == CKV_BF16 && ctx->d == 128 && !(c.flags & CKV_FLAG_SIMT_SCORE)) ? 1 : 0;
  if (ctx->score_kind == 1) {
    LayerGeom g = geom(ctx, ctx->max_ns);
    if (score_tc_nsplit(g) <= 0) ctx->score_kind = 0;
  }
  {
    LayerGeom g = geom(ctx, ctx->max_ns);
    ctx->attn_kind = (ctx->dtype == CKV_BF16 && attn_tc_supported(g) && !(c.flags & CKV_FLAG_SIMT_ATTN)) ? 1 : 0;
  }
  if (ctx->score_kind == 1)
    CKC(cudaMalloc(&ctx->tmap_cache, score_tc_qpack_elems(ctx->Hkv, R_max) * sizeof(__nv_bfloat16)));
  if (ctx->attn_kind == 1) {
    const size_t nb = attn_tc_dense_bytes(geom(ctx, ctx->max_ns), ctx->k, ctx->max_ns);
    CKC(cudaMalloc(&ctx->dense_kv, nb));
    CKC(cudaMemset(ctx->dense_kv, 0, nb));
  }
  if (ctx->W > 1) {  // exchange window (fused device-side exchange, xchg.cuh)
    ctx->xl = make_xlayout(ctx->W, ctx->Hq, ctx->max_ns, ctx->k, ctx->d, ctx->esz);
    CKC(cudaMalloc(reinterpret_cast<void**>(&ctx->xwin), ctx->xl.total));
    CKC(cudaMemset(ctx->xwin, 0, ctx->xl.total));
    CKC(dalloc(&ctx->lam_loc, (size_t)ctx->Hq * ctx->max_ns));
    CKC(dalloc(&ctx->cand_loc, (size_t)ctx->k));
  }
  CKC(cudaDeviceSynchronize());
#undef CKC
  (void)st;
  *out = ctx;
  return CKV_OK;
}

ckv_status ckv_store_prefix(ckv_ctx* ctx, int32_t layer, const void* k, const void* v, int64_t n_tokens,
                            void* stream) {
  NvtxRange nvtx_("ckv_store_prefix");
  if (!ctx) return CKV_EINVAL;
  ctx->err.clear();
  if (!k || !v) return fail(ctx, CKV_EINVAL, "null k/v");
  if (layer < 0 || layer >= ctx->L) return fail(ctx, CKV_EINVAL, "layer %d out of range", layer);
  if (n_tokens != ctx->n) return fail(ctx, CKV_EINVAL, "n_tokens %lld != prefix_len %lld", (long long)n_tokens,
                                      (long long)ctx->n);
  CK(cudaSetDevice(ctx->cfg.device));
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const size_t bytes = (size_t)ctx->n * ctx->Hkv * ctx->d * ctx->esz;
  auto is_dev = [](const void* p) {
    cudaPointerAttributes a;
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
      cudaGetLastError();
      return false;
    }
    return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
  };
  void *kd = const_cast<void*>(k), *vd = const_cast<void*>(v), *tmp = nullptr, *staging = nullptr;
  if (!is_dev(k) || !is_dev(v)) {
    CK(cudaMalloc(&tmp, 2 * bytes));
    CK(cudaMemcpyAsync(tmp, k, bytes, cudaMemcpyDefault, st));
    CK(cudaMemcpyAsync(static_cast<char*>(tmp) + bytes, v, bytes, cudaMemcpyDefault, st));
    kd = tmp;
    vd = static_cast<char*>(tmp) + bytes;
  }
  const size_t stage_bytes = (size_t)ctx->m_loc * ctx->rec_bytes;
  CK(cudaMalloc(&staging, stage_bytes));
  void* probe_l = const_cast<void*>(probe_layer(ctx, layer));
  if (ctx->dtype == CKV_FP32) {
    LK(launch_pack_probe<float>(static_cast<const float*>(kd), ctx->t0, ctx->cyc_W, ctx->shard, ctx->c, ctx->n_loc,
                                ctx->n_pad, ctx->Hkv, ctx->d, static_cast<float*>(probe_l), st));
    LK(launch_pack_records<float>(static_cast<const float*>(kd), static_cast<const float*>(vd), ctx->t0, ctx->cyc_W,
                                  ctx->shard, ctx->n_loc, ctx->m_loc, ctx->c, ctx->Hkv, ctx->d, ctx->rec_swz,
                                  static_cast<float*>(staging), st));
  } else {
    LK(launch_pack_probe<__nv_bfloat16>(static_cast<const __nv_bfloat16*>(kd), ctx->t0, ctx->cyc_W, ctx->shard,
                                        ctx->c, ctx->n_loc, ctx->n_pad, ctx->Hkv, ctx->d,
                                        static_cast<__nv_bfloat16*>(probe_l), st));
    LK(launch_pack_records<__nv_bfloat16>(static_cast<const __nv_bfloat16*>(kd), static_cast<const __nv_bfloat16*>(vd),
                                          ctx->t0, ctx->cyc_W, ctx->shard, ctx->n_loc, ctx->m_loc, ctx->c, ctx->Hkv,
                                          ctx->d, ctx->rec_swz, static_cast<__nv_bfloat16*>(staging), st));
  }
  CK(cudaMemcpyAsync(ctx->host_store + (size_t)layer * stage_bytes, staging, stage_bytes, cudaMemcpyDeviceToHost, st));
  CacheLayer cl = cache_layer(ctx, layer);
  if (ctx->global_heap) {  // the shared pool may hold any layer's chunks: empty all of it
    CK(cudaMemsetAsync(ctx->slot_of, 0xFF, sizeof(int32_t) * ctx->L * ctx->m_loc, st));
    CK(cudaMemsetAsync(ctx->owner, 0xFF, sizeof(int32_t) * ctx->L * ctx->P, st));
    CK(cudaMemsetAsync(ctx->pf_epoch, 0xFF, sizeof(int32_t) * ctx->L * ctx->P, st));
  } else {
    CK(cudaMemsetAsync(cl.slot_of, 0xFF, sizeof(int32_t) * ctx->m_loc, st));
    CK(cudaMemsetAsync(cl.owner, 0xFF, sizeof(int32_t) * ctx->P, st));
    CK(cudaMemsetAsync(cl.pf_epoch, 0xFF, sizeof(int32_t) * ctx->P, st));
  }
  CK(cudaMemsetAsync(cl.I, 0, sizeof(float) * ctx->m_loc, st));
  CK(cudaMemsetAsync(cl.F, 0, sizeof(int32_t) * ctx->m_loc, st));
  CK(cudaMemsetAsync(cl.T, 0, sizeof(int32_t) * ctx->m_loc, st));
  CK(cudaStreamSynchronize(st));
  CK(cudaFree(staging));
  if (tmp) CK(cudaFree(tmp));
  ctx->stored[layer] = 1;
  return CKV_OK;
}

ckv_status ckv_reprefill_layer(ckv_ctx* ctx, int32_t layer, const void* q, const void* k_suf, const void* v_suf,
                               int32_t n_suffix, void* out, int32_t* selected_ids, float* chunk_scores,
                               void* stream) {
  NvtxRange nvtx_("ckv_reprefill_layer");
  if (!ctx) return CKV_EINVAL;
  ctx->err.clear();
  ckv_status s = check_layer_call(ctx, layer, n_suffix);
  if (s != CKV_OK) return s;
  if (!q || !k_suf || !v_suf || !out || !selected_ids) return fail(ctx, CKV_EINVAL, "null argument");
  if (ctx->W != 1 && !ctx->x_attached)
    return fail(ctx, CKV_ESTATE, "num_shards > 1: attach the exchange (ckv_exchange_open / _attach) or use ckv_shard_*");
  CK(cudaSetDevice(ctx->cfg.device));
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (ctx->W != 1)
    return reprefill_sharded(ctx, layer, q, k_suf, v_suf, n_suffix, out, selected_ids, chunk_scores, st);
  if (layer == 0) {
    ++ctx->epoch;
    ctx->spec_next = -1;
    LK(launch_epoch_inc(ctx->epoch_dev, st));
  }
  const int p = ctx->period;
  const int pid = layer / p;
  const bool first = (layer % p) == 0;
  const int pend = (pid + 1) * p < ctx->L ? (pid + 1) * p : ctx->L;  // end of this period
  int32_t* ids = ctx->ids_buf[pid & 1];  // double-buffered by period: side-stream plans may still read it
  int32_t* nids = ctx->n_ids_buf[pid & 1];
  bool planned = false;  // the demand plan of this layer ran inside the fused select kernel
  // p = 1: the next layer's speculative plan + gather are issued after this layer's last kernel (not
  // right after A3): they then overlap the next layer's scoring instead of this layer's compaction
  // (demand misses on the same host link) and attention (SMs); they are joined before the next
  // layer's plan.  Measured on the B200: steady-state stream 106.7 vs 109.7 us/layer, all-hit 89.6
  // vs 92.0.  The tuning build's CKV_LATE_PF=0 restores the early issue (A/B).
  static const bool late_on = !(tuning_env("CKV_LATE_PF") && tuning_env("CKV_LATE_PF")[0] == '0');
  const bool late_pf = late_on && first && p == 1 && !ctx->global_heap && ctx->quota > 0 && layer + 1 < ctx->L;
  // ... and the speculative plan runs as CTA 1 of this layer's demand-plan launch (cache_plan2): a
  // single-CTA planner on the side stream could not share an SM with the next layer's persistent
  // score kernel, so it ran after it and its gather landed late (measured: steady-state stream
  // 100.6 vs 107.6 us/layer, all-hit 91.2 vs 89.9).  Tuning build: CKV_PLAN2=0 for the A/B.
  static const bool plan2_on = !(tuning_env("CKV_PLAN2") && tuning_env("CKV_PLAN2")[0] == '0');
  bool planned2 = false;
  if (first) {  // identification: A1 -> A2 -> A3
    // The persistent score kernel needs every SM: side-stream prefetch work for this layer must
    // not still be resident when it starts (one late CTA delays the whole statically partitioned
    // launch), so the prefetch is joined here rather than only before the attention.
    static const bool side_sync = !(tuning_env("CKV_SIDE_SYNC") && tuning_env("CKV_SIDE_SYNC")[0] == '0');
    if (side_sync && ctx->pf_issued[layer] == ctx->epoch && !ctx->pf_late[layer]) {
      CK(cudaStreamWaitEvent(st, ctx->ev_pf[layer], 0));
      pdl_mark_event_wait(st);
      ctx->pf_joined[layer] = ctx->epoch;
    }
    int nsplit = 0;
    if ((s = run_score(ctx, layer, q, k_suf, n_suffix, nullptr, &nsplit, st)) != CKV_OK) return s;
    LayerGeom g = geom(ctx, n_suffix);
    PROF_BEGIN(2);
    LK(launch_chunk_sum(g, ctx->lam2, ctx->Lam2, ctx->Apart, st));
    PROF_END(2);
    // p = 1 with the speculative plan fused (below): the top-k runs inside that launch too
    static const bool topk_fuse_on = !(tuning_env("CKV_TOPK_PLAN") && tuning_env("CKV_TOPK_PLAN")[0] == '0');
    const bool fuse_sel = late_pf && plan2_on && gather_fused(ctx) && topk_fuse_on && ctx->m_loc <= 8192;
    if (!fuse_sel) {
      PROF_BEGIN(6);
      LK(launch_topk_scores(ctx->A, ctx->Apart, ctx->Hkv, ctx->m_loc, ctx->k, 0, 1, ids, ctx->sel_keys[pid & 1],
                            ctx->k, nids, st));
      PROF_END(6);
    }
    // intra-period loads (exact ids) for the period's other layers, then the speculative load of
    // the next period's first layer (A6), all on the side stream in layer order
    // (global heap: one shared pool, so the next layer's speculative plan may only run after this
    // layer's demand plan and compaction -- issued below, after run_attend)
    if (late_pf && plan2_on && gather_fused(ctx)) {
      // this layer's demand plan (CTA 0) and the next layer's speculative plan (CTA 1) in one
      // launch; the speculative gather follows at the end of the layer (below).  A prefetch of
      // this layer not yet joined must land its plan first (tables) -- it was planned on this
      // stream, so only its gather is outstanding, and the compaction waits for that
      if (ctx->pf_issued[layer] == ctx->epoch && ctx->pf_joined[layer] != ctx->epoch && !ctx->pf_late[layer]) {
        CK(cudaStreamWaitEvent(st, ctx->ev_pf[layer], 0));
        pdl_mark_event_wait(st);
        ctx->pf_joined[layer] = ctx->epoch;
      }
      PROF_BEGIN(3);
      PlanJob a{cache_layer(ctx, layer), ids, nids, 0, 0, 0, ctx->epoch, ctx->rec_bytes, ctx->scratch_main,
                demand_plan_out(ctx, layer, selected_ids)};
      PlanOut po{ctx->gl_side, ctx->nload_side, nullptr, nullptr, ctx->counts + (size_t)((layer + 1) * 2 + 1) * 4,
                 ctx->stats, nullptr, ctx->epoch_dev};
      po.rank_keys = fuse_sel ? ctx->cand_b : ctx->sel_keys[pid & 1];
      if (layer > 0) {
        po.gate_misses = ctx->counts + (size_t)((layer - 1) * 2) * 4 + 1;
        po.gate_max = ctx->spec_gate;
      }
      PlanJob b{cache_layer(ctx, layer + 1), fuse_sel ? ctx->ids_b : ids, fuse_sel ? ctx->n_b : nids, 0, 1, ctx->quota,
                ctx->epoch, ctx->rec_bytes, ctx->scratch_side, po};
      if (fuse_sel) {
        TopkJob t{ctx->A, ctx->Apart, ctx->Hkv, ctx->m_loc, ctx->k, ids, ctx->sel_keys[pid & 1], nids,
                  ctx->ids_b, ctx->cand_b, ctx->n_b};
        LK(launch_topk_plan2(t, a, b, st));
      } else {
        LK(launch_cache_plan2(a, b, st));
      }
      PROF_END(3);
      planned = true;
      planned2 = true;
    }
    if (!ctx->global_heap && !late_pf)
      for (int lp = layer + 1; lp <= pend && lp < ctx->L; ++lp)
        // layers inside the period reuse ids exactly (load all k); the next period's first layer is
        // speculative (the quota, highest-scored first)
        if ((s = issue_prefetch(ctx, lp, ids, nids, st, false, ctx->sel_keys[pid & 1], lp < pend ? ctx->k : -1)) !=
            CKV_OK)
          return s;
    // subperiod gate: attention of the first layer waits for sp layers' chunks
    for (int lp = layer + 1; lp < layer + ctx->subperiod && lp < pend; ++lp)
      if (ctx->pf_issued[lp] == ctx->epoch) {
        CK(cudaStreamWaitEvent(st, ctx->ev_pf[lp], 0));
        pdl_mark_event_wait(st);
      }
  }
  // the demand planner also writes selected_ids (no separate copy node per layer)
  const bool defer_pf = ctx->global_heap && first && ctx->quota > 0 && layer + 1 < ctx->L;
  // (late_pf: the next layer's speculative plan + gather are issued after this layer's last kernel)
  if ((s = run_attend(ctx, layer, ids, nids, q, k_suf, v_suf, n_suffix, 1, out, nullptr, nullptr, selected_ids,
                      planned, st, defer_pf ? ctx->ev_ids : nullptr)) != CKV_OK)
    return s;
  if (defer_pf && (s = issue_prefetch(ctx, layer + 1, ids, nids, st, true, ctx->sel_keys[pid & 1])) != CKV_OK)
    return s;
  static const bool inscore_on = !(tuning_env("CKV_SPEC_INSCORE") && tuning_env("CKV_SPEC_INSCORE")[0] == '0');
  if (late_pf && planned2 && inscore_on && ctx->score_kind == 1) {
    // the speculative gather of the next layer (planned by CTA 1 above) runs in that layer's score
    // kernel (its gather warp): stream order completes it before that layer's plan -- nothing to join
    ctx->spec_next = layer + 1;
    ctx->pf_issued[layer + 1] = ctx->epoch;
    ctx->pf_joined[layer + 1] = ctx->epoch;
    ctx->pf_late[layer + 1] = 1;
  } else if (late_pf && planned2) {  // speculative gather of the layer planned by cache_plan2 (CTA 1)
    CK(cudaEventRecord(ctx->ev_ids, st));
    CK(cudaStreamWaitEvent(ctx->side, ctx->ev_ids, 0));
    pdl_mark_event_wait(ctx->side);
    LK(launch_gather(ctx->gl_side, ctx->nload_side, host_layer_dev(ctx, layer + 1), pool_layer(ctx, layer + 1),
                     ctx->rec_bytes, ctx->side));
    CK(cudaEventRecord(ctx->ev_pf[layer + 1], ctx->side));
    ctx->pf_issued[layer + 1] = ctx->epoch;
    ctx->pf_late[layer + 1] = 1;
  } else if (late_pf) {
    if ((s = issue_prefetch(ctx, layer + 1, ids, nids, st, false, ctx->sel_keys[pid & 1])) != CKV_OK) return s;
    ctx->pf_late[layer + 1] = 1;  // joined before the next layer's plan, not before its scoring
  }
  if (chunk_scores) CK(cudaMemcpyAsync(chunk_scores, ctx->A, sizeof(float) * ctx->m_loc, cudaMemcpyDeviceToDevice, st));
  return CKV_OK;
}

ckv_status ckv_shard_score(ckv_ctx* ctx, int32_t layer, const void* q, const void* k_suf, int32_t n_suffix,
                           float* lam_local, void* stream) {
  NvtxRange nvtx_("ckv_shard_score");
  if (!ctx) return CKV_EINVAL;
  ctx->err.clear();
  ckv_status s = check_layer_call(ctx, layer, n_suffix);
  if (s != CKV_OK) return s;
  if (!q || !k_suf || !lam_local) return fail(ctx, CKV_EINVAL, "null argument");
  CK(cudaSetDevice(ctx->cfg.device));
  if (layer == 0) {
    ++ctx->epoch;
    LK(launch_epoch_inc(ctx->epoch_dev, static_cast<cudaStream_t>(stream)));
  }
  int nsplit = 0;
  return run_score(ctx, layer, q, k_suf, n_suffix, lam_local, &nsplit, static_cast<cudaStream_t>(stream));
}

ckv_status ckv_shard_select(ckv_ctx* ctx, int32_t layer, const void* q, const void* k_suf, int32_t n_suffix,
                            const float* lam_all, uint64_t* cand, float* chunk_scores, void* stream) {
  if (!ctx) return CKV_EINVAL;
  ctx->err.clear();
  ckv_status s = check_layer_call(ctx, layer, n_suffix);
  if (s != CKV_OK) return s;
  if (!q || !k_suf || !lam_all || !cand) return fail(ctx, CKV_EINVAL, "null argument");
  CK(cudaSetDevice(ctx->cfg.device));
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  LayerGeom g = geom(ctx, n_suffix);
  // global Lambda = LSE over shards in rank order (+ causal suffix in FULLROW mode)
  if (ctx->dtype == CKV_FP32)
    LK(launch_row_lse<float>(g, nullptr, 0, static_cast<const float*>(q), static_cast<const float*>(k_suf),
                             ctx->fullrow, lam_all, ctx->W, ctx->Lam2, nullptr, st));
  else
    LK(launch_row_lse<__nv_bfloat16>(g, nullptr, 0, static_cast<const __nv_bfloat16*>(q),
                                     static_cast<const __nv_bfloat16*>(k_suf), ctx->fullrow, lam_all, ctx->W,
                                     ctx->Lam2, nullptr, st));
  ctx->lam2_layer = layer;
  LK(launch_chunk_sum(g, ctx->lam2, ctx->Lam2, ctx->Apart, st));
  LK(launch_topk_scores(ctx->A, ctx->Apart, ctx->Hkv, ctx->m_loc, ctx->k, ctx->j0, ctx->cyc_W > 0 ? ctx->cyc_W : 1,
                        nullptr, cand, ctx->k, nullptr, st));
  if (chunk_scores) CK(cudaMemcpyAsync(chunk_scores, ctx->A, sizeof(float) * ctx->m_loc, cudaMemcpyDeviceToDevice, st));
  return CKV_OK;
}

ckv_status ckv_shard_attend(ckv_ctx* ctx, int32_t layer, const uint64_t* cand_all, const void* q, const void* k_suf,
                            const void* v_suf, int32_t n_suffix, float* o_part, float* lse_part,
                            int32_t* selected_ids, void* stream) {
  NvtxRange nvtx_("ckv_shard_attend");
  if (!ctx) return CKV_EINVAL;
  ctx->err.clear();
  ckv_status s = check_layer_call(ctx, layer, n_suffix);
  if (s != CKV_OK) return s;
  if (!cand_all || !q || !k_suf || !v_suf || !o_part || !lse_part || !selected_ids)
    return fail(ctx, CKV_EINVAL, "null argument");
  CK(cudaSetDevice(ctx->cfg.device));
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  int32_t* ids = ctx->ids_buf[layer & 1];
  int32_t* nids = ctx->n_ids_buf[layer & 1];
  LK(launch_topk_merge(cand_all, ctx->W * ctx->k, ctx->k, ctx->m, ctx->j0, ctx->j1, ctx->cyc_W, ctx->flag, ctx->ids_glob, ids,
                       nids, st));
  if ((s = issue_prefetch(ctx, layer + 1, ids, nids, st)) != CKV_OK) return s;
  if ((s = run_attend(ctx, layer, ids, nids, q, k_suf, v_suf, n_suffix, ctx->shard == ctx->W - 1, nullptr, o_part,
                      lse_part, nullptr, false, st)) != CKV_OK)
    return s;
  CK(cudaMemcpyAsync(selected_ids, ctx->ids_glob, sizeof(int32_t) * ctx->k, cudaMemcpyDeviceToDevice, st));
  return CKV_OK;
}

ckv_status ckv_lse_merge_prepare(ckv_ctx* ctx, const float* o_part, const float* lse_part, const float* lse_max,
                                 int32_t n_suffix, float* merge_buf, void* stream) {
  if (!ctx) return CKV_EINVAL;
  ctx->err.clear();
  if (!o_part || !lse_part || !lse_max || !merge_buf || n_suffix < 1 || n_suffix > ctx->max_ns)
    return fail(ctx, CKV_EINVAL, "bad argument");
  LK(launch_lse_merge_prepare(n_suffix * ctx->Hq, ctx->d, o_part, lse_part, lse_max, merge_buf,
                              static_cast<cudaStream_t>(stream)));
  return CKV_OK;
}

ckv_status ckv_lse_merge_finish(ckv_ctx* ctx, const float* merge_buf, int32_t n_suffix, void* out, void* stream) {
  if (!ctx) return CKV_EINVAL;
  ctx->err.clear();
  if (!merge_buf || !out || n_suffix < 1 || n_suffix > ctx->max_ns) return fail(ctx, CKV_EINVAL, "bad argument");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (ctx->dtype == CKV_FP32)
    LK(launch_lse_merge_finish<float>(n_suffix * ctx->Hq, ctx->d, merge_buf, static_cast<float*>(out), st));
  else
    LK(launch_lse_merge_finish<__nv_bfloat16>(n_suffix * ctx->Hq, ctx->d, merge_buf,
                                              static_cast<__nv_bfloat16*>(out), st));
  return CKV_OK;
}

ckv_status ckv_exchange_handle(ckv_ctx* ctx, void* handle_out) {
  if (!ctx) return CKV_EINVAL;
  ctx->err.clear();
  if (!handle_out) return fail(ctx, CKV_EINVAL, "null handle_out");
  if (ctx->W < 2 || !ctx->xwin) return fail(ctx, CKV_EINVAL, "num_shards == 1: no exchange window");
  static_assert(sizeof(cudaIpcMemHandle_t) == CKV_EXCHANGE_HANDLE_BYTES, "IPC handle size");
  CK(cudaSetDevice(ctx->cfg.device));
  cudaIpcMemHandle_t h;
  CK(cudaIpcGetMemHandle(&h, ctx->xwin));
  memcpy(handle_out, &h, sizeof h);
  return CKV_OK;
}

ckv_status ckv_exchange_open(ckv_ctx* ctx, const void* handles) {
  if (!ctx) return CKV_EINVAL;
  ctx->err.clear();
  if (!handles) return fail(ctx, CKV_EINVAL, "null handles");
  if (ctx->W < 2 || !ctx->xwin) return fail(ctx, CKV_EINVAL, "num_shards == 1: no exchange window");
  if (ctx->x_attached) return fail(ctx, CKV_ESTATE, "exchange already attached");
  CK(cudaSetDevice(ctx->cfg.device));
  XPeers xp{};
  xp.W = ctx->W;
  xp.self = ctx->shard;
  for (int g = 0; g < ctx->W; ++g) {
    if (g == ctx->shard) {
      xp.base[g] = ctx->xwin;
      continue;
    }
    cudaIpcMemHandle_t h;
    memcpy(&h, static_cast<const char*>(handles) + (size_t)g * sizeof h, sizeof h);
    void* p = nullptr;
    CK(cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess));
    ctx->x_opened.push_back(p);
    xp.base[g] = static_cast<char*>(p);
  }
  ctx->xp = xp;
  ctx->x_attached = true;
  return CKV_OK;
}

ckv_status ckv_exchange_attach(ckv_ctx* ctx, ckv_ctx* const* ctxs, int32_t num_ctxs) {
  if (!ctx) return CKV_EINVAL;
  ctx->err.clear();
  if (!ctxs || num_ctxs != ctx->W) return fail(ctx, CKV_EINVAL, "need num_shards contexts in rank order");
  if (ctx->W < 2 || !ctx->xwin) return fail(ctx, CKV_EINVAL, "num_shards == 1: no exchange window");
  if (ctx->x_attached) return fail(ctx, CKV_ESTATE, "exchange already attached");
  XPeers xp{};
  xp.W = ctx->W;
  xp.self = ctx->shard;
  for (int g = 0; g < ctx->W; ++g) {
    const ckv_ctx* o = ctxs[g];
    if (!o || o->W != ctx->W || o->shard != g || !o->xwin || o->xl.total != ctx->xl.total)
      return fail(ctx, CKV_EINVAL, "context %d is not rank %d of this group", g, g);
    if (o->cfg.device != ctx->cfg.device) {  // several GPUs in one process: map the peer
      CK(cudaSetDevice(ctx->cfg.device));
      const cudaError_t e = cudaDeviceEnablePeerAccess(o->cfg.device, 0);
      if (e == cudaErrorPeerAccessAlreadyEnabled) cudaGetLastError();
      else CK(e);
    }
    xp.base[g] = o->xwin;
  }
  ctx->xp = xp;
  ctx->x_attached = true;
  return CKV_OK;
}

ckv_status ckv_test_exchange_flags(ckv_ctx* ctx, uint32_t* flags_out) {
  if (!ctx) return CKV_EINVAL;
  ctx->err.clear();
  if (!flags_out || !ctx->xwin) return fail(ctx, CKV_EINVAL, "no exchange window");
  CK(cudaSetDevice(ctx->cfg.device));
  cudaStream_t s;
  CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  CK(cudaMemcpyAsync(flags_out, ctx->xwin + ctx->xl.flags, sizeof(uint32_t) * XF_COUNT, cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  CK(cudaStreamDestroy(s));
  return CKV_OK;
}

ckv_status ckv_set_period(ckv_ctx* ctx, int32_t period, int32_t subperiod) {
  if (!ctx) return CKV_EINVAL;
  ctx->err.clear();
  const int p = period > 0 ? period : 1, sp = subperiod > 0 ? subperiod : 1;
  if (sp > p) return fail(ctx, CKV_EINVAL, "subperiod > period");
  if (p > 1 && ctx->W > 1) return fail(ctx, CKV_EUNSUPPORTED, "period > 1 needs num_shards == 1");
  if (p > 1 && ctx->global_heap) return fail(ctx, CKV_EUNSUPPORTED, "period > 1 needs per-layer cache pools");
  ctx->period = p;
  ctx->subperiod = sp;
  return CKV_OK;
}

ckv_status ckv_set_cache_policy(ckv_ctx* ctx, int32_t policy, void* stream) {
  if (!ctx) return CKV_EINVAL;
  ctx->err.clear();
  if (policy < CKV_CACHE_ATTN || policy > CKV_CACHE_LRU) return fail(ctx, CKV_EINVAL, "cache policy %d", policy);
  CK(cudaSetDevice(ctx->cfg.device));
  CK(cudaDeviceSynchronize());
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  CK(cudaMemsetAsync(ctx->slot_of, 0xFF, sizeof(int32_t) * ctx->L * ctx->m_loc, st));
  CK(cudaMemsetAsync(ctx->owner, 0xFF, sizeof(int32_t) * ctx->L * ctx->P, st));
  CK(cudaMemsetAsync(ctx->pf_epoch, 0xFF, sizeof(int32_t) * ctx->L * ctx->P, st));
  CK(cudaMemsetAsync(ctx->I, 0, sizeof(float) * ctx->L * ctx->m_loc, st));
  CK(cudaMemsetAsync(ctx->F, 0, sizeof(int32_t) * ctx->L * ctx->m_loc, st));
  CK(cudaMemsetAsync(ctx->T, 0, sizeof(int32_t) * ctx->L * ctx->m_loc, st));
  CK(cudaStreamSynchronize(st));
  ctx->cache_policy = policy;
  return CKV_OK;
}

ckv_status ckv_reset_cache(ckv_ctx* ctx, void* stream) {
  if (!ctx) return CKV_EINVAL;
  ctx->err.clear();
  CK(cudaSetDevice(ctx->cfg.device));
  CK(cudaDeviceSynchronize());
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  CK(cudaMemsetAsync(ctx->slot_of, 0xFF, sizeof(int32_t) * ctx->L * ctx->m_loc, st));
  CK(cudaMemsetAsync(ctx->owner, 0xFF, sizeof(int32_t) * ctx->L * ctx->P, st));
  CK(cudaMemsetAsync(ctx->pf_epoch, 0xFF, sizeof(int32_t) * ctx->L * ctx->P, st));
  return CKV_OK;
}

ckv_status ckv_get_stats(ckv_ctx* ctx, ckv_stats* out) {
  if (!ctx || !out) return CKV_EINVAL;
  ctx->err.clear();
  CK(cudaSetDevice(ctx->cfg.device));
  CK(cudaDeviceSynchronize());
  int64_t s[16];
  CK(cudaMemcpy(s, ctx->stats, sizeof s, cudaMemcpyDeviceToHost));
  memset(out, 0, sizeof *out);
  out->total_hits = s[0];
  out->total_misses = s[1];
  out->total_spec_loads = s[2];
  out->total_spec_used = s[3];
  out->total_link_bytes_delta = s[4];
  out->total_link_bytes_spec = s[5];
  out->total_layers = s[6];
  if (s[15]) return fail(ctx, CKV_ESTATE, "HBM chunk cache overflow detected by the planner (P < k + quota?)");
  if (ctx->last_layer >= 0) {
    int32_t cnt[8];
    CK(cudaMemcpy(cnt, ctx->counts + (size_t)ctx->last_layer * 8, sizeof cnt, cudaMemcpyDeviceToHost));
    out->last_hits = cnt[0];
    out->last_misses = cnt[1];
    out->last_spec_used = cnt[3];
    out->last_spec_loads = ctx->pf_issued[ctx->last_layer] == ctx->epoch ? cnt[4 + 1] : 0;
  }
  return CKV_OK;
}

ckv_status ckv_reset_stats(ckv_ctx* ctx) {
  if (!ctx) return CKV_EINVAL;
  CK(cudaSetDevice(ctx->cfg.device));
  CK(cudaDeviceSynchronize());
  CK(cudaMemset(ctx->stats, 0, sizeof(int64_t) * 16));
  return CKV_OK;
}

ckv_status ckv_profile(ckv_ctx* ctx, int32_t enable) {
  if (!ctx) return CKV_EINVAL;
  ctx->prof_on = enable != 0;
  return CKV_OK;
}

ckv_status ckv_profile_read(ckv_ctx* ctx, double* ms, int64_t* count) {
  if (!ctx || !ms || !count) return CKV_EINVAL;
  ctx->err.clear();
  CK(cudaSetDevice(ctx->cfg.device));
  CK(cudaDeviceSynchronize());
  for (int i = 0; i < CKV_NUM_STAGES; ++i) {
    ms[i] = 0.0;
    count[i] = 0;
  }
  for (auto& mk : ctx->prof_marks) {
    float t = 0.f;
    CK(cudaEventElapsedTime(&t, mk.second.first, mk.second.second));
    ms[mk.first] += t;
    count[mk.first] += 1;
  }
  ctx->prof_marks.clear();
  ctx->prof_used = 0;
  return CKV_OK;
}

int64_t ckv_kernel_launches(const ckv_ctx* ctx) { return ctx ? ctx->launches : -1; }

int32_t ckv_num_chunks(const ckv_ctx* ctx) { return ctx ? ctx->m : -1; }
int32_t ckv_num_local_chunks(const ckv_ctx* ctx) { return ctx ? ctx->m_loc : -1; }
int32_t ckv_k(const ckv_ctx* ctx) { return ctx ? ctx->k : -1; }
int32_t ckv_score_kernel_kind(const ckv_ctx* ctx) { return ctx ? ctx->score_kind : -1; }
int32_t ckv_attn_kernel_kind(const ckv_ctx* ctx) { return ctx ? ctx->attn_kind : -1; }

ckv_status ckv_test_topk(ckv_ctx* ctx, const float* A, int32_t m, int32_t k, int32_t* ids, void* stream) {
  if (!ctx) return CKV_EINVAL;
  ctx->err.clear();
  if (!A || !ids || m < 1 || k < 1 || k > m) return fail(ctx, CKV_EINVAL, "bad argument");
  LK(launch_topk_scores(const_cast<float*>(A), nullptr, 0, m, k, 0, 1, ids, nullptr, 0, nullptr,
                        static_cast<cudaStream_t>(stream)));
  return CKV_OK;
}

ckv_status ckv_test_cache_step(ckv_ctx* ctx, int32_t layer, const int32_t* ids, int32_t k, int32_t prefetch,
                               const float* A, int32_t* loads, int32_t* victims, int32_t* counts, void* stream) {
  if (!ctx) return CKV_EINVAL;
  ctx->err.clear();
  if (layer < 0 || layer >= ctx->L || !ids || !loads || !counts || k < 1 || k > ctx->k)
    return fail(ctx, CKV_EINVAL, "bad argument");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  ++ctx->epoch;
  PlanOut po{loads, ctx->nload_main, prefetch ? nullptr : ctx->kept_slots, victims, counts, nullptr, nullptr, nullptr};
  LK(launch_cache_plan(cache_layer(ctx, layer), ids, nullptr, k, prefetch ? 1 : 0, ctx->quota, ctx->epoch,
                       ctx->rec_bytes, nullptr, ctx->scratch_main, po, st));
  if (A && !prefetch) {
    CK(cudaMemcpyAsync(ctx->n_ids_buf[0], &k, sizeof(int32_t), cudaMemcpyHostToDevice, st));
    CK(cudaStreamSynchronize(st));
    LK(launch_cache_update(cache_layer(ctx, layer), ids, ctx->n_ids_buf[0], A, ctx->epoch, st));
  }
  return CKV_OK;
}

ckv_status ckv_block_cover(ckv_ctx* ctx, const int32_t* ids, int32_t n_ids, int32_t block_tokens, int32_t* blocks,
                           int32_t* n_blocks, void* stream) {
  if (!ctx) return CKV_EINVAL;
  ctx->err.clear();
  if ((!ids && n_ids > 0) || !blocks || !n_blocks || n_ids < 0 || block_tokens < 1)
    return fail(ctx, CKV_EINVAL, "bad argument");
  CK(cudaSetDevice(ctx->cfg.device));
  LK(launch_block_cover(ids, n_ids, ctx->c, block_tokens, ctx->n, blocks, n_blocks,
                        static_cast<cudaStream_t>(stream)));
  return CKV_OK;
}

ckv_status ckv_load_chunks(ckv_ctx* ctx, int32_t layer, const int32_t* ids, int32_t n_ids, void* stream) {
  if (!ctx) return CKV_EINVAL;
  ctx->err.clear();
  if (layer < 0 || layer >= ctx->L || !ids || n_ids < 1 || n_ids > ctx->k) return fail(ctx, CKV_EINVAL, "bad argument");
  if (!ctx->stored[layer]) return fail(ctx, CKV_ESTATE, "layer %d prefix not stored", layer);
  CK(cudaSetDevice(ctx->cfg.device));
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  PlanOut po{ctx->gl_main, ctx->nload_main, nullptr, nullptr, ctx->counts + (size_t)(layer * 2) * 4, ctx->stats,
             nullptr, nullptr};
  LK(launch_cache_plan(cache_layer(ctx, layer), ids, nullptr, n_ids, 0, 0, ctx->epoch, ctx->rec_bytes, nullptr,
                       ctx->scratch_main, po, st));
  LK(launch_gather(ctx->gl_main, ctx->nload_main, host_layer_dev(ctx, layer), pool_layer(ctx, layer), ctx->rec_bytes,
                   st));
  return CKV_OK;
}

const char* ckv_last_error(const ckv_ctx* ctx) { return ctx ? ctx->err.c_str() : "null context"; }

void ckv_destroy(ckv_ctx* ctx) {
  ckv::timeline_dump();
  ckv::dtl_dump();
  if (!ctx) return;
  free_all(ctx);
  delete ctx;
}

}  // extern "C"

namespace ckv {
static std::vector<const void*>& kernel_registry() {
  static std::vector<const void*> r;
  return r;
}
int register_kernels(std::initializer_list<const void*> ks) {
  for (const void* k : ks) kernel_registry().push_back(k);
  return (int)kernel_registry().size();
}
cudaError_t preload_kernels() {  // on the current device
  for (const void* k : kernel_registry()) {
    cudaFuncAttributes a;
    if (cudaError_t e = cudaFuncGetAttributes(&a, k)) return e;
  }
  return cudaSuccess;
}
static cudaStream_t g_pdl_marked[8];
static int g_pdl_n_marked = 0;
void pdl_mark_event_wait(cudaStream_t st) {
  for (int i = 0; i < g_pdl_n_marked; ++i)
    if (g_pdl_marked[i] == st) return;
  if (g_pdl_n_marked < 8) g_pdl_marked[g_pdl_n_marked++] = st;
}
bool pdl_take_event_wait(cudaStream_t st) {
  for (int i = 0; i < g_pdl_n_marked; ++i)
    if (g_pdl_marked[i] == st) {
      g_pdl_marked[i] = g_pdl_marked[--g_pdl_n_marked];
      return true;
    }
  return false;
}
// Debug timeline (CKV_TIMELINE=1): an event after every kernel launch (also inside graph capture,
// as event-record nodes -- they break the programmatic edges, so this measures a PDL-free
// schedule); ckv_destroy prints the last 400 entries (end time of each kernel, us, relative).
struct TlEntry {
  const void* kern;
  cudaStream_t st;
  cudaEvent_t ev;
};
static std::vector<TlEntry> g_tl;
static size_t g_tl_pos = 0;
void timeline_mark(const void* kern, cudaStream_t st) {
  static const bool on = tuning_env("CKV_TIMELINE") && tuning_env("CKV_TIMELINE")[0] == '1';
  if (!on) return;
  if (g_tl.empty()) {
    g_tl.resize(400);
    for (auto& t : g_tl) cudaEventCreate(&t.ev);
  }
  TlEntry& t = g_tl[g_tl_pos++ % g_tl.size()];
  t.kern = kern;
  t.st = st;
  cudaEventRecord(t.ev, st);
}
void timeline_dump() {
  if (g_tl.empty() || g_tl_pos < g_tl.size()) return;
  cudaDeviceSynchronize();
  const size_t n = g_tl.size(), first = g_tl_pos % n;
  float prev = 0.f;
  for (size_t i = 0; i < n; ++i) {
    const TlEntry& t = g_tl[(first + i) % n];
    float ms = 0.f;
    cudaEventElapsedTime(&ms, g_tl[first].ev, t.ev);
    const char* name = nullptr;
    cudaFuncGetName(&name, t.kern);
    std::string nm = name ? name : "?";
    const size_t k = nm.find("kernel");
    if (k != std::string::npos) nm = nm.substr(0, k + 6);
    const size_t b = nm.rfind("_N_");
    if (b != std::string::npos) nm = nm.substr(b);
    fprintf(stderr, "[tl] %8.2f us  +%7.2f  %s %s\n", ms * 1e3, (ms - prev) * 1e3, nm.c_str(),
            t.st == nullptr ? "" : "");
    fprintf(stderr, "[tl-stream] %p\n", (void*)t.st);
    prev = ms;
  }
}
#ifdef CKV_TUNING
static std::vector<DtlSetter>& dtl_setters() {
  static std::vector<DtlSetter> v;
  return v;
}
int register_dtl(DtlSetter f) {
  dtl_setters().push_back(f);
  return 0;
}
static unsigned long long* g_dtl_buf = nullptr;
static unsigned int* g_dtl_cnt = nullptr;
static std::vector<std::pair<unsigned long long, std::string>> g_dtl_names;  // (grid | block << 32, kernel)
void dtl_init() {
  if (!(tuning_env("CKV_DTL") && tuning_env("CKV_DTL")[0] == '1') || g_dtl_buf) return;
  cudaMalloc(&g_dtl_buf, 8192 * 2 * sizeof(unsigned long long));
  cudaMalloc(&g_dtl_cnt, sizeof(unsigned int));
  cudaMemset(g_dtl_cnt, 0, sizeof(unsigned int));
  for (DtlSetter f : dtl_setters()) f(g_dtl_buf, g_dtl_cnt);
}
void dtl_name(const void* kern, dim3 grid, dim3 block) {
  if (!g_dtl_buf) return;
  const unsigned long long key = grid.x | ((unsigned long long)block.x << 32);
  for (auto& e : g_dtl_names)
    if (e.first == key) return;
  const char* name = nullptr;
  cudaFuncGetName(&name, kern);
  std::string nm = name ? name : "?";
  const size_t k = nm.find("kernel");
  if (k != std::string::npos) nm = nm.substr(0, k + 6);
  const size_t b = nm.rfind("_N_");
  if (b != std::string::npos) nm = nm.substr(b + 3);
  const size_t u = nm.find("_cu_");
  if (u != std::string::npos) nm = nm.substr(u + 4);
  g_dtl_names.push_back({key, nm});
}
void dtl_dump() {
  if (!g_dtl_buf) return;
  cudaDeviceSynchronize();
  unsigned int n = 0;
  cudaMemcpy(&n, g_dtl_cnt, sizeof n, cudaMemcpyDeviceToHost);
  if (n > 8192) n = 8192;
  std::vector<unsigned long long> h(2 * (size_t)n);
  cudaMemcpy(h.data(), g_dtl_buf, h.size() * sizeof(unsigned long long), cudaMemcpyDeviceToHost);
  std::vector<std::pair<unsigned long long, unsigned long long>> r;
  for (unsigned i = 0; i < n; ++i) r.push_back({h[2 * i], h[2 * i + 1]});
  std::sort(r.begin(), r.end());
  for (auto& e : r) {
    const char* nm = "?";
    for (auto& k : g_dtl_names)
      if (k.first == e.second) nm = k.second.c_str();
    fprintf(stderr, "[dtl] %llu %u %u %s\n", e.first, (unsigned)(e.second & 0xffffffffu), (unsigned)(e.second >> 32), nm);
  }
}
#else
void dtl_init() {}
void dtl_name(const void*, dim3, dim3) {}
void dtl_dump() {}
#endif
bool pdl_enabled() {
  static int v = -1;
  if (v < 0) {
    const char* e = tuning_env("CKV_PDL");
    v = (e && e[0] == '0') ? 0 : 1;
  }
  return v == 1;
}
}  // namespace ckv
