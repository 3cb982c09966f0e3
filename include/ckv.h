/*
 * ckv.h -- C-ABI of the B200-native ContiguousKV Re-Prefill hot path.
 *
 * Paper: "ContiguousKV: Accelerating LLM Prefill with Granularity-Aligned KV
 * Cache Management", arXiv 2601.13631.  Per layer the library runs
 * the data-parallel hot path of the Re-Prefill phase (Def. 1):
 *
 *   A1/A2  score every ContiguousChunk (Def. 2) by the
 *          attention mass the suffix queries put on it (Eq. 1);
 *   A3     select the top-k chunks under the token budget;
 *   A4/A5  look them up in the HBM chunk cache (attention-guided retention,
 *          PAPER.md:424-455, Eq. 2) and gather the misses as whole chunks from the
 *          pinned, chunk-contiguous host store;
 *   A6     speculatively prefetch the next layer's chunks from this layer's ids
 *          (inter-period prefetch at p = 1): planned with this
 *          layer's plan, copied by a warp of the next layer's score kernel (bf16,
 *          tcgen05 path) or on a side stream (periods, fp32 / SIMT path);
 *   A7/A8  exact softmax attention of the suffix queries over the kept chunks plus
 *          the causal suffix, split-K with an LSE combine;
 *   A9     cache-score update I_j += A_j, F_j += 1.
 *
 * Readings of the paper's silent points (normalisation domain, summation axis,
 * 1/sqrt(d), GQA aggregation, chunk range, k from a budget, ties) are
 * SURVEY.md §8(c) Q1-Q16, restated in DESIGN.md §2.
 *
 * Conventions (all entry points):
 *  - No C++ exception crosses this boundary.  Every call returns a ckv_status;
 *    arguments are validated before anything is enqueued; the message of the last
 *    failure is available from ckv_last_error(ctx) until the next call on ctx.
 *  - "device" pointers are CUDA device (or managed) pointers on cfg.device; "host"
 *    pointers are ordinary CPU pointers.  Tensors are dense, row-major, with the
 *    element type cfg.dtype (CKV_BF16: IEEE bfloat16 bit patterns; CKV_FP32: float).
 *  - Work is enqueued asynchronously on the caller's `stream` (cudaStream_t passed
 *    as void*; NULL = legacy default stream).  Input buffers must stay live and
 *    unmodified, and output buffers must not be read, until the stream reaches the
 *    point of the call.  The caller owns every pointer passed in; the library owns
 *    everything it allocates (host store, probe keys, slot pool, workspaces,
 *    side stream, events) and frees it in ckv_destroy.
 *  - A context is not re-entrant: one host thread and one caller stream per ctx.
 *  - CUDA failures map to CKV_ECUDA; asynchronous kernel faults surface on a later
 *    call (or the caller's stream synchronisation).
 */
#ifndef CKV_H_
#define CKV_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct ckv_ctx ckv_ctx; /* opaque, owned by the library */

typedef enum {
  CKV_OK = 0,
  CKV_EINVAL = 1,     /* invalid argument (shape, range, null pointer) */
  CKV_ENOMEM = 2,     /* host or device allocation failed */
  CKV_ECUDA = 3,      /* CUDA runtime / driver error */
  CKV_ESTATE = 5,     /* call not valid in the current state (e.g. prefix not stored) */
  CKV_EUNSUPPORTED = 7 /* shape outside what the compiled kernels support */
} ckv_status;

typedef enum { CKV_BF16 = 0, CKV_FP32 = 1 } ckv_dtype;

/* Softmax normalisation domain of the chunk scores. */
typedef enum { CKV_NORM_PREFIX = 0, CKV_NORM_FULLROW = 1 } ckv_norm;

/* cfg.flags */
#define CKV_FLAG_SIMT_SCORE 0x1u  /* force the SIMT (FFMA) scoring kernel in bf16 mode */
#define CKV_FLAG_SIMT_ATTN 0x2u   /* force the SIMT attention kernel in bf16 mode */
#define CKV_FLAG_CYCLIC_SHARDS 0x4u /* num_shards > 1: shard g owns chunks j with j mod W == g (balanced
                                       sharding) instead of a contiguous range */
#define CKV_FLAG_V_ONLY_STORE 0x10u /* bf16, d = 128, c % 8 == 0: host records and cache slots hold V only;
                                       the kept chunks' K is read from the HBM probe array (which holds every
                                       prefix key anyway), halving host-link bytes per miss (SURVEY §8(a) A5
                                       variant).  CKV_EUNSUPPORTED otherwise. */
#define CKV_FLAG_GLOBAL_HEAP 0x8u   /* one HBM chunk cache of L * cache_slots slots shared by every layer
                                       ("a single global GPU heap"): victims are the lowest
                                       (S, layer, chunk) residents of any layer; default: per-layer pools.
                                       The next layer's speculative plan then runs only after this layer's
                                       compaction; needs period 1 and one shard (CKV_EUNSUPPORTED otherwise) */

typedef struct {
  int32_t num_layers;      /* L >= 1 */
  int32_t num_q_heads;     /* Hq >= 1 */
  int32_t num_kv_heads;    /* Hkv >= 1, Hq % Hkv == 0 (GQA) */
  int32_t head_dim;        /* d: 64 or 128 (multiple of 16, <= 128 in SIMT mode) */
  int32_t dtype;           /* ckv_dtype */
  int32_t chunk_size;      /* c >= 1 (Def. 2) */
  int64_t prefix_len;      /* n >= 1, fixed per ctx; m = ceil(n / c) */
  int32_t max_suffix_len;  /* capacity for n_s */
  int32_t budget_chunks;   /* k >= 1; 0 => ckv_budget_chunks(n, c, budget_bp) */
  int32_t budget_bp;       /* budget ratio in basis points 1..10000 (used iff budget_chunks == 0) */
  int32_t score_norm;      /* ckv_norm */
  int32_t cache_slots;     /* HBM chunk-cache slots per layer (P); 0 => 2k + prefetch_chunks;
                              must be >= k + prefetch_chunks (global heap: the pool holds L * P) */
  int32_t prefetch_chunks; /* speculative next-layer prefetch quota per layer (chunks); 0 = off */
  int32_t device;          /* CUDA device ordinal */
  int32_t shard_index;     /* position shard owned by this ctx; 0 for one GPU */
  int32_t num_shards;      /* W >= 1; shard g owns chunks [g*ceil(m/W), min((g+1)*ceil(m/W), m)), or
                              j mod W == g with CKV_FLAG_CYCLIC_SHARDS */
  uint32_t flags;          /* CKV_FLAG_* */
  int32_t period;          /* p >= 1 (0 => 1): layers [P p, (P+1) p) reuse the chunk ids identified at
                              layer P p (Def. 3); the other layers skip A1-A3 and
                              their chunks are prefetched right after identification (intra-period
                              prefetch).  p > 1 needs num_shards == 1. */
  int32_t subperiod;       /* sp in [1, p] (0 => 1): the first layer of a period starts attention only
                              after the chunks of sp layers are loaded (subperiod_size) */
} ckv_config;

/* Counters of the last completed ckv_reprefill_layer / ckv_shard_attend call plus
 * running totals since ckv_create / ckv_reset_stats (host-readable; the call
 * synchronises the library's streams). */
typedef struct {
  int32_t last_hits, last_misses;      /* selected chunks found / not found in HBM at plan time */
  int32_t last_spec_loads;             /* chunks speculatively prefetched for this layer */
  int32_t last_spec_used;              /* of those, selected by this layer */
  int64_t total_hits, total_misses, total_spec_loads, total_spec_used;
  int64_t total_link_bytes_delta;      /* host->HBM bytes gathered on the critical path */
  int64_t total_link_bytes_spec;       /* host->HBM bytes gathered speculatively */
  int64_t total_layers;
} ckv_stats;

/* k = max(1, min(m, floor(budget_bp * n / (10000 * c)))), m = ceil(n / c)
 * ("top-k chunks under the token budget"; budget ratios PAPER.md:516).
 * Returns -1 on invalid arguments. */
int32_t ckv_budget_chunks(int64_t n, int32_t c, int32_t budget_bp);

/* Create a context on cfg->device: allocates the pinned, mapped, chunk-contiguous
 * host store (L * m_local records of 2*Hkv*c*d elements: [K|V][Hkv][c][d] per
 * chunk), the HBM probe-key array [L][Hkv][n_local][d], the HBM slot pool
 * [L][P] records, the cache tables and the workspaces.  *out receives the ctx.
 * Errors: CKV_EINVAL (bad config), CKV_ENOMEM, CKV_ECUDA, CKV_EUNSUPPORTED. */
ckv_status ckv_create(const ckv_config* cfg, ckv_ctx** out);

/* Store one layer's prefix K/V (the pre-computed prefix KV cache).
 * k, v: [n_tokens, Hkv, d] token-major, host or device memory (detected), cfg.dtype.
 * n_tokens must equal cfg.prefix_len; the ctx keeps only its shard's chunks.
 * Writes the probe keys into HBM, the chunk records into the host store, and
 * resets layer `layer`'s cache slots and (I, F) table.  Copies: the source may be
 * reused once `stream` passes this call.  Setup path (not part of the hot path).
 * Errors: CKV_EINVAL (layer out of range, n_tokens != prefix_len, null), CKV_ECUDA. */
ckv_status ckv_store_prefix(ckv_ctx* ctx, int32_t layer, const void* k, const void* v,
                            int64_t n_tokens, void* stream);

/* One layer of the Re-Prefill hot path, A1-A9: on one GPU (num_shards == 1), or on one rank of
 * a position-sharded group (num_shards > 1, after ckv_exchange_open / ckv_exchange_attach: the
 * exchanges of SURVEY §8(e) run inside the call over peer memory, see below; every rank
 * returns the identical global ids and the identical merged `out`).
 *  q      device [n_suffix, Hq, d]  suffix queries (post-RoPE), cfg.dtype
 *  k_suf  device [n_suffix, Hkv, d] suffix keys;  v_suf same shape: suffix values
 *  out    device [n_suffix, Hq, d]  attention output, cfg.dtype
 *  selected_ids  device int32 [k]   selected chunk ids, ascending (global ids)
 *  chunk_scores  device float [m] or NULL: A_j (Eq. 1) for parity/debug
 * Layer 0 starts a new request; layers must be called in order, and the calls of one request on
 * one stream (or stream-ordered by the caller: a call reads what the previous one enqueued,
 * e.g. the speculative copy list).  With period p = 1 every
 * layer runs A1-A9; if prefetch_chunks > 0 and layer + 1 < L the call also plans the
 * speculative prefetch of layer + 1 (this layer's ids); its copy runs inside the next call's
 * score kernel (tcgen05 path) or on the side stream.  With p > 1 only the
 * first layer of a period identifies chunks; it then enqueues the loads of the period's other
 * layers (exact ids) and the speculative load of the next period's first layer; the other
 * layers reuse the ids (selected_ids / chunk_scores report the period's).
 * Errors: CKV_EINVAL (null/range, 1 <= n_suffix <= max_suffix_len), CKV_ESTATE
 * (layer not stored, or num_shards > 1 without an attached exchange), CKV_ECUDA. */
ckv_status ckv_reprefill_layer(ckv_ctx* ctx, int32_t layer, const void* q, const void* k_suf,
                               const void* v_suf, int32_t n_suffix, void* out,
                               int32_t* selected_ids, float* chunk_scores, void* stream);

/* ---- position-sharded form; the caller runs the collectives ----
 * Per layer on every rank, with replicated q/k_suf/v_suf:
 *  1. ckv_shard_score       -> lam_local [Hq*n_s] float: base-2 log partition of
 *                              each suffix row over this shard's prefix keys
 *  2. caller: allgather lam_local over ranks (rank order) -> lam_all [W][Hq*n_s]
 *  3. ckv_shard_select      -> cand [k] uint64 (device): local top-min(k, m_g) candidates as
 *                              (float bits of A_j << 32) | (0xFFFFFFFF - global id),
 *                              padded with 0; chunk_scores (device float [m_g] or NULL)
 *                              receives this shard's A_j computed with the global normaliser
 *  4. caller: allgather cand -> cand_all [W*k]
 *  5. ckv_shard_attend      -> global selected ids (identical on all ranks), and this
 *                              shard's normalised partial output o_part [n_s,Hq,d]
 *                              float and lse_part [n_s*Hq] float (natural log,
 *                              -inf where the shard has no key for the row)
 *  6. caller: allreduce(MAX) of lse_part -> lse_max; ckv_lse_merge_prepare packs
 *     merge_buf [n_s*Hq*(d+1)] float = [o*e^(lse-M) | e^(lse-M)];
 *     caller: allreduce(SUM) of merge_buf; ckv_lse_merge_finish writes out.
 * The causal suffix keys are attended by the last shard only. */
ckv_status ckv_shard_score(ckv_ctx* ctx, int32_t layer, const void* q, const void* k_suf,
                           int32_t n_suffix, float* lam_local, void* stream);
ckv_status ckv_shard_select(ckv_ctx* ctx, int32_t layer, const void* q, const void* k_suf,
                            int32_t n_suffix, const float* lam_all, uint64_t* cand,
                            float* chunk_scores, void* stream);
ckv_status ckv_shard_attend(ckv_ctx* ctx, int32_t layer, const uint64_t* cand_all,
                            const void* q, const void* k_suf, const void* v_suf,
                            int32_t n_suffix, float* o_part, float* lse_part,
                            int32_t* selected_ids, void* stream);
ckv_status ckv_lse_merge_prepare(ckv_ctx* ctx, const float* o_part, const float* lse_part,
                                 const float* lse_max, int32_t n_suffix, float* merge_buf,
                                 void* stream);
ckv_status ckv_lse_merge_finish(ckv_ctx* ctx, const float* merge_buf, int32_t n_suffix,
                                void* out, void* stream);

/* ---- fused device-side exchange (SURVEY §8(e) + §8(f) NEXT-3) ----
 * The same position-sharded algorithm as the split-phase calls above, but the exchanges run
 * inside the library over peer memory (NVLink on a multi-GPU node), so a sharded layer is one
 * ckv_reprefill_layer call per rank, capturable in one CUDA graph per rank:
 * every ctx with num_shards = W > 1 owns an exchange WINDOW (device memory, identical layout on
 * every rank).  Per layer, after each producing kernel the library broadcasts (or, for the
 * partial outputs, scatters by row slice) its result straight into the peers' windows and
 * increments a per-exchange counter in every peer's window (release at system scope); the
 * consuming stream waits for the counter to reach W with a stream memory operation (no SM is
 * held while waiting) and re-arms it.  Four exchanges per layer:
 *   1. row normalisers  lam_g [Hq*n_s] float  -> all ranks     (global Lambda, rank order)
 *   2. candidates       cand_g [k] uint64     -> all ranks     (identical merged top-k)
 *   3. partial outputs  (O_g, lse_g) rows of slice s -> rank s (reduce-scatter over rows:
 *                       rank s merges rows [s*ceil(n_s*Hq/W), ...) of every rank's partial)
 *   4. merged rows      out slice s (cfg.dtype) -> all ranks   (all-gather), copied into `out`
 * Bytes over the peer links per rank and layer (W ranks, n_s*Hq = N rows):
 *   4*N*(W-1) + 8*k*(W-1) + (W-1)/W * N*(4d + 4) + (W-1)/W * N*d*e.
 * Setup, once per ctx, after every rank's ckv_create:
 *   multi-process (one process per GPU): ckv_exchange_handle on every rank -> all-gather the
 *     64-byte handles in rank order (e.g. torch.distributed) -> ckv_exchange_open(handles);
 *   one process driving several ranks (tests; several GPUs or logical ranks on one GPU):
 *     ckv_exchange_attach(ctxs) with the W contexts in rank order.
 * The peers must call ckv_reprefill_layer for the same layers in the same order with the
 * same n_suffix (it is collective); each rank's stream blocks until its peers contribute.
 * Errors: CKV_EINVAL (null, wrong count, num_shards == 1), CKV_ESTATE (already attached),
 * CKV_ECUDA (IPC / peer-access failure), CKV_EUNSUPPORTED (W > 8). */
#define CKV_EXCHANGE_HANDLE_BYTES 64
ckv_status ckv_exchange_handle(ckv_ctx* ctx, void* handle_out /* host, 64 bytes */);
ckv_status ckv_exchange_open(ckv_ctx* ctx, const void* handles /* host, W * 64 bytes, rank order */);
ckv_status ckv_exchange_attach(ckv_ctx* ctx, ckv_ctx* const* ctxs /* host, W contexts, rank order */,
                               int32_t num_ctxs);

/* Change the Period p and subperiod sp (same meaning and limits as ckv_config.period /
 * .subperiod) between requests (before the next layer-0 call).  CKV_EINVAL / CKV_EUNSUPPORTED
 * as in ckv_create. */
ckv_status ckv_set_period(ckv_ctx* ctx, int32_t period, int32_t subperiod);

/* Eviction score of the HBM chunk cache (A4).  CKV_CACHE_ATTN is the paper's
 * attention-guided policy S_j = I_j * F_j (Eq. 2); CKV_CACHE_LFU
 * (S_j = F_j) and CKV_CACHE_LRU (S_j = request index of the last selection) are the
 * ablation baselines of PAPER.md:610-613 ("w/o AC": "LFU as the cache policy").
 * Victims are always the lowest (S, j) residents that are not requested and not pinned. */
typedef enum { CKV_CACHE_ATTN = 0, CKV_CACHE_LFU = 1, CKV_CACHE_LRU = 2 } ckv_cache_policy;

/* Select the eviction policy.  Synchronises the device, empties every slot and zeroes
 * the (I, F, last-use) tables of every layer, so each policy starts from the same cold
 * state (performance only: results never depend on the cache).  Call between requests.
 * Errors: CKV_EINVAL (unknown policy), CKV_ECUDA. */
ckv_status ckv_set_cache_policy(ckv_ctx* ctx, int32_t policy, void* stream);

/* Cache control / introspection. */
ckv_status ckv_reset_cache(ckv_ctx* ctx, void* stream); /* empty every slot; keep (I, F) */
ckv_status ckv_get_stats(ckv_ctx* ctx, ckv_stats* out);  /* synchronises the library's streams */
ckv_status ckv_reset_stats(ckv_ctx* ctx);
int32_t ckv_num_chunks(const ckv_ctx* ctx);        /* m (global) */
int32_t ckv_num_local_chunks(const ckv_ctx* ctx);  /* m_g of this shard */
int32_t ckv_k(const ckv_ctx* ctx);                 /* k */
int32_t ckv_score_kernel_kind(const ckv_ctx* ctx); /* A1 kernel: 0 = SIMT, 1 = tcgen05 */
int32_t ckv_attn_kernel_kind(const ckv_ctx* ctx);  /* A7 kernel: 0 = SIMT, 1 = tcgen05 */

/* Stage profiling: when enabled, CUDA events are recorded on the caller's stream
 * around each stage of every hot-path call.  ckv_profile_read synchronises, returns
 * the summed device time (ms) and the number of timed launches per stage, and
 * clears the record.  Stages: 0 A1 score, 1 A2 row normaliser, 2 A2 chunk sum,
 * 3 A4 plan, 4 A5 delta gather, 5 A7+A8 attention + combine, 6 A3 top-k,
 * 7 A9 update.  ms and count: host arrays of CKV_NUM_STAGES. */
#define CKV_NUM_STAGES 8
ckv_status ckv_profile(ckv_ctx* ctx, int32_t enable);
ckv_status ckv_profile_read(ckv_ctx* ctx, double* ms, int64_t* count);
/* Number of CUDA kernels this ctx has launched since creation (all streams). */
int64_t ckv_kernel_launches(const ckv_ctx* ctx);

/* ---- granularity accounting ----
 * ckv_block_cover: the blocks of a coarse store of block_tokens-token blocks (e.g. the 64-token
 *   chunks of IMPRESS / AttentionStore) that hold at least one token of the
 *   selected chunks of this ctx (chunk j = tokens [j*c, min((j+1)*c, n)), Eq. 1 range):
 *   read amplification RA = tokens of those blocks / tokens of the chunks (PAPER.md:209-221,
 *   325-327; RA = 1 when block_tokens == c).
 *   ids     device int32 [n_ids], ascending global chunk ids (n_ids may be 0; ids may then be NULL)
 *   blocks  device int32, capacity ceil(n / block_tokens): ascending block ids (written)
 *   n_blocks device int32 [1]: number of blocks (written)
 * ckv_load_chunks: plan (A4) and gather (A5) an explicit ascending list of local chunk ids of
 *   `layer` into the HBM cache (demand load, no (I, F) update); the link bytes and
 *   hits/misses accumulate into ckv_get_stats.  1 <= n_ids <= k.  Used to time whole-block
 *   loads from a coarse store (a ctx with chunk_size = block size) on the same gather engine.
 * Errors: CKV_EINVAL (null / range), CKV_ESTATE (layer not stored), CKV_ECUDA. */
ckv_status ckv_block_cover(ckv_ctx* ctx, const int32_t* ids, int32_t n_ids, int32_t block_tokens,
                           int32_t* blocks, int32_t* n_blocks, void* stream);
ckv_status ckv_load_chunks(ckv_ctx* ctx, int32_t layer, const int32_t* ids, int32_t n_ids, void* stream);

/* ---- test entry points (parity of integer work, no allocation) ----
 * ckv_test_topk: ids[k] (device int32, ascending) = top-k of A[m] (device float, A >= 0)
 *   with lower-index tie-break, by the same radix-select kernel the hot path uses.
 * ckv_test_cache_step: run the cache planner (A4) on layer `layer` for the given
 *   ascending ids[k] (device int32); prefetch != 0 plans a speculative load (quota
 *   cfg.prefetch_chunks) instead of a demand load; when A (device float [m_local])
 *   is non-NULL the A9 update I += A, F += 1 follows.  loads (device int32
 *   [2*k]: chunk, slot pairs in ascending chunk order), victims (device int32 [k]: evicted
 *   entries as table indices layer * m_local + chunk) and counts (device int32 [4]:
 *   hits, loads, victims, 0) are written; no data is copied. */
ckv_status ckv_test_topk(ckv_ctx* ctx, const float* A, int32_t m, int32_t k, int32_t* ids,
                         void* stream);
/* ckv_test_exchange_flags: the XF_COUNT (4) exchange counters of this rank's window (host
 *   uint32 [4]: row normalisers, candidates, partial outputs, merged rows), read on a private
 *   non-blocking stream (does not wait for the caller's stream).  num_shards > 1 only. */
ckv_status ckv_test_exchange_flags(ckv_ctx* ctx, uint32_t* flags_out);
ckv_status ckv_test_cache_step(ckv_ctx* ctx, int32_t layer, const int32_t* ids, int32_t k,
                               int32_t prefetch, const float* A, int32_t* loads,
                               int32_t* victims, int32_t* counts, void* stream);

const char* ckv_last_error(const ckv_ctx* ctx); /* never NULL; "" if no error */
void ckv_destroy(ckv_ctx* ctx);                 /* NULL is a no-op; synchronises first */

#ifdef __cplusplus
}
#endif
#endif /* CKV_H_ */
