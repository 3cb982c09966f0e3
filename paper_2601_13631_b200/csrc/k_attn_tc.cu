// A7 split-K exact attention on tcgen05 (bf16, d = 128), flash-attention style, in two kernels.
//
// Same contract as attn_simt_kernel (k_attn.cu): for every GQA-packed suffix row and every
// key split, a normalised partial O and its base-2 LSE over the kept prefix chunks (all
// visible, partial-chunk padding masked) and the causal suffix keys t <= r
// (Q6, Q9).  A8 (attn_combine) merges the splits.
//
// 1. compact_kv_kernel: the kept chunks' K / V (from their HBM cache slots, records stored
//    pre-swizzled, rec_elem) and the suffix K / V are copied into a dense per-layer tile image
//    dense[kvh][tile][K|V][half][128 keys][64] (128-byte swizzle), one warp per 2 KB piece.
//    Measured on B200: the per-copy issue cost of the bulk-copy engine (~55 ns per copy) made
//    gathering 2 KB pieces inside the attention kernel (32 copies per tile, for each of the
//    7 row tiles that reuse a tile) the attention's bound; tensor-core MMAs cost >= ~60 cycles
//    each whatever N, so per-chunk N = c MMAs are no way around it.
// 2. attn_tc_kernel: per work item (kv head, 128-row tile, key split), 1 CTA per SM, 576 threads.
//    TMEM: S0 [0,128) S1 [128,256) (P(j) is written over S(j) as bf16 pairs), O [256,384),
//    Q [384,448).
//   warp 0      producer: one 64 KB bulk copy per key tile from the dense image, 3 stages.
//   warp 1      TMEM alloc + MMA issue: S = Q K^T (M 128, N 128, K 128) with Q (A) from TMEM,
//               then O += P V with P (A) from TMEM and V (B) MN-major from smem, software-
//               pipelined one tile behind S.  tcgen05 MMAs execute in issue order, so S(j+2)
//               (same TMEM buffer) follows PV(j).
//   warps 2..17 softmax: one row per thread, four warps per TMEM lane quadrant (32 key
//               columns and 32 O columns each); P = 2^(s - m) as bf16 into TMEM (each warp writes
//               its 16 P columns over the first half of its own 32 S columns, so no warp waits
//               for another before overwriting S).  The reference m of a row is its prefix LSE
//               Lambda2 from A2 when the layer was scored (lam_ref): every prefix logit is <= it
//               (an LSE bounds the max), so prefix tiles need no row max, no cross-warp exchange
//               and no rescale; the suffix tile (or a layer without lam_ref) computes the row max
//               through shared memory with a lazy O rescale (only when the running max grows by
//               > 8 in log2 units).  They also load each item's Q rows from q into TMEM.
#include <algorithm>
#include <cstdio>
#include <cstdlib>

#include "common.cuh"
#include "tc_ptx.cuh"

namespace ckv {
namespace {

constexpr int BM = 128, BN = 128, D = 128;
constexpr int kSoftWarps = 16;
constexpr int NWQ = kSoftWarps / 4;  // softmax warps per TMEM lane quadrant
constexpr int CPW = BN / NWQ;        // key / O columns per softmax warp
constexpr int kThreads = 64 + 32 * kSoftWarps;
constexpr int kStages = 3;
constexpr uint32_t kKVBytes = 2 * BN * D * 2;   // K + V of a 128-key tile = 64 KB
constexpr uint32_t kPartBytes = kKVBytes / 4;   // one (K|V, half) block: 128 rows x 128 B
constexpr size_t kSmem = kStages * kKVBytes + 1024 /*align*/ + 256 /*barriers*/;
constexpr uint32_t kOBlockBytes = BM * 32 * 4;  // O staging: [128 rows][32 floats], 128-byte swizzle
constexpr float kRescaleThresh = 8.f;  // log2 units
constexpr uint32_t kColO = 256, kColQ = 384;

struct AttnParams {
  LayerGeom g;
  const __nv_bfloat16* q;  // [ns][Hq][128]
  const int32_t* kept_ids;
  const int32_t* n_kept_dev;
  int include_suffix;
  int nsplit;
  int MT;
  int NTp_cap, NTs, T_cap;
  const char* dense;  // [Hkv][T_cap][64 KB]
  int n_items;
  float scale;
  float* o_part;
  float* lse_part;
  const float* lam_ref;  // Lambda2 [Hkv][R] of this layer (log2 units, >= every prefix logit) or null
  unsigned long long* trace;  // debug: %globaltimer events of CTA 0 (CKV_ATTN_TRACE=1), else null
};

// debug timeline: event e (0 start, 1 q_full seen by MMA, 2 kv_full seen by MMA, 3 s_full seen by
// softmax, 4 p_full arrived, 5 o_full seen by softmax, 6 epilogue stored), occurrence i
__device__ __forceinline__ void trace_ev(const AttnParams& p, int e, int i) {
  if (p.trace && blockIdx.x == 0 && i < 32) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    p.trace[e * 32 + i] = t;
  }
}

struct Tiles {
  int t0, t1;  // [t0, t1) in the tile index space of the item's KV head
  int NTp;     // prefix tiles actually present
};

__device__ __forceinline__ Tiles item_tiles(const AttnParams& p, int sp, int n_kept) {
  Tiles t;
  t.t0 = (int)((int64_t)sp * p.T_cap / p.nsplit);
  t.t1 = (int)((int64_t)(sp + 1) * p.T_cap / p.nsplit);
  t.NTp = (n_kept * p.g.c + BN - 1) / BN;
  return t;
}
// skip prefix tiles past the kept chunks; suffix tiles live at [NTp_cap, NTp_cap + NTs)
__device__ __forceinline__ bool tile_present(const AttnParams& p, const Tiles& tl, int t) {
  return (t < p.NTp_cap) ? (t < tl.NTp) : (p.include_suffix != 0);
}

// Dense tile image of the kept chunks and the suffix (see the file comment).  Warp items:
// prefix (kvh, kept chunk i, part = K h0 | K h1 | V h0 | V h1): c rows of 128 B copied as is
// (record rows are swizzled by (row & 7) and c % 8 == 0, so they land swizzled);
// suffix (kvh, key t, K|V): one 256 B row of k_suf / v_suf, 16-byte units swizzled on the way.
// A kept chunk the planner marked as a miss (slot encoded as -(s + 2)) is read from the mapped
// host store instead (A5 fused: whole records) and also written to its cache
// slot s, so the layer has no separate gather launch on its critical path.
// V-only store (rec_swz 2): the K pieces come from the HBM probe array ([Hkv][n_pad][128], rows of
// the chunk's local tokens), swizzled on the way; the records (slots, host) hold V alone.
__global__ void __launch_bounds__(256, 3) compact_kv_kernel(LayerGeom g, char* __restrict__ pool,
                                                         const char* __restrict__ host_layer,
                                                         const __nv_bfloat16* __restrict__ probe,
                                                         const int32_t* __restrict__ kept_ids,
                                                         int64_t rec_bytes, const int32_t* __restrict__ kept_slots,
                                                         const int32_t* __restrict__ n_kept_dev, int k_cap,
                                                         const __nv_bfloat16* __restrict__ k_suf,
                                                         const __nv_bfloat16* __restrict__ v_suf, int include_suffix,
                                                         int NTp_cap, int T_cap, char* __restrict__ dense) {
  pdl_wait();
  pdl_trigger();
  const int n_kept = *n_kept_dev;
  const int lane = threadIdx.x & 31;
  const int64_t nwarps = (int64_t)gridDim.x * (blockDim.x >> 5);
  const int64_t n_pre = (int64_t)g.Hkv * k_cap * 4;
  const int64_t n_suf = include_suffix ? (int64_t)g.Hkv * g.ns * 2 : 0;
  const uint32_t piece = (uint32_t)g.c * 128u;  // bytes of one (K|V, half) block of a chunk
  for (int64_t w = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; w < n_pre + n_suf; w += nwarps) {
    if (w < n_pre) {
      const int part = (int)(w & 3);
      const int64_t ci = w >> 2;
      const int kvh = (int)(ci / k_cap), i = (int)(ci % k_cap);
      if (i >= n_kept) continue;
      const int slot = kept_slots[i];
      if (slot == -1) continue;  // not loaded (planner capacity failure, reported in the stats)
      const int key = i * g.c;
      uint4* dst = reinterpret_cast<uint4*>(dense + ((int64_t)kvh * T_cap + key / BN) * kKVBytes +
                                            part * kPartBytes + (key % BN) * 128);
      if (g.rec_swz == 2 && part < 2) {  // K half `part` of the chunk's rows, from the probe array
        const uint4* src = reinterpret_cast<const uint4*>(probe + ((int64_t)kvh * g.n_pad + (int64_t)kept_ids[i] * g.c) * 128);
        const int nu = g.c * 8;  // 16-byte units: c rows x 8
        for (int u0 = 0; u0 < nu; u0 += 32 * 4) {
          uint4 v[4];
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const int idx = u0 + lane + 32 * q;  // row idx / 8, unit idx % 8 of this half
            if (idx < nu) v[q] = __ldg(src + (idx >> 3) * 16 + part * 8 + (idx & 7));
          }
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const int idx = u0 + lane + 32 * q;
            if (idx < nu) dst[(idx >> 3) * 8 + ((idx & 7) ^ ((idx >> 3) & 7))] = v[q];
          }
        }
        continue;
      }
      // record offset of this piece: swizzled [Hkv][K|V][half] pieces, or V-only [Hkv][half]
      const int64_t off = g.rec_swz == 2 ? ((int64_t)kvh * 2 + (part - 2)) * piece : (int64_t)kvh * 4 * piece + part * piece;
      // record rows are swizzled by (row in chunk) & 7; in the tile a row sits at key + p, so for
      // c % 8 != 0 (chunk sizes 1, 2, 4) each 16-byte unit is re-swizzled on the way
      const int rs = key & 7;  // 0 whenever c % 8 == 0: units copy as they are
      auto dunit = [&](int idx) {  // destination unit of source unit idx (row idx / 8, unit idx % 8)
        const int p8 = idx >> 3, us = idx & 7;
        return rs == 0 ? idx : p8 * 8 + ((us ^ (p8 & 7)) ^ ((rs + p8) & 7));
      };
      if (slot >= 0) {
        const uint4* src = reinterpret_cast<const uint4*>(pool + (int64_t)slot * rec_bytes + off);
        const int nu = (int)(piece / 16);
        for (int u0 = 0; u0 < nu; u0 += 32 * 4) {  // 4 independent 16-byte loads in flight per lane
          uint4 v[4];
#pragma unroll
          for (int q = 0; q < 4; ++q)
            if (u0 + lane + 32 * q < nu) v[q] = __ldcg(src + u0 + lane + 32 * q);
#pragma unroll
          for (int q = 0; q < 4; ++q)
            if (u0 + lane + 32 * q < nu) dst[dunit(u0 + lane + 32 * q)] = v[q];
        }
      } else {
        const uint4* src = reinterpret_cast<const uint4*>(host_layer + (int64_t)kept_ids[i] * rec_bytes + off);
        uint4* cdst = reinterpret_cast<uint4*>(pool + (int64_t)(-slot - 2) * rec_bytes + off);
        const int nu = (int)(piece / 16);
        for (int u0 = 0; u0 < nu; u0 += 32 * 4) {  // 4 host loads in flight per lane (whole 2 KB piece)
          uint4 v[4];
#pragma unroll
          for (int q = 0; q < 4; ++q)
            if (u0 + lane + 32 * q < nu) v[q] = __ldg(src + u0 + lane + 32 * q);
#pragma unroll
          for (int q = 0; q < 4; ++q)
            if (u0 + lane + 32 * q < nu) {
              dst[dunit(u0 + lane + 32 * q)] = v[q];
              cdst[u0 + lane + 32 * q] = v[q];
            }
        }
      }
    } else {
      const int64_t si = w - n_pre;
      const int kv = (int)(si & 1);
      const int64_t rt = si >> 1;
      const int kvh = (int)(rt / g.ns), t = (int)(rt % g.ns);
      if (lane >= 16) continue;
      const __nv_bfloat16* row = (kv ? v_suf : k_suf) + ((int64_t)t * g.Hkv + kvh) * D;
      const uint4 val = reinterpret_cast<const uint4*>(row)[lane];
      const int tile = NTp_cap + t / BN, r = t % BN, half = lane >> 3, u = (lane & 7) ^ (r & 7);
      uint4* dst = reinterpret_cast<uint4*>(dense + ((int64_t)kvh * T_cap + tile) * kKVBytes +
                                            (kv * 2 + half) * kPartBytes + r * 128 + u * 16);
      *dst = val;
    }
  }
}

// O += P V for the tile that was scored one step earlier (MMA thread): P (A) from the tile's
// S buffer in TMEM, V (B) the MN-major [half][128 keys][64] block of the stage.
__device__ __forceinline__ void issue_pv(uint32_t tmem, uint8_t* kvbuf0, uint64_t* p_full, uint64_t* pv_done,
                                         uint64_t* o_empty, uint64_t* v_full, uint64_t* kv_empty, uint32_t idesc_o,
                                         int jj, int stage, int vphase, int sbuf, int nkeys, int icount, int& pcount) {
  ptx::mbar_wait(p_full, pcount & 1);
  if (jj == 0) ptx::mbar_wait(o_empty, (icount & 1) ^ 1);
  ptx::mbar_wait(&v_full[stage], vphase);
  ptx::tc_fence_after();
  const uint32_t va0 = ptx::smem_u32(kvbuf0 + stage * kKVBytes + 2 * kPartBytes);
  const int ksteps = (nkeys + 15) / 16;  // key steps past the tile's valid keys are skipped
  for (int k = 0; k < ksteps; ++k)
    // P of keys [16k, 16k + 16): written by softmax warp k / 2 at its S columns 32 (k / 2) + 8 (k % 2)
    ptx::mma_bf16_ts(tmem + kColO, tmem + sbuf * BN + (k >> 1) * 32 + (k & 1) * 8,
                     ptx::umma_desc_sw128_mn(va0 + k * 16 * 128, kPartBytes),
                     idesc_o, k > 0 || jj > 0 ? 1u : 0u);
  ptx::mma_commit(pv_done);
  ptx::mma_commit(&kv_empty[stage]);
  ++pcount;
}

__global__ void __launch_bounds__(kThreads, 1) attn_tc_kernel(const __grid_constant__ CUtensorMap tmO, AttnParams p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* kvbuf0 = smem;
  __shared__ float red_m[2][NWQ * 128];  // [tile parity][warp of a quadrant][128 rows]
  __shared__ float red_l[NWQ * 128];
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + kStages * kKVBytes);
  // K and V halves of a stage have their own barriers: K(t) is released as soon as S(t) is
  // computed, so the K of later tiles streams in while the softmax and PV of earlier tiles run
  uint64_t* k_full = bars + 0;              // [kStages]
  uint64_t* kv_empty = bars + kStages;      // [kStages] V half released (after PV)
  uint64_t* v_full = bars + 2 * kStages;    // [kStages]
  uint64_t* k_empty = bars + 3 * kStages;   // [kStages] K half released (after S)
  uint64_t* s_full = bars + 4 * kStages;    // [2]
  uint64_t* p_full = s_full + 2;
  uint64_t* pv_done = p_full + 1;
  uint64_t* o_full = pv_done + 1;
  uint64_t* o_empty = o_full + 1;
  uint64_t* q_full = o_empty + 1;
  uint64_t* epi_done = q_full + 1;  // the item's O staging (in stage 0) has been stored
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(epi_done + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) trace_ev(p, 0, 0);

  if (threadIdx.x == 0) {
    for (int i = 0; i < kStages; ++i) {
      ptx::mbar_init(&k_full[i], 1);
      ptx::mbar_init(&kv_empty[i], 1);
      ptx::mbar_init(&v_full[i], 1);
      ptx::mbar_init(&k_empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) ptx::mbar_init(&s_full[i], 1);
    ptx::mbar_init(p_full, kSoftWarps);
    ptx::mbar_init(pv_done, 1);
    ptx::mbar_init(o_full, 1);
    ptx::mbar_init(o_empty, kSoftWarps);
    ptx::mbar_init(q_full, kSoftWarps);
    ptx::mbar_init(epi_done, 1);
    ptx::fence_mbar_init();
  }
  if (warp == 1) ptx::tmem_alloc<512>(tmem_slot);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    // ------------------------------------------------------------ bulk-copy producer
    if (lane == 0) {
      pdl_wait();
      const int n_kept = *p.n_kept_dev;
      int kvcount = 0, icount = 0;
      for (int it = blockIdx.x; it < p.n_items; it += gridDim.x, ++icount) {
        const int sp = it % p.nsplit, kvh = it / (p.nsplit * p.MT);
        const Tiles tl = item_tiles(p, sp, n_kept);
        // stage 0 doubles as the previous item's O staging buffer
        if (icount > 0) ptx::mbar_wait(epi_done, (icount - 1) & 1);
        for (int t = tl.t0; t < tl.t1; ++t) {
          if (!tile_present(p, tl, t)) continue;
          const int st = kvcount % kStages;
          const uint32_t par = ((kvcount / kStages) & 1) ^ 1;
          const char* src = p.dense + ((int64_t)kvh * p.T_cap + t) * kKVBytes;
          ptx::mbar_wait(&k_empty[st], par);
          ptx::mbar_expect_tx(&k_full[st], kKVBytes / 2);
          ptx::bulk_g2s(kvbuf0 + st * kKVBytes, src, kKVBytes / 2, &k_full[st]);
          ptx::mbar_wait(&kv_empty[st], par);
          ptx::mbar_expect_tx(&v_full[st], kKVBytes / 2);
          ptx::bulk_g2s(kvbuf0 + st * kKVBytes + kKVBytes / 2, src + kKVBytes / 2, kKVBytes / 2, &v_full[st]);
          ++kvcount;
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer
    if (lane == 0) {
      pdl_wait();
      pdl_trigger();  // after this CTA's own dependency is resolved (see common.cuh)
      const int n_kept = *p.n_kept_dev;
      int n_valid_prefix = 0;  // keys of the kept prefix (the last kept chunk may be partial)
      if (n_kept > 0)
        n_valid_prefix = (n_kept - 1) * p.g.c + min(p.g.c, p.g.n_loc - p.kept_ids[n_kept - 1] * p.g.c);
      constexpr uint32_t idesc_s = ptx::idesc_bf16_f32(BM, BN, false);
      constexpr uint32_t idesc_o = ptx::idesc_bf16_f32(BM, D, true);
      int icount = 0, kvcount = 0, scount = 0, pcount = 0;
      for (int it = blockIdx.x; it < p.n_items; it += gridDim.x, ++icount) {
        const int sp = it % p.nsplit;
        const Tiles tl = item_tiles(p, sp, n_kept);
        ptx::mbar_wait(q_full, icount & 1);
        trace_ev(p, 1, icount);
        int j = 0, prev_stage = 0, prev_sb = 0, prev_keys = 0, prev_vph = 0;
        for (int t = tl.t0; t < tl.t1; ++t) {
          if (!tile_present(p, tl, t)) continue;
          const int st = kvcount % kStages;
          ptx::mbar_wait(&k_full[st], (kvcount / kStages) & 1);
          trace_ev(p, 2, kvcount);
          ptx::tc_fence_after();
          const int sb = scount & 1;
          const uint32_t ka = ptx::smem_u32(kvbuf0 + st * kKVBytes);
#pragma unroll
          for (int k = 0; k < D / 16; ++k)
            ptx::mma_bf16_ts(tmem + sb * BN, tmem + kColQ + k * 8,
                             ptx::umma_desc_sw128(ka + (k >> 2) * kPartBytes + (k & 3) * 32), idesc_s, k > 0 ? 1u : 0u);
          ptx::mma_commit(&s_full[sb]);
          ptx::mma_commit(&k_empty[st]);
          ++scount;
          if (j > 0)
            issue_pv(tmem, kvbuf0, p_full, pv_done, o_empty, v_full, kv_empty, idesc_o, j - 1, prev_stage, prev_vph,
                     prev_sb, prev_keys, icount, pcount);
          prev_vph = (kvcount / kStages) & 1;
          prev_stage = st;
          prev_sb = sb;
          prev_keys = (t < p.NTp_cap) ? min(BN, n_valid_prefix - t * BN) : min(BN, p.g.ns - (t - p.NTp_cap) * BN);
          ++kvcount;
          ++j;
        }
        if (j > 0)
          issue_pv(tmem, kvbuf0, p_full, pv_done, o_empty, v_full, kv_empty, idesc_o, j - 1, prev_stage, prev_vph,
                   prev_sb, prev_keys, icount, pcount);
        ptx::mma_commit(o_full);
      }
    }
  } else {
    // ------------------------------------------------------------ softmax / epilogue
    // kSoftWarps = 16: four warps per TMEM lane quadrant, each owning CPW = 32 key columns
    // of S (= 16 P columns), the same 32 columns of O and 32 elements (16 columns) of Q.
    const int e = warp - 2, quad = warp & 3, h = e >> 2;
    const int rit = quad * 32 + lane;  // row in tile
    const uint32_t lane_off = (uint32_t)(quad * 32) << 16;
    const uint32_t bar_id = 1 + quad;  // named barrier of the quadrant's NWQ warps
    int icount = 0, scount = 0, pcount = 0, nx = 0;  // nx: row-max exchanges (red_m parity)
    int n_kept = -1, n_valid_prefix = 0;
    const float sc = p.scale;
    for (int it = blockIdx.x; it < p.n_items; it += gridDim.x, ++icount) {
      const int sp = it % p.nsplit, mt = (it / p.nsplit) % p.MT, kvh = it / (p.nsplit * p.MT);
      const int rho = mt * BM + rit;
      const bool row_ok = rho < p.g.R;
      const int gq = rho / p.g.ns, r = rho - gq * p.g.ns;
      {  // Q rows of this item -> TMEM (the previous item's MMAs are all complete: o_full)
        uint32_t qv[16];
        if (row_ok) {
          const uint4* src = reinterpret_cast<const uint4*>(p.q + ((size_t)r * p.g.Hq + kvh * p.g.G + gq) * D + h * 32);
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            const uint4 u = src[i];
            qv[4 * i] = u.x;
            qv[4 * i + 1] = u.y;
            qv[4 * i + 2] = u.z;
            qv[4 * i + 3] = u.w;
          }
        } else {
#pragma unroll
          for (int i = 0; i < 16; ++i) qv[i] = 0u;
        }
        if (n_kept < 0) {  // first item: issued while the Q loads are in flight
          pdl_wait();
          n_kept = *p.n_kept_dev;
          if (n_kept > 0)
            n_valid_prefix = (n_kept - 1) * p.g.c + min(p.g.c, p.g.n_loc - p.kept_ids[n_kept - 1] * p.g.c);
        }
        ptx::tmem_st16_nowait(tmem + kColQ + h * 16 + lane_off, qv);
        ptx::tmem_wait_st();
        ptx::tc_fence_before();
        __syncwarp();
        if (lane == 0) ptx::mbar_arrive(q_full);
      }
      const Tiles tl = item_tiles(p, sp, n_kept);
      float m_ref = -INFINITY, l = 0.f;
      // prefix LSE as the reference (uniform over the quadrant's 4 warps: they share these rows)
      bool ref_ok = false;
      if (p.lam_ref) {
        const float lr = row_ok ? p.lam_ref[(size_t)kvh * p.g.R + rho] : 0.f;
        ref_ok = __all_sync(0xffffffffu, lr > -INFINITY && lr < INFINITY);
        if (ref_ok) m_ref = lr;
      }
      int j = 0;
      for (int t = tl.t0; t < tl.t1; ++t) {
        if (!tile_present(p, tl, t)) continue;
        const int sb = scount & 1;
        ptx::mbar_wait(&s_full[sb], (scount >> 1) & 1);
        if (warp == 2 && lane == 0) trace_ev(p, 3, scount);
        ptx::tc_fence_after();
        float x[CPW];
        ptx::tmem_ld32p(tmem + sb * BN + h * CPW + lane_off, x);
        ++scount;
        const bool pre = t < p.NTp_cap;
        const int b0 = (pre ? t * BN : (t - p.NTp_cap) * BN) + h * CPW;
        const int lim = pre ? n_valid_prefix : min(r + 1, p.g.ns);  // key valid iff index < lim
        if (b0 + CPW > lim) {
#pragma unroll
          for (int i = 0; i < CPW; ++i)
            if (b0 + i >= lim) x[i] = -INFINITY;
        }
        float f = 1.f;
        bool resc = false;
        if (!(ref_ok && pre)) {  // row max needed: suffix tile, or no prefix-LSE reference
          float mx[CPW / 2];
#pragma unroll
          for (int i = 0; i < CPW / 2; ++i) mx[i] = fmaxf(x[i], x[i + CPW / 2]);
#pragma unroll
          for (int n = CPW / 4; n >= 1; n >>= 1)
#pragma unroll
            for (int i = 0; i < n; ++i) mx[i] = fmaxf(mx[i], mx[i + n]);
          // red_m is double-buffered by tile parity: a warp can only overwrite a buffer two
          // exchanges later, after the next barrier, which every reader of these values has passed
          float* rm = red_m[nx & 1];
          ++nx;
          rm[h * 128 + rit] = mx[0];
          ptx::named_bar_sync(bar_id, 32 * NWQ);
          float tmax = rm[rit];
#pragma unroll
          for (int w = 1; w < NWQ; ++w) tmax = fmaxf(tmax, rm[w * 128 + rit]);
          tmax *= sc;
          const float m_new = fmaxf(m_ref, tmax);
          resc = (j > 0) && (m_ref != -INFINITY) && (m_new > m_ref + kRescaleThresh);
          f = resc ? fast_exp2(m_ref - m_new) : 1.f;
          if (j == 0 || m_ref == -INFINITY || resc) m_ref = m_new;
        }
        const float msub = (m_ref == -INFINITY) ? 0.f : m_ref;
        float ls[4] = {0.f, 0.f, 0.f, 0.f};
        uint32_t pk[CPW / 2];
#pragma unroll
        for (int i = 0; i < CPW / 2; ++i) {
          // 1 pair in 8 on the FMA pipe (polynomial exp2), the rest on MUFU
          const float a0 = fmaf(x[2 * i], sc, -msub), a1 = fmaf(x[2 * i + 1], sc, -msub);
          const float p0 = (i & 7) == 0 ? exp2_poly(a0) : fast_exp2(a0);
          const float p1 = (i & 7) == 0 ? exp2_poly(a1) : fast_exp2(a1);
          ls[i & 3] += p0 + p1;
          __nv_bfloat162 b2 = __floats2bfloat162_rn(p0, p1);
          pk[i] = *reinterpret_cast<uint32_t*>(&b2);
        }
        const float lsum = (ls[0] + ls[1]) + (ls[2] + ls[3]);
        if (__any_sync(0xffffffffu, resc)) {
          // lazy rescale: O must hold PV(j-1) before it is multiplied by 2^(m_old - m_new)
          ptx::mbar_wait(pv_done, (pcount - 1) & 1);
          ptx::tc_fence_after();
          float o[32];
          const uint32_t ta = tmem + kColO + h * CPW + lane_off;
          ptx::tmem_ld32(ta, o);
#pragma unroll
          for (int i = 0; i < 32; ++i) o[i] *= f;
          ptx::tmem_st32(ta, o);
        }
        l = l * f + lsum;
        // P(j) over S(j): keys [h*32, h*32+32) -> columns [h*32, h*32+16) of the S buffer (this
        // warp's own S columns, already in its registers)
        ptx::tmem_st16_nowait(tmem + sb * BN + h * CPW + lane_off, pk);
        ptx::tmem_wait_st();
        ptx::tc_fence_before();
        __syncwarp();
        if (lane == 0) ptx::mbar_arrive(p_full);
        if (warp == 2 && lane == 0) trace_ev(p, 4, pcount);
        ++pcount;
        ++j;
      }
      // final O of this item
      ptx::mbar_wait(o_full, icount & 1);
      if (warp == 2 && lane == 0) trace_ev(p, 5, icount);
      ptx::tc_fence_after();
      red_l[h * 128 + rit] = l;
      ptx::named_bar_sync(bar_id, 32 * NWQ);
      float ltot = 0.f;
#pragma unroll
      for (int w = 0; w < NWQ; ++w) ltot += red_l[w * 128 + rit];
      ptx::named_bar_sync(bar_id, 32 * NWQ);
      float o[32];
      if (j > 0) ptx::tmem_ld32(tmem + kColO + h * CPW + lane_off, o);
      ptx::tc_fence_before();
      __syncwarp();
      if (lane == 0) ptx::mbar_arrive(o_empty);
      // O rows -> swizzled staging in stage 0 (free: every MMA of the item is complete and the
      // producer waits epi_done before the next item) -> four TMA box stores (rows >= R clipped)
      {
        const float inv = (j > 0 && ltot > 0.f) ? 1.f / ltot : 0.f;
        const uint32_t srow = ptx::smem_u32(kvbuf0) + h * kOBlockBytes + rit * 128;
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const uint32_t a = srow + (uint32_t)((u ^ (rit & 7)) * 16);
          if (j > 0)
            ptx::st_shared_v4(a, __float_as_uint(o[4 * u] * inv), __float_as_uint(o[4 * u + 1] * inv),
                              __float_as_uint(o[4 * u + 2] * inv), __float_as_uint(o[4 * u + 3] * inv));
          else
            ptx::st_shared_v4(a, 0u, 0u, 0u, 0u);
        }
        if (row_ok && h == 0)
          p.lse_part[((size_t)sp * p.g.Hkv + kvh) * p.g.R + rho] =
              (j > 0 && ltot > 0.f) ? m_ref + fast_log2(ltot) : -INFINITY;
      }
      ptx::fence_proxy_async_smem();
      ptx::named_bar_sync(5, 32 * kSoftWarps);
      if (warp == 2 && lane == 0) {
#pragma unroll
        for (int b = 0; b < 4; ++b)
          ptx::tma_store_3d(&tmO, kvbuf0 + b * kOBlockBytes, b * 32, mt * BM, sp * p.g.Hkv + kvh);
        ptx::bulk_commit();
        ptx::bulk_wait_read0();
        ptx::mbar_arrive(epi_done);
      }
      if (warp == 2 && lane == 0) trace_ev(p, 6, icount);
    }
  }
  if (warp == 2 && lane == 0) ptx::bulk_wait0();
  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc<512>(tmem);
  }
}

int sm_count() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
  }
  return n;
}

const int kReg = register_kernels({(const void*)compact_kv_kernel, (const void*)attn_tc_kernel});

}  // namespace

bool attn_tc_supported(const LayerGeom& g) {
  // chunk blocks must tile the 128-key tiles (c | 128)
  // (any c dividing 128: c % 8 != 0 re-swizzles the record rows in the compaction; V-only needs c % 8 == 0)
  return g.d == D && (g.rec_swz == 1 || (g.rec_swz == 2 && g.c % 8 == 0)) && g.c >= 1 && g.c <= BN &&
         (BN % g.c) == 0;
}

int attn_tc_nsplit(const LayerGeom& g, int k_cap, int include_suffix) {
  const int MT = (g.R + BM - 1) / BM;
  const int T_cap = (k_cap * g.c + BN - 1) / BN + (include_suffix ? (g.ns + BN - 1) / BN : 0);
  int s = sm_count() / (g.Hkv * MT);
  static int force = -1;  // tuning knob CKV_ATTN_SPLITS (results unchanged, only the split count)
  if (force < 0) {
    const char* e = tuning_env("CKV_ATTN_SPLITS");
    force = (e && atoi(e) > 0) ? atoi(e) : 0;
  }
  if (force > 0) s = force;
  if (s < 1) s = 1;
  if (s > T_cap) s = T_cap;
  return s < 1 ? 1 : s;
}

size_t attn_tc_dense_bytes(const LayerGeom& g, int k_cap, int max_ns) {
  const int T_cap = (k_cap * g.c + BN - 1) / BN + (max_ns + BN - 1) / BN;
  return (size_t)g.Hkv * T_cap * kKVBytes;
}

cudaError_t launch_attn_tc(const LayerGeom& g, const __nv_bfloat16* q, const __nv_bfloat16* k_suf,
                           const __nv_bfloat16* v_suf, const __nv_bfloat16* pool_layer, const int32_t* kept_slots,
                           const int32_t* kept_ids, const int32_t* n_kept_dev, int k_cap, int include_suffix,
                           int nsplit, float* o_part, float* lse_part, void* dense_ws, const char* host_layer,
                           const __nv_bfloat16* probe_layer, cudaEvent_t after_compact, const float* lam_ref,
                           cudaStream_t st) {
  if (!attn_tc_supported(g) || !dense_ws) return cudaErrorNotSupported;
  AttnParams p;
  p.g = g;
  p.q = q;
  p.kept_ids = kept_ids;
  p.n_kept_dev = n_kept_dev;
  p.include_suffix = include_suffix;
  p.nsplit = nsplit;
  p.MT = (g.R + BM - 1) / BM;
  p.NTp_cap = (k_cap * g.c + BN - 1) / BN;
  p.NTs = (g.ns + BN - 1) / BN;
  p.T_cap = p.NTp_cap + (include_suffix ? p.NTs : 0);
  p.dense = static_cast<const char*>(dense_ws);
  p.n_items = g.Hkv * p.MT * nsplit;
  p.scale = kLog2e / sqrtf((float)g.d);
  p.o_part = o_part;
  p.lse_part = lse_part;
  p.lam_ref = lam_ref;
  const int64_t rec_bytes = (int64_t)(g.rec_swz == 2 ? 1 : 2) * g.Hkv * g.c * D * 2;
  const int64_t n_warps = (int64_t)g.Hkv * k_cap * 4 + (include_suffix ? (int64_t)g.Hkv * g.ns * 2 : 0);
  const int cblocks = (int)std::min<int64_t>((n_warps + 7) / 8, 3 * sm_count());  // one resident wave (3 CTAs / SM)
  if (cudaError_t e_ = launch_kernel(compact_kv_kernel, cblocks, 256, 0, st, g,
                                     reinterpret_cast<char*>(const_cast<__nv_bfloat16*>(pool_layer)), host_layer,
                                     probe_layer,
                                     kept_ids, rec_bytes, kept_slots,
                                             n_kept_dev, k_cap, k_suf, v_suf, include_suffix, p.NTp_cap, p.T_cap,
                                             static_cast<char*>(dense_ws))) return e_;
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  if (after_compact) {  // the cache slots of this layer are no longer read after this point
    if ((e = cudaEventRecord(after_compact, st)) != cudaSuccess) return e;
    pdl_mark_event_wait(st);  // an event node between the kernels: no programmatic edge across it
  }
  static bool attr = false;
  if (!attr) {
    e = cudaFuncSetAttribute(attn_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmem);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  const int grid = p.n_items < sm_count() ? p.n_items : sm_count();
  static int trace_mode = -1;
  static unsigned long long* trace_buf = nullptr;
  if (trace_mode < 0) {
    const char* ev = tuning_env("CKV_ATTN_TRACE");
    trace_mode = (ev && ev[0] == '1') ? 1 : 0;
    if (trace_mode) cudaMalloc(&trace_buf, 7 * 32 * sizeof(unsigned long long));
  }
  p.trace = trace_buf;
  if (trace_buf) cudaMemsetAsync(trace_buf, 0, 7 * 32 * sizeof(unsigned long long), st);
  CUtensorMap tmO;
  if (!make_tmap_f32_3d_store(&tmO, o_part, D, (uint64_t)g.R, (uint64_t)nsplit * g.Hkv, BM))
    return cudaErrorInvalidValue;
  if (cudaError_t e_ = launch_kernel(attn_tc_kernel, grid, kThreads, kSmem, st, tmO, p)) return e_;
  if (trace_buf) {  // debug only: synchronous dump of CTA 0's event times (us since kernel start)
    unsigned long long h[7 * 32];
    cudaStreamSynchronize(st);
    cudaMemcpy(h, trace_buf, sizeof h, cudaMemcpyDeviceToHost);
    const char* nm[7] = {"start", "q_full", "kv_full", "s_full", "p_full", "o_full", "stored"};
    for (int e = 1; e < 7; ++e) {
      fprintf(stderr, "[attn trace] %-8s", nm[e]);
      for (int i = 0; i < 10; ++i) fprintf(stderr, " %6.2f", h[e * 32 + i] ? (h[e * 32 + i] - h[0]) * 1e-3 : -1.0);
      fprintf(stderr, "\n");
    }
  }
  return cudaGetLastError();
}

}  // namespace ckv
