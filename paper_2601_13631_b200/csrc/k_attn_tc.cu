// A7 split-K exact attention on tcgen05 (bf16, d = 128), flash-attention style.
//
// Same contract as attn_simt_kernel (k_attn.cu): for every GQA-packed suffix row and every
// key split, a normalised partial O and its base-2 LSE over the kept prefix chunks (all
// visible, partial-chunk padding masked) and the causal suffix keys t <= r
// (Q6, Q9).  A8 (attn_combine) merges the splits.
//
// Per work item (kv head, 128-row tile, key split), 1 CTA per SM, 576 threads:
//   warp 0      producer: Q tile by TMA (the GQA-packed [Hkv][R_pad][128] Q left by the score
//               kernel); per 128-key tile the K and V halves of up to 128/c kept chunks straight
//               from their HBM cache slots, one 1-D bulk copy per (chunk, K|V, half) issued by
//               many lanes at once (records are stored pre-swizzled, rec_elem), or the suffix
//               tile through a 3-D TMA map over k_suf / v_suf.  Two 64 KB stages; K and V of a
//               stage have separate barriers (K(j+2) lands as soon as S(j) is done).
//   warp 1      TMEM alloc + MMA issue: S = Q K^T (M 128, N 128, K 128; K-major / K-major) into one
//               of two TMEM S buffers, then O += P V (P K-major from smem, V MN-major) into the TMEM
//               O accumulator, software-pipelined one tile behind S.
//   warps 2..17 softmax: one row per thread, four warps per TMEM lane quadrant (32 key columns
//               and 32 O columns each); row max exchanged through shared memory; lazy O rescale
//               (only when the running max grows by > 8 in log2 units) via tcgen05.ld/st;
//               P = 2^(s - m) written as bf16 in the 128-byte-swizzled K-major layout.
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
constexpr uint32_t kQBytes = BM * D * 2;           // 32 KB
constexpr uint32_t kKVBytes = 2 * BN * D * 2;      // K + V = 64 KB
constexpr uint32_t kPBytes = BM * BN * 2;          // 32 KB
constexpr size_t kSmem = kQBytes + 2 * kKVBytes + kPBytes + 4096 + 1024;
constexpr float kRescaleThresh = 8.f;
constexpr int kSlotBuf = 1024;              // log2 units

struct AttnParams {
  LayerGeom g;
  const int32_t* kept_slots;
  const int32_t* kept_ids;
  const int32_t* n_kept_dev;
  int k_cap;
  int include_suffix;
  int nsplit;
  int MT, R_pad;
  int NTp_cap, NTs, T_cap;
  const char* pool;      // this layer's slot pool (swizzled records, rec_elem)
  int64_t rec_bytes;
  uint32_t chunk_bytes;  // one (chunk, kv head) K+V block = 4 * c * 128 bytes
  int n_items;
  float scale;
  float* o_part;
  float* lse_part;
  unsigned long long* trace;  // debug: per-event %globaltimer of CTA 0 (CKV_ATTN_TRACE=1), else null
};

__device__ __forceinline__ void trace_ev(const AttnParams& p, int ev, int i) {
  if (p.trace && blockIdx.x == 0 && i < 64) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    p.trace[ev * 64 + i] = t;
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

// O += P V for the tile that was scored one step earlier (MMA thread).  Prefix tiles hold
// `nv` chunk blocks [K h0|K h1|V h0|V h1] of c rows each; suffix tiles hold [K h0|K h1|V h0|V h1]
// of 128 rows each.  V is the MN-major B operand (d contiguous), P the K-major A operand.
__device__ __forceinline__ void issue_pv(const AttnParams& p, uint32_t tmem_O, uint32_t pa, uint8_t* kvbuf0,
                                         uint64_t* p_full, uint64_t* p_empty, uint64_t* o_empty, uint64_t* kv_empty,
                                         uint64_t* v_full, uint32_t idesc_o, int jj, int stage, int stage_use,
                                         bool prefix, int nv, int icount, int& pcount) {
  ptx::mbar_wait(&v_full[stage], (stage_use >> 1) & 1);
  ptx::mbar_wait(p_full, pcount & 1);
  if (jj == 0) ptx::mbar_wait(o_empty, (icount & 1) ^ 1);
  ptx::tc_fence_after();
  const uint32_t sa = ptx::smem_u32(kvbuf0 + stage * kKVBytes);
  uint32_t acc = jj > 0 ? 1u : 0u;
  const int ksteps = prefix ? (nv * p.g.c + 15) / 16 : BN / 16;  // keys of absent chunks are skipped
  for (int k = 0; k < ksteps; ++k) {
    const uint64_t adesc = ptx::umma_desc_sw128(pa + (k >> 2) * (kPBytes / 2) + (k & 3) * 32);
    const uint64_t bdesc = ptx::umma_desc_sw128_mn(sa + kKVBytes / 2 + k * 16 * 128, kKVBytes / 4);
    ptx::mma_bf16(tmem_O, adesc, bdesc, idesc_o, acc);
    acc = 1u;
  }
  ptx::mma_commit(p_empty);
  ptx::mma_commit(&kv_empty[stage]);
  ++pcount;
}

__global__ void __launch_bounds__(kThreads, 1)
    attn_tc_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmKs,
                   const __grid_constant__ CUtensorMap tmVs, AttnParams p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* qbuf = smem;
  uint8_t* kvbuf0 = smem + kQBytes;
  uint8_t* pbuf = kvbuf0 + 2 * kKVBytes;
  __shared__ float red_m[NWQ * 128], red_l[NWQ * 128];  // [warp of a quadrant][128 rows]
  __shared__ int slot_of_pos[16];          // producer: slot of each chunk position of a tile
  __shared__ int slot_buf[kSlotBuf];       // producer: slot ids of the current item
  uint64_t* bars = reinterpret_cast<uint64_t*>(pbuf + kPBytes);
  uint64_t* q_full = bars + 0;
  uint64_t* q_empty = bars + 1;
  uint64_t* k_full = bars + 2;    // [2] K half of a stage landed
  uint64_t* k_empty = bars + 14;  // [2] S(j) done with K of the stage
  uint64_t* v_full = bars + 18;   // [2] V half landed
  uint64_t* kv_empty = bars + 4;  // [2] PV(j) done with V of the stage
  uint64_t* s_full = bars + 6;    // [2]
  uint64_t* s_empty = bars + 8;   // [2]
  uint64_t* p_full = bars + 10;
  uint64_t* p_empty = bars + 11;
  uint64_t* o_full = bars + 12;
  uint64_t* o_empty = bars + 13;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 16);  // bars 16, 17 hold the slot

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int n_kept = *p.n_kept_dev;
  if (threadIdx.x == 0) trace_ev(p, 5, 0);

  if (threadIdx.x == 0) {
    ptx::mbar_init(q_full, 1);
    ptx::mbar_init(q_empty, 1);
    for (int i = 0; i < 2; ++i) {
      ptx::mbar_init(&k_full[i], 1);
      ptx::mbar_init(&k_empty[i], 1);
      ptx::mbar_init(&v_full[i], 1);
      ptx::mbar_init(&kv_empty[i], 1);
      ptx::mbar_init(&s_full[i], 1);
      ptx::mbar_init(&s_empty[i], kSoftWarps);
    }
    ptx::mbar_init(p_full, kSoftWarps);
    ptx::mbar_init(p_empty, 1);
    ptx::mbar_init(o_full, 1);
    ptx::mbar_init(o_empty, kSoftWarps);
    ptx::fence_mbar_init();
  }
  if (warp == 1) ptx::tmem_alloc<512>(tmem_slot);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t tmem_O = tmem + 256;

  if (warp == 0) {
    // ------------------------------------------------------------ TMA producer (whole warp:
    // lanes fetch the tile's slot ids in parallel, lane 0 issues the copies)
    if (lane == 0) {
      ptx::tma_prefetch_desc(&tmQ);
    }
    int icount = 0, kvcount = 0;
    const int cpt = BN / p.g.c;  // chunks per key tile (<= 16)
    for (int it = blockIdx.x; it < p.n_items; it += gridDim.x, ++icount) {
      const int sp = it % p.nsplit, mt = (it / p.nsplit) % p.MT, kvh = it / (p.nsplit * p.MT);
      const Tiles tl = item_tiles(p, sp, n_kept);
      if (lane == 0) {
        ptx::mbar_wait(q_empty, (icount & 1) ^ 1);
        ptx::mbar_expect_tx(q_full, kQBytes);
        const int yq = kvh * p.R_pad + mt * BM;
        ptx::tma_load_2d(qbuf, &tmQ, q_full, 0, yq);
        ptx::tma_load_2d(qbuf + kQBytes / 2, &tmQ, q_full, 64, yq);
      }
      // all slot ids of the item's kept chunks, staged in shared memory once per item
      const int c_beg = min(tl.t0, p.NTp_cap) * cpt;
      const int c_end = min(min(tl.t1, p.NTp_cap) * cpt, n_kept);
      for (int i = c_beg + lane; i < c_end && i - c_beg < kSlotBuf; i += 32) slot_buf[i - c_beg] = p.kept_slots[i];
      __syncwarp();
      for (int t = tl.t0; t < tl.t1; ++t) {
        if (!tile_present(p, tl, t)) continue;
        const int st = kvcount & 1;
        uint8_t* kb = kvbuf0 + st * kKVBytes;
        const bool prefix = t < p.NTp_cap;
        const int nv = prefix ? min(cpt, n_kept - t * cpt) : 0;
        // c = 8 with an odd chunk count: the last 16-key MMA step also spans the next (absent)
        // chunk position, so fill it with a duplicate (finite V; its P is masked to 0)
        const int ncopy = (prefix && (nv * p.g.c) % 16) ? nv + 1 : nv;
        // K and V of a stage have separate barriers: K(j+2) may land as soon as S(j) is done,
        // V(j+2) once PV(j) is done
        const uint32_t hb = p.g.c * 128u;  // bytes of one (K|V, half) block
        if (prefix && lane < cpt && lane < nv) {
          const int ci = t * cpt + lane;
          slot_of_pos[lane] = (ci - c_beg < kSlotBuf) ? slot_buf[ci - c_beg] : p.kept_slots[ci];
        }
        for (int kv = 0; kv < 2; ++kv) {
          uint64_t* full = kv == 0 ? &k_full[st] : &v_full[st];
          if (lane == 0) {
            ptx::mbar_wait(kv == 0 ? &k_empty[st] : &kv_empty[st], ((kvcount >> 1) & 1) ^ 1);
            ptx::mbar_expect_tx(full, prefix ? ncopy * 2 * hb : kKVBytes / 2);
            if (kv == 0) trace_ev(p, 0, kvcount);
          }
          __syncwarp();  // slot ids visible; expect_tx precedes every complete_tx of this phase
          uint8_t* dstb = kb + kv * (kKVBytes / 2);
          if (prefix) {
            // two contiguous bulk copies per kept chunk and operand (h0, h1 of the swizzled
            // record image, rec_elem) into rows [q c, (q+1) c) of the [half][128 keys][128 B]
            // tile; issued by many lanes at once (one issuing thread serialises them)
            for (int w = lane; w < ncopy * 2; w += 32) {
              const int q = w >> 1, hh = w & 1;
              const int sl = slot_of_pos[q < nv ? q : nv - 1];
              const char* src = p.pool + (int64_t)sl * p.rec_bytes + (int64_t)kvh * p.chunk_bytes + (kv * 2 + hh) * hb;
              ptx::bulk_g2s(dstb + hh * (kKVBytes / 4) + q * hb, src, hb, full);
            }
          } else if (lane == 0) {
            const int ts0 = (t - p.NTp_cap) * BN;
            const CUtensorMap* m = kv == 0 ? &tmKs : &tmVs;
            ptx::tma_load_3d(dstb, m, full, 0, kvh, ts0);
            ptx::tma_load_3d(dstb + kKVBytes / 4, m, full, 64, kvh, ts0);
          }
        }
        __syncwarp();
        ++kvcount;
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer
    if (lane == 0) {
      constexpr uint32_t idesc_s = ptx::idesc_bf16_f32(BM, BN, false);
      constexpr uint32_t idesc_o = ptx::idesc_bf16_f32(BM, D, true);
      const int cpt = BN / p.g.c;
      int icount = 0, kvcount = 0, scount = 0, pcount = 0;
      const uint32_t qa = ptx::smem_u32(qbuf);
      const uint32_t pa = ptx::smem_u32(pbuf);
      for (int it = blockIdx.x; it < p.n_items; it += gridDim.x, ++icount) {
        const int sp = it % p.nsplit;
        const Tiles tl = item_tiles(p, sp, n_kept);
        ptx::mbar_wait(q_full, icount & 1);
        int j = 0, prev_stage = 0, prev_nv = 0, prev_use = 0;
        bool prev_prefix = false;
        for (int t = tl.t0; t < tl.t1; ++t) {
          if (!tile_present(p, tl, t)) continue;
          const int st = kvcount & 1;
          ptx::mbar_wait(&k_full[st], (kvcount >> 1) & 1);
          trace_ev(p, 1, kvcount);
          const int sb = scount & 1;
          ptx::mbar_wait(&s_empty[sb], ((scount >> 1) & 1) ^ 1);
          ptx::tc_fence_after();
          const uint32_t ka = ptx::smem_u32(kvbuf0 + st * kKVBytes);
          const bool prefix = t < p.NTp_cap;
          const int nv = prefix ? min(cpt, n_kept - t * cpt) : 0;
#pragma unroll
          for (int k = 0; k < D / 16; ++k) {
            const uint32_t off_q = (k >> 2) * (kQBytes / 2) + (k & 3) * 32;
            const uint32_t off_k = (k >> 2) * (kKVBytes / 4) + (k & 3) * 32;
            ptx::mma_bf16(tmem + sb * BN, ptx::umma_desc_sw128(qa + off_q), ptx::umma_desc_sw128(ka + off_k),
                          idesc_s, k > 0 ? 1u : 0u);
          }
          ptx::mma_commit(&s_full[sb]);
          ptx::mma_commit(&k_empty[st]);
          trace_ev(p, 2, scount);
          ++scount;
          if (j > 0)
            issue_pv(p, tmem_O, pa, kvbuf0, p_full, p_empty, o_empty, kv_empty, v_full, idesc_o, j - 1, prev_stage,
                     prev_use, prev_prefix, prev_nv, icount, pcount);
          prev_stage = st;
          prev_use = kvcount;
          prev_prefix = prefix;
          prev_nv = nv;
          ++kvcount;
          ++j;
        }
        if (j > 0)
          issue_pv(p, tmem_O, pa, kvbuf0, p_full, p_empty, o_empty, kv_empty, v_full, idesc_o, j - 1, prev_stage,
                   prev_use, prev_prefix, prev_nv, icount, pcount);
        ptx::mma_commit(q_empty);
        ptx::mma_commit(o_full);
      }
    }
  } else {
    // ------------------------------------------------------------ softmax / epilogue
    // kSoftWarps = 16: four warps per TMEM lane quadrant, each owning CPW = 32 key columns
    // of S, the same 32 columns of O, and 32 keys (64 bytes) of every P row.
    const int e = warp - 2, quad = warp & 3, h = e >> 2;
    const int rit = quad * 32 + lane;  // row in tile
    const uint32_t lane_off = (uint32_t)(quad * 32) << 16;
    const uint32_t bar_id = 1 + quad;  // named barrier of the quadrant's NWQ warps
    int icount = 0, scount = 0, pcount = 0;
    const float sc = p.scale;
    int n_valid_prefix = 0;
    if (n_kept > 0) {
      const int last = p.kept_ids[n_kept - 1];
      n_valid_prefix = (n_kept - 1) * p.g.c + min(p.g.c, p.g.n_loc - last * p.g.c);
    }
    for (int it = blockIdx.x; it < p.n_items; it += gridDim.x, ++icount) {
      const int sp = it % p.nsplit, mt = (it / p.nsplit) % p.MT, kvh = it / (p.nsplit * p.MT);
      const Tiles tl = item_tiles(p, sp, n_kept);
      const int rho = mt * BM + rit;
      const bool row_ok = rho < p.g.R;
      const int r = rho % p.g.ns;
      float m_ref = -INFINITY, l = 0.f;
      int j = 0;
      for (int t = tl.t0; t < tl.t1; ++t) {
        if (!tile_present(p, tl, t)) continue;
        const int sb = scount & 1;
        ptx::mbar_wait(&s_full[sb], (scount >> 1) & 1);
        if (warp == 2 && lane == 0) trace_ev(p, 3, scount);
        ptx::tc_fence_after();
        float x[CPW];
        ptx::tmem_ld32p(tmem + sb * BN + h * CPW + lane_off, x);
        ptx::tc_fence_before();
        __syncwarp();
        if (lane == 0) ptx::mbar_arrive(&s_empty[sb]);  // S buffer consumed into registers
        ++scount;
        const bool pre = t < p.NTp_cap;
        const int b0 = (pre ? t * BN : (t - p.NTp_cap) * BN) + h * CPW;
        const int lim = pre ? n_valid_prefix : min(r + 1, p.g.ns);  // key valid iff index < lim
        if (b0 + CPW > lim) {
#pragma unroll
          for (int i = 0; i < CPW; ++i)
            if (b0 + i >= lim) x[i] = -INFINITY;
        }
        float mx[CPW / 2];
#pragma unroll
        for (int i = 0; i < CPW / 2; ++i) mx[i] = fmaxf(x[i], x[i + CPW / 2]);
#pragma unroll
        for (int n = CPW / 4; n >= 1; n >>= 1)
#pragma unroll
          for (int i = 0; i < n; ++i) mx[i] = fmaxf(mx[i], mx[i + n]);
        red_m[h * 128 + rit] = mx[0];
        ptx::named_bar_sync(bar_id, 32 * NWQ);
        float tmax = red_m[rit];
#pragma unroll
        for (int w = 1; w < NWQ; ++w) tmax = fmaxf(tmax, red_m[w * 128 + rit]);
        tmax *= sc;
        ptx::named_bar_sync(bar_id, 32 * NWQ);  // red_m reusable
        const float m_new = fmaxf(m_ref, tmax);
        const bool resc = (j > 0) && (m_ref != -INFINITY) && (m_new > m_ref + kRescaleThresh);
        const float f = resc ? fast_exp2(m_ref - m_new) : 1.f;
        if (j == 0 || m_ref == -INFINITY || resc) m_ref = m_new;
        const float msub = (m_ref == -INFINITY) ? 0.f : m_ref;
        float ls[4] = {0.f, 0.f, 0.f, 0.f};
        uint32_t pk[CPW / 2];
#pragma unroll
        for (int i = 0; i < CPW / 2; ++i) {
          const float p0 = fast_exp2(fmaf(x[2 * i], sc, -msub));
          const float p1 = fast_exp2(fmaf(x[2 * i + 1], sc, -msub));
          ls[i & 3] += p0 + p1;
          __nv_bfloat162 b2 = __floats2bfloat162_rn(p0, p1);
          pk[i] = *reinterpret_cast<uint32_t*>(&b2);
        }
        const float lsum = (ls[0] + ls[1]) + (ls[2] + ls[3]);
        if (__any_sync(0xffffffffu, resc)) {
          // lazy rescale: O must hold PV(j-1) before it is multiplied by 2^(m_old - m_new)
          ptx::mbar_wait(p_empty, (pcount - 1) & 1);
          ptx::tc_fence_after();
          float o[32];
          const uint32_t ta = tmem_O + h * CPW + lane_off;
          ptx::tmem_ld32(ta, o);
#pragma unroll
          for (int i = 0; i < 32; ++i) o[i] *= f;
          ptx::tmem_st32(ta, o);
        }
        l = l * f + lsum;
        // P buffer free (PV(j-1) done reading it)?  keys [h*32, h*32+32) = half h/2, units
        // 4*(h&1) .. 4*(h&1)+3 of the 128-byte row, swizzled by (row & 7)
        ptx::mbar_wait(p_empty, (pcount & 1) ^ 1);
        const uint32_t prow = ptx::smem_u32(pbuf) + (h >> 1) * (kPBytes / 2) + rit * 128;
#pragma unroll
        for (int c16 = 0; c16 < CPW / 8; ++c16) {
          const uint32_t phys = (uint32_t)(((h & 1) * 4 + c16) ^ (rit & 7));
          ptx::st_shared_v4(prow + phys * 16, pk[4 * c16], pk[4 * c16 + 1], pk[4 * c16 + 2], pk[4 * c16 + 3]);
        }
        ptx::fence_proxy_async_smem();
        ptx::tc_fence_before();
        __syncwarp();
        if (lane == 0) ptx::mbar_arrive(p_full);
        if (warp == 2 && lane == 0) trace_ev(p, 4, pcount);
        ++pcount;
        ++j;
      }
      // final O of this item
      ptx::mbar_wait(o_full, icount & 1);
      ptx::tc_fence_after();
      red_l[h * 128 + rit] = l;
      ptx::named_bar_sync(bar_id, 32 * NWQ);
      float ltot = 0.f;
#pragma unroll
      for (int w = 0; w < NWQ; ++w) ltot += red_l[w * 128 + rit];
      ptx::named_bar_sync(bar_id, 32 * NWQ);
      float o[32];
      if (j > 0) ptx::tmem_ld32(tmem_O + h * CPW + lane_off, o);
      ptx::tc_fence_before();
      __syncwarp();
      if (lane == 0) ptx::mbar_arrive(o_empty);
      if (row_ok) {
        const float inv = (j > 0 && ltot > 0.f) ? 1.f / ltot : 0.f;
        float* dst = p.o_part + (((size_t)sp * p.g.Hkv + kvh) * p.g.R + rho) * D + h * CPW;
#pragma unroll
        for (int i = 0; i < CPW; i += 4)
          *reinterpret_cast<float4*>(dst + i) =
              (j > 0) ? make_float4(o[i] * inv, o[i + 1] * inv, o[i + 2] * inv, o[i + 3] * inv)
                      : make_float4(0.f, 0.f, 0.f, 0.f);
        if (h == 0)
          p.lse_part[((size_t)sp * p.g.Hkv + kvh) * p.g.R + rho] =
              (j > 0 && ltot > 0.f) ? m_ref + fast_log2(ltot) : -INFINITY;
      }
    }
  }
  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc<512>(tmem);
  }
}

__global__ void pack_q_attn_kernel(LayerGeom g, int R_pad, const __nv_bfloat16* __restrict__ q,
                                   __nv_bfloat16* __restrict__ qpack) {
  const int64_t total = (int64_t)g.Hkv * R_pad * (D / 8);
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int x8 = (int)(i % (D / 8));
    const int64_t row = i / (D / 8);
    const int kvh = (int)(row / R_pad), rho = (int)(row % R_pad);
    uint4 val = make_uint4(0, 0, 0, 0);
    if (rho < g.R) {
      const int gq = rho / g.ns, r = rho % g.ns;
      val = *reinterpret_cast<const uint4*>(q + ((int64_t)r * g.Hq + kvh * g.G + gq) * D + x8 * 8);
    }
    *reinterpret_cast<uint4*>(qpack + row * D + x8 * 8) = val;
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

}  // namespace

bool attn_tc_supported(const LayerGeom& g) {
  // chunk blocks (c rows, 8-row swizzle atoms) must tile 128 keys
  return g.d == D && g.rec_swz == 1 && g.c >= 8 && g.c <= BN && (BN % g.c) == 0;
}

int attn_tc_nsplit(const LayerGeom& g, int k_cap, int include_suffix) {
  const int MT = (g.R + BM - 1) / BM;
  const int T_cap = (k_cap * g.c + BN - 1) / BN + (include_suffix ? (g.ns + BN - 1) / BN : 0);
  int s = sm_count() / (g.Hkv * MT);
  if (s < 1) s = 1;
  if (s > T_cap) s = T_cap;
  return s < 1 ? 1 : s;
}

cudaError_t launch_attn_tc(const LayerGeom& g, const __nv_bfloat16* q, const __nv_bfloat16* k_suf,
                           const __nv_bfloat16* v_suf, const __nv_bfloat16* pool_layer, int P_slots,
                           const int32_t* kept_slots, const int32_t* kept_ids, const int32_t* n_kept_dev, int k_cap,
                           int include_suffix, int nsplit, float* o_part, float* lse_part, void* qpack_ws,
                           bool qpack_ready, cudaStream_t st) {
  if (!attn_tc_supported(g) || !qpack_ws) return cudaErrorNotSupported;
  AttnParams p;
  p.g = g;
  p.kept_slots = kept_slots;
  p.kept_ids = kept_ids;
  p.n_kept_dev = n_kept_dev;
  p.k_cap = k_cap;
  p.include_suffix = include_suffix;
  p.nsplit = nsplit;
  p.MT = (g.R + BM - 1) / BM;
  p.R_pad = p.MT * BM;
  p.NTp_cap = (k_cap * g.c + BN - 1) / BN;
  p.NTs = (g.ns + BN - 1) / BN;
  p.T_cap = p.NTp_cap + (include_suffix ? p.NTs : 0);
  p.pool = reinterpret_cast<const char*>(pool_layer);
  p.rec_bytes = (int64_t)2 * g.Hkv * g.c * D * 2;
  p.chunk_bytes = 4u * g.c * 128u;
  (void)P_slots;
  p.n_items = g.Hkv * p.MT * nsplit;
  p.scale = kLog2e / sqrtf((float)g.d);
  p.o_part = o_part;
  p.lse_part = lse_part;
  auto* qpack = static_cast<__nv_bfloat16*>(qpack_ws);
  cudaError_t e = cudaSuccess;
  if (!qpack_ready) {  // the tcgen05 score kernel already packed this layer's Q otherwise
    pack_q_attn_kernel<<<256, 256, 0, st>>>(g, p.R_pad, q, qpack);
    e = cudaGetLastError();
    if (e != cudaSuccess) return e;
  }
  CUtensorMap tmQ, tmKs, tmVs;
  if (!make_tmap_bf16_2d(&tmQ, qpack, D, (uint64_t)g.Hkv * p.R_pad, BM)) return cudaErrorInvalidValue;
  if (!make_tmap_bf16_3d(&tmKs, k_suf, D, g.Hkv, g.ns, BN)) return cudaErrorInvalidValue;
  if (!make_tmap_bf16_3d(&tmVs, v_suf, D, g.Hkv, g.ns, BN)) return cudaErrorInvalidValue;
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
    const char* ev = getenv("CKV_ATTN_TRACE");
    trace_mode = (ev && ev[0] == '1') ? 1 : 0;
    if (trace_mode) cudaMalloc(&trace_buf, 6 * 64 * sizeof(unsigned long long));
  }
  p.trace = trace_buf;
  if (trace_buf) cudaMemsetAsync(trace_buf, 0, 6 * 64 * sizeof(unsigned long long), st);
  attn_tc_kernel<<<grid, kThreads, kSmem, st>>>(tmQ, tmKs, tmVs, p);
  if (trace_buf) {  // debug only: synchronous dump of CTA 0's event times (ns since kernel start)
    unsigned long long h[6 * 64];
    cudaStreamSynchronize(st);
    cudaMemcpy(h, trace_buf, sizeof h, cudaMemcpyDeviceToHost);
    const unsigned long long t0 = h[5 * 64];
    const char* nm[5] = {"tma_issue", "kv_full", "s_commit", "s_full@sm", "p_full@sm"};
    for (int e = 0; e < 5; ++e) {
      fprintf(stderr, "[attn trace] %-10s", nm[e]);
      for (int i = 0; i < 12; ++i) fprintf(stderr, " %7.2f", h[e * 64 + i] ? (h[e * 64 + i] - t0) * 1e-3 : -1.0);
      fprintf(stderr, "\n");
    }
  }
  return cudaGetLastError();
}

}  // namespace ckv
