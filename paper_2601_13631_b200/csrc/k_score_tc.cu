// A1 score-partial on the 5th-generation tensor cores (tcgen05 + TMEM + TMA), bf16, d = 128.
//
// Same contract as the SIMT kernel (k_score_simt.cu): for every (KV head, suffix row rho,
// chunk j) it writes lam2 = log2 sum_{i in chunk j} 2^(l_i log2 e), l_i = q.k_i / sqrt(d)
// (Q2-Q5), and per (row, 64-key quarter tile) a partial base-2 LSE.
//
// Layout / schedule (persistent, one CTA per SM, 576 threads):
//   warp 0      TMA producer: K tiles [256 keys x 128] (64 KB, double-buffered, loaded once per
//               (kv head, key tile) = K-stationary) and Q tiles [128 rows x 128] (32 KB, 2 stages)
//               from a GQA-packed Q [Hkv][R_pad][128]; 128-byte swizzle.
//   warp 1      TMEM allocator + single-thread MMA issuer: D[128 x 256] fp32 in TMEM
//               (two accumulators = all 512 columns), 8 x tcgen05.mma kind::f16 (K = 16 each).
//   warp 18     speculative gather (A6): the whole-chunk records the previous layer's plan chose
//               for this layer, host store -> HBM slots, one 4 KiB segment per warp iteration
//               (the link transfer overlaps this layer's scoring on the SMs it already holds, so
//               it needs no side stream, no event join and no SM of its own); idle otherwise.
//   warps 2..17 epilogue: tcgen05.ld 32 columns at a time, one suffix row per thread (TMEM lane),
//               four warps per lane quadrant (64 columns each); per-chunk LSE in registers,
//               coalesced lam2 stores ([kvh][chunk][row] layout).
// Work units (kv head, key tile, row tile) are linearised with the row tile fastest and split
// into contiguous ranges per CTA, so each K tile crosses HBM about once.
#include <cstdio>
#include <cstdlib>

#include "common.cuh"
#include "tc_ptx.cuh"

namespace ckv {
namespace {

constexpr int BM = 128, BN = 256, D = 128;
constexpr int kEpiWarps = 16;  // 4 per TMEM lane quadrant, 64 key columns each
constexpr int kColSplit = kEpiWarps / 4;
constexpr int kGatherWarp = 2 + kEpiWarps;
constexpr int kThreads = 96 + 32 * kEpiWarps;
constexpr int kGatherSeg = 4096;  // bytes per gather work item (as gather_kernel, k_cache.cu)
constexpr uint32_t kKBytes = BN * D * 2;  // 65536
constexpr uint32_t kQBytes = BM * D * 2;  // 32768
// Ring depths: the default (several row tiles per KV head) streams a new Q tile per unit through
// 3 stages (TMA latency of a Q tile, ~2 us, spans more than one unit's MMAs) and keeps 2 K tiles;
// with one row tile per KV head (G * n_s <= 128, e.g. the n_s = 8 HBM probe) Q is loaded once per
// KV head and every unit needs a new 64 KB K tile, so the smem goes to a 3-deep K ring instead.
template <int KS, int QS>
constexpr size_t smem_bytes() { return KS * kKBytes + QS * kQBytes + 1024 /*align*/ + 256 /*barriers*/; }

struct TcParams {
  LayerGeom g;
  float* lam2;
  float* lampart;
  int nsplit;   // = kColSplit * NKT (one partial normaliser per row, key tile and column quarter)
  int NKT;      // key tiles per kv head
  int MT;       // row tiles per kv head
  int R_pad;
  int q_direct;  // 1: Q tiles straight from q [ns][Hq][128] by a 3-D map (n_s % 128 == 0), no pack
  int perm;      // 1 (one row tile per KV head, R <= 128): packed row of rho = (rho % 4) * 32 + rho / 4, so
                 // the valid rows spread over all four TMEM lane quadrants (= all four SM sub-partitions)
  int n_units;  // Hkv * NKT * MT
  float scale;  // log2(e) / sqrt(d)
  int epi_sleep;  // epilogue warps wait for their accumulator with a suspend-time hint
  unsigned long long* trace;  // tuning build (CKV_SCORE_TRACE=1): %globaltimer events of CTA 0, else null
  SpecGather spec;  // A6 speculative gather of this layer (list null: none)
  int dbg;  // tuning build (CKV_SCORE_DBG): 1 = no epilogue math, 2 = no MMAs, 3 = no stores (results invalid)
};

// ---- packed fp32x2 arithmetic (sm_100: FFMA2 / FADD2 issue two fp32 lanes per instruction) ----
__device__ __forceinline__ uint64_t f2(float a, float b) {
  uint64_t r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b));
  return r;
}
__device__ __forceinline__ void f2_split(uint64_t r, float& a, float& b) {
  asm("mov.b64 {%0, %1}, %2;" : "=f"(a), "=f"(b) : "l"(r));
}
__device__ __forceinline__ uint64_t f2_fma(uint64_t a, uint64_t b, uint64_t c) {
  uint64_t d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
  return d;
}
__device__ __forceinline__ uint64_t f2_add(uint64_t a, uint64_t b) {
  uint64_t d;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}
__device__ __forceinline__ uint64_t f2_sub(uint64_t a, uint64_t b) {
  uint64_t d;
  asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}

// 2^x for a pair of x <= 0 on the FMA pipe: x clamped to -125 (flushes like ex2.approx.ftz
// would, to within 2^-125), round-to-nearest split x = i + f with the 1.5 * 2^23 trick,
// degree-4 minimax polynomial of 2^f on [-0.5, 0.5] (max rel. error 2.7e-6 in fp32), and i
// added to the exponent field in the integer domain ((bits(r) << 23) == i << 23 mod 2^32).
__device__ __forceinline__ uint64_t exp2_poly_x2(uint64_t x) {
  float a, b;
  f2_split(x, a, b);
  x = f2(fmaxf(a, -125.f), fmaxf(b, -125.f));
  const uint64_t M = f2(12582912.f, 12582912.f);
  const uint64_t r = f2_add(x, M);
  const uint64_t f = f2_sub(x, f2_sub(r, M));
  uint64_t q = f2_fma(f, f2(9.570068679749966e-3f, 9.570068679749966e-3f),
                      f2(5.5917806923389435e-2f, 5.5917806923389435e-2f));
  q = f2_fma(q, f, f2(0.240247443318367f, 0.240247443318367f));
  q = f2_fma(q, f, f2(0.6931218504905701f, 0.6931218504905701f));
  q = f2_fma(q, f, f2(0.9999992847442627f, 0.9999992847442627f));
  float qa, qb, ra, rb;
  f2_split(q, qa, qb);
  f2_split(r, ra, rb);
  return f2(__int_as_float(__float_as_int(qa) + (__float_as_int(ra) << 23)),
            __int_as_float(__float_as_int(qb) + (__float_as_int(rb) << 23)));
}

// Sum of 2*NP consecutive values held as NP packed pairs (pairwise tree on FADD2, then one
// FADD of the two lanes); NP a power of two.
template <int NP>
__device__ __forceinline__ float pair_sum(uint64_t* P) {
#pragma unroll
  for (int h = NP / 2; h >= 1; h /= 2) {
#pragma unroll
    for (int i = 0; i < h; ++i) P[i] = f2_add(P[i], P[i + h]);
  }
  float a, b;
  f2_split(P[0], a, b);
  return a + b;
}

// One warp's 64 key columns of one row tile (this thread: one suffix row): a single max over
// the 64 scores is the reference for every exponential (no running rescale).  Per score the
// issue slots are: 1/2 FMNMX3 (max), 1/2 FFMA2 (scale and shift), 1/2 FADD2 (chunk sums) and
// either one MUFU.EX2 or, for NPX of every 8 pairs, the FFMA2 polynomial above -- the split
// balances the MUFU pipe (16 ex2/clk/SM) against the issue slots (4 warp-instructions/clk/SM).
template <int C, int NPX, bool MASK>
__device__ __forceinline__ void epilogue_unit(const TcParams& p, float (&v)[64], int key0, float* lamrow,
                                              float* lampart_out, bool row_ok) {
  if constexpr (MASK) {  // only the shard's last key tile (a separate instantiation)
#pragma unroll
    for (int j = 0; j < 64; ++j)
      if (key0 + j >= p.g.n_loc) v[j] = -INFINITY;
  }
  float m[22];
#pragma unroll
  for (int i = 0; i < 21; ++i) m[i] = fmaxf(fmaxf(v[3 * i], v[3 * i + 1]), v[3 * i + 2]);
  m[21] = v[63];
#pragma unroll
  for (int i = 0; i < 7; ++i) m[i] = fmaxf(fmaxf(m[3 * i], m[3 * i + 1]), m[3 * i + 2]);
  m[0] = fmaxf(fmaxf(m[0], m[1]), m[2]);
  m[3] = fmaxf(fmaxf(m[3], m[4]), m[5]);
  m[6] = fmaxf(m[6], m[21]);
  const float gm = fmaxf(fmaxf(m[0], m[3]), m[6]);
  const float ms = (gm == -INFINITY) ? 0.f : gm * p.scale;
  const uint64_t SC = f2(p.scale, p.scale), NMS = f2(-ms, -ms);
  uint64_t P[32];
#pragma unroll
  for (int j = 0; j < 32; ++j) {
    const uint64_t t = f2_fma(f2(v[2 * j], v[2 * j + 1]), SC, NMS);
    if ((j & 7) < NPX) {
      P[j] = exp2_poly_x2(t);
    } else {
      float a, b;
      f2_split(t, a, b);
      P[j] = f2(fast_exp2(a), fast_exp2(b));
    }
  }
  constexpr int CG = C < 64 ? C : 64;  // keys per chunk piece inside these 64 columns
  constexpr int NC = 64 / CG;          // chunk pieces
  float cs[NC];
  if constexpr (CG == 1) {
#pragma unroll
    for (int j = 0; j < 32; ++j) f2_split(P[j], cs[2 * j], cs[2 * j + 1]);
  } else {
#pragma unroll
    for (int i = 0; i < NC; ++i) cs[i] = pair_sum<CG / 2>(P + i * (CG / 2));
  }
  float tot;
  {
    float t2[NC];
#pragma unroll
    for (int i = 0; i < NC; ++i) t2[i] = cs[i];
#pragma unroll
    for (int h = NC / 2; h >= 1; h /= 2) {
#pragma unroll
      for (int i = 0; i < h; ++i) t2[i] += t2[i + h];
    }
    tot = t2[0];
  }
  if (!row_ok) return;
#ifdef CKV_TUNING
  if (p.dbg == 3 && tot != -1.f) return;  // all the math, no stores (tot is never -1)
#endif
#pragma unroll
  for (int i = 0; i < NC; ++i) {
    if (MASK && key0 / C + i >= p.g.m_loc) break;
    lamrow[(size_t)i * p.g.R] = (cs[i] > 0.f) ? ms + fast_log2(cs[i]) : -INFINITY;
  }
  *lampart_out = (tot > 0.f) ? ms + fast_log2(tot) : -INFINITY;
}

// Unit index bookkeeping without integer division in the loops: unit u = pr * MT + r covers
// (kv head, key tile) pair pr = kvh * NKT + kt and row tile mt = (r + pr) mod MT.
struct UnitIter {
  int r, pr, prm, kvh, kt;
  __device__ __forceinline__ UnitIter(int u, int MT, int NKT) {
    pr = u / MT;
    r = u - pr * MT;
    prm = pr % MT;
    kvh = pr / NKT;
    kt = pr - kvh * NKT;
  }
  __device__ __forceinline__ int mt(int MT) const { return r + prm >= MT ? r + prm - MT : r + prm; }
  __device__ __forceinline__ bool last_of_pair(int MT) const { return r + 1 == MT; }
  __device__ __forceinline__ void next(int MT, int NKT) {
    if (++r == MT) {
      r = 0;
      ++pr;
      if (++prm == MT) prm = 0;
      if (++kt == NKT) {
        kt = 0;
        ++kvh;
      }
    }
  }
};

// tuning build only: event e of unit i (< 32) of CTA 0
__device__ __forceinline__ void trace_ev(const TcParams& p, int e, int i) {
#ifdef CKV_TUNING
  if (p.trace && blockIdx.x == 0 && i < 32) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    p.trace[e * 32 + i] = t;
  }
#endif
}

template <int C, int NP, int KS, int QS>
__global__ void __launch_bounds__(kThreads, 1)
    score_tc_kernel(const __grid_constant__ CUtensorMap tmK, const __grid_constant__ CUtensorMap tmQ, TcParams p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* kbuf0 = smem;
  uint8_t* qbuf0 = smem + KS * kKBytes;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + KS * kKBytes + QS * kQBytes);
  uint64_t* k_full = bars + 0;             // [KS]
  uint64_t* k_empty = bars + KS;           // [KS]
  uint64_t* acc_full = bars + 2 * KS;      // [2]
  uint64_t* acc_empty = bars + 2 * KS + 2; // [2]
  uint64_t* q_full = bars + 2 * KS + 4;    // [QS]
  uint64_t* q_empty = q_full + QS;         // [QS]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(q_empty + QS);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
#ifdef CKV_TUNING
  if (p.trace && threadIdx.x == 0) {  // per-CTA start (slot 5) / end (slot 6) events
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    p.trace[5 * 32 + blockIdx.x] = t;
  }
#endif
  // units: (kv head, key tile) pairs x row tiles; the row-tile order is rotated by the pair index
  // (a bijection inside every pair, whichever CTAs share it) so the CTAs working on one KV head
  // at a time do not all fetch the same Q tile from L2 at once
  const int u0 = (int)((int64_t)blockIdx.x * p.n_units / gridDim.x);
  const int u1 = (int)((int64_t)(blockIdx.x + 1) * p.n_units / gridDim.x);

  if (threadIdx.x == 0) {
    for (int i = 0; i < KS; ++i) {
      ptx::mbar_init(&k_full[i], 1);
      ptx::mbar_init(&k_empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      ptx::mbar_init(&acc_full[i], 1);
      ptx::mbar_init(&acc_empty[i], kEpiWarps / 2);  // one epilogue group per buffer
    }
    for (int i = 0; i < QS; ++i) {
      ptx::mbar_init(&q_full[i], 1);
      ptx::mbar_init(&q_empty[i], 1);
    }
    ptx::fence_mbar_init();
  }
  if (warp == 1) ptx::tmem_alloc<512>(tmem_slot);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      ptx::tma_prefetch_desc(&tmK);
      ptx::tma_prefetch_desc(&tmQ);
      int kcount = 0, qcount = 0, cur = -1, qcur = -1;
      UnitIter it(u0, p.MT, p.NKT);
      for (int u = u0; u < u1; ++u, it.next(p.MT, p.NKT)) {
        const int pr = it.pr, mt = it.mt(p.MT), kvh = it.kvh, kt = it.kt;
        if (pr != cur) {
          const int kb = kcount % KS;
          ptx::mbar_wait_sleep(&k_empty[kb], ((kcount / KS) & 1) ^ 1);
          ptx::mbar_expect_tx(&k_full[kb], kKBytes);
          const int y = kvh * p.g.n_pad + kt * BN;
          uint8_t* dst = kbuf0 + kb * kKBytes;
          ptx::tma_load_2d(dst, &tmK, &k_full[kb], 0, y);
          ptx::tma_load_2d(dst + kKBytes / 2, &tmK, &k_full[kb], 64, y);
          cur = pr;
          ++kcount;
        }
        const int qid = kvh * p.MT + mt;
        if (qid == qcur) continue;  // same Q tile as the previous unit (one row tile per KV head)
        qcur = qid;
        const int qs = qcount % QS;
        ptx::mbar_wait_sleep(&q_empty[qs], ((qcount / QS) & 1) ^ 1);
        if (qcount == 0) pdl_wait();  // Q is the previous kernel's output (the probe keys are not)
        ptx::mbar_expect_tx(&q_full[qs], kQBytes);
        uint8_t* dq = qbuf0 + qs * kQBytes;
        if (p.q_direct) {  // a 128-row tile is 128 consecutive tokens of one query head
          const int rho0 = mt * BM, gq = rho0 / p.g.ns, r0 = rho0 - gq * p.g.ns, head = kvh * p.g.G + gq;
          ptx::tma_load_3d(dq, &tmQ, &q_full[qs], 0, head, r0);
          ptx::tma_load_3d(dq + kQBytes / 2, &tmQ, &q_full[qs], 64, head, r0);
        } else {
          const int yq = kvh * p.R_pad + mt * BM;
          ptx::tma_load_2d(dq, &tmQ, &q_full[qs], 0, yq);
          ptx::tma_load_2d(dq + kQBytes / 2, &tmQ, &q_full[qs], 64, yq);
        }
        ++qcount;
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t idesc = ptx::idesc_bf16_f32(BM, BN);
      int kcount = 0, qcount = 0, acount = 0, cur = -1, kb = 0, qcur = -1, qs = 0;
      UnitIter it(u0, p.MT, p.NKT);
      for (int u = u0; u < u1; ++u, it.next(p.MT, p.NKT)) {
        const int pr = it.pr;
        if (pr != cur) {
          kb = kcount % KS;
          ptx::mbar_wait_sleep(&k_full[kb], (kcount / KS) & 1);
          ++kcount;
          cur = pr;
        }
        const int qid = it.kvh * p.MT + it.mt(p.MT);
        if (qid != qcur) {  // a new Q tile (the producer loads one only when the tile changes)
          qcur = qid;
          qs = qcount % QS;
          ptx::mbar_wait_sleep(&q_full[qs], (qcount / QS) & 1);
          ++qcount;
        }
        trace_ev(p, 0, acount);  // Q (and K) of the unit landed
        const int ab = acount & 1;
        ptx::mbar_wait_sleep(&acc_empty[ab], ((acount >> 1) & 1) ^ 1);
        trace_ev(p, 1, acount);  // accumulator free: MMAs issued
        ptx::tc_fence_after();
        const uint32_t d_tmem = tmem_base + ab * BN;
        const uint32_t qa = ptx::smem_u32(qbuf0 + qs * kQBytes);
        const uint32_t ka = ptx::smem_u32(kbuf0 + kb * kKBytes);
#ifdef CKV_TUNING
        if (p.dbg != 2)
#endif
#pragma unroll
        for (int k = 0; k < D / 16; ++k) {
          const uint32_t off_q = (k >> 2) * (kQBytes / 2) + (k & 3) * 32;
          const uint32_t off_k = (k >> 2) * (kKBytes / 2) + (k & 3) * 32;
          ptx::mma_bf16(d_tmem, ptx::umma_desc_sw128(qa + off_q), ptx::umma_desc_sw128(ka + off_k), idesc,
                        k > 0 ? 1u : 0u);
        }
        // release the Q stage when the next unit uses another Q tile (or this is the CTA's last)
        UnitIter nx = it;
        nx.next(p.MT, p.NKT);
        if (u + 1 == u1 || nx.kvh * p.MT + nx.mt(p.MT) != qid) ptx::mma_commit(&q_empty[qs]);
        ptx::mma_commit(&acc_full[ab]);
        const bool last_of_pair = (u + 1 == u1) || it.last_of_pair(p.MT);
        if (last_of_pair) ptx::mma_commit(&k_empty[kb]);
        ++acount;
      }
    }
  } else if (warp == kGatherWarp) {
    if (p.spec.list) {
      pdl_wait();  // the list and count come from the previous layer's plan
      const int n = *p.spec.n_load;
      const int64_t rb = p.spec.rec_bytes;
      const int nseg = (int)((rb + kGatherSeg - 1) / kGatherSeg);
      for (int it = blockIdx.x; it < n * nseg; it += gridDim.x) {
        const int e = it / nseg, sg = it - e * nseg;
        const int j = p.spec.list[2 * e], s = p.spec.list[2 * e + 1];
        const int64_t off = (int64_t)sg * kGatherSeg;
        const int cnt = (int)(min((int64_t)kGatherSeg, rb - off) / 16);
        const int4* src = reinterpret_cast<const int4*>(p.spec.host_layer + (int64_t)j * rb + off);
        int4* dst = reinterpret_cast<int4*>(p.spec.pool_layer + (int64_t)s * rb + off);
        int4 v[kGatherSeg / 16 / 32];
#pragma unroll
        for (int u = 0; u < kGatherSeg / 16 / 32; ++u)
          if (lane + 32 * u < cnt) v[u] = __ldg(src + lane + 32 * u);
#pragma unroll
        for (int u = 0; u < kGatherSeg / 16 / 32; ++u)
          if (lane + 32 * u < cnt) dst[lane + 32 * u] = v[u];
      }
    }
  } else {
    pdl_wait();
    pdl_trigger();  // after this CTA's own dependency is resolved (see common.cuh)
    // Two epilogue groups of 8 warps, one per accumulator buffer: group g drains the units
    // whose accumulator is buffer g (every other unit), so the groups run one MMA apart and the
    // exp2 phase of one overlaps the TMEM-load / max / sum / store phases of the other (with
    // every warp on every unit, all sixteen hit the MUFU pipe at once and leave it idle after).
    // In a group, the 2 warps of each TMEM lane quadrant take 128 columns each, in two passes
    // of 64; the accumulator is released after the second pass's TMEM load.
    const int e = warp - 2;
    const int quad = warp & 3;                // TMEM lane quadrant (warp id % 4)
    const int grp = (e >> 2) & 1;             // accumulator buffer drained by this warp
    const int chalf = e >> 3;                 // 128-column half of the 256 columns
    const int row_in_tile = quad * 32 + lane;
    const uint32_t lane_off = (uint32_t)(quad * 32) << 16;
    const int nfull = p.g.n_loc / BN;  // key tiles without a ragged tail
    int acount = 0;
    UnitIter it(u0, p.MT, p.NKT);
    for (int u = u0; u < u1; ++u, it.next(p.MT, p.NKT), ++acount) {
      const int ab = acount & 1;
      if (ab != grp) continue;
      const int mt = it.mt(p.MT), kvh = it.kvh, kt = it.kt;
      if (p.epi_sleep)
        ptx::mbar_wait_sleep(&acc_full[ab], (acount >> 1) & 1);
      else
        ptx::mbar_wait(&acc_full[ab], (acount >> 1) & 1);
      ptx::tc_fence_after();
      if (lane == 0 && e < 8 && (e & 3) == 0) trace_ev(p, 2, acount);  // group's first warp: MMA done
      if (p.perm ? quad >= p.g.R : mt * BM + quad * 32 >= p.g.R) {  // warp-uniform: quadrant all padding
        ptx::tc_fence_before();
        __syncwarp();
        if (lane == 0) ptx::mbar_arrive(&acc_empty[ab]);
        continue;
      }
      const int rho = p.perm ? lane * 4 + quad : mt * BM + row_in_tile;
      const bool row_ok = rho < p.g.R;
#pragma unroll 1
      for (int pass = 0; pass < 2; ++pass) {
        const int cq = chalf * 2 + pass;  // 64-column quarter of the key tile
        float v[64];
        {
          uint32_t r0[32], r1[32];
          const uint32_t ta = tmem_base + (uint32_t)(ab * BN + cq * (BN / kColSplit)) + lane_off;
          ptx::tmem_ld32_nowait(ta, r0);
          ptx::tmem_ld32_nowait(ta + 32, r1);
          ptx::tmem_wait_ld_tied(r0);
          ptx::tmem_wait_ld_tied(r1);
#pragma unroll
          for (int j = 0; j < 32; ++j) {
            v[j] = __uint_as_float(r0[j]);
            v[32 + j] = __uint_as_float(r1[j]);
          }
        }
        if (pass == 1) {  // both quarters read: release the accumulator to the MMA warp
          ptx::tc_fence_before();
          __syncwarp();
          if (lane == 0) ptx::mbar_arrive(&acc_empty[ab]);
          if (lane == 0 && e < 8 && (e & 3) == 0) trace_ev(p, 3, acount);
        }
#ifdef CKV_TUNING
        if (p.dbg == 1) {
          if (row_ok && v[0] + v[63] == 12345.f) p.lam2[0] = v[1];  // keep the loads alive
          continue;
        }
#endif
        const int key0 = kt * BN + cq * (BN / kColSplit);
        float* lamrow = p.lam2 + ((size_t)kvh * p.g.m_loc + key0 / C) * p.g.R + rho;
        float* lp = p.lampart + ((size_t)kvh * p.nsplit + kt * kColSplit + cq) * p.g.R + rho;
        if (kt >= nfull) {  // warp-uniform: the last key tile only
          epilogue_unit<C, NP, true>(p, v, key0, lamrow, lp, row_ok);
        } else {
          epilogue_unit<C, NP, false>(p, v, key0, lamrow, lp, row_ok);
        }
      }
      if (lane == 0 && e < 8 && (e & 3) == 0) trace_ev(p, 4, acount);  // epilogue of the unit done
    }
  }
  ptx::tc_fence_before();
  __syncthreads();
#ifdef CKV_TUNING
  if (p.trace && threadIdx.x == 0) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    p.trace[5 * 32 + 160 + blockIdx.x] = t;
  }
#endif
  if (warp == 1) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc<512>(tmem_base);
#ifdef CKV_TUNING
    if (p.trace && lane == 0) {  // after the dealloc (slot 352 + CTA)
      unsigned long long t;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      p.trace[5 * 32 + 352 + blockIdx.x] = t;
    }
#endif
  }
}

#ifdef CKV_TUNING
__global__ void stamp_kernel(unsigned long long* t) {
  unsigned long long v;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(v));
  *t = v;
}
// calibration: a 576-thread CTA per SM that records its start / end like the score kernel
__global__ void __launch_bounds__(kThreads, 1) null_kernel(unsigned long long* t) {
  unsigned long long v;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(v));
  __syncthreads();
  if (threadIdx.x == 0) t[blockIdx.x] = v;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(v));
  if (threadIdx.x == 0) t[160 + blockIdx.x] = v;
}
#endif

// GQA row packing: qpack[kvh][rho][x] = q[r][kvh*G + g][x], rho = g*ns + r, zero rows past R.
__global__ void pack_q_kernel(LayerGeom g, int R_pad, int perm, const __nv_bfloat16* __restrict__ q,
                              __nv_bfloat16* __restrict__ qpack) {
  pdl_wait();
  pdl_trigger();
  const int64_t total = (int64_t)g.Hkv * R_pad * (D / 8);
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int x8 = (int)(i % (D / 8));
    const int64_t row = i / (D / 8);
    const int kvh = (int)(row / R_pad), slot = (int)(row % R_pad);
    const int rho = perm ? (slot & 31) * 4 + (slot >> 5) : slot;  // inverse of slot = (rho % 4) * 32 + rho / 4
    uint4 val = make_uint4(0, 0, 0, 0);
    if (rho < g.R) {
      const int gq = rho / g.ns, r = rho % g.ns;
      val = *reinterpret_cast<const uint4*>(q + ((int64_t)r * g.Hq + kvh * g.G + gq) * D + x8 * 8);
    }
    *reinterpret_cast<uint4*>(qpack + row * D + x8 * 8) = val;
  }
}

int num_sms() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
  }
  return n;
}

template <int C, int NP, int KS, int QS>
cudaError_t launch_cpq(const CUtensorMap& tmK, const CUtensorMap& tmQ, const TcParams& p, int grid, cudaStream_t st) {
  constexpr size_t kSmem = smem_bytes<KS, QS>();
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(score_tc_kernel<C, NP, KS, QS>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)kSmem);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  if (cudaError_t e_ = launch_kernel(score_tc_kernel<C, NP, KS, QS>, grid, kThreads, kSmem, st, tmK, tmQ, p)) return e_;
  return cudaGetLastError();
}
template <int C, int NP>
cudaError_t launch_cp(const CUtensorMap& tmK, const CUtensorMap& tmQ, const TcParams& p, int grid, cudaStream_t st) {
  if (p.MT == 1) return launch_cpq<C, NP, 3, 1>(tmK, tmQ, p, grid, st);  // one row tile per KV head
  return launch_cpq<C, NP, 2, 3>(tmK, tmQ, p, grid, st);
}

// pairs of every 8 (i.e. exponentials of every 16) evaluated by the FFMA2 polynomial instead of
// MUFU.EX2; the tuning build's CKV_SCORE_POLY overrides it for A/B sweeps.  Measured on B200: 2 at
// c = 16 (C3: 87.1 vs 87.9 us/layer with 3), 3 for c <= 8 (C5 c = 4: 497 vs 525 us of A1 with 2 --
// its 16 lg2 per 64-key pass already load the MUFU pipe)
constexpr int kPolyPairs = 2;
template <int C>
constexpr int poly_pairs_c() { return C <= 8 ? 3 : kPolyPairs; }
int poly_pairs() {
  static int np = -1;
  if (np < 0) {
    const char* e = tuning_env("CKV_SCORE_POLY");
    np = e ? atoi(e) : kPolyPairs;
    if (np < 0 || np > 8) np = kPolyPairs;
  }
  return np;
}

template <int C>
cudaError_t launch_c(const CUtensorMap& tmK, const CUtensorMap& tmQ, const TcParams& p, int grid, cudaStream_t st) {
#ifdef CKV_TUNING
  switch (poly_pairs()) {
    case 0: return launch_cp<C, 0>(tmK, tmQ, p, grid, st);
    case 1: return launch_cp<C, 1>(tmK, tmQ, p, grid, st);
    case 2: return launch_cp<C, 2>(tmK, tmQ, p, grid, st);
    case 3: return launch_cp<C, 3>(tmK, tmQ, p, grid, st);
    case 4: return launch_cp<C, 4>(tmK, tmQ, p, grid, st);
    case 5: return launch_cp<C, 5>(tmK, tmQ, p, grid, st);
    case 6: return launch_cp<C, 6>(tmK, tmQ, p, grid, st);
    default: break;
  }
#endif
  (void)poly_pairs;
  return launch_cp<C, poly_pairs_c<C>()>(tmK, tmQ, p, grid, st);
}

#define CKV_SC(C) (const void*)score_tc_kernel<C, poly_pairs_c<C>(), 2, 3>, (const void*)score_tc_kernel<C, poly_pairs_c<C>(), 3, 1>
const int kReg = register_kernels({CKV_SC(1), CKV_SC(2), CKV_SC(4), CKV_SC(8), CKV_SC(16), CKV_SC(32), CKV_SC(64),
                                   (const void*)pack_q_kernel});
#undef CKV_SC

}  // namespace

int score_tc_nsplit(const LayerGeom& g) {
  if (g.d != D) return 0;
  if (g.c < 1 || g.c > BN / kColSplit || ((BN / kColSplit) % g.c) != 0) return 0;
  return kColSplit * ((g.n_loc + BN - 1) / BN);
}

int score_tc_packs_q(const LayerGeom& g) { return (g.ns % BM) != 0 || g.R <= BM; }

size_t score_tc_qpack_elems(int Hkv, int R_max) { return (size_t)Hkv * ((R_max + BM - 1) / BM) * BM * D; }

cudaError_t launch_score_tc(const LayerGeom& g, const __nv_bfloat16* q, const __nv_bfloat16* probe_layer, float* lam2,
                            float* lampart, int nsplit, void* qpack_ws, const SpecGather& spec, cudaStream_t st) {
  if (score_tc_nsplit(g) == 0 || nsplit != score_tc_nsplit(g) || !qpack_ws) return cudaErrorNotSupported;
  TcParams p;
  p.g = g;
  p.lam2 = lam2;
  p.lampart = lampart;
  p.spec = spec;
  p.nsplit = nsplit;
  p.NKT = nsplit / kColSplit;
  p.MT = (g.R + BM - 1) / BM;
  p.R_pad = p.MT * BM;
  p.n_units = g.Hkv * p.NKT * p.MT;
  p.scale = kLog2e / sqrtf((float)g.d);
  p.trace = nullptr;
  p.epi_sleep = 1;
  p.dbg = 0;
#ifdef CKV_TUNING
  if (const char* es = tuning_env("CKV_SCORE_DBG")) p.dbg = atoi(es);
  if (const char* es = tuning_env("CKV_SCORE_EPI_SLEEP")) p.epi_sleep = atoi(es);
#endif
#ifdef CKV_TUNING
  static unsigned long long* trace_buf = nullptr;
  if (tuning_env("CKV_SCORE_TRACE")) {
    if (!trace_buf) cudaMalloc(&trace_buf, (5 * 32 + 352 + 160) * sizeof(unsigned long long));
    cudaMemsetAsync(trace_buf, 0, (5 * 32 + 352 + 160) * sizeof(unsigned long long), st);
    p.trace = trace_buf;
  }
#endif
  auto* qpack = static_cast<__nv_bfloat16*>(qpack_ws);
  p.perm = p.MT == 1 ? 1 : 0;
  p.q_direct = ((g.ns % BM) == 0 && !p.perm) ? 1 : 0;
  if (!p.q_direct)
    if (cudaError_t e_ = launch_kernel(pack_q_kernel, 256, 256, 0, st, g, p.R_pad, p.perm, q, qpack)) return e_;
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  CUtensorMap tmK, tmQ;
  if (!make_tmap_bf16_2d(&tmK, probe_layer, D, (uint64_t)g.Hkv * g.n_pad, BN)) return cudaErrorInvalidValue;
  if (p.q_direct) {
    if (!make_tmap_bf16_3d(&tmQ, q, D, g.Hq, g.ns, BM)) return cudaErrorInvalidValue;
  } else if (!make_tmap_bf16_2d(&tmQ, qpack, D, (uint64_t)g.Hkv * p.R_pad, BM)) {
    return cudaErrorInvalidValue;
  }
  const int grid = p.n_units < num_sms() ? p.n_units : num_sms();
  cudaError_t el;
#ifdef CKV_TUNING
  cudaEvent_t tev0 = nullptr, tev1 = nullptr;
  if (p.trace) {
    cudaEventCreate(&tev0);
    cudaEventCreate(&tev1);
    cudaStreamSynchronize(st);
    cudaEventRecord(tev0, st);
    stamp_kernel<<<1, 1, 0, st>>>(p.trace + 5 * 32 + 318);
  }
#endif
  switch (g.c) {
    case 1: el = launch_c<1>(tmK, tmQ, p, grid, st); break;
    case 2: el = launch_c<2>(tmK, tmQ, p, grid, st); break;
    case 4: el = launch_c<4>(tmK, tmQ, p, grid, st); break;
    case 8: el = launch_c<8>(tmK, tmQ, p, grid, st); break;
    case 16: el = launch_c<16>(tmK, tmQ, p, grid, st); break;
    case 32: el = launch_c<32>(tmK, tmQ, p, grid, st); break;
    case 64: el = launch_c<64>(tmK, tmQ, p, grid, st); break;
    default: return cudaErrorNotSupported;
  }
#ifdef CKV_TUNING
  if (p.trace && el == cudaSuccess) {  // synchronous dump of CTA 0's events (us since its first)
    unsigned long long h[5][32], cta[320];
    stamp_kernel<<<1, 1, 0, st>>>(p.trace + 5 * 32 + 319);
    cudaEventRecord(tev1, st);
    cudaStreamSynchronize(st);
    float tev_ms = 0.f;
    cudaEventElapsedTime(&tev_ms, tev0, tev1);
    fprintf(stderr, "[score trace] launch event time %.2f us (stream idle before)\n", tev_ms * 1e3);
    cudaEventDestroy(tev0);
    cudaEventDestroy(tev1);
    cudaMemcpy(h, p.trace, sizeof h, cudaMemcpyDeviceToHost);
    cudaMemcpy(cta, p.trace + 5 * 32, sizeof cta, cudaMemcpyDeviceToHost);
    {
      unsigned long long s0 = ~0ull, s1 = 0, e0 = ~0ull, e1 = 0, dmax = 0;
      {
        unsigned long long dl[160];
        cudaMemcpy(dl, p.trace + 5 * 32 + 352, sizeof dl, cudaMemcpyDeviceToHost);
        for (int b = 0; b < grid; ++b) dmax = dl[b] > dmax ? dl[b] : dmax;
      }
      for (int b = 0; b < grid; ++b) {
        s0 = cta[b] < s0 ? cta[b] : s0;
        s1 = cta[b] > s1 ? cta[b] : s1;
        e0 = cta[160 + b] < e0 ? cta[160 + b] : e0;
        e1 = cta[160 + b] > e1 ? cta[160 + b] : e1;
      }
      fprintf(stderr, "[score trace] stamp before -> first CTA start %.2f us; last CTA end -> stamp after %.2f us; "
              "last dealloc -> stamp after %.2f us\n",
              ((long long)s0 - (long long)cta[318]) * 1e-3, ((long long)cta[319] - (long long)e1) * 1e-3,
              ((long long)cta[319] - (long long)dmax) * 1e-3);
      fprintf(stderr, "[score trace] CTA start spread %.2f us, end %.2f..%.2f us after first start; CTA0 start %.2f end %.2f\n",
              (s1 - s0) * 1e-3, (e0 - s0) * 1e-3, (e1 - s0) * 1e-3, (cta[0] - s0) * 1e-3, (cta[160] - s0) * 1e-3);
    }
    unsigned long long t0 = ~0ull;
    for (auto& r : h)
      for (unsigned long long t : r)
        if (t && t < t0) t0 = t;
    {
      unsigned long long* cal = nullptr;
      cudaMalloc(&cal, 320 * sizeof(unsigned long long));
      stamp_kernel<<<1, 1, 0, st>>>(cal + 318);
      null_kernel<<<grid, kThreads, 0, st>>>(cal);
      stamp_kernel<<<1, 1, 0, st>>>(cal + 319);
      unsigned long long hc[320];
      cudaMemcpy(hc, cal, sizeof hc, cudaMemcpyDeviceToHost);
      unsigned long long c0 = ~0ull, c1 = 0;
      for (int b = 0; b < grid; ++b) {
        c0 = hc[b] < c0 ? hc[b] : c0;
        c1 = hc[160 + b] > c1 ? hc[160 + b] : c1;
      }
      fprintf(stderr, "[score trace] calibration null kernel: stamp -> start %.2f us, end -> stamp %.2f us\n",
              ((long long)c0 - (long long)hc[318]) * 1e-3, ((long long)hc[319] - (long long)c1) * 1e-3);
      cudaFree(cal);
    }
    const char* nm[5] = {"q_land", "acc_free", "mma_done", "release", "epi_done"};
    for (int ev = 0; ev < 5; ++ev) {
      fprintf(stderr, "[score trace] %-8s", nm[ev]);
      for (int i = 0; i < 32; ++i) fprintf(stderr, " %6.2f", h[ev][i] ? (h[ev][i] - t0) * 1e-3 : -1.0);
      fprintf(stderr, "\n");
    }
  }
#endif
  return el;
}

}  // namespace ckv
