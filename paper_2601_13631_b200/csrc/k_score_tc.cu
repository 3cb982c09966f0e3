// A1 score-partial on the 5th-generation tensor cores (tcgen05 + TMEM + TMA), bf16, d = 128.
//
// Same contract as the SIMT kernel (k_score_simt.cu): for every (KV head, suffix row rho,
// chunk j) it writes lam2 = log2 sum_{i in chunk j} 2^(l_i log2 e), l_i = q.k_i / sqrt(d)
// (Q2-Q5), and per (row, 64-key quarter tile) a partial base-2 LSE.
//
// Layout / schedule (persistent, one CTA per SM, 576 threads):
//   Work unit = (kv head, row group, 128-key tile); a row group is up to MG = 4 GQA-packed
//   128-row tiles of Q, kept resident in shared memory (MG x 32 KB) while the CTA streams its
//   contiguous range of key tiles, so neither Q nor K is re-read per row tile.
//   warp 0      TMA producer: the row group's Q tiles once per group; K tiles [128 keys x 128]
//               (32 KB, double-buffered), 128-byte swizzle.
//   warp 1      TMEM allocator + single-thread MMA issuer: one D[128 x 128] fp32 accumulator
//               per resident row tile (4 x 128 = all 512 TMEM columns), 8 x tcgen05.mma
//               kind::f16 (K = 16) per accumulator.
//   warps 2..17 epilogue: warp group g (4 warps, one per TMEM lane quadrant) drains
//               accumulator g: one suffix row per thread, tcgen05.ld 32 columns at a time;
//               per-chunk LSE in registers, coalesced lam2 stores ([kvh][chunk][row] layout),
//               one partial row LSE per (row, key tile).
#include <cstdio>
#include <cstdlib>

#include "common.cuh"
#include "tc_ptx.cuh"

namespace ckv {
namespace {

constexpr int BM = 128, BN = 256, D = 128, MG = 2;
constexpr int kEpiWarps = 16;  // 2 groups (one per accumulator) x 4 lane quadrants x 2 column halves
constexpr int QC = BN / 2;     // key columns per epilogue warp
constexpr int kThreads = 64 + 32 * kEpiWarps;
constexpr uint32_t kKBytes = BN * D * 2;  // 64 KB
constexpr uint32_t kQBytes = BM * D * 2;  // 32 KB per row tile
constexpr size_t kSmem = 2 * kKBytes + MG * kQBytes + 1024 /*align*/ + 256 /*barriers*/;

struct TcParams {
  LayerGeom g;
  float* lam2;
  float* lampart;
  int nsplit;   // = NKT (one partial row LSE per key tile)
  int NKT;      // key tiles per kv head
  int MT;       // row tiles per kv head
  int NRG;      // row groups per kv head
  int R_pad;
  int n_units;  // Hkv * NRG * NKT
  float scale;  // log2(e) / sqrt(d)
  unsigned long long* trace;  // debug (CKV_SCORE_TRACE=1): %globaltimer events of CTA 0, else null
};

__device__ __forceinline__ void strace(const TcParams& p, int ev, int i) {
  if (p.trace && blockIdx.x == 0 && i < 64) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    p.trace[ev * 64 + i] = t;
  }
}

// In-place pairwise tree: after the call a[0..N/G) hold sums of consecutive groups of G.
template <int N, int G>
__device__ __forceinline__ void tree_sum(float* a) {
  if constexpr (G > 1) {
    tree_sum<N, G / 2>(a);
#pragma unroll
    for (int i = 0; i < N / G; ++i) a[i] = a[2 * i] + a[2 * i + 1];
  }
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

// One 32-key group of one row: masked max -> 2^(l - max) (MUFU or exp2_poly) -> chunk sums.
// Writes lam2 for chunks inside the group (C <= 32); returns the group's (max, sum) in log2
// units so the caller can assemble larger chunks and the row's partial LSE.
template <int C, int NP>
__device__ __forceinline__ void epilogue_group(const TcParams& p, float (&v)[32], int key0, int kvh, int rho,
                                               bool row_ok, float& gms_out, float& gs_out) {
  const float sc = p.scale;
  if (key0 + 32 > p.g.n_loc) {  // only the shard's last key tile (warp-uniform)
#pragma unroll
    for (int j = 0; j < 32; ++j)
      if (key0 + j >= p.g.n_loc) v[j] = -INFINITY;
  }
  float m[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) m[i] = fmaxf(v[2 * i], v[2 * i + 1]);
#pragma unroll
  for (int n = 8; n >= 1; n >>= 1)
#pragma unroll
    for (int i = 0; i < n; ++i) m[i] = fmaxf(m[2 * i], m[2 * i + 1]);
  const float gm = m[0];
  const float gms = (gm == -INFINITY) ? 0.f : gm * sc;
#pragma unroll
  for (int j = 0; j < 32; ++j) {
    const float t = fmaf(v[j], sc, -gms);
    v[j] = ((j & 7) < NP) ? exp2_poly(t) : fast_exp2(t);  // NP of every 8 on the FMA pipe
  }
  constexpr int CG = C < 32 ? C : 32;  // chunk piece inside this group
  tree_sum<32, CG>(v);                 // v[0 .. 32/CG) = chunk (piece) sums
  float cs[32 / CG];
#pragma unroll
  for (int i = 0; i < 32 / CG; ++i) cs[i] = v[i];
  tree_sum<32 / CG, 32 / CG>(v);
  gms_out = gms;
  gs_out = v[0];
  if constexpr (C <= 32) {
    float* lam = p.lam2 + (size_t)kvh * p.g.m_loc * p.g.R + rho;
#pragma unroll
    for (int i = 0; i < 32 / C; ++i) {
      const int chunk = key0 / C + i;
      if (row_ok && chunk < p.g.m_loc)
        lam[(size_t)chunk * p.g.R] = (cs[i] > 0.f) ? gms + fast_log2(cs[i]) : -INFINITY;
    }
  }
}

__device__ __forceinline__ void lse2_merge(float& M, float& S, float m, float s) {
  if (s <= 0.f) return;
  if (S <= 0.f) {
    M = m;
    S = s;
  } else {
    const float nm = fmaxf(M, m);
    S = S * fast_exp2(M - nm) + s * fast_exp2(m - nm);
    M = nm;
  }
}

template <int C, int NP>
__global__ void __launch_bounds__(kThreads, 1)
    score_tc_kernel(const __grid_constant__ CUtensorMap tmK, const __grid_constant__ CUtensorMap tmQ, TcParams p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* kbuf0 = smem;
  uint8_t* qbuf0 = smem + 2 * kKBytes;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + 2 * kKBytes + MG * kQBytes);
  uint64_t* k_full = bars + 0;        // [2]
  uint64_t* k_empty = bars + 2;       // [2]
  uint64_t* q_full = bars + 4;
  uint64_t* q_empty = bars + 5;
  uint64_t* acc_full = bars + 6;      // [MG]
  uint64_t* acc_empty = bars + 6 + MG;  // [MG]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 6 + 2 * MG);
  __shared__ float2 xchg[2 * MG * 2 * 128];  // [iteration parity][group][column half][row]

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int u0 = (int)((int64_t)blockIdx.x * p.n_units / gridDim.x);
  const int u1 = (int)((int64_t)(blockIdx.x + 1) * p.n_units / gridDim.x);

  if (threadIdx.x == 0) {
    for (int i = 0; i < 2; ++i) {
      ptx::mbar_init(&k_full[i], 1);
      ptx::mbar_init(&k_empty[i], 1);
    }
    ptx::mbar_init(q_full, 1);
    ptx::mbar_init(q_empty, 1);
    for (int i = 0; i < MG; ++i) {
      ptx::mbar_init(&acc_full[i], 1);
      ptx::mbar_init(&acc_empty[i], kEpiWarps / MG);
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
      int kcount = 0, qcount = 0, cur = -1;
      for (int u = u0; u < u1; ++u) {
        const int grp = u / p.NKT, kt = u % p.NKT;
        const int kvh = grp / p.NRG, rg = grp % p.NRG;
        if (grp != cur) {  // new row group: its Q tiles, once
          const int nm = min(MG, p.MT - rg * MG);
          ptx::mbar_wait(q_empty, (qcount & 1) ^ 1);
          ptx::mbar_expect_tx(q_full, nm * kQBytes);
          for (int m = 0; m < nm; ++m) {
            const int yq = kvh * p.R_pad + (rg * MG + m) * BM;
            uint8_t* dq = qbuf0 + m * kQBytes;
            ptx::tma_load_2d(dq, &tmQ, q_full, 0, yq);
            ptx::tma_load_2d(dq + kQBytes / 2, &tmQ, q_full, 64, yq);
          }
          cur = grp;
          ++qcount;
        }
        const int kb = kcount & 1;
        ptx::mbar_wait(&k_empty[kb], ((kcount >> 1) & 1) ^ 1);
        ptx::mbar_expect_tx(&k_full[kb], kKBytes);
        strace(p, 0, kcount);
        const int y = kvh * p.g.n_pad + kt * BN;
        uint8_t* dst = kbuf0 + kb * kKBytes;
        ptx::tma_load_2d(dst, &tmK, &k_full[kb], 0, y);
        ptx::tma_load_2d(dst + kKBytes / 2, &tmK, &k_full[kb], 64, y);
        ++kcount;
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t idesc = ptx::idesc_bf16_f32(BM, BN);
      int kcount = 0, qcount = 0, cur = -1, nm = 0;
      int acount[MG] = {};
      for (int u = u0; u < u1; ++u) {
        const int grp = u / p.NKT;
        if (grp != cur) {
          if (cur >= 0) ptx::mma_commit(q_empty);  // previous row group's Q fully consumed
          nm = min(MG, p.MT - (grp % p.NRG) * MG);
          ptx::mbar_wait(q_full, qcount & 1);
          ++qcount;
          cur = grp;
        }
        const int kb = kcount & 1;
        ptx::mbar_wait(&k_full[kb], (kcount >> 1) & 1);
        strace(p, 1, kcount);
        const uint32_t ka = ptx::smem_u32(kbuf0 + kb * kKBytes);
        for (int m = 0; m < nm; ++m) {
          ptx::mbar_wait(&acc_empty[m], ((acount[m] >> 0) & 1) ^ 1);
          ptx::tc_fence_after();
          const uint32_t qa = ptx::smem_u32(qbuf0 + m * kQBytes);
#pragma unroll
          for (int k = 0; k < D / 16; ++k) {
            const uint32_t off = (k >> 2) * (kQBytes / 2) + (k & 3) * 32;
            const uint32_t offk = (k >> 2) * (kKBytes / 2) + (k & 3) * 32;
            ptx::mma_bf16(tmem_base + m * BN, ptx::umma_desc_sw128(qa + off), ptx::umma_desc_sw128(ka + offk), idesc,
                          k > 0 ? 1u : 0u);
          }
          ptx::mma_commit(&acc_full[m]);
          ++acount[m];
        }
        ptx::mma_commit(&k_empty[kb]);
        strace(p, 2, kcount);
        ++kcount;
      }
    }
  } else {
    // warp group m (8 warps: 4 lane quadrants x 2 column halves) drains accumulator m; the two
    // groups run out of phase (their accumulators complete one M-tile MMA apart), so one
    // group's exponentials overlap the other's reductions on every SM sub-partition
    const int e = warp - 2;
    const int m = e >> 3;               // accumulator / resident row tile of this warp group
    const int quad = warp & 3;          // TMEM lane quadrant -> rows quad*32 .. +31
    const int colq = (e >> 2) & 1;      // key columns colq*QC .. +QC-1 of the tile
    const int rit = quad * 32 + lane;
    const uint32_t bar_id = 1 + m * 4 + quad;  // the 2 warps sharing (group, quadrant)
    int acount = 0;
    int it = 0;
    for (int u = u0; u < u1; ++u) {
      const int grp = u / p.NKT, kt = u % p.NKT;
      const int kvh = grp / p.NRG, rg = grp % p.NRG;
      const int nm = min(MG, p.MT - rg * MG);
      if (m < nm) {
        ++it;
        ptx::mbar_wait(&acc_full[m], acount & 1);
        ++acount;
        ptx::tc_fence_after();
        const int rho = (rg * MG + m) * BM + rit;
        const bool row_ok = rho < p.g.R;
        // this warp: key columns [colq*QC, (colq+1)*QC) of the tile, in 32-key groups
        const int key0 = kt * BN + colq * QC;
        float gms = -INFINITY, gs = 0.f;  // (max, sum) of the warp's QC keys for this row
        float CM = -INFINITY, CS = 0.f;   // running chunk piece for 32 < C <= QC
        if constexpr (NP == 11) {  // tuning skeleton: pipeline only
          gms = 0.f;
          gs = 1.f;
          __syncwarp();
          if (lane == 0) ptx::mbar_arrive(&acc_empty[m]);
        } else {
          float v[QC / 32][32];
#pragma unroll
          for (int gi = 0; gi < QC / 32; ++gi)
            ptx::tmem_ld32(tmem_base + (uint32_t)(m * BN + colq * QC + gi * 32) + ((uint32_t)(quad * 32) << 16), v[gi]);
          ptx::tc_fence_before();
          __syncwarp();
          if (lane == 0) ptx::mbar_arrive(&acc_empty[m]);  // accumulator columns now in registers
#pragma unroll
          for (int gi = 0; gi < QC / 32; ++gi) {
            float g_m = 0.f, g_s = 0.f;
            if constexpr (NP == 10) {  // tuning: TMEM drain only
              g_s = v[gi][0] + v[gi][31];
            } else {
              epilogue_group<C, NP>(p, v[gi], key0 + gi * 32, kvh, rho, row_ok, g_m, g_s);
            }
            lse2_merge(gms, gs, g_m, g_s);
            if constexpr (C > 32 && C <= QC) {  // chunk spans groups of this warp only
              lse2_merge(CM, CS, g_m, g_s);
              if (((gi + 1) * 32) % C == 0) {
                const int chunk = (key0 + gi * 32) / C;
                if (row_ok && chunk < p.g.m_loc)
                  p.lam2[((size_t)kvh * p.g.m_loc + chunk) * p.g.R + rho] =
                      (CS > 0.f) ? CM + fast_log2(CS) : -INFINITY;
                CM = -INFINITY;
                CS = 0.f;
              }
            }
          }
        }
        // exchange the two QC-key pieces of each row within the (group, quadrant) warp pair
        float2* xb = xchg + ((it & 1) * MG + m) * (2 * 128);
        xb[colq * 128 + rit] = make_float2(gms, gs);
        ptx::named_bar_sync(bar_id, 64);
        if constexpr (C > QC) {  // chunks spanning several warps' pieces
          constexpr int PW = C / QC;
          if ((colq % PW) == 0) {
            float M2 = -INFINITY, S2 = 0.f;
#pragma unroll
            for (int w = 0; w < PW; ++w) {
              const float2 pc = xb[(colq + w) * 128 + rit];
              lse2_merge(M2, S2, pc.x, pc.y);
            }
            const int chunk = key0 / C;
            if (row_ok && chunk < p.g.m_loc)
              p.lam2[((size_t)kvh * p.g.m_loc + chunk) * p.g.R + rho] = (S2 > 0.f) ? M2 + fast_log2(S2) : -INFINITY;
          }
        }
        if (colq == 0) {  // the row's partial normaliser over this key tile
          float HM = -INFINITY, HS = 0.f;
#pragma unroll
          for (int w = 0; w < 2; ++w) {
            const float2 pc = xb[w * 128 + rit];
            lse2_merge(HM, HS, pc.x, pc.y);
          }
          if (row_ok) p.lampart[((size_t)kvh * p.nsplit + kt) * p.g.R + rho] = (HS > 0.f) ? HM + fast_log2(HS) : -INFINITY;
        }
      }
    }
  }
  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc<512>(tmem_base);
  }
}

__global__ void trace_start_kernel(unsigned long long* t) {
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(*t));
}

// GQA row packing: qpack[kvh][rho][x] = q[r][kvh*G + g][x], rho = g*ns + r, zero rows past R.
__global__ void pack_q_kernel(LayerGeom g, int R_pad, const __nv_bfloat16* __restrict__ q,
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

template <int C, int NP>
cudaError_t launch_cp(const CUtensorMap& tmK, const CUtensorMap& tmQ, const TcParams& p, int grid, cudaStream_t st) {
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(score_tc_kernel<C, NP>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmem);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  static int trace_mode = -1;
  static unsigned long long* tbuf = nullptr;
  if (trace_mode < 0) {
    const char* ev = getenv("CKV_SCORE_TRACE");
    trace_mode = (ev && ev[0] == '1') ? 1 : 0;
    if (trace_mode) cudaMalloc(&tbuf, 7 * 64 * sizeof(unsigned long long));
  }
  TcParams pp = p;
  pp.trace = tbuf;
  if (tbuf) cudaMemsetAsync(tbuf, 0, 7 * 64 * sizeof(unsigned long long), st);
  if (tbuf) {  // kernel start reference: recorded by a 1-thread marker launched just before
    trace_start_kernel<<<1, 1, 0, st>>>(tbuf + 6 * 64);
  }
  score_tc_kernel<C, NP><<<grid, kThreads, kSmem, st>>>(tmK, tmQ, pp);
  if (tbuf) {
    unsigned long long h[7 * 64];
    cudaStreamSynchronize(st);
    cudaMemcpy(h, tbuf, sizeof h, cudaMemcpyDeviceToHost);
    const unsigned long long t0 = h[6 * 64];
    const char* nm[6] = {"k_issue", "k_full", "mma_done", "acc0_full", "acc3_full", "acc0_free"};
    for (int e = 0; e < 6; ++e) {
      fprintf(stderr, "[score trace] %-9s", nm[e]);
      for (int i = 0; i < 14; ++i) fprintf(stderr, " %6.2f", h[e * 64 + i] ? (h[e * 64 + i] - t0) * 1e-3 : -1.0);
      fprintf(stderr, "\n");
    }
  }
  return cudaGetLastError();
}

// share of exponentials evaluated by exp2_poly (of every 8); CKV_SCORE_POLY overrides (tuning)
int poly_share() {
  static int np = -1;
  if (np < 0) {
    const char* e = getenv("CKV_SCORE_POLY");
    np = e ? atoi(e) : 2;
    if (np != 0 && np != 2 && np != 3 && np != 10 && np != 11) np = 2;
  }
  return np;
}

template <int C>
cudaError_t launch_c(const CUtensorMap& tmK, const CUtensorMap& tmQ, const TcParams& p, int grid, cudaStream_t st) {
  switch (poly_share()) {
    case 0: return launch_cp<C, 0>(tmK, tmQ, p, grid, st);
    case 3: return launch_cp<C, 3>(tmK, tmQ, p, grid, st);
    case 10: return launch_cp<C, 10>(tmK, tmQ, p, grid, st);  // tuning only: results invalid
    case 11: return launch_cp<C, 11>(tmK, tmQ, p, grid, st);  // tuning only: results invalid
    default: return launch_cp<C, 2>(tmK, tmQ, p, grid, st);
  }
}

}  // namespace

int score_tc_nsplit(const LayerGeom& g) {
  if (g.d != D) return 0;
  if (g.c < 1 || g.c > BN || (BN % g.c) != 0) return 0;
  return (g.n_loc + BN - 1) / BN;
}

size_t score_tc_qpack_elems(int Hkv, int R_max) { return (size_t)Hkv * ((R_max + BM - 1) / BM) * BM * D; }

cudaError_t launch_score_tc(const LayerGeom& g, const __nv_bfloat16* q, const __nv_bfloat16* probe_layer, float* lam2,
                            float* lampart, int nsplit, void* qpack_ws, cudaStream_t st) {
  if (score_tc_nsplit(g) == 0 || nsplit != score_tc_nsplit(g) || !qpack_ws) return cudaErrorNotSupported;
  TcParams p;
  p.g = g;
  p.lam2 = lam2;
  p.lampart = lampart;
  p.nsplit = nsplit;
  p.NKT = nsplit;
  p.MT = (g.R + BM - 1) / BM;
  p.R_pad = p.MT * BM;
  p.NRG = (p.MT + MG - 1) / MG;
  p.n_units = g.Hkv * p.NRG * p.NKT;
  p.scale = kLog2e / sqrtf((float)g.d);
  auto* qpack = static_cast<__nv_bfloat16*>(qpack_ws);
  pack_q_kernel<<<256, 256, 0, st>>>(g, p.R_pad, q, qpack);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  CUtensorMap tmK, tmQ;
  if (!make_tmap_bf16_2d(&tmK, probe_layer, D, (uint64_t)g.Hkv * g.n_pad, BN)) return cudaErrorInvalidValue;  // box 64 x 128
  if (!make_tmap_bf16_2d(&tmQ, qpack, D, (uint64_t)g.Hkv * p.R_pad, BM)) return cudaErrorInvalidValue;
  const int grid = p.n_units < num_sms() ? p.n_units : num_sms();
  switch (g.c) {
    case 1: return launch_c<1>(tmK, tmQ, p, grid, st);
    case 2: return launch_c<2>(tmK, tmQ, p, grid, st);
    case 4: return launch_c<4>(tmK, tmQ, p, grid, st);
    case 8: return launch_c<8>(tmK, tmQ, p, grid, st);
    case 16: return launch_c<16>(tmK, tmQ, p, grid, st);
    case 32: return launch_c<32>(tmK, tmQ, p, grid, st);
    case 64: return launch_c<64>(tmK, tmQ, p, grid, st);
    case 128: return launch_c<128>(tmK, tmQ, p, grid, st);
    default: return cudaErrorNotSupported;
  }
}

}  // namespace ckv
