// Single-CTA radix select and block scan used by top-k (A3) and the cache planner (A4).
#pragma once
#include "common.cuh"

namespace ckv {

struct SelectSmem {
  int hist[256];
  int warp_tot[32];
  int state[3];
  alignas(16) int hist3[3][256];  // rotating histograms of the one-barrier-per-pass select
  int wc[8][32];      // per-(key slot, warp) flag counts of the one-barrier compaction
};

// Exclusive prefix sum of v over the block (threadIdx order); *tot = block total.
// Every thread of the block must call it.
template <int NT>
__device__ __forceinline__ int block_excl_scan(int v, int& tot, SelectSmem& ss) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  int incl = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    int y = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += y;
  }
  __syncthreads();  // protect warp_tot from a previous call
  if (lane == 31) ss.warp_tot[wid] = incl;
  __syncthreads();
  if (wid == 0) {
    int w = (lane < NT / 32) ? ss.warp_tot[lane] : 0;
    int wi = w;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      int y = __shfl_up_sync(0xffffffffu, wi, o);
      if (lane >= o) wi += y;
    }
    if (lane < NT / 32) ss.warp_tot[lane] = wi - w;  // exclusive warp offsets
    if (lane == 31) ss.state[0] = wi;
  }
  __syncthreads();
  tot = ss.state[0];
  return ss.warp_tot[wid] + incl - v;
}

// k-th largest (1-based) of n keys key(i); keys must be unique among those that can
// reach the top k.  MSB-first 8-bit digits, 8 passes.  Every thread must call it.
template <int NT, typename KeyFn>
__device__ uint64_t block_kth_largest(KeyFn key, int n, int k, SelectSmem& ss) {
  uint64_t prefix = 0, mask = 0;
  int krem = k;
  for (int shift = 56; shift >= 0; shift -= 8) {
    for (int b = threadIdx.x; b < 256; b += NT) ss.hist[b] = 0;
    __syncthreads();
    for (int i0 = 0; i0 < n; i0 += NT) {  // whole warps per iteration (warp-aggregated counts)
      const int i = i0 + threadIdx.x;
      uint64_t kv = 0;
      bool in = false;
      if (i < n) {
        kv = key(i);
        in = (kv & mask) == prefix;
      }
      const unsigned act = __ballot_sync(0xffffffffu, in);
      if (in) {
        const unsigned dig = (unsigned)(kv >> shift) & 255u;
        const unsigned peers = __match_any_sync(act, dig);
        if ((threadIdx.x & 31) == __ffs(peers) - 1) atomicAdd(&ss.hist[dig], __popc(peers));
      }
    }
    __syncthreads();
    if (threadIdx.x < 32) {
      const int lane = threadIdx.x;
      int cnt[8], tot = 0;
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        cnt[j] = ss.hist[255 - 8 * lane - j];
        tot += cnt[j];
      }
      int incl = tot;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        int y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
      }
      const int excl = incl - tot;
      const unsigned bal = __ballot_sync(0xffffffffu, excl < krem && incl >= krem);
      if (lane == __ffs(bal) - 1) {
        int cum = excl;
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          if (cum + cnt[j] >= krem) {
            ss.state[0] = 255 - 8 * lane - j;
            ss.state[1] = krem - cum;
            ss.state[2] = (cnt[j] == krem - cum);  // the whole bin is taken: threshold found
            break;
          }
          cum += cnt[j];
        }
      }
    }
    __syncthreads();
    prefix |= (uint64_t)ss.state[0] << shift;
    mask |= (uint64_t)255u << shift;
    krem = ss.state[1];
    const bool done = ss.state[2] != 0;
    __syncthreads();
    // every key of the chosen bin is selected: keys >= prefix (low digits 0) are exactly k
    if (done) break;
  }
  return prefix;
}

// Same select over keys held in registers: thread t owns keys i = t + NT*u (u < KPT), valid iff
// i < n.  No memory traffic per pass (the hot-path top-k over m <= NT*KPT chunk scores).
template <int NT, int KPT>
__device__ uint64_t block_kth_largest_regs(const uint64_t (&keys)[KPT], int n, int k, SelectSmem& ss) {
  uint64_t prefix = 0, mask = 0;
  int krem = k;
  for (int shift = 56; shift >= 0; shift -= 8) {
    for (int b = threadIdx.x; b < 256; b += NT) ss.hist[b] = 0;
    __syncthreads();
#pragma unroll
    for (int u = 0; u < KPT; ++u) {
      const int i = threadIdx.x + NT * u;
      const bool in = i < n && (keys[u] & mask) == prefix;
      // warp-aggregated: early passes put most keys in a few bins (same float exponent)
      const unsigned act = __ballot_sync(0xffffffffu, in);
      if (in) {
        const unsigned dig = (unsigned)(keys[u] >> shift) & 255u;
        const unsigned peers = __match_any_sync(act, dig);
        if ((threadIdx.x & 31) == __ffs(peers) - 1) atomicAdd(&ss.hist[dig], __popc(peers));
      }
    }
    __syncthreads();
    if (threadIdx.x < 32) {
      const int lane = threadIdx.x;
      int cnt[8], tot = 0;
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        cnt[j] = ss.hist[255 - 8 * lane - j];
        tot += cnt[j];
      }
      int incl = tot;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        int y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
      }
      const int excl = incl - tot;
      const unsigned bal = __ballot_sync(0xffffffffu, excl < krem && incl >= krem);
      if (lane == __ffs(bal) - 1) {
        int cum = excl;
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          if (cum + cnt[j] >= krem) {
            ss.state[0] = 255 - 8 * lane - j;
            ss.state[1] = krem - cum;
            ss.state[2] = (cnt[j] == krem - cum);
            break;
          }
          cum += cnt[j];
        }
      }
    }
    __syncthreads();
    prefix |= (uint64_t)ss.state[0] << shift;
    mask |= (uint64_t)255u << shift;
    krem = ss.state[1];
    const bool done = ss.state[2] != 0;
    if (done) break;
    // the next pass's histogram clear is ordered after every thread read state (the clear
    // touches hist only, and state is rewritten only after the next pass's second barrier)
  }
  __syncthreads();
  return prefix;
}

// Keys in registers (KPT per thread, m <= NT * KPT): A_j is summed from the per-KV-head partials
// once, and the eight radix passes and the compaction run without memory traffic.

// One barrier per radix pass (keys in registers, NT == 1024): three rotating histograms (the one
// for pass p+1 is cleared during pass p; it was last read in pass p-2, which every warp finished
// before barrier p-1), and EVERY warp scans the 256 bins itself after the pass's barrier, so the
// threshold digit needs no broadcast barrier.  Returns the k-th largest key.
template <int NT, int KPT>
__device__ uint64_t block_kth_largest_regs1(const uint64_t (&keys)[KPT], int n, int k, SelectSmem& ss) {
  static_assert(NT == 1024, "one warp per lane of the per-warp scans");
  const int lane = threadIdx.x & 31;
  if (threadIdx.x < 256) ss.hist3[0][threadIdx.x] = 0;
  __syncthreads();
  uint64_t prefix = 0, mask = 0;
  int krem = k;
  for (int p = 0, shift = 56; shift >= 0; ++p, shift -= 8) {
    int* h = ss.hist3[p % 3];
    if (threadIdx.x < 256) ss.hist3[(p + 1) % 3][threadIdx.x] = 0;
#pragma unroll
    for (int u = 0; u < KPT; ++u) {
      const int i = threadIdx.x + NT * u;
      const bool in = i < n && (keys[u] & mask) == prefix;
      if (p == 0) {  // the top byte (sign + exponent bits): few distinct digits per warp -> aggregate
        const unsigned act = __ballot_sync(0xffffffffu, in);
        if (in) {
          const unsigned dig = (unsigned)(keys[u] >> shift) & 255u;
          const unsigned peers = __match_any_sync(act, dig);
          if (lane == __ffs(peers) - 1) atomicAdd(&h[dig], __popc(peers));
        }
      } else if (in) {  // mantissa bytes: digits nearly distinct in a warp -> one atomic per key
        atomicAdd(&h[(unsigned)(keys[u] >> shift) & 255u], 1);
      }
    }
    __syncthreads();
    // lane l owns bins [248 - 8l, 256 - 8l), read as two 16-byte vectors (no bank conflicts),
    // cnt[j] = bin 255 - 8l - j (descending)
    const int4 lo = *reinterpret_cast<const int4*>(h + 248 - 8 * lane);
    const int4 hi = *reinterpret_cast<const int4*>(h + 252 - 8 * lane);
    const int cnt[8] = {hi.w, hi.z, hi.y, hi.x, lo.w, lo.z, lo.y, lo.x};
    const int tot = (cnt[0] + cnt[1] + cnt[2] + cnt[3]) + (cnt[4] + cnt[5] + cnt[6] + cnt[7]);
    int incl = tot;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += y;
    }
    const int excl = incl - tot;
    const unsigned bal = __ballot_sync(0xffffffffu, excl < krem && incl >= krem);
    const int src = __ffs(bal) - 1;
    int sel = 0, knew = 0, done = 0;
    if (lane == src) {
      int cum = excl;
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        if (cum + cnt[j] >= krem) {
          sel = 255 - 8 * lane - j;
          knew = krem - cum;
          done = cnt[j] == krem - cum;
          break;
        }
        cum += cnt[j];
      }
    }
    sel = __shfl_sync(0xffffffffu, sel, src);
    knew = __shfl_sync(0xffffffffu, knew, src);
    done = __shfl_sync(0xffffffffu, done, src);
    dtl_mark(10 + p);  // tuning build: end of radix pass p
    prefix |= (uint64_t)sel << shift;
    mask |= (uint64_t)255u << shift;
    krem = knew;
    if (done) break;  // uniform across the block: every warp computed the same histogram scan
  }
  return prefix;
}

// Ascending compaction of the keys >= T held in registers (slot u of thread t = index t + NT*u)
// with one barrier: warp ballots give in-warp positions, per-(slot, warp) counts go to shared
// memory, and every warp derives its block offsets from them.  Returns the number written.
template <int NT, int KPT, typename Emit>
__device__ int block_compact_regs1(const uint64_t (&keys)[KPT], int n, uint64_t T, SelectSmem& ss, Emit emit) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  bool f[KPT];
  int pos[KPT];
#pragma unroll
  for (int u = 0; u < KPT; ++u) {
    f[u] = (threadIdx.x + NT * u < n) && keys[u] >= T;
    const unsigned b = __ballot_sync(0xffffffffu, f[u]);
    pos[u] = __popc(b & ((1u << lane) - 1u));
    if (lane == 0) ss.wc[u][wid] = __popc(b);
  }
  __syncthreads();
  int base = 0;
#pragma unroll
  for (int u = 0; u < KPT; ++u) {
    const int v = ss.wc[u][lane];
    int incl = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += y;
    }
    const int woff = __shfl_sync(0xffffffffu, incl - v, wid);
    const int tot = __shfl_sync(0xffffffffu, incl, 31);
    if (f[u]) emit(base + woff + pos[u], threadIdx.x + NT * u, keys[u]);
    base += tot;
  }
  return base;
}

// Apart is read with ld.global.cg: in the fused kernel other CTAs of the same grid wrote it.
template <int NT, int KPT>
__device__ void topk_body(float* __restrict__ A, const float* __restrict__ Apart, int nparts, int m, int k,
                          int id_offset, int id_mul, int32_t* __restrict__ ids, uint64_t* __restrict__ cand, int n_cand_out,
                          int32_t* __restrict__ n_out, SelectSmem& ss, float* As = nullptr, int32_t* ids_s = nullptr) {
  uint64_t key[KPT];
#pragma unroll
  for (int u = 0; u < KPT; ++u) {
    const int j = threadIdx.x + NT * u;
    key[u] = 0ull;
    if (j < m) {
      float a;
      if (Apart) {  // A_j = sum over KV heads of the chunk-sum partials, fixed order
        a = 0.f;
        for (int h = 0; h < nparts; ++h) a += __ldcg(Apart + (size_t)h * m + j);
        if (A) A[j] = a;  // (null: a private copy of the select, topk_plan2_kernel's CTA 1)
        if (As) As[j] = a;  // shared-memory copy for a planner in the same CTA
      } else {
        a = A[j];
      }
      key[u] = ((uint64_t)__float_as_uint(a) << 32) | (uint64_t)(0xFFFFFFFFu - (uint32_t)(j * id_mul + id_offset));
    }
  }
  dtl_mark(4);
  const int kk = min(k, m);
  const uint64_t T = block_kth_largest_regs1<NT, KPT>(key, m, kk, ss);
  dtl_mark(5);
  // ascending compaction
  const int base = block_compact_regs1<NT, KPT>(key, m, T, ss, [&](int pos, int j, uint64_t kv) {
    if (ids) ids[pos] = j * id_mul + id_offset;
    if (ids_s) ids_s[pos] = j * id_mul + id_offset;
    if (cand) cand[pos] = kv;
  });
  if (cand)
    for (int t = kk + threadIdx.x; t < n_cand_out; t += NT) cand[t] = 0ull;
  if (n_out && threadIdx.x == 0) *n_out = base;
}

}  // namespace ckv
