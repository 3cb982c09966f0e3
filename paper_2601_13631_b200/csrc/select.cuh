// Single-CTA radix select and block scan used by top-k (A3) and the cache planner (A4).
#pragma once
#include "common.cuh"

namespace ckv {

struct SelectSmem {
  int hist[256];
  int warp_tot[32];
  int state[3];
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
// Apart is read with ld.global.cg: in the fused kernel other CTAs of the same grid wrote it.
template <int NT, int KPT>
__device__ void topk_body(float* __restrict__ A, const float* __restrict__ Apart, int nparts, int m, int k,
                          int id_offset, int id_mul, int32_t* __restrict__ ids, uint64_t* __restrict__ cand, int n_cand_out,
                          int32_t* __restrict__ n_out, SelectSmem& ss) {
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
        A[j] = a;
      } else {
        a = A[j];
      }
      key[u] = ((uint64_t)__float_as_uint(a) << 32) | (uint64_t)(0xFFFFFFFFu - (uint32_t)(j * id_mul + id_offset));
    }
  }
  const int kk = min(k, m);
  const uint64_t T = block_kth_largest_regs<NT, KPT>(key, m, kk, ss);
  // ascending compaction
  int base = 0;
#pragma unroll
  for (int u = 0; u < KPT; ++u) {
    if (NT * u >= m) break;
    const int j = threadIdx.x + NT * u;
    const bool f = (j < m) && key[u] >= T;
    int tot;
    const int pos = block_excl_scan<NT>(f ? 1 : 0, tot, ss);
    if (f) {
      if (ids) ids[base + pos] = j * id_mul + id_offset;
      if (cand) cand[base + pos] = key[u];
    }
    base += tot;
  }
  if (cand)
    for (int t = kk + threadIdx.x; t < n_cand_out; t += NT) cand[t] = 0ull;
  if (n_out && threadIdx.x == 0) *n_out = base;
}

}  // namespace ckv
