// A4 cache plan (+ fused A9) as a device function of one CTA, shared by the standalone planner
// kernel (k_cache.cu) and the fused chunk-sum -> top-k -> plan kernel (k_reduce.cu).
//
// HBM chunk cache (§4.4, 424-455): per (layer, chunk) the cumulative importance
// I_j and access count F_j live in a table that survives eviction; the
// cache score is S_j = I_j * F_j (Eq. 2).  Selected chunks are checked
// against the cache before loading; misses take free slots first, then the
// slots of the lowest-(S, j) residents that are neither requested nor pinned by an
// in-flight prefetch ("Both heaps will evict low-scored ContiguousChunks").
#pragma once
#include "common.cuh"
#include "select.cuh"

namespace ckv {

__device__ __forceinline__ bool bsearch_ids(const int32_t* ids, int n, int j) {
  int lo = 0, hi = n - 1;
  while (lo <= hi) {
    int mid = (lo + hi) >> 1;
    int v = ids[mid];
    if (v == j) return true;
    if (v < j) lo = mid + 1; else hi = mid - 1;
  }
  return false;
}

constexpr int kPlanKPT = 4;  // victim keys per thread held in registers (P <= 4 * NT)
constexpr int kPlanSmemKeysMax = 24 * 1024;  // larger pools: keys in dynamic shared memory (192 KB)

// Shared-memory copies of one layer's cache tables (the fused top-k / plan kernel, k_cache.cu):
// copied with cp.async while the top-k runs, so the planner's lookups (hit / miss, spec-used, A9
// read-modify-write, free slots, victim candidates) cost no dependent global round trip.  Any
// pointer may be null (read global memory); the planner's writes always go to global memory.
struct PlanTables {
  const int32_t* ids = nullptr;       // [n_ids] the plan's ids (this CTA's top-k output)
  const float* A = nullptr;           // [m_loc] chunk scores (the fused A9's I += A)
  const int32_t* slot_of = nullptr;   // [m_loc]
  const float* I = nullptr;           // [m_loc]
  const int32_t* F = nullptr;         // [m_loc]
  const int32_t* owner = nullptr;     // [P]
  const int32_t* pf_epoch = nullptr;  // [P]
};
__device__ __forceinline__ void cp_async4(void* dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"((uint32_t)__cvta_generic_to_shared(dst)), "l"(src)
               : "memory");
}

struct PlanSmem {
  SelectSmem ss;
  int hits, spec_used;
  uint32_t req_bits[kPlanSmemKeysMax / 32];  // slots holding a requested chunk (pools <= kPlanSmemKeysMax)
};

// The A4 planner (+ fused A9) run by one CTA of NT threads (every thread must call it).
template <int NT>
__device__ void cache_plan_body(const CacheLayer& cl, const int32_t* __restrict__ ids, int n_ids, int prefetch,
                                int quota, int epoch, int64_t rec_bytes, int32_t* __restrict__ scratch,
                                const PlanOut& out, PlanSmem& ps, uint64_t* skeys = nullptr,
                                const PlanTables& tc = PlanTables()) {
  SelectSmem& ss = ps.ss;
  int& s_hits = ps.hits;
  int& s_spec_used = ps.spec_used;
  if (out.epoch_dev) epoch = *out.epoch_dev;
  int32_t* miss = scratch;            // [n_ids]
  int32_t* freel = scratch + n_ids;   // [P]
  int32_t* vict = freel + cl.P;       // [P]
  int32_t* mpos = vict + cl.P;        // [n_ids]: position in ids of each miss
  if (threadIdx.x == 0) { s_hits = 0; s_spec_used = 0; }
  const bool use_bits = cl.P <= kPlanSmemKeysMax;
  if (use_bits)
    for (int w = threadIdx.x; w < (cl.P + 31) / 32; w += NT) ps.req_bits[w] = 0u;
  __syncthreads();

  // 1. hit / miss, misses compacted in ascending chunk order.  Hits write their kept slot now;
  //    a miss's position in ids is kept (mpos) so step 4 writes its slot without another lookup.
  //    The A9 update is fused here: it touches only requested chunks, which
  //    are never eviction candidates, so the victims are those of an update after planning.
  int n_miss = 0;
  for (int b = 0; b < n_ids; b += NT) {
    const int t = b + threadIdx.x;
    bool is_miss = false;
    int j = -1;
    if (t < n_ids) {
      j = tc.ids ? tc.ids[t] : ids[t];
      const int s = tc.slot_of ? tc.slot_of[j] : cl.slot_of[j];
      is_miss = s < 0;
      if (!is_miss) {
        atomicAdd(&s_hits, 1);
        if (use_bits) atomicOr(&ps.req_bits[s >> 5], 1u << (s & 31));
        if (!prefetch && (tc.pf_epoch ? tc.pf_epoch[s] : cl.pf_epoch[s]) == epoch) atomicAdd(&s_spec_used, 1);
      }
      if (out.kept_slots) out.kept_slots[t] = s;  // misses: -1 until step 4 assigns a slot
      if (out.ids_out) out.ids_out[t] = j;
      if (out.upd_A) {
        cl.I[j] = (tc.I ? tc.I[j] : cl.I[j]) + (tc.A ? tc.A[j] : out.upd_A[j]);
        cl.F[j] = (tc.F ? tc.F[j] : cl.F[j]) + 1;
        cl.T[j] = epoch;
      }
    }
    int tot;
    const int pos = block_excl_scan<NT>(is_miss ? 1 : 0, tot, ss);
    if (is_miss) {
      miss[n_miss + pos] = j;
      mpos[n_miss + pos] = t;
    }
    n_miss += tot;
  }
  // adaptive speculation: when the previous layer's demand plan missed (almost) nothing, the HBM
  // cache already serves this request and a speculative load would only take link bytes and
  // slots (in a warm multi-request stream only ~3% of them were used); speculate again as soon as
  // the demand misses grow (cold cache, a new topic)
  if (prefetch && out.gate_misses && *out.gate_misses <= out.gate_max) n_miss = 0;
  if (prefetch && n_miss > quota) {
    if (out.rank_keys) {
      // speculation is a bet that layer l+1 reuses layer l's chunks: spend the
      // quota on the misses layer l scored highest (kept in ascending chunk order)
      auto rkey = [&](int t) -> uint64_t { return out.rank_keys[mpos[t]]; };
      const uint64_t T = block_kth_largest<NT>(rkey, n_miss, quota, ss);
      int n2 = 0;
      for (int b = 0; b < n_miss; b += NT) {
        const int t = b + threadIdx.x;
        const bool f = t < n_miss && rkey(t) >= T;
        const int jm = f ? miss[t] : 0, pm = f ? mpos[t] : 0;
        int tot;
        const int pos = block_excl_scan<NT>(f ? 1 : 0, tot, ss);  // barriers: reads precede writes
        if (f) {
          miss[n2 + pos] = jm;
          mpos[n2 + pos] = pm;
        }
        n2 += tot;
      }
      n_miss = n2;
    } else {
      n_miss = quota;
    }
  }
  // 2. free slots, ascending (only needed when something is loaded)
  int n_free = 0;
  if (n_miss > 0)
    for (int b = 0; b < cl.P; b += NT) {
      const int s = b + threadIdx.x;
      const bool f = s < cl.P && (tc.owner ? tc.owner[s] : cl.owner[s]) < 0;
      int tot;
      const int pos = block_excl_scan<NT>(f ? 1 : 0, tot, ss);
      if (f) freel[n_free + pos] = s;
      n_free += tot;
    }
  // 3. victims: the `need` lowest (S, j) evictable residents
  int need = n_miss - n_free;
  int n_vict = 0;
  if (need > 0) {
    auto key = [&](int s) -> uint64_t {
      const int e = tc.owner ? tc.owner[s] : cl.owner[s];  // table index layer * m_loc + j
      if (e < 0) return 0ull;
      if (use_bits) {  // requested by this plan = the slot of a hit (marked in step 1)
        if (ps.req_bits[s >> 5] & (1u << (s & 31))) return 0ull;
      } else {
        const int jl = e - cl.lbase;
        if (jl >= 0 && jl < cl.m_loc && bsearch_ids(ids, n_ids, jl)) return 0ull;
      }
      if (!prefetch && (tc.pf_epoch ? tc.pf_epoch[s] : cl.pf_epoch[s]) == epoch) return 0ull;
      // Eq. 2 by default; the ablation policies of PAPER.md:610-613.  Ties by
      // (S, layer, j) = (S, e)
      // (I, F of this layer's residents from the shared-memory copies when present: per-layer pools
      // hold this layer's chunks only, and the fused A9 touches requested chunks, never candidates)
      const int jl = e - cl.lbase;
      const bool tl = tc.I && jl >= 0 && jl < cl.m_loc;
      const float I = tl ? tc.I[jl] : cl.I0[e];
      const int F = tl ? tc.F[jl] : cl.F0[e];
      const float S = cl.policy == 0 ? I * (float)F : cl.policy == 1 ? (float)F : (float)cl.T0[e];
      return ~(((uint64_t)__float_as_uint(S) << 32) | (uint64_t)(uint32_t)e);
    };
    if (cl.P <= NT * kPlanKPT) {
      // keys evaluated once into registers (slot s = threadIdx.x + NT*u): the radix passes then
      // cost no memory traffic (integer LFU / LRU scores tie a lot and run all 8 passes)
      uint64_t kr[kPlanKPT];
      int ev = 0;
#pragma unroll
      for (int u = 0; u < kPlanKPT; ++u) {
        const int s = threadIdx.x + NT * u;
        kr[u] = s < cl.P ? key(s) : 0ull;
        ev += kr[u] != 0ull;
      }
      int n_evictable;
      block_excl_scan<NT>(ev, n_evictable, ss);
      if (need > n_evictable) {  // capacity guard (cannot trigger when P >= k + quota): loud, not a crash
        if (threadIdx.x == 0 && out.stats) out.stats[15] = 1;
        need = n_evictable;
        n_miss = n_free + need;
      }
      const uint64_t T = need > 0 ? block_kth_largest_regs<NT, kPlanKPT>(kr, cl.P, need, ss) : ~0ull;
#pragma unroll
      for (int u = 0; u < kPlanKPT; ++u) {
        if (NT * u >= cl.P) break;
        const bool f = kr[u] != 0ull && kr[u] >= T;
        int tot;
        const int pos = block_excl_scan<NT>(f ? 1 : 0, tot, ss);
        if (f) vict[n_vict + pos] = threadIdx.x + NT * u;
        n_vict += tot;
      }
    } else if (skeys) {
      // large pools (global heap): keys evaluated once into shared memory, passes read them there
      int ev = 0;
      for (int s = threadIdx.x; s < cl.P; s += NT) {
        const uint64_t kv = key(s);
        skeys[s] = kv;
        ev += kv != 0ull;
      }
      int n_evictable;
      block_excl_scan<NT>(ev, n_evictable, ss);  // its barriers also publish skeys
      if (need > n_evictable) {
        if (threadIdx.x == 0 && out.stats) out.stats[15] = 1;
        need = n_evictable;
        n_miss = n_free + need;
      }
      auto skey = [&](int s) -> uint64_t { return skeys[s]; };
      const uint64_t T = need > 0 ? block_kth_largest<NT>(skey, cl.P, need, ss) : ~0ull;
      for (int b = 0; b < cl.P; b += NT) {
        const int s = b + threadIdx.x;
        const uint64_t kv = s < cl.P ? skeys[s] : 0ull;
        const bool f = kv != 0ull && kv >= T;
        int tot;
        const int pos = block_excl_scan<NT>(f ? 1 : 0, tot, ss);
        if (f) vict[n_vict + pos] = s;
        n_vict += tot;
      }
    } else {
      int n_evictable = 0;
      for (int b = 0; b < cl.P; b += NT) {
        const int s = b + threadIdx.x;
        int tot;
        block_excl_scan<NT>((s < cl.P && key(s) != 0ull) ? 1 : 0, tot, ss);
        n_evictable += tot;
      }
      if (need > n_evictable) {
        if (threadIdx.x == 0 && out.stats) out.stats[15] = 1;
        need = n_evictable;
        n_miss = n_free + need;
      }
      const uint64_t T = need > 0 ? block_kth_largest<NT>(key, cl.P, need, ss) : ~0ull;
      for (int b = 0; b < cl.P; b += NT) {
        const int s = b + threadIdx.x;
        uint64_t kv = 0ull;
        if (s < cl.P) kv = key(s);
        const bool f = kv != 0ull && kv >= T;
        int tot;
        const int pos = block_excl_scan<NT>(f ? 1 : 0, tot, ss);
        if (f) vict[n_vict + pos] = s;
        n_vict += tot;
      }
    }
    __syncthreads();
    for (int t = threadIdx.x; t < n_vict; t += NT) {
      const int s = vict[t];
      const int e = tc.owner ? tc.owner[s] : cl.owner[s];
      if (out.victims) out.victims[t] = e;
      cl.slot_of0[e] = -1;
      cl.owner[s] = -1;
    }
  }
  __syncthreads();
  // 4. assign slots to misses: free slots, then victim slots (both ascending)
  for (int t = threadIdx.x; t < n_miss; t += NT) {
    const int s = (t < n_free) ? freel[t] : vict[t - n_free];
    const int j = miss[t];
    cl.slot_of[j] = s;
    cl.owner[s] = cl.lbase + j;
    cl.pf_epoch[s] = prefetch ? epoch : -1;
    out.gather_list[2 * t] = j;
    out.gather_list[2 * t + 1] = s;
    if (out.kept_slots) out.kept_slots[mpos[t]] = out.mark_miss ? -(s + 2) : s;
  }
  if (threadIdx.x == 0) {
    *out.n_load = n_miss;
    if (out.counts) {
      out.counts[0] = s_hits;
      out.counts[1] = n_miss;
      out.counts[2] = n_vict;
      out.counts[3] = s_spec_used;
    }
    if (out.stats) {
      unsigned long long* st = reinterpret_cast<unsigned long long*>(out.stats);
      if (prefetch) {
        atomicAdd(st + 2, (unsigned long long)n_miss);
        atomicAdd(st + 5, (unsigned long long)((int64_t)n_miss * rec_bytes));
      } else {
        atomicAdd(st + 0, (unsigned long long)s_hits);
        atomicAdd(st + 1, (unsigned long long)n_miss);
        atomicAdd(st + 3, (unsigned long long)s_spec_used);
        atomicAdd(st + 4, (unsigned long long)((int64_t)n_miss * rec_bytes));
        atomicAdd(st + 6, 1ull);
      }
    }
  }
}

}  // namespace ckv
