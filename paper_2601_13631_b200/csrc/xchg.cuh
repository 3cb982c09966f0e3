// Fused device-side exchange of the position-sharded path (
// include/ckv.h "fused device-side exchange").
//
// Every rank owns one exchange WINDOW in device memory with the same layout on every rank.
// Producers write their results straight into the peers' windows (NVLink stores on a
// multi-GPU node, plain stores for logical ranks on one GPU) and then increment one counter
// per exchange in every peer's window with a system-scope release; the consumer's stream
// waits for its own counter to reach W with a stream memory operation and re-arms it to 0.
//
// Re-arming is race-free because the exchanges of a layer form a chain: a rank re-arms
// counter x right after its wait and, in stream order, before it signals exchange x+1; a
// peer can only reach its next signal of counter x after it has observed that later signal.
#pragma once
#include <cstddef>
#include <cstdint>

namespace ckv {

constexpr int kMaxPeers = 8;
enum { XF_LAM = 0, XF_CAND = 1, XF_PART = 2, XF_OUT = 3, XF_COUNT = 4 };

// Byte offsets inside a window (identical on every rank of a group).
struct XLayout {
  size_t flags;     // uint32 [XF_COUNT] (padded)
  size_t lam;       // float  [W][Hq * max_ns]: slot g = rank g's row normalisers (log2)
  size_t cand;      // uint64 [W][k]: slot g = rank g's candidates
  size_t part_o;    // float  [W][rps_max][d]: slot g = rank g's partial rows of MY slice
  size_t part_lse;  // float  [W][rps_max]: their natural-log LSE (-inf: no key on rank g)
  size_t outs;      // cfg.dtype [max_ns * Hq][d]: the merged output, slice s written by rank s
  size_t total;
  int lam_stride;   // floats per lam slot (Hq * max_ns)
  int rps_max;      // rows per slice at max_ns: ceil(max_ns * Hq / W)
};

inline size_t xalign(size_t x) { return (x + 255) & ~size_t(255); }

inline XLayout make_xlayout(int W, int Hq, int max_ns, int k, int d, int esz) {
  XLayout L;
  L.lam_stride = Hq * max_ns;
  L.rps_max = (max_ns * Hq + W - 1) / W;
  size_t o = 0;
  L.flags = o;
  o = xalign(o + sizeof(uint32_t) * XF_COUNT);
  L.lam = o;
  o = xalign(o + sizeof(float) * (size_t)W * L.lam_stride);
  L.cand = o;
  o = xalign(o + sizeof(uint64_t) * (size_t)W * k);
  L.part_o = o;
  o = xalign(o + sizeof(float) * (size_t)W * L.rps_max * d);
  L.part_lse = o;
  o = xalign(o + sizeof(float) * (size_t)W * L.rps_max);
  L.outs = o;
  o = xalign(o + (size_t)esz * max_ns * Hq * d);
  L.total = o;
  return L;
}

// Window bases of all ranks as seen from this process (own window included).
struct XPeers {
  char* base[kMaxPeers];
  int W;
  int self;
};

// Where the partial-output rows of this rank go (the reduce-scatter half of the LSE merge):
// row i of [n_s * Hq] belongs to slice s = i / rps, stored at row i - s * rps of slot `self`
// of rank s's window.
struct XPartDst {
  XPeers xp;
  size_t part_o, part_lse;  // window offsets
  int rps;                  // rows per slice of this call
  int rps_max;              // slot stride (rows)
  int d;
};

#ifdef __CUDACC__
__device__ __forceinline__ void red_release_sys_add(uint32_t* p, uint32_t v) {
  asm volatile("red.release.sys.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
#endif

}  // namespace ckv
