// Fused device-side exchange kernels and stream waits (xchg.cuh).
//   put_signal_kernel  broadcast a small local buffer (row normalisers, candidates) into slot
//                      `self` of every rank's window, then bump counter `flag` in every window
//   merge_slice_kernel LSE-merge the W partial outputs of this rank's row slice (read from the
//                      own window) and broadcast the merged rows (caller dtype) into every
//                      rank's output image: the reduce-scatter + all-gather of the PAPER.md:99
//                      softmax split over shards
//   wait_reset_kernel  one thread waits (acquire) until the own counter reaches W, re-arms it
//                      (one warp of one SM while waiting; as an ordinary kernel node the whole
//                      exchange stays PDL-ordered and capturable in a CUDA graph)
#include "common.cuh"
#include "xchg.cuh"

namespace ckv {
namespace {

constexpr int kPutThreads = 1024;

// One CTA: its stores precede (barrier + system fence) the counter increments of thread 0.
// With programmatic launch, griddepcontrol.wait makes the producing kernel's writes (including
// its own peer stores) visible first.
__global__ void __launch_bounds__(kPutThreads) put_signal_kernel(XPeers xp, const uint32_t* __restrict__ src,
                                                                 int n_words, size_t dst_off, size_t flag_off) {
  pdl_wait();
  pdl_trigger();
  for (int g = 0; g < xp.W; ++g) {
    uint32_t* dst = reinterpret_cast<uint32_t*>(xp.base[g] + dst_off);
    for (int i = threadIdx.x; i < n_words; i += kPutThreads) dst[i] = src[i];
  }
  __threadfence_system();
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence_system();
    for (int g = 0; g < xp.W; ++g) red_release_sys_add(reinterpret_cast<uint32_t*>(xp.base[g] + flag_off), 1u);
  }
}

// One warp per row of this rank's slice: rows [self * rps, min((self + 1) * rps, N)) of the
// [n_s * Hq] output rows.  Rank g's partial (normalised O_g, natural-log lse_g) sits in slot g
// of the own window; O = sum_g e^(lse_g - M) O_g / sum_g e^(lse_g - M) (ranks in order).
template <typename T>
__global__ void __launch_bounds__(256) merge_slice_kernel(XPeers xp, XLayout xl, int N, int rps, int d) {
  pdl_wait();
  pdl_trigger();
  const int lane = threadIdx.x & 31;
  const int lr = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;  // row inside the slice
  const int row = xp.self * rps + lr;
  if (lr >= rps || row >= N) return;
  const char* own = xp.base[xp.self];
  const float* lse = reinterpret_cast<const float*>(own + xl.part_lse);
  const float* po = reinterpret_cast<const float*>(own + xl.part_o);
  const float lg = lane < xp.W ? lse[(size_t)lane * xl.rps_max + lr] : -INFINITY;
  float M = lg;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) M = fmaxf(M, __shfl_xor_sync(0xffffffffu, M, o));
  const float w = (lg == -INFINITY) ? 0.f : __expf(lg - M);
  float den = w;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) den += __shfl_xor_sync(0xffffffffu, den, o);
  const float inv = den > 0.f ? 1.f / den : 0.f;
  for (int x = lane; x < d; x += 32) {
    float acc = 0.f;
    for (int g = 0; g < xp.W; ++g) {
      const float wg = __shfl_sync(0xffffffffu, w, g);
      if (wg != 0.f) acc += wg * po[((size_t)g * xl.rps_max + lr) * d + x];
    }
    const T v = from_f<T>(acc * inv);
    for (int g = 0; g < xp.W; ++g) reinterpret_cast<T*>(xp.base[g] + xl.outs)[(size_t)row * d + x] = v;
  }
}

// One thread spins (acquire, system scope) until this rank's counter reaches `target` -- all W
// ranks have published -- then re-arms it.  It does not trigger its dependents early: the next
// kernel starts only once the wait is over (and its griddepcontrol.wait sees the data).
__global__ void wait_reset_kernel(uint32_t* flag, uint32_t target) {
  pdl_wait();
  if (threadIdx.x == 0) {
    uint32_t v;
    int ns = 32;
    for (;;) {
      asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(flag) : "memory");
      if (v >= target) break;
      __nanosleep(ns);
      if (ns < 256) ns *= 2;
    }
    *flag = 0u;
    __threadfence_system();
  }
}

const int kReg = register_kernels({(const void*)put_signal_kernel, (const void*)merge_slice_kernel<float>,
                                   (const void*)merge_slice_kernel<__nv_bfloat16>, (const void*)wait_reset_kernel});

}  // namespace

cudaError_t launch_xchg_put(const XPeers& xp, const void* src, size_t bytes, size_t dst_off, size_t flag_off,
                            cudaStream_t st) {
  if (bytes % 4) return cudaErrorInvalidValue;
  if (cudaError_t e = launch_kernel(put_signal_kernel, 1, kPutThreads, 0, st, xp,
                                    static_cast<const uint32_t*>(src), (int)(bytes / 4), dst_off, flag_off))
    return e;
  return cudaGetLastError();
}

template <typename T>
cudaError_t launch_xchg_merge(const XPeers& xp, const XLayout& xl, int N, int rps, int d, cudaStream_t st) {
  const int blocks = (rps * 32 + 255) / 256;
  if (cudaError_t e = launch_kernel(merge_slice_kernel<T>, blocks > 0 ? blocks : 1, 256, 0, st, xp, xl, N, rps, d))
    return e;
  return cudaGetLastError();
}
template cudaError_t launch_xchg_merge<float>(const XPeers&, const XLayout&, int, int, int, cudaStream_t);
template cudaError_t launch_xchg_merge<__nv_bfloat16>(const XPeers&, const XLayout&, int, int, int, cudaStream_t);

cudaError_t xchg_wait(cudaStream_t st, void* flag_dev, uint32_t target) {
  if (cudaError_t e = launch_kernel(wait_reset_kernel, 1, 32, 0, st, static_cast<uint32_t*>(flag_dev), target))
    return e;
  return cudaGetLastError();
}

}  // namespace ckv
