// Fused device-side exchange kernels and stream waits (xchg.cuh).
//   put_signal_kernel  broadcast a small local buffer (row normalisers, candidates) into slot
//                      `self` of every rank's window, then bump counter `flag` in every window
//   merge_slice_kernel LSE-merge the W partial outputs of this rank's row slice (read from the
//                      own window) and broadcast the merged rows (caller dtype) into every
//                      rank's output image: the reduce-scatter + all-gather of the PAPER.md:99
//                      softmax split over shards
//   xchg_wait          stream memory operation: wait until own counter >= W, re-arm to 0
#include <cuda.h>

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

using PFN_wait32 = CUresult (*)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
using PFN_write32 = CUresult (*)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);

template <typename F>
F driver_fn(const char* name) {
  void* p = nullptr;
  cudaDriverEntryPointQueryResult q;
  if (cudaGetDriverEntryPoint(name, &p, cudaEnableDefault, &q) != cudaSuccess || q != cudaDriverEntryPointSuccess)
    return nullptr;
  return reinterpret_cast<F>(p);
}

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
  static PFN_wait32 wait = driver_fn<PFN_wait32>("cuStreamWaitValue32");
  static PFN_write32 write = driver_fn<PFN_write32>("cuStreamWriteValue32");
  if (!wait || !write) return cudaErrorNotSupported;
  const CUdeviceptr a = reinterpret_cast<CUdeviceptr>(flag_dev);
  if (wait(reinterpret_cast<CUstream>(st), a, target, CU_STREAM_WAIT_VALUE_GEQ) != CUDA_SUCCESS)
    return cudaErrorUnknown;
  if (write(reinterpret_cast<CUstream>(st), a, 0u, CU_STREAM_WRITE_VALUE_DEFAULT) != CUDA_SUCCESS)
    return cudaErrorUnknown;
  pdl_mark_event_wait(st);  // the next kernel must not launch programmatically across the wait
  return cudaSuccess;
}

}  // namespace ckv
