// A3 top-k (exact radix select, lowest-index tie-break, ascending ids) and the
// candidate merge of the position-sharded path.
//
// Keys are 64-bit composites (float bits of A_j << 32) | (0xFFFFFFFF - j): A_j >= 0 so the
// float bit pattern orders like the value, and the index part makes every key unique
// (larger key = larger score, then lower index), so exactly k keys are >= the k-th
// largest key T.  T is found by eight 8-bit MSB-first histogram passes in one CTA.
#include "common.cuh"
#include "select.cuh"

namespace ckv {
namespace {

constexpr int NT = 1024;

template <int KPT>
__global__ void __launch_bounds__(NT) topk_scores_kernel(float* __restrict__ A, const float* __restrict__ Apart,
                                                         int nparts, int m, int k, int id_offset, int id_mul,
                                                         int32_t* __restrict__ ids, uint64_t* __restrict__ cand,
                                                         int n_cand_out, int32_t* __restrict__ n_out) {
  pdl_wait();
  pdl_trigger();
  __shared__ SelectSmem ss;
  topk_body<NT, KPT>(A, Apart, nparts, m, k, id_offset, id_mul, ids, cand, n_cand_out, n_out, ss);
}

// Large m (> NT * 8 chunks): keys re-read from A every pass.
__global__ void __launch_bounds__(NT) topk_scores_big_kernel(float* __restrict__ A, const float* __restrict__ Apart,
                                                             int nparts, int m, int k, int id_offset, int id_mul,
                                                             int32_t* __restrict__ ids, uint64_t* __restrict__ cand,
                                                             int n_cand_out, int32_t* __restrict__ n_out) {
  pdl_wait();
  pdl_trigger();
  __shared__ SelectSmem ss;
  if (Apart) {  // A_j = sum over KV heads of the chunk-sum partials, fixed order
    for (int j = threadIdx.x; j < m; j += NT) {
      float a = 0.f;
      for (int h = 0; h < nparts; ++h) a += Apart[(size_t)h * m + j];
      A[j] = a;
    }
    __syncthreads();
  }
  auto key = [&](int j) -> uint64_t {
    return ((uint64_t)__float_as_uint(A[j]) << 32) | (uint64_t)(0xFFFFFFFFu - (uint32_t)(j * id_mul + id_offset));
  };
  const int kk = min(k, m);
  const uint64_t T = block_kth_largest<NT>(key, m, kk, ss);
  int base = 0;
  for (int j0 = 0; j0 < m; j0 += NT) {
    const int j = j0 + threadIdx.x;
    const bool f = (j < m) && key(j) >= T;
    int tot;
    const int pos = block_excl_scan<NT>(f ? 1 : 0, tot, ss);
    if (f) {
      if (ids) ids[base + pos] = j * id_mul + id_offset;
      if (cand) cand[base + pos] = key(j);
    }
    base += tot;
  }
  if (cand)
    for (int t = kk + threadIdx.x; t < n_cand_out; t += NT) cand[t] = 0ull;
  if (n_out && threadIdx.x == 0) *n_out = base;
}

// Global top-k over the gathered candidates of all shards; ids_glob ascending (identical
// on every rank), ids_local = the selected ids this shard owns, as local chunk indices.
__global__ void __launch_bounds__(NT) topk_merge_kernel(const uint64_t* __restrict__ cand_all, int n_cand, int k,
                                                        int m_glob, int j0, int j1, int cyc_W,
                                                        int32_t* __restrict__ flag,
                                                        int32_t* __restrict__ ids_glob, int32_t* __restrict__ ids_local,
                                                        int32_t* __restrict__ n_local) {
  pdl_wait();
  pdl_trigger();
  __shared__ SelectSmem ss;
  for (int j = threadIdx.x; j < m_glob; j += NT) flag[j] = 0;
  auto key = [&](int i) -> uint64_t { return cand_all[i]; };
  const uint64_t T = block_kth_largest<NT>(key, n_cand, k, ss);
  __syncthreads();
  for (int i = threadIdx.x; i < n_cand; i += NT) {
    const uint64_t kv = cand_all[i];
    if (kv != 0ull && kv >= T) flag[0xFFFFFFFFu - (uint32_t)(kv & 0xFFFFFFFFull)] = 1;
  }
  __syncthreads();
  int base = 0, lbase = 0;
  for (int jb = 0; jb < m_glob; jb += NT) {
    const int j = jb + threadIdx.x;
    const bool f = (j < m_glob) && flag[j];
    int tot;
    const int pos = block_excl_scan<NT>(f ? 1 : 0, tot, ss);
    if (f) ids_glob[base + pos] = j;
    base += tot;
    // owned by this shard: [j0, j1) (contiguous) or j % cyc_W == j0 (cyclic; local id j / cyc_W)
    const bool fl = f && (cyc_W > 0 ? (j % cyc_W) == j0 : (j >= j0 && j < j1));
    int ltot;
    const int lpos = block_excl_scan<NT>(fl ? 1 : 0, ltot, ss);
    if (fl) ids_local[lbase + lpos] = cyc_W > 0 ? j / cyc_W : j - j0;
    lbase += ltot;
  }
  if (threadIdx.x == 0) *n_local = lbase;
}

// NEXT-4 granularity accounting: the ascending ids of the B-token
// blocks of a coarse block store that hold at least one token of the selected u-token units
// (ids ascending; unit j = tokens [j*u, min((j+1)*u, n))).  Because the ids ascend, the block
// range of unit t only has to be clipped against the last block of unit t-1 to stay unique.
__global__ void __launch_bounds__(NT) block_cover_kernel(const int32_t* __restrict__ ids, int n_ids, int u, int B,
                                                         int64_t n, int32_t* __restrict__ blocks,
                                                         int32_t* __restrict__ n_blocks) {
  pdl_wait();
  pdl_trigger();
  __shared__ SelectSmem ss;
  auto last_block = [&](int j) -> int64_t { return (min((int64_t)(j + 1) * u, n) - 1) / B; };
  int base = 0;
  for (int t0 = 0; t0 < n_ids; t0 += NT) {
    const int t = t0 + threadIdx.x;
    int64_t start = 0, nb = 0;
    if (t < n_ids) {
      const int j = ids[t];
      start = (int64_t)j * u / B;
      if (t > 0) start = max(start, last_block(ids[t - 1]) + 1);
      nb = max((int64_t)0, last_block(j) - start + 1);
    }
    int tot;
    const int pos = block_excl_scan<NT>((int)nb, tot, ss);
    for (int i = 0; i < (int)nb; ++i) blocks[base + pos + i] = (int32_t)(start + i);
    base += tot;
  }
  if (threadIdx.x == 0) *n_blocks = base;
}

const int kReg = register_kernels({(const void*)topk_scores_kernel<1>, (const void*)topk_scores_kernel<2>,
                                   (const void*)topk_scores_kernel<4>, (const void*)topk_scores_kernel<8>,
                                   (const void*)topk_scores_big_kernel, (const void*)topk_merge_kernel,
                                   (const void*)block_cover_kernel});

}  // namespace

cudaError_t launch_block_cover(const int32_t* ids, int n_ids, int u, int B, int64_t n, int32_t* blocks,
                               int32_t* n_blocks, cudaStream_t st) {
  if (cudaError_t e_ = launch_kernel(block_cover_kernel, 1, NT, 0, st, ids, n_ids, u, B, n, blocks, n_blocks)) return e_;
  return cudaGetLastError();
}

cudaError_t launch_topk_scores(float* A, const float* Apart, int nparts, int m, int k, int id_offset, int id_mul, int32_t* ids,
                               uint64_t* cand_out, int n_cand_out, int32_t* n_out, cudaStream_t st) {
  cudaError_t e_;
  if (m <= NT)
    e_ = launch_kernel(topk_scores_kernel<1>, 1, NT, 0, st, A, Apart, nparts, m, k, id_offset, id_mul, ids, cand_out, n_cand_out, n_out);
  else if (m <= 2 * NT)
    e_ = launch_kernel(topk_scores_kernel<2>, 1, NT, 0, st, A, Apart, nparts, m, k, id_offset, id_mul, ids, cand_out, n_cand_out, n_out);
  else if (m <= 4 * NT)
    e_ = launch_kernel(topk_scores_kernel<4>, 1, NT, 0, st, A, Apart, nparts, m, k, id_offset, id_mul, ids, cand_out, n_cand_out, n_out);
  else if (m <= 8 * NT)
    e_ = launch_kernel(topk_scores_kernel<8>, 1, NT, 0, st, A, Apart, nparts, m, k, id_offset, id_mul, ids, cand_out, n_cand_out, n_out);
  else
    e_ = launch_kernel(topk_scores_big_kernel, 1, NT, 0, st, A, Apart, nparts, m, k, id_offset, id_mul, ids, cand_out, n_cand_out, n_out);
  if (e_) return e_;
  return cudaGetLastError();
}

cudaError_t launch_topk_merge(const uint64_t* cand_all, int n_cand, int k, int m_glob, int j0, int j1, int cyc_W,
                              int32_t* flag_scratch, int32_t* ids_glob, int32_t* ids_local, int32_t* n_local,
                              cudaStream_t st) {
  if (cudaError_t e_ = launch_kernel(topk_merge_kernel, 1, NT, 0, st, cand_all, n_cand, k, m_glob, j0, j1, cyc_W, flag_scratch, ids_glob, ids_local,
                                      n_local)) return e_;
  return cudaGetLastError();
}

}  // namespace ckv
