// A1 score-partial on tcgen05 (placeholder until the tensor-core kernel lands).
#include "common.cuh"
namespace ckv {
int score_tc_nsplit(const LayerGeom&) { return 0; }
cudaError_t launch_score_tc(const LayerGeom&, const __nv_bfloat16*, const __nv_bfloat16*, float*, float*, int, void*,
                            cudaStream_t) {
  return cudaErrorNotSupported;
}
}  // namespace ckv
