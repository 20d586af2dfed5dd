// LFB_VARIANT_FUSED — production kernel (placeholder until implemented).
#include "lfb_common.cuh"

namespace lfb {

bool fused_available(int, int) { return false; }

int volume_fused_f64(int, int64_t, double, double, double, const double *,
                     double *, const double *, const double *, const double *,
                     cudaStream_t) {
  return LFB_ERR_BAD_VARIANT;
}

int volume_fused_f32(int, int64_t, float, float, float, const float *, float *,
                     const float *, const float *, const float *, cudaStream_t) {
  return LFB_ERR_BAD_VARIANT;
}

}  // namespace lfb
