// Shared device helpers for the volume-term kernels.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "lfb_volume.h"

namespace lfb {

// Point-wise physics of Euler set 2C (reference oracle
// lf/bench/reference.py:15-33, Fortran lf/bench/data/volume.f90:29-52).
//
// The contravariant flux of field b along reference direction dir is
//   F_dir,b = sum_a g(a,dir) f_ab
// and with V_dir = sum_a g(a,dir) U_a (contravariant momentum) it factors as
//   b = 0      : V_dir
//   b = 1..3   : V_dir * (U_b / rho) + g(b,dir) * p
//   b = 4..7   : V_dir * (q_b / rho)
// which is the same sum regrouped (fp64 rounding differences ~1e-16 relative,
// far inside the 1e-12 parity bound).

__device__ __forceinline__ double pressure(double th, double p0, double R,
                                           double gam) {
  return p0 * pow(R * th / p0, gam);
}
__device__ __forceinline__ float pressure(float th, float p0, float R,
                                          float gam) {
  return p0 * powf(R * th / p0, gam);
}

__device__ __forceinline__ double recip(double x) { return 1.0 / x; }
__device__ __forceinline__ float recip(float x) { return 1.0f / x; }

template <typename T>
__device__ __forceinline__ bool aligned_to(const void *p) {
  return (reinterpret_cast<uintptr_t>(p) % sizeof(T)) == 0;
}

}  // namespace lfb

// Launch helpers return these codes (see include/lfb_volume.h).
#define LFB_CHECK_LAUNCH()                                   \
  do {                                                       \
    cudaError_t _e = cudaGetLastError();                     \
    if (_e != cudaSuccess) return LFB_ERR_LAUNCH;            \
  } while (0)
