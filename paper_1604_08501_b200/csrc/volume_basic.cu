// LFB_VARIANT_BASIC — the straightforward fused volume kernel.
//
// Structure of the reference's level-3..5 OpenCL kernel (lanes = (i, j),
// sequential k per lane, one work-group per element; lf/bench/recipes.py:30-94):
//   * one thread per (i, j) column of an element, EPB elements per CTA;
//   * per field b: every thread computes the r/s/t contravariant fluxes of
//     its column, parks F_r and F_s in shared memory, keeps F_t in
//     registers (the t-line is the thread's own column), then after one
//     barrier contracts all three with D and updates rhsq += Jinv * sum.
//   * point-wise quantities (1/rho, p, V) are recomputed per field from
//     global memory (L1/L2 hits after the first field).
// Generic in Nq (1..16) and dtype; it is the parity workhorse for small
// Nq and the baseline rung of the variant ladder.

#include "lfb_common.cuh"

namespace lfb {
namespace {

template <typename T, int NQ>
__device__ __forceinline__ void field_flux(int b, int pt, const T *__restrict__ qe,
                                           const T *__restrict__ ge, T p0, T R,
                                           T gam, T &Fr, T &Fs, T &Ft) {
  constexpr int NPT = NQ * NQ * NQ;
  const T rho = qe[pt];
  const T u1 = qe[1 * NPT + pt], u2 = qe[2 * NPT + pt], u3 = qe[3 * NPT + pt];
  T V[3];
#pragma unroll
  for (int d = 0; d < 3; ++d)
    V[d] = ge[(d * 3 + 0) * NPT + pt] * u1 + ge[(d * 3 + 1) * NPT + pt] * u2 +
           ge[(d * 3 + 2) * NPT + pt] * u3;
  T F[3];
  if (b == 0) {
#pragma unroll
    for (int d = 0; d < 3; ++d) F[d] = V[d];
  } else {
    const T s = qe[b * NPT + pt] * recip(rho);
    if (b <= 3) {
      const T p = pressure(qe[4 * NPT + pt], p0, R, gam);
#pragma unroll
      for (int d = 0; d < 3; ++d) F[d] = V[d] * s + ge[(d * 3 + (b - 1)) * NPT + pt] * p;
    } else {
#pragma unroll
      for (int d = 0; d < 3; ++d) F[d] = V[d] * s;
    }
  }
  Fr = F[0];
  Fs = F[1];
  Ft = F[2];
}

template <typename T, int NQ, int EPB>
__global__ void __launch_bounds__(NQ *NQ *EPB)
    volume_basic_kernel(int64_t ne, T p0, T R, T gam, const T *__restrict__ q,
                        T *__restrict__ rhsq, const T *__restrict__ D,
                        const T *__restrict__ g, const T *__restrict__ jinv) {
  constexpr int NPT = NQ * NQ * NQ;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T *sD = reinterpret_cast<T *>(smem_raw);             // [n][i]
  T *sFr = sD + NQ * NQ + (NQ * NQ % 2);               // [EPB][NPT]
  T *sFs = sFr + EPB * NPT;                            // [EPB][NPT]

  const int tid = threadIdx.x + threadIdx.y * NQ * NQ;
  for (int t = tid; t < NQ * NQ; t += NQ * NQ * EPB) sD[t] = D[t];

  const int i = threadIdx.x % NQ, j = threadIdx.x / NQ, slot = threadIdx.y;
  const int64_t e = (int64_t)blockIdx.x * EPB + slot;
  const bool active = e < ne;
  const T *qe = q + e * 8 * NPT;
  const T *ge = g + e * 9 * NPT;
  const T *je = jinv + e * NPT;
  T *re = rhsq + e * 8 * NPT;
  T *fr = sFr + slot * NPT, *fs = sFs + slot * NPT;
  __syncthreads();

  for (int b = 0; b < 8; ++b) {
    T ft[NQ];
    if (active) {
#pragma unroll
      for (int k = 0; k < NQ; ++k) {
        const int pt = (k * NQ + j) * NQ + i;
        T a, s, t;
        field_flux<T, NQ>(b, pt, qe, ge, p0, R, gam, a, s, t);
        fr[pt] = a;
        fs[pt] = s;
        ft[k] = t;
      }
    }
    __syncthreads();
    if (active) {
#pragma unroll
      for (int k = 0; k < NQ; ++k) {
        T acc = T(0);
#pragma unroll
        for (int n = 0; n < NQ; ++n) {
          acc += sD[n * NQ + i] * fr[(k * NQ + j) * NQ + n];
          acc += sD[n * NQ + j] * fs[(k * NQ + n) * NQ + i];
          acc += sD[n * NQ + k] * ft[n];
        }
        const int pt = (k * NQ + j) * NQ + i;
        re[b * NPT + pt] += je[pt] * acc;
      }
    }
    __syncthreads();
  }
}

template <typename T, int NQ>
int launch_basic(int64_t ne, T p0, T R, T gam, const T *q, T *rhsq, const T *D,
                 const T *g, const T *jinv, cudaStream_t stream) {
  constexpr int EPB = (NQ * NQ >= 128) ? 1 : (128 / (NQ * NQ));
  constexpr int NPT = NQ * NQ * NQ;
  const size_t smem = sizeof(T) * (NQ * NQ + 1 + 2 * EPB * NPT);
  auto kern = volume_basic_kernel<T, NQ, EPB>;
  if (smem > 48 * 1024) {
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)smem) != cudaSuccess)
      return LFB_ERR_CUDA;
  }
  const int64_t blocks = (ne + EPB - 1) / EPB;
  if (blocks == 0) return LFB_OK;
  dim3 block(NQ * NQ, EPB);
  kern<<<(unsigned)blocks, block, smem, stream>>>(ne, p0, R, gam, q, rhsq, D, g,
                                                  jinv);
  LFB_CHECK_LAUNCH();
  return LFB_OK;
}

template <typename T>
int dispatch_basic(int nq, int64_t ne, T p0, T R, T gam, const T *q, T *rhsq,
                   const T *D, const T *g, const T *jinv, cudaStream_t s) {
  switch (nq) {
#define LFB_CASE(N) \
  case N:           \
    return launch_basic<T, N>(ne, p0, R, gam, q, rhsq, D, g, jinv, s);
    LFB_CASE(1) LFB_CASE(2) LFB_CASE(3) LFB_CASE(4) LFB_CASE(5) LFB_CASE(6)
    LFB_CASE(7) LFB_CASE(8) LFB_CASE(9) LFB_CASE(10) LFB_CASE(11) LFB_CASE(12)
    LFB_CASE(13) LFB_CASE(14) LFB_CASE(15) LFB_CASE(16)
#undef LFB_CASE
    default:
      return LFB_ERR_BAD_NQ;
  }
}

}  // namespace

int volume_basic_f64(int nq, int64_t ne, double p0, double R, double gam,
                     const double *q, double *rhsq, const double *D,
                     const double *g, const double *jinv, cudaStream_t s) {
  return dispatch_basic<double>(nq, ne, p0, R, gam, q, rhsq, D, g, jinv, s);
}

int volume_basic_f32(int nq, int64_t ne, float p0, float R, float gam,
                     const float *q, float *rhsq, const float *D,
                     const float *g, const float *jinv, cudaStream_t s) {
  return dispatch_basic<float>(nq, ne, p0, R, gam, q, rhsq, D, g, jinv, s);
}

}  // namespace lfb
