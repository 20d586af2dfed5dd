// LFB_VARIANT_FUSED — the production volume kernel.
//
// Design: the reference's level-8 structure
// (lf/bench/recipes.py:97-117: q read once, point-wise quantities in
// private registers, rhsq buffered on chip, 1/J at write-back) re-derived
// for B200:
//
//  * one thread owns one (i, j) column of an element (all Nq points along
//    k); EPB elements per CTA; persistent grid, CTAs stride over element
//    groups;
//  * phase 1 (once per element): 1/rho, p = p0 (R Theta/p0)^gam and the
//    contravariant momenta V_d = sum_a g(a,d) U_a of the thread's column
//    stay in registers (q and g read once from HBM);
//  * phase 2 (per field b): fluxes F_r, F_s, F_t of the column; the
//    t-derivative is the thread's own column (register scatter against the
//    D column, D broadcast from shared memory); F_r and F_s go to
//    XOR-swizzled shared tiles (double-buffered across fields: one barrier
//    per field) and the r/s derivative lines are read back with 128-bit
//    broadcast loads; D(i,.) and D(j,.) live in registers;
//  * write-back rhsq += Jinv * acc, coalesced (i fastest);
//  * the next element group's q/g/Jinv/rhsq is streamed into L2 with
//    cp.async.bulk.prefetch.L2 while the current one computes, so HBM
//    stays busy without needing more resident warps.
// No intermediate flux ever reaches HBM: traffic is the 272 B/pt minimum.

#include <stdlib.h>

#include "lfb_common.cuh"

namespace lfb {
namespace {

__device__ __forceinline__ void prefetch_l2(const void *p, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes)
               : "memory");
}

// Shared flux tile for one element and one field: [k][row][col] with the
// 16-byte chunk index XOR-swizzled by row so both the column-parallel
// stores and the line loads hit distinct bank groups (NQ = 8: 4 chunks per
// row, swizzle (row >> 1) & 3).
template <typename T, int NQ>
struct Tile {
  static constexpr int VEC = 16 / sizeof(T);  // elements per 16-byte chunk
  static constexpr int CHUNKS = NQ / VEC;
  __device__ static __forceinline__ int swz(int row) {
    return CHUNKS >= 4 ? ((row >> 1) & (CHUNKS - 1)) : (CHUNKS == 2 ? ((row >> 1) & 1) : 0);
  }
  // element (row, col) of plane k
  __device__ static __forceinline__ int at(int k, int row, int col) {
    const int c = col / VEC, w = col % VEC;
    return (k * NQ + row) * NQ + ((c ^ swz(row)) * VEC) + w;
  }
};

template <typename T>
struct Vec2;
template <>
struct Vec2<double> {
  using type = double2;
};
template <>
struct Vec2<float> {
  using type = float4;
};

template <typename T, int NQ, int EPB, bool PREFETCH, int MINB>
__global__ void __launch_bounds__(NQ *NQ *EPB, MINB)
    volume_fused_kernel(int64_t ne, T p0, T R, T gam, const T *__restrict__ q,
                        T *__restrict__ rhsq, const T *__restrict__ D,
                        const T *__restrict__ g, const T *__restrict__ jinv) {
  static_assert(NQ % (16 / sizeof(T)) == 0, "rows must be whole 16-byte chunks");
  constexpr int NPT = NQ * NQ * NQ;
  constexpr int VEC = 16 / sizeof(T);
  using V16 = typename Vec2<T>::type;
  using TileT = Tile<T, NQ>;

  extern __shared__ __align__(16) unsigned char smem_raw[];
  T *sD = reinterpret_cast<T *>(smem_raw);  // sD[n*NQ + i] = D(i, n)
  T *sFlux = sD + NQ * NQ;                  // [2 buf][EPB][2 (r,s)][NPT]

  const int tid = threadIdx.x + threadIdx.y * NQ * NQ;
  for (int t = tid; t < NQ * NQ; t += NQ * NQ * EPB) sD[t] = D[t];

  const int i = threadIdx.x % NQ, j = threadIdx.x / NQ, slot = threadIdx.y;
  const int64_t ngroups = (ne + EPB - 1) / EPB;
  __syncthreads();

  // D(i, n) and D(j, n): the thread's rows for the r and s lines.
  T Di[NQ], Dj[NQ];
#pragma unroll
  for (int n = 0; n < NQ; ++n) {
    Di[n] = sD[n * NQ + i];
    Dj[n] = sD[n * NQ + j];
  }

  int buf = 0;
  for (int64_t grp = blockIdx.x; grp < ngroups; grp += gridDim.x) {
    if (PREFETCH && tid < 4) {
      const int64_t nxt = grp + gridDim.x;
      if (nxt < ngroups) {
        const int64_t e0 = nxt * EPB;
        const int64_t cnt = (e0 + EPB <= ne) ? EPB : (ne - e0);
        const T *base;
        uint64_t bytes;
        if (tid == 0) { base = q + e0 * 8 * NPT; bytes = cnt * 8 * NPT * sizeof(T); }
        else if (tid == 1) { base = g + e0 * 9 * NPT; bytes = cnt * 9 * NPT * sizeof(T); }
        else if (tid == 2) { base = jinv + e0 * NPT; bytes = cnt * NPT * sizeof(T); }
        else { base = rhsq + e0 * 8 * NPT; bytes = cnt * 8 * NPT * sizeof(T); }
        prefetch_l2(base, (uint32_t)bytes);
      }
    }

    const int64_t e = grp * EPB + slot;
    const bool active = e < ne;
    const int64_t ec = active ? e : (ne - 1);  // clamp: inactive slots compute junk, never store
    const T *qe = q + ec * 8 * NPT;
    const T *ge = g + ec * 9 * NPT;
    const T *je = jinv + ec * NPT;
    T *re = rhsq + ec * 8 * NPT;
    const int col = j * NQ + i;

    // ---- phase 1: point-wise quantities of the column --------------------
    T rinv[NQ], pr[NQ], V0[NQ], V1[NQ], V2[NQ];
#pragma unroll
    for (int k = 0; k < NQ; ++k) {
      const int pt = k * NQ * NQ + col;
      const T rho = __ldg(qe + pt);
      const T u1 = __ldg(qe + 1 * NPT + pt), u2 = __ldg(qe + 2 * NPT + pt),
              u3 = __ldg(qe + 3 * NPT + pt), th = __ldg(qe + 4 * NPT + pt);
      T gg[9];
#pragma unroll
      for (int x = 0; x < 9; ++x) gg[x] = __ldg(ge + x * NPT + pt);
      rinv[k] = recip(rho);
      pr[k] = pressure(th, p0, R, gam);
      // g layout [dir][a]: gg[dir*3 + a]
      V0[k] = gg[0] * u1 + gg[1] * u2 + gg[2] * u3;
      V1[k] = gg[3] * u1 + gg[4] * u2 + gg[5] * u3;
      V2[k] = gg[6] * u1 + gg[7] * u2 + gg[8] * u3;
    }

    // ---- phase 2: per field ---------------------------------------------
#pragma unroll 1
    for (int b = 0; b < 8; ++b) {
      T *sFr = sFlux + ((buf * EPB + slot) * 2 + 0) * NPT;
      T *sFs = sFlux + ((buf * EPB + slot) * 2 + 1) * NPT;
      T acc[NQ];
#pragma unroll
      for (int k = 0; k < NQ; ++k) acc[k] = T(0);

#pragma unroll
      for (int k = 0; k < NQ; ++k) {
        const int pt = k * NQ * NQ + col;
        T fr, fs, ft;
        if (b == 0) {
          fr = V0[k]; fs = V1[k]; ft = V2[k];
        } else {
          const T s = __ldg(qe + b * NPT + pt) * rinv[k];
          fr = V0[k] * s; fs = V1[k] * s; ft = V2[k] * s;
          if (b <= 3) {
            const T pk = pr[k];
            fr += __ldg(ge + (0 * 3 + (b - 1)) * NPT + pt) * pk;
            fs += __ldg(ge + (1 * 3 + (b - 1)) * NPT + pt) * pk;
            ft += __ldg(ge + (2 * 3 + (b - 1)) * NPT + pt) * pk;
          }
        }
        // r line along i: tile rows j, cols i;  s line along j: rows i, cols j
        sFr[TileT::at(k, j, i)] = fr;
        sFs[TileT::at(k, i, j)] = fs;
        // t line is this thread's column: scatter against column k of D
        const V16 *dcol = reinterpret_cast<const V16 *>(sD + k * NQ);
#pragma unroll
        for (int c = 0; c < NQ / VEC; ++c) {
          const V16 d = dcol[c];
          if constexpr (VEC == 2) {
            acc[2 * c + 0] += d.x * ft;
            acc[2 * c + 1] += d.y * ft;
          } else {
            acc[4 * c + 0] += d.x * ft;
            acc[4 * c + 1] += d.y * ft;
            acc[4 * c + 2] += d.z * ft;
            acc[4 * c + 3] += d.w * ft;
          }
        }
      }
      __syncthreads();

#pragma unroll
      for (int k = 0; k < NQ; ++k) {
        T a = acc[k];
#pragma unroll
        for (int c = 0; c < NQ / VEC; ++c) {
          const V16 fr = *reinterpret_cast<const V16 *>(sFr + TileT::at(k, j, c * VEC));
          const V16 fs = *reinterpret_cast<const V16 *>(sFs + TileT::at(k, i, c * VEC));
          if constexpr (VEC == 2) {
            a += Di[2 * c] * fr.x + Di[2 * c + 1] * fr.y;
            a += Dj[2 * c] * fs.x + Dj[2 * c + 1] * fs.y;
          } else {
            a += Di[4 * c] * fr.x + Di[4 * c + 1] * fr.y + Di[4 * c + 2] * fr.z +
                 Di[4 * c + 3] * fr.w;
            a += Dj[4 * c] * fs.x + Dj[4 * c + 1] * fs.y + Dj[4 * c + 2] * fs.z +
                 Dj[4 * c + 3] * fs.w;
          }
        }
        acc[k] = a;
      }
      if (active) {
#pragma unroll
        for (int k = 0; k < NQ; ++k) {
          const int pt = k * NQ * NQ + col;
          T *dst = re + b * NPT + pt;
          *dst = *dst + __ldg(je + pt) * acc[k];
        }
      }
      buf ^= 1;
    }
  }
}

template <typename T, int NQ>
struct FusedCfg {
  static constexpr int EPB = (NQ * NQ >= 128) ? 1 : (128 / (NQ * NQ));
  static constexpr size_t smem() {
    return sizeof(T) * (NQ * NQ + 2 * EPB * 2 * NQ * NQ * NQ);
  }
};

template <typename T, int NQ>
int launch_fused(int64_t ne, T p0, T R, T gam, const T *q, T *rhsq, const T *D,
                 const T *g, const T *jinv, cudaStream_t stream) {
  using C = FusedCfg<T, NQ>;
  constexpr int EPB = C::EPB;
  const size_t smem = C::smem();
  // the measured best: 4 CTAs/SM bound, no L2 prefetch (prefetching a whole
  // CTA group ahead overflowed L2 and doubled DRAM reads)
  auto kern = volume_fused_kernel<T, NQ, EPB, false, 4>;
  if (smem > 48 * 1024 &&
      cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           (int)smem) != cudaSuccess)
    return LFB_ERR_CUDA;
  int dev = 0, sms = 0, per_sm = 0;
  if (cudaGetDevice(&dev) != cudaSuccess ||
      cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess ||
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, NQ * NQ * EPB, smem) !=
          cudaSuccess)
    return LFB_ERR_CUDA;
  if (per_sm < 1) return LFB_ERR_LAUNCH;
  const int64_t groups = (ne + EPB - 1) / EPB;
  const int64_t grid = groups < (int64_t)sms * per_sm ? groups : (int64_t)sms * per_sm;
  if (grid == 0) return LFB_OK;
  kern<<<(unsigned)grid, dim3(NQ * NQ, EPB), smem, stream>>>(ne, p0, R, gam, q, rhsq, D,
                                                             g, jinv);
  LFB_CHECK_LAUNCH();
  return LFB_OK;
}

template <typename T>
int dispatch_fused(int nq, int64_t ne, T p0, T R, T gam, const T *q, T *rhsq,
                   const T *D, const T *g, const T *jinv, cudaStream_t s) {
  switch (nq) {
    case 4: return launch_fused<T, 4>(ne, p0, R, gam, q, rhsq, D, g, jinv, s);
    case 8: return launch_fused<T, 8>(ne, p0, R, gam, q, rhsq, D, g, jinv, s);
    default: break;
  }
  if constexpr (sizeof(T) == 8) {
    if (nq == 6) return launch_fused<T, 6>(ne, p0, R, gam, q, rhsq, D, g, jinv, s);
  }
  return LFB_ERR_BAD_VARIANT;
}

}  // namespace

bool fused_available(int dtype_bytes, int nq) {
  if (dtype_bytes == 8) return nq == 4 || nq == 6 || nq == 8;
  if (dtype_bytes == 4) return nq == 4 || nq == 8;
  return false;
}

int volume_fused_f64(int nq, int64_t ne, double p0, double R, double gam,
                     const double *q, double *rhsq, const double *D,
                     const double *g, const double *jinv, cudaStream_t s) {
  if (!fused_available(8, nq)) return LFB_ERR_BAD_VARIANT;
  return dispatch_fused<double>(nq, ne, p0, R, gam, q, rhsq, D, g, jinv, s);
}

int volume_fused_f32(int nq, int64_t ne, float p0, float R, float gam,
                     const float *q, float *rhsq, const float *D,
                     const float *g, const float *jinv, cudaStream_t s) {
  if (!fused_available(4, nq)) return LFB_ERR_BAD_VARIANT;
  return dispatch_fused<float>(nq, ne, p0, R, gam, q, rhsq, D, g, jinv, s);
}

}  // namespace lfb
