// LFB_VARIANT_COL — column-owner kernel in the storage precision: FFMA for
// fp32 storage (the reference's own f32 pipeline, tolerance 1e-5), DFMA for
// fp64.
//
// Why (profiles/r01_tc_nq8_f32.json): the tc kernel computes
// the fp32 variant in fp64 — DMMA on the shared fp64/tensor-DP pipe (50 % of
// its cycles at Nq=8) plus 34 f32<->f64 conversions per point — and reaches
// only 0.72 of HBM. At 136 B/pt the fp32 path needs ~5.6 SM-cycles per point;
// its 24·Nq = 192 FMAs/pt are 1.5 cycles on the FP32 pipe (128 lanes/SM).
//
// Decomposition (element = Nq^3 points, KS*Nq^2 threads per element, EPB
// elements per CTA, persistent grid):
//   thread (i, j, h) owns the column points (i, j, k), k in [h·KP, (h+1)·KP);
//   phase 1 (per element): q and g of the own points are read once from
//     HBM (coalesced: a warp covers consecutive (i, j) at fixed k) and
//     1/rho, p, V_r, V_s, V_t stay in registers;
//   per field b: the three fluxes of the own points (q_b and g(b, .) are
//     re-read from L1 — the element's lines were just fetched) go to three
//     shared tiles, F_r as rows along i, F_s as rows along j, F_t as columns
//     along k (double-buffered across fields: ONE barrier per field); every
//     own point then contracts its three lines with 16-byte vector loads
//     (D(i,.), D(j,.) in registers, D(k,.) broadcast from shared memory) and
//     rhsq_b += Jinv · (R + S + T) is written back coalesced.
// Row strides are padded to an odd number of 16-byte chunks so the line
// loads of a warp (rows at distinct j, i or (i, j)) hit distinct bank groups.
// No intermediate flux reaches HBM: traffic is the 34 values/pt minimum.

#include <stdint.h>
#include <stdlib.h>

#include "lfb_common.cuh"
#include "lfb_math.cuh"

namespace lfb {
bool col_available(int dtype_bytes, int nq);
namespace {

__device__ __forceinline__ void col_prefetch_l2(const void *p, uint64_t bytes) {
  uintptr_t lo = reinterpret_cast<uintptr_t>(p) & ~(uintptr_t)15;
  const uintptr_t hi = (reinterpret_cast<uintptr_t>(p) + bytes + 15) & ~(uintptr_t)15;
  while (lo < hi) {
    const uint32_t n = (uint32_t)((hi - lo) > 65536 ? 65536 : (hi - lo));
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(lo), "r"(n) : "memory");
    lo += n;
  }
}

template <typename T, int NQ, int KS, int EPB>
struct ColCfg {
  static constexpr int NPT = NQ * NQ * NQ;
  static constexpr int KP = (NQ + KS - 1) / KS;  // points per thread (last h: fewer)
  static constexpr int TPE = NQ * NQ * KS;  // threads per element
  static constexpr int THREADS = (EPB * TPE + 31) / 32 * 32;
  static constexpr int VEC = 16 / (int)sizeof(T);
  // odd Nq: scalar line accesses with the odd line stride Nq (every
  // row-strided access of a warp conflict-free, no vector tail); even Nq:
  // 16-byte vector loads with an odd number of 16-byte chunks per line
  // (A/B at 1e8 points: fp64 Nq 3 / 5 / 9 0.355 / 0.661 / 0.316 -> 0.387 /
  // 0.67 / 0.33, fp32 Nq 5 / 9 0.541 / 0.419 -> 0.598 / 0.427; even Nq lose)
  static constexpr bool SC = (NQ % 2) == 1;
  // fp32 Nq = 2 mod 4: 8-byte line accesses with an odd number of 8-byte units
  // per line (a 16-byte chunk stride leaves a 2-float tail whose 8-byte reads
  // conflict 2-4 ways): Nq 6 / 10 0.596 / 0.424 -> 0.627 / 0.476
  static constexpr bool S2 = sizeof(T) == 4 && NQ % 4 == 2;
  static constexpr int LV = SC ? 1 : S2 ? 2 : VEC;    // line access width (values)
  static constexpr int RV = (NQ + VEC - 1) / VEC;      // 16-byte chunks per line
  static constexpr int RSC = (RV % 2) ? RV : RV + 1;   // odd chunk stride
  static constexpr int RS = SC ? (NQ | 1) : S2 ? ((NQ / 2) % 2 ? NQ : NQ + 2) : RSC * VEC;
  // per-direction line strides: RS, except where the bank model of the
  // scalar patterns (tools/col_banks.py) finds a better one for the F_s rows
  // / F_t columns: fp64 Nq 5 F_s 13, F_t 9 (0.676 -> 0.688 of HBM); fp32
  // Nq 5 F_s 19, F_t 9
  static constexpr bool ALT5 = SC && NQ == 5;
  static constexpr int RSS = ALT5 ? (sizeof(T) == 8 ? 13 : 19) : RS, RST = ALT5 ? 9 : RS;
  static constexpr int TILE = NQ * NQ * RS;            // F_r, one element
  static constexpr int TILES = NQ * NQ * RSS;          // F_s
  static constexpr int TILET = NQ * NQ * RST;          // F_t
  static constexpr int ETILE = TILE + TILES + TILET;   // one element, three directions
  static constexpr int BUF = ETILE * EPB;              // one field buffer
  // + D(i, n) as given ([n][i]) and transposed with padded rows ([k][n])
  static constexpr size_t smem() { return sizeof(T) * (2 * BUF + NQ * NQ + NQ * RS); }
};

template <typename T>
struct V16;
template <>
struct V16<float> {
  using type = float4;
};
template <>
struct V16<double> {
  using type = double2;
};

// n-th value of a 16-byte vector
template <typename V>
__device__ __forceinline__ auto vget(const V &v, int n) -> decltype(v.x) {
  if constexpr (sizeof(v) / sizeof(v.x) == 4) {
    return n == 0 ? v.x : n == 1 ? v.y : n == 2 ? v.z : v.w;
  } else {
    return n == 0 ? v.x : v.y;
  }
}

template <typename T>
__device__ __forceinline__ void col_scalars(T rho, T th, T p0, T Rp0, T gam, T &rinv, T &p) {
  if constexpr (sizeof(T) == 4) {
    rinv = __frcp_rn(rho);
    p = p0 * exp2f(gam * __log2f(Rp0 * th));
  } else {
    rinv = fast_rcp(rho);
    p = p0 * pos_pow(Rp0 * th, gam);
  }
}

// the NQ values of one padded shared line: 16-byte vector loads (LV = VEC)
// or scalar loads (LV = 1)
template <typename T, int NQ, int LV>
__device__ __forceinline__ void load_line(const T *line, T (&out)[NQ]) {
  if constexpr (LV == 1) {
#pragma unroll
    for (int n = 0; n < NQ; ++n) out[n] = line[n];
  } else if constexpr (LV == 2 && sizeof(T) == 4) {  // pairs of floats
#pragma unroll
    for (int c = 0; c < NQ / 2; ++c) {
      const float2 v = *reinterpret_cast<const float2 *>(line + 2 * c);
      out[2 * c] = v.x;
      out[2 * c + 1] = v.y;
    }
  } else {
    using V = typename V16<T>::type;
#pragma unroll
    for (int c = 0; c < (NQ + LV - 1) / LV; ++c) {
      const V v = *reinterpret_cast<const V *>(line + c * LV);
#pragma unroll
      for (int u = 0; u < LV; ++u)
        if (c * LV + u < NQ) out[c * LV + u] = vget(v, u);
    }
  }
}

// sum_n d[n] * line[n] over one padded shared line
template <typename T, int NQ, int LV>
__device__ __forceinline__ T line_dot(const T *line, const T (&d)[NQ], T acc) {
  T x[NQ];
  load_line<T, NQ, LV>(line, x);
#pragma unroll
  for (int n = 0; n < NQ; ++n) acc = fma(d[n], x[n], acc);
  return acc;
}

template <typename T, int NQ, int KS, int EPB, bool PF, int MINB>
__global__ void __launch_bounds__(ColCfg<T, NQ, KS, EPB>::THREADS, MINB)
    volume_col_kernel(int64_t ne, T p0, T R, T gam, const T *__restrict__ q,
                      T *__restrict__ rhsq, const T *__restrict__ D, const T *__restrict__ g,
                      const T *__restrict__ jinv) {
  using C = ColCfg<T, NQ, KS, EPB>;
  constexpr int NPT = C::NPT, KP = C::KP, RS = C::RS, TILE = C::TILE, VEC = C::VEC, LV = C::LV;
  using V = typename V16<T>::type;

  extern __shared__ __align__(16) unsigned char smem_raw[];
  T *const sbuf = reinterpret_cast<T *>(smem_raw);  // [2][EPB][3][TILE]
  T *const sDT = sbuf + 2 * C::BUF;                  // sDT[k*RS + n] = D(k, n) (16-B rows)
  T *const sD = sDT + NQ * RS;                       // sD[n*NQ + i] = D(i, n)

  const int tid = threadIdx.x;
  for (int t = tid; t < NQ * NQ; t += C::THREADS) {
    sD[t] = D[t];
    sDT[(t % NQ) * RS + t / NQ] = D[t];
  }

  const int slot = tid / C::TPE;  // element within the CTA's group
  const int te = tid % C::TPE;
  const int i = te % NQ, j = (te / NQ) % NQ, h = te / (NQ * NQ);  // dead threads: h < KS
  const int k0 = h * KP;
  const bool thread_live = slot < EPB;  // threads past EPB*TPE only join barriers
  const int64_t ngroups = (ne + EPB - 1) / EPB;
  const T Rp0 = R / p0;
  __syncthreads();

  // one own point per thread (KP = 1): its D(k, .) row lives in registers —
  // loop-invariant, but a shared-memory load cannot be hoisted across the
  // per-field barriers (+8-9 % at Nq 5, 6; with KP = 2 the extra registers
  // spill and it loses, profiles/r01_col_configs.txt)
  constexpr bool DKREG = KP == 1;
  T Di[NQ], Dj[NQ], Dkr[DKREG ? KP : 1][DKREG ? NQ : 1];
#pragma unroll
  for (int n = 0; n < NQ; ++n) {
    Di[n] = sD[n * NQ + i];
    Dj[n] = sD[n * NQ + j];
    if constexpr (DKREG) {
#pragma unroll
      for (int kk = 0; kk < KP; ++kk)
        Dkr[kk][n] = sD[n * NQ + (k0 + kk < NQ ? k0 + kk : 0)];
    }
  }
  // own points' offsets inside an element slab, and tile positions
  const int col = j * NQ + i;
  T *const tr0 = sbuf + slot * C::ETILE;                 // F_r rows (k, j) along i
  T *const ts0 = tr0 + TILE;                              // F_s rows (k, i) along j
  T *const tt0 = ts0 + C::TILES;                          // F_t columns (j, i) along k

  int buf = 0;
  for (int64_t grp = blockIdx.x; grp < ngroups; grp += gridDim.x) {
    if (PF && tid < 4) {
      const int64_t nx = grp + gridDim.x;
      if (nx < ngroups) {
        const int64_t ea = nx * EPB;
        const int64_t cnt = (ea + EPB <= ne) ? EPB : ne - ea;
        if (tid == 0) col_prefetch_l2(q + ea * 8 * NPT, (uint64_t)cnt * 8 * NPT * sizeof(T));
        if (tid == 1) col_prefetch_l2(g + ea * 9 * NPT, (uint64_t)cnt * 9 * NPT * sizeof(T));
        if (tid == 2) col_prefetch_l2(rhsq + ea * 8 * NPT, (uint64_t)cnt * 8 * NPT * sizeof(T));
        if (tid == 3) col_prefetch_l2(jinv + ea * NPT, (uint64_t)cnt * NPT * sizeof(T));
      }
    }
    const int64_t e = grp * EPB + slot;
    const bool live = thread_live && e < ne;
    const int64_t ec = live ? e : 0;  // dead slots compute on element 0, never store
    const T *qe = q + ec * 8 * NPT;
    const T *ge = g + ec * 9 * NPT;
    T *re = rhsq + ec * 8 * NPT;

    // ---- phase 1: point-wise state of the own points -----------------------
    T rinv[KP], pr[KP], V0[KP], V1[KP], V2[KP], jv[KP];
#pragma unroll
    for (int kk = 0; kk < KP; ++kk) {
      if (k0 + kk >= NQ) break;
      const int pt = (k0 + kk) * NQ * NQ + col;
      const T rho = __ldg(qe + pt), u1 = __ldg(qe + NPT + pt), u2 = __ldg(qe + 2 * NPT + pt),
              u3 = __ldg(qe + 3 * NPT + pt), th = __ldg(qe + 4 * NPT + pt);
      T gg[9];
#pragma unroll
      for (int x = 0; x < 9; ++x) gg[x] = __ldg(ge + x * NPT + pt);
      jv[kk] = __ldg(jinv + ec * NPT + pt);
      col_scalars<T>(rho, th, p0, Rp0, gam, rinv[kk], pr[kk]);
      V0[kk] = gg[0] * u1 + gg[1] * u2 + gg[2] * u3;  // g layout [dir][a]
      V1[kk] = gg[3] * u1 + gg[4] * u2 + gg[5] * u3;
      V2[kk] = gg[6] * u1 + gg[7] * u2 + gg[8] * u3;
    }

    // ---- per field -----------------------------------------------------------
#pragma unroll
    for (int b = 0; b < 8; ++b) {
      T *const tr = tr0 + buf * C::BUF;
      T *const ts = ts0 + buf * C::BUF;
      T *const tt = tt0 + buf * C::BUF;
      T rh[KP], ftv[KP];
#pragma unroll
      for (int kk = 0; kk < KP; ++kk) {
        const int k = k0 + kk, pt = k * NQ * NQ + col;
        if (!thread_live || k >= NQ) break;
        rh[kk] = re[b * NPT + pt];
        T fr = V0[kk], fs = V1[kk], ft = V2[kk];
        if (b > 0) {
          const T s = __ldg(qe + b * NPT + pt) * rinv[kk];
          fr *= s;
          fs *= s;
          ft *= s;
          if (b <= 3) {  // + g(b, dir) p
            fr = fma(__ldg(ge + (0 * 3 + b - 1) * NPT + pt), pr[kk], fr);
            fs = fma(__ldg(ge + (1 * 3 + b - 1) * NPT + pt), pr[kk], fs);
            ft = fma(__ldg(ge + (2 * 3 + b - 1) * NPT + pt), pr[kk], ft);
          }
        }
        tr[(k * NQ + j) * RS + i] = fr;
        ts[(k * NQ + i) * C::RSS + j] = fs;
        ftv[kk] = ft;
      }
      if (thread_live) {
        // F_t: the own KP points are contiguous in the column -> 16-byte stores
        T *const dst = tt + (j * NQ + i) * C::RST + k0;
        if constexpr (!C::SC && !C::S2 && (KP * sizeof(T)) % 16 == 0 && (NQ % KP) == 0) {
#pragma unroll
          for (int c = 0; c < KP / VEC; ++c) {
            V v;
            if constexpr (VEC == 4) {
              v.x = ftv[4 * c]; v.y = ftv[4 * c + 1]; v.z = ftv[4 * c + 2]; v.w = ftv[4 * c + 3];
            } else {
              v.x = ftv[2 * c]; v.y = ftv[2 * c + 1];
            }
            *reinterpret_cast<V *>(dst + c * VEC) = v;
          }
        } else {
#pragma unroll
          for (int kk = 0; kk < KP; ++kk)
            if (k0 + kk < NQ) dst[kk] = ftv[kk];
        }
      }
      __syncthreads();
      if (thread_live) {
      // T: the own column along k, against D(k, n) broadcast from sD
      T ftc[NQ];
      load_line<T, NQ, LV>(tt + (j * NQ + i) * C::RST, ftc);
#pragma unroll
      for (int kk = 0; kk < KP; ++kk) {
        const int k = k0 + kk;
        if (k >= NQ) break;
        T acc = T(0);
        if constexpr (DKREG) {  // the thread's D(k, .) rows live in registers
#pragma unroll
          for (int n = 0; n < NQ; ++n) acc = fma(Dkr[kk][n], ftc[n], acc);
        } else {  // D(k, .) row, broadcast within the warp (one k per warp)
          T dk[NQ];
          load_line<T, NQ, LV>(sDT + k * RS, dk);
#pragma unroll
          for (int n = 0; n < NQ; ++n) acc = fma(dk[n], ftc[n], acc);
        }
        acc = line_dot<T, NQ, LV>(tr + (k * NQ + j) * RS, Di, acc);
        acc = line_dot<T, NQ, LV>(ts + (k * NQ + i) * C::RSS, Dj, acc);
        if (live) re[b * NPT + k * NQ * NQ + col] = fma(jv[kk], acc, rh[kk]);
      }
      }
      buf ^= 1;
    }
  }
}

#define LFB_ARGS(KS_, EPB_, MB_) KS_, EPB_, MB_

template <typename T, int NQ, int KS, int EPB, int MINB>
int launch_col(int64_t ne, T p0, T R, T gam, const T *q, T *rhsq, const T *D, const T *g,
               const T *jinv, cudaStream_t stream) {
  using C = ColCfg<T, NQ, KS, EPB>;
  auto kern = volume_col_kernel<T, NQ, KS, EPB, true, MINB>;
  const size_t smem = C::smem();
  if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) !=
      cudaSuccess)
    return LFB_ERR_CUDA;
  int dev = 0, sms = 0, per_sm = 0;
  if (cudaGetDevice(&dev) != cudaSuccess ||
      cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess ||
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, C::THREADS, smem) !=
          cudaSuccess)
    return LFB_ERR_CUDA;
  if (per_sm < 1) return LFB_ERR_LAUNCH;
  const int64_t groups = (ne + EPB - 1) / EPB;
  const int64_t slots = (int64_t)sms * per_sm;
  const int64_t grid = groups < slots ? groups : slots;
  if (grid == 0) return LFB_OK;
  kern<<<(unsigned)grid, C::THREADS, smem, stream>>>(ne, p0, R, gam, q, rhsq, D, g, jinv);
  LFB_CHECK_LAUNCH();
  return LFB_OK;
}

// (KS, EPB, MINB) per (dtype, Nq): threads per element = KS Nq^2, EPB
// elements per CTA — the measured best of the alternatives in
// profiles/r01_col_configs.txt.
template <typename T>
int dispatch_col(int nq, int64_t ne, T p0, T R, T gam, const T *q, T *rhsq, const T *D,
                 const T *g, const T *jinv, cudaStream_t s) {
  constexpr bool F64 = sizeof(T) == 8;
#define LFB_L(NQ_, KS_, EPB_, MB_) \
  return launch_col<T, NQ_, KS_, EPB_, MB_>(ne, p0, R, gam, q, rhsq, D, g, jinv, s)
// A0 = the shipped (KS, EPB, MINB) per Nq; A1, A2 = the measured runners-up
// (COL_ALT selects one for A/B builds). Re-measured after the odd-Nq scalar
// lines (1e8 points): fp32 Nq 5 (5,1,8) 0.649 vs (5,2,4) 0.597, fp32 Nq 9
// (9,1,1) 0.432 vs (3,1,2) 0.426, fp64 Nq 7 (2,1,2) 0.425 vs (7,1,2) 0.377
#ifndef COL_ALT
#define COL_ALT 0
#endif
#if COL_ALT == 1
#define LFB_COL3(NQ_, A0, A1, A2) \
  case NQ_:                       \
    LFB_L(NQ_, A1);
#elif COL_ALT == 2
#define LFB_COL3(NQ_, A0, A1, A2) \
  case NQ_:                       \
    LFB_L(NQ_, A2);
#else
#define LFB_COL3(NQ_, A0, A1, A2) \
  case NQ_:                       \
    LFB_L(NQ_, A0);
#endif
  if constexpr (F64) {
    switch (nq) {
      LFB_COL3(2, LFB_ARGS(1, 32, 2), LFB_ARGS(1, 32, 2), LFB_ARGS(1, 32, 2))
      LFB_COL3(3, LFB_ARGS(1, 14, 2), LFB_ARGS(1, 14, 2), LFB_ARGS(1, 14, 2))
      LFB_COL3(4, LFB_ARGS(2, 4, 2), LFB_ARGS(4, 2, 3), LFB_ARGS(1, 8, 2))
      LFB_COL3(5, LFB_ARGS(5, 1, 4), LFB_ARGS(5, 1, 5), LFB_ARGS(5, 1, 6))
      LFB_COL3(6, LFB_ARGS(3, 1, 4), LFB_ARGS(3, 1, 5), LFB_ARGS(6, 1, 4))
      LFB_COL3(7, LFB_ARGS(2, 1, 2), LFB_ARGS(7, 1, 2), LFB_ARGS(4, 1, 3))
      LFB_COL3(8, LFB_ARGS(4, 1, 2), LFB_ARGS(8, 1, 1), LFB_ARGS(2, 1, 2))
      LFB_COL3(9, LFB_ARGS(3, 1, 2), LFB_ARGS(9, 1, 1), LFB_ARGS(3, 1, 2))
      LFB_COL3(10, LFB_ARGS(5, 1, 1), LFB_ARGS(10, 1, 1), LFB_ARGS(5, 1, 1))
      LFB_COL3(11, LFB_ARGS(4, 1, 1), LFB_ARGS(6, 1, 1), LFB_ARGS(4, 1, 1))
      LFB_COL3(12, LFB_ARGS(4, 1, 1), LFB_ARGS(6, 1, 1), LFB_ARGS(4, 1, 1))
      default: return LFB_ERR_BAD_VARIANT;
    }
  } else {
    switch (nq) {
      LFB_COL3(2, LFB_ARGS(1, 32, 4), LFB_ARGS(1, 32, 4), LFB_ARGS(1, 32, 4))
      LFB_COL3(3, LFB_ARGS(1, 14, 4), LFB_ARGS(1, 14, 4), LFB_ARGS(1, 14, 4))
      LFB_COL3(4, LFB_ARGS(4, 2, 6), LFB_ARGS(2, 4, 4), LFB_ARGS(1, 8, 4))
      LFB_COL3(5, LFB_ARGS(5, 1, 8), LFB_ARGS(5, 2, 4), LFB_ARGS(1, 5, 4))
      LFB_COL3(6, LFB_ARGS(6, 1, 4), LFB_ARGS(3, 1, 6), LFB_ARGS(2, 2, 4))
      LFB_COL3(7, LFB_ARGS(2, 1, 4), LFB_ARGS(7, 1, 4), LFB_ARGS(1, 3, 4))
      LFB_COL3(8, LFB_ARGS(2, 1, 4), LFB_ARGS(4, 1, 4), LFB_ARGS(8, 1, 2))
      LFB_COL3(9, LFB_ARGS(9, 1, 1), LFB_ARGS(3, 1, 2), LFB_ARGS(3, 1, 3))
      LFB_COL3(10, LFB_ARGS(2, 1, 2), LFB_ARGS(2, 1, 3), LFB_ARGS(5, 1, 2))
      LFB_COL3(11, LFB_ARGS(4, 1, 1), LFB_ARGS(3, 1, 2), LFB_ARGS(6, 1, 1))
      LFB_COL3(12, LFB_ARGS(4, 1, 1), LFB_ARGS(3, 1, 1), LFB_ARGS(6, 1, 1))
      LFB_COL3(13, LFB_ARGS(4, 1, 1), LFB_ARGS(3, 1, 1), LFB_ARGS(5, 1, 1))
      LFB_COL3(14, LFB_ARGS(4, 1, 1), LFB_ARGS(3, 1, 1), LFB_ARGS(5, 1, 1))
      LFB_COL3(15, LFB_ARGS(4, 1, 1), LFB_ARGS(3, 1, 1), LFB_ARGS(3, 1, 1))
      LFB_COL3(16, LFB_ARGS(4, 1, 1), LFB_ARGS(3, 1, 1), LFB_ARGS(2, 1, 1))
      default: return LFB_ERR_BAD_VARIANT;
    }
  }
#undef LFB_COL3
#undef LFB_L
}

}  // namespace

// fp64 stops at Nq = 12 (register state per column point); fp32 covers 2..16.
// The file is compiled twice (LFB_COL_DTYPE = 8 | 4, see the Makefile) so the
// two dtypes' template instances build in parallel.
#if !defined(LFB_COL_DTYPE) || LFB_COL_DTYPE == 8
bool col_available(int dtype_bytes, int nq) {
  if (dtype_bytes == 8) return nq >= 2 && nq <= 12;
  return dtype_bytes == 4 && nq >= 2 && nq <= 16;
}

int volume_col_f64(int nq, int64_t ne, double p0, double R, double gam, const double *q,
                   double *rhsq, const double *D, const double *g, const double *jinv,
                   cudaStream_t s) {
  if (!col_available(8, nq)) return LFB_ERR_BAD_VARIANT;
  return dispatch_col<double>(nq, ne, p0, R, gam, q, rhsq, D, g, jinv, s);
}
#endif

#if !defined(LFB_COL_DTYPE) || LFB_COL_DTYPE == 4
int volume_col_f32(int nq, int64_t ne, float p0, float R, float gam, const float *q,
                   float *rhsq, const float *D, const float *g, const float *jinv,
                   cudaStream_t s) {
  if (!col_available(4, nq)) return LFB_ERR_BAD_VARIANT;
  return dispatch_col<float>(nq, ne, p0, R, gam, q, rhsq, D, g, jinv, s);
}
#endif

}  // namespace lfb
