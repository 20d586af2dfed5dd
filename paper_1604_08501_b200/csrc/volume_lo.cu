// LFB_VARIANT_LO — "line owners", Nq 9..12, FMA in the storage precision.
//
// Why: at Nq >= 9 the column kernel (volume_col.cu) is
// bound by its shared-memory pipe — every point re-reads the three Nq-long
// flux lines it contracts, ~3 Nq values per point and field — and the
// tensor-core line kernels (volume_lt*.cu, volume_ltu.cu) by the register
// footprint of one 1000-1700 point element per SM. Here the contractions are
// done by LINE owners, so D(o, .) is the only operand that changes along a
// contraction and is read as a warp-wide broadcast; fluxes and write-back
// are done by POINT owners, so every global access is coalesced.
//
//   CTA = one element, ceil(Nq^2 / 32) warps, several CTAs per SM;
//   point owners: x = tid + THREADS u; line owner te < Nq^2 owns R-line
//     (j, k), S-line (i, k) and T-line (i, j) with (te % Nq, te / Nq);
//   phase 1 (per element, point owners): W_d = V_d / rho (V_d = sum_a
//     g(a,d) U_a) and p -> shared state rows by point;
//   per field b:
//     A  point owners: F_r, F_s, F_t -> the R / S / T tiles (rows = lines);
//        q of the next field and rhsq_b go to registers          | barrier
//     B  line owners: load the three rows, then per output index o one
//        broadcast D(o, .) row against three dot products, the outputs
//        written over the own rows                                | barrier
//     C  point owners: rhsq_b += Jinv (R + S + T)                 | barrier
//   the next element's phase-1 slabs are L2-prefetched at field 7.
// Shared traffic per point and field is ~0.5 wavefronts (12 scalar accesses
// + the state reads + one broadcast per output row); tile row strides from
// the bank model tools/lo_banks.py. HBM traffic is the 34 values/pt minimum
// (q, g, Jinv read once from HBM; the per-field re-reads hit L2).

#include <stdint.h>

#include "lfb_common.cuh"
#include "lfb_math.cuh"
#include "lfb_tma.cuh"

#ifndef LO_PF  // L2 prefetch of the next element's phase-1 inputs at field LO_PF_FIELD
// (A/B, profiles/r02b_lo_pf_ab.txt: none / field 0 / 4 / 5 / 6 / 7 — 7 leads,
// fp64 Nq 9 0.47 -> 0.545; also prefetching the next element's q_5..7 and
// rhsq there was no better)
#define LO_PF 1
#endif
#ifndef LO_PF_FIELD
#define LO_PF_FIELD 7
#endif
#ifndef LO_CS  // streaming cache operator on last-use loads and the rhsq stores
#define LO_CS 1
#endif
#ifndef LO_RPF  // rhsq into L2: 0 the element's 8 slabs at its start, 1 a field
#define LO_RPF 2  // ahead, 2 a field ahead for fp64 only (profiles/r02b_lo_l2_ab.txt)
#endif
#ifndef LO_MINB32  // fp32 CTAs per SM the registers are budgeted for
#define LO_MINB32 3
#endif
#ifndef LO_OUNROLL  // unroll of the output-row loop of the line contractions (0: full;
// profiles/r02b_lo_unroll_ab.txt: 1 / 2 / 3 / 6 / 9 / full, full +1-4 %)
#define LO_OUNROLL 0
#endif

namespace lfb {
bool lo_available(int dtype_bytes, int nq);
namespace {

// tile row strides (values) from the bank model tools/lo_banks.py, per
// (dtype bytes, Nq 9..12): point-owner and line-owner accesses of each tile
// (fp32 Nq 11: S at 15, the model's runner-up at a third of the tile size of
// its optimum 35 — measured 0.485 / 0.513 / 0.506 / 0.498 at S = 11 / 15 /
// 27 / 35, profiles/r02b_lo_strides_ab.txt)
constexpr int lo_rsr(int nq, int bytes) { return nq == 12 ? 13 : nq; }
constexpr int lo_rss(int nq, int bytes) {
  return bytes == 4 ? (nq == 9 ? 25 : nq == 10 ? 17 : nq == 11 ? 15 : 15)
                    : (nq == 9 ? 9 : nq == 10 ? 13 : nq == 11 ? 19 : 13);
}
constexpr int lo_rst(int nq, int bytes) {
  return bytes == 4 ? (nq == 9 ? 17 : nq == 10 ? 11 : nq == 11 ? 11 : 13)
                    : (nq == 9 ? 17 : nq == 10 ? 11 : nq == 11 ? 25 : 13);
}

template <typename T, int NQ>
struct LoCfg {
  static constexpr int NPT = NQ * NQ * NQ;
  static constexpr int TPE = NQ * NQ;                     // lines per direction
  static constexpr int THREADS = (TPE + 31) / 32 * 32;    // one line triple each (B)
  static constexpr int NPP = (NPT + THREADS - 1) / THREADS;  // points per thread (A, C)
  static constexpr int VEC = 16 / (int)sizeof(T);
  static constexpr int CH0 = (NQ + VEC - 1) / VEC;        // 16-byte chunks of a D row
  static constexpr int SP = ((CH0 % 2) ? CH0 : CH0 + 1) * VEC;  // D row stride
  static constexpr int RSR = lo_rsr(NQ, sizeof(T));
  static constexpr int RSS = lo_rss(NQ, sizeof(T)), RST = lo_rst(NQ, sizeof(T));
  // state [4][NPT] (W_r, W_s, W_t, p by point; Jinv is read from global at
  // the write-back — a fifth row cost CTAs per SM, profiles/r02b_lo_jg_ab.txt),
  // R / S / T tiles [TPE][RS*], D rows [NQ][SP] (row o = D(o, .))
  static constexpr int ST = (NPT + VEC - 1) / VEC * VEC;
  static constexpr int NSR = 4;  // state rows
  static constexpr int DOFF = (NSR * ST + TPE * (RSR + RSS + RST) + VEC - 1) / VEC * VEC;
  static constexpr size_t SMEM = sizeof(T) * ((size_t)DOFF + NQ * SP);
  // fp64: 3 CTAs' registers at Nq <= 10 (fp64 Nq 10 0.495 -> 0.511; at
  // Nq 11, 12 the 168-register cap spills, 0.48 -> 0.43)
  static constexpr int MINB = sizeof(T) == 4 ? LO_MINB32 : (NQ <= 10 ? 3 : 2);
};

template <typename T>
struct LoVec;
template <>
struct LoVec<float> {
  using type = float4;
};
template <>
struct LoVec<double> {
  using type = double2;
};

// last-use loads / write-once stores with the streaming (evict-first) cache
// operator, so an element's dead lines leave L2 before the live ones
template <typename T>
__device__ __forceinline__ T lo_ld_last(const T *p) {
  return LO_CS ? __ldcs(p) : __ldg(p);
}
template <typename T>
__device__ __forceinline__ void lo_st_once(T *p, T v) {
  if (LO_CS) __stcs(p, v); else *p = v;
}

template <typename T>
__device__ __forceinline__ void lo_scalars(T rho, T th, T p0, T Rp0, T gam, T &rinv, T &p) {
  if constexpr (sizeof(T) == 4) {
    rinv = __frcp_rn(rho);
    p = p0 * exp2f(gam * __log2f(Rp0 * th));
  } else {
    rinv = fast_rcp(rho);
    p = p0 * pos_pow(Rp0 * th, gam);
  }
}

template <typename T, int NQ>
__global__ void __launch_bounds__(LoCfg<T, NQ>::THREADS, LoCfg<T, NQ>::MINB)
    volume_lo_kernel(int64_t ne, T p0, T R, T gam, const T *__restrict__ q, T *__restrict__ rhsq,
                     const T *__restrict__ D, const T *__restrict__ g,
                     const T *__restrict__ jinv) {
  using C = LoCfg<T, NQ>;
  constexpr int NPT = C::NPT, TPE = C::TPE, SP = C::SP, ST = C::ST, NPP = C::NPP;
  constexpr int RSR = C::RSR, RSS = C::RSS, RST = C::RST, VEC = C::VEC, OUN = LO_OUNROLL ? LO_OUNROLL : NQ;
  constexpr int NTH = C::THREADS;
  constexpr bool RPF = LO_RPF == 1 || (LO_RPF == 2 && sizeof(T) == 8);
  using V = typename LoVec<T>::type;
  extern __shared__ __align__(16) unsigned char lo_raw[];
  T *const sst = reinterpret_cast<T *>(lo_raw);  // state [4][ST]
  T *const sR = sst + C::NSR * ST;                // R tile [TPE][RSR]: row (k,j), pos i
  T *const sS = sR + TPE * RSR;                   // S tile [TPE][RSS]: row (k,i), pos j
  T *const sT = sS + TPE * RSS;                   // T tile [TPE][RST]: row (j,i), pos k
  T *const sD = sst + C::DOFF;                    // D rows [NQ][SP] (16-byte aligned)

  const int tid = threadIdx.x;
  for (int x = tid; x < NQ * SP; x += NTH) {
    const int o = x / SP, n = x % SP;
    T dv = T(0);
    if (n < NQ) dv = D[n * NQ + o];  // D[n*NQ + i] = D(i, n); no load past the Nq^2 values
    sD[x] = dv;
  }
  // own points x = tid + NTH u (A, C): tile positions
  int pR[NPP], pS[NPP], pT[NPP];
#pragma unroll
  for (int u = 0; u < NPP; ++u) {
    const int x = tid + NTH * u < NPT ? tid + NTH * u : NPT - 1;
    const int i = x % NQ, j = (x / NQ) % NQ, k = x / (NQ * NQ);
    pR[u] = (k * NQ + j) * RSR + i;
    pS[u] = (k * NQ + i) * RSS + j;
    pT[u] = (j * NQ + i) * RST + k;
  }
  auto own = [&](int u) { return NPP * NTH == NPT || tid + NTH * u < NPT; };
  const bool live = tid < TPE;  // line owner (B)
  const T Rp0 = R / p0;
  __syncthreads();

  for (int64_t e = blockIdx.x; e < ne; e += gridDim.x) {
    const T *qe = q + e * 8 * NPT + tid;
    const T *ge = g + e * 9 * NPT + tid;
    const T *je = jinv + e * NPT + tid;
    T *re = rhsq + e * 8 * NPT + tid;
    if (tid == 0) {  // the slabs first touched in the field loop
      prefetch_l2_range(q + e * 8 * NPT + 5 * NPT, 3ull * NPT * sizeof(T));
      if (!RPF) prefetch_l2_range(rhsq + e * 8 * NPT, 8ull * NPT * sizeof(T));
      else prefetch_l2_range(rhsq + e * 8 * NPT, 1ull * NPT * sizeof(T));
    }
    // ---- phase 1 (point owners): W_d, p -> state ----------------------------
#pragma unroll
    for (int u = 0; u < NPP; ++u) {
      if (own(u)) {
        const int o = NTH * u;
        const T rho = __ldg(qe + o), th = __ldg(qe + 4 * NPT + o);
        T U[3], gv[9];
#pragma unroll
        for (int c = 0; c < 3; ++c) U[c] = __ldg(qe + (1 + c) * NPT + o);
#pragma unroll
        for (int k = 0; k < 9; ++k) gv[k] = __ldg(ge + k * NPT + o);
        T rinv, p;
        lo_scalars(rho, th, p0, Rp0, gam, rinv, p);
#pragma unroll
        for (int d = 0; d < 3; ++d)
          sst[d * ST + tid + o] = fma(gv[3 * d], U[0], fma(gv[3 * d + 1], U[1], gv[3 * d + 2] * U[2])) * rinv;
        sst[3 * ST + tid + o] = p;
      }
    }
    T qv[NPP];  // q_b at the own points, loaded a field ahead
#pragma unroll
    for (int u = 0; u < NPP; ++u) qv[u] = own(u) ? __ldg(qe + NTH * u) : T(0);

#pragma unroll 1
    for (int b = 0; b < 8; ++b) {
      if (LO_PF && b == LO_PF_FIELD && tid == 32 && e + gridDim.x < ne) {
        // the next element's phase-1 inputs (q_0..4, g, Jinv) into L2
        const int64_t en = e + gridDim.x;
        prefetch_l2_range(q + en * 8 * NPT, 5ull * NPT * sizeof(T));
        prefetch_l2_range(g + en * 9 * NPT, 9ull * NPT * sizeof(T));
        prefetch_l2_range(jinv + en * NPT, 1ull * NPT * sizeof(T));
      }
      // ---- A (point owners): fluxes -> R, S, T tiles --------------------------
      const bool mom = b >= 1 && b <= 3;
      T rh[NPP];  // rhsq_b, consumed in C
#pragma unroll
      for (int u = 0; u < NPP; ++u) rh[u] = own(u) ? lo_ld_last(re + b * NPT + NTH * u) : T(0);
      if (RPF && tid == 0 && b < 7) prefetch_l2_range(rhsq + (e * 8 + b + 1) * NPT, 1ull * NPT * sizeof(T));
#pragma unroll
      for (int u = 0; u < NPP; ++u) {
        if (own(u)) {
          const int o = NTH * u;
          T f[3];
#pragma unroll
          for (int d = 0; d < 3; ++d) f[d] = sst[d * ST + tid + o] * qv[u];
          if (mom) {
            const T pv = sst[3 * ST + tid + o];
#pragma unroll
            for (int d = 0; d < 3; ++d) f[d] = fma(lo_ld_last(ge + (3 * d + b - 1) * NPT + o), pv, f[d]);
          }
          sR[pR[u]] = f[0];
          sS[pS[u]] = f[1];
          sT[pT[u]] = f[2];
        }
      }
      if (b < 7) {
#pragma unroll
        for (int u = 0; u < NPP; ++u) qv[u] = own(u) ? lo_ld_last(qe + (b + 1) * NPT + NTH * u) : T(0);
      }
      __syncthreads();
      // ---- B (line owners): contractions, outputs over the own rows ----------
      if (live) {
        T Fr[NQ], Fs[NQ], Ft[NQ];
#pragma unroll
        for (int n = 0; n < NQ; ++n) {
          Fr[n] = sR[tid * RSR + n];
          Fs[n] = sS[tid * RSS + n];
          Ft[n] = sT[tid * RST + n];
        }
#pragma unroll OUN
        for (int o = 0; o < NQ; ++o) {
          T ar = T(0), as = T(0), at = T(0);
#pragma unroll
          for (int c = 0; c < C::CH0; ++c) {
            const V dv = *reinterpret_cast<const V *>(sD + o * SP + c * VEC);
            const T *pd = reinterpret_cast<const T *>(&dv);
#pragma unroll
            for (int v = 0; v < VEC; ++v) {
              const int n = c * VEC + v;
              if (n < NQ) {
                ar = fma(pd[v], Fr[n], ar);
                as = fma(pd[v], Fs[n], as);
                at = fma(pd[v], Ft[n], at);
              }
            }
          }
          sR[tid * RSR + o] = ar;
          sS[tid * RSS + o] = as;
          sT[tid * RST + o] = at;
        }
      }
      __syncthreads();
      // ---- C (point owners): rhsq_b += Jinv (R + S + T) ------------------------
#pragma unroll
      for (int u = 0; u < NPP; ++u) {
        if (own(u)) {
          const int o = NTH * u;
          lo_st_once(re + b * NPT + o, fma(__ldg(je + o), sR[pR[u]] + sS[pS[u]] + sT[pT[u]], rh[u]));
        }
      }
      __syncthreads();
    }
  }
}

template <typename T, int NQ>
int launch_lo(int64_t ne, T p0, T R, T gam, const T *q, T *rhsq, const T *D, const T *g,
              const T *jinv, cudaStream_t s) {
  using C = LoCfg<T, NQ>;
  auto kern = volume_lo_kernel<T, NQ>;
  if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::SMEM) !=
      cudaSuccess)
    return LFB_ERR_CUDA;
  int dev = 0, sms = 0, per_sm = 0;
  if (cudaGetDevice(&dev) != cudaSuccess ||
      cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess ||
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, C::THREADS, C::SMEM) !=
          cudaSuccess ||
      per_sm < 1)
    return LFB_ERR_LAUNCH;
  const int64_t slots = (int64_t)sms * per_sm;
  const int64_t grid = ne < slots ? ne : slots;
  if (grid == 0) return LFB_OK;
  kern<<<(unsigned)grid, C::THREADS, C::SMEM, s>>>(ne, p0, R, gam, q, rhsq, D, g, jinv);
  LFB_CHECK_LAUNCH();
  return LFB_OK;
}

template <typename T>
int dispatch_lo(int nq, int64_t ne, T p0, T R, T gam, const T *q, T *rhsq, const T *D,
                const T *g, const T *jinv, cudaStream_t s) {
  switch (nq) {
    case 9: return launch_lo<T, 9>(ne, p0, R, gam, q, rhsq, D, g, jinv, s);
    case 10: return launch_lo<T, 10>(ne, p0, R, gam, q, rhsq, D, g, jinv, s);
    case 11: return launch_lo<T, 11>(ne, p0, R, gam, q, rhsq, D, g, jinv, s);
    case 12: return launch_lo<T, 12>(ne, p0, R, gam, q, rhsq, D, g, jinv, s);
    default: return LFB_ERR_BAD_VARIANT;
  }
}

}  // namespace

bool lo_available(int dtype_bytes, int nq) {
  return (dtype_bytes == 4 || dtype_bytes == 8) && nq >= 9 && nq <= 12;
}

int volume_lo_f64(int nq, int64_t ne, double p0, double R, double gam, const double *q,
                  double *rhsq, const double *D, const double *g, const double *jinv,
                  cudaStream_t s) {
  if (!lo_available(8, nq)) return LFB_ERR_BAD_VARIANT;
  return dispatch_lo<double>(nq, ne, p0, R, gam, q, rhsq, D, g, jinv, s);
}

int volume_lo_f32(int nq, int64_t ne, float p0, float R, float gam, const float *q,
                  float *rhsq, const float *D, const float *g, const float *jinv,
                  cudaStream_t s) {
  if (!lo_available(4, nq)) return LFB_ERR_BAD_VARIANT;
  return dispatch_lo<float>(nq, ne, p0, R, gam, q, rhsq, D, g, jinv, s);
}

}  // namespace lfb
