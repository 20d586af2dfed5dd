// LFB_VARIANT_LINES — large Nq (9..13): the three derivatives as DMMA
// "line GEMMs" over shared-memory flux tiles.
//
// At Nq >= 9 an element no longer fits the tc kernel's scheme (one element's
// q+g is 99 KB at Nq=9 and 235 KB at Nq=12 in fp64, and the virtual Nq=8
// planes do not cover it). Here every direction is treated as a GEMM over
// flattened lines, for one field at a time:
//   R:  C[i][line(j,k)] = sum_n D(i,n) F_r[n][line]      (lines = Nq^2)
//   S:  C[j][line(i,k)] = sum_n D(j,n) F_s[n][line]
//   T:  C[k][line(i,j)] = sum_n D(k,n) F_t[n][line]
// with m8n8k4 fp64 tiles: M = output position (ceil(Nq/8) tiles, rows >= Nq
// masked), N = 8 consecutive lines, K = contraction index in steps of 4.
// Each flux tile is stored line-major with the position fastest, so one
// B-fragment load is 4 positions x 8 lines. The three results land in three
// line-major accumulators that the write-back gathers per point.
//
// Per element (one CTA of 8 warps per SM, persistent, the next element
// L2-prefetched with cp.async.bulk.prefetch.L2):
//   once:      1/rho, p, V_r, V_s, V_t per point -> shared state (q, g read
//              once from HBM);
//   per field: fluxes -> 3 tiles | barrier | DMMA line GEMMs -> 3 tiles |
//              barrier | rhsq += Jinv (R + S + T), coalesced RMW.
// HBM traffic is the 272 B/pt minimum (q_b and g are re-read per field from
// L1/L2, not HBM).

#include <stdint.h>
#include <stdlib.h>

#include "lfb_common.cuh"
#include "lfb_math.cuh"

namespace lfb {
namespace {


__device__ __forceinline__ void prefetch_l2_lines(const void *p, uint64_t bytes) {
  // 16-byte aligned superset, split into <= 32 KB requests
  uintptr_t lo = reinterpret_cast<uintptr_t>(p) & ~(uintptr_t)15;
  const uintptr_t hi = (reinterpret_cast<uintptr_t>(p) + bytes + 15) & ~(uintptr_t)15;
  while (lo < hi) {
    const uint32_t n = (uint32_t)((hi - lo) > 32768 ? 32768 : (hi - lo));
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(lo), "r"(n) : "memory");
    lo += n;
  }
}

// L2 eviction-priority loads: an element's q and g are read in the state
// pass and re-read (last use) in the per-field passes; keeping the first
// touch evict_last and the last touch evict_first keeps the re-reads in L2
// instead of HBM (profiles/r01_lines_l2.txt).
__device__ __forceinline__ uint64_t l2_policy(bool last) {
  uint64_t p;
  if (last)
    asm("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  else
    asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ double ldh(const double *p, uint64_t pol) {
  double v;
  asm volatile("ld.global.nc.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v) : "l"(p), "l"(pol));
  return v;
}
__device__ __forceinline__ float ldh(const float *p, uint64_t pol) {
  float v;
  asm volatile("ld.global.nc.L2::cache_hint.f32 %0, [%1], %2;" : "=f"(v) : "l"(p), "l"(pol));
  return v;
}
__device__ __forceinline__ double ldh_rw(const double *p, uint64_t pol) {
  double v;
  asm volatile("ld.global.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v) : "l"(p), "l"(pol));
  return v;
}
__device__ __forceinline__ float ldh_rw(const float *p, uint64_t pol) {
  float v;
  asm volatile("ld.global.L2::cache_hint.f32 %0, [%1], %2;" : "=f"(v) : "l"(p), "l"(pol));
  return v;
}

__device__ __forceinline__ void dmma_ln(double &d0, double &d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

template <typename T>
__device__ __forceinline__ void scalars(double rho, double th, double p0, double Rp0, double gam,
                                        double &rinv, double &p) {
  if constexpr (sizeof(T) == 4) {
    rinv = (double)__frcp_rn((float)rho);
    p = p0 * (double)exp2f((float)gam * log2f((float)Rp0 * (float)th));
  } else {
    rinv = fast_rcp(rho);
    p = p0 * pos_pow(Rp0 * th, gam);
  }
}

// threads per CTA: 16 warps for the large tiles (1 CTA/SM by shared
// memory), 8 warps x 2 CTAs/SM where two elements' tiles fit
template <int NQ>
struct LinesCfg {
  static constexpr int THREADS = NQ >= 11 ? 512 : 256;
  static constexpr int MINB = NQ >= 11 ? 1 : 2;
};

constexpr int stride_mod16(int nq, int r1, int r2) {
  int l = nq;
  while (l % 16 != r1 && l % 16 != r2) ++l;
  return l;
}

// MODE 0: one odd line stride for every tile. MODE 1 (default): per tile
// kind, chosen for its fragment access (64-bit accesses are served 16 lanes
// = 16 double slots at a time; conflict-free iff addr mod 16 distinct):
//   flux tiles, read as B fragments (line 8lt+g, pos 4ks+c; g, c < 4 per
//     half-warp): stride = 4 or 12 mod 16 -> {12g + c} distinct;
//   accumulator tiles, written as C fragments (lines 8lt+2c(+1), pos 8mt+g):
//     stride = 2 mod 16 -> {4c + g} distinct.
// (profiles/r01_lines_banks.txt: MODE 0 makes a third of the shared
// wavefronts bank-conflict replays, but MODE 1 is slower — see launch_lines.)
// contraction index n held by lane column c at k-step ks of a line GEMM: the
// order of the K dimension is free (A = D fragments and B = flux fragments
// use the same map), so at Nq 9 it is permuted to make the B-fragment reads
// of 4 consecutive lines hit distinct banks (exhaustive search over the K
// partitions with the half-warp bank model: 2-way -> none; 0.458 -> 0.465
// of HBM); -1 = padding
__device__ __forceinline__ int lines_kidx(int nq, int ks, int c) {
  // packed 4-bit tables (15 = padding), one nibble per (ks, c)
  // (Nq 10's best map, 0xFF7654329810, measured slower: 0.483 -> 0.473)
  const uint64_t t = nq == 9 ? 0xF763F852F410ull : 0;
  if (t == 0) return 4 * ks + c;
  const int v = (int)((t >> (4 * (4 * ks + c))) & 15);
  return v == 15 ? -1 : v;
}

template <int NQ, int MODE, int TH = LinesCfg<NQ>::THREADS>
struct LinesGeom {
  static constexpr int NPT = NQ * NQ * NQ;
  static constexpr int NL = NQ * NQ;                 // lines per direction
  static constexpr int MT = (NQ + 7) / 8;            // output-position tiles
  static constexpr int KS = (NQ + 3) / 4;            // k-steps
  static constexpr int LT = (NL + 7) / 8;            // line tiles
  // MODE 0 line stride: odd, except Nq = 10 where the even stride 10 puts the
  // B-fragment reads, C-fragment writes and owner accesses on fewer
  // conflicted wavefronts (bank model 490 -> 424 / 466 -> 377 per element
  // field, tools/lines_banks.py; measured 0.467 -> 0.483 of HBM)
  static constexpr int LS0 = NQ == 10 ? 10 : (NQ | 1);
  static constexpr int LSF = MODE == 0 ? LS0 : stride_mod16(NQ, 4, 12);
  static constexpr int LSA = MODE == 0 ? LS0 : stride_mod16(NQ, 2, 2);
  static constexpr int PPT = (NPT + TH - 1) / TH;
  static constexpr int TSF = NL * LSF;               // one flux tile
  static constexpr int TSA = NL * LSA;               // one accumulator tile
};

// shared: state[5][NPT] (1/rho, p, V_r, V_s, V_t), flux[3][TSF], acc[3][TSA]
template <int NQ, int MODE>
constexpr size_t lines_smem() {
  using Gm = LinesGeom<NQ, MODE>;
  return sizeof(double) * ((size_t)5 * Gm::NPT + (size_t)3 * (Gm::TSF + Gm::TSA));
}

// TH: threads per CTA (LinesCfg default; other values are A/B instances)
template <typename T, int NQ, int MODE, int TH = LinesCfg<NQ>::THREADS>
__global__ void __launch_bounds__(TH, (TH == LinesCfg<NQ>::THREADS) ? LinesCfg<NQ>::MINB : 1)
    volume_lines_kernel(int64_t ne, double p0, double R, double gam, const T *__restrict__ q,
                        T *__restrict__ rhsq, const T *__restrict__ D, const T *__restrict__ g,
                        const T *__restrict__ jinv, int pf_mode, bool hint) {
  using Gm = LinesGeom<NQ, MODE, TH>;
  constexpr int LN_THREADS = TH;
  constexpr int NPT = Gm::NPT, NL = Gm::NL, MT = Gm::MT, KS = Gm::KS, LT = Gm::LT;
  constexpr int LSF = Gm::LSF, LSA = Gm::LSA, TSF = Gm::TSF, TSA = Gm::TSA, PPT = Gm::PPT;
  extern __shared__ __align__(16) double lsm[];
  double *st = lsm;                  // [5][NPT]
  double *fl = lsm + 5 * NPT;        // [3][TSF] line-major: fl[d][line*LSF + pos]
  double *ac = fl + 3 * TSF;         // [3][TSA] line-major: ac[d][line*LSA + pos]

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int gq = lane >> 2, c = lane & 3;
  const double Rp0 = R / p0;
  const uint64_t keep = l2_policy(hint), drop = l2_policy(false);
  auto ld1 = [&](const T *p) -> double { return hint ? (double)ldh(p, keep) : (double)__ldg(p); };
  auto ld2 = [&](const T *p) -> double { return hint ? (double)ldh(p, drop) : (double)__ldg(p); };

  // A fragments: A[g][c] = D(pos = 8 mt + g, n = 4 ks + c), zero outside [0,NQ)
  // Nq 9: the second output tile would hold 1 valid position of 8 — it goes
  // to the DFMA pipe instead (from the B fragment each lane already holds,
  // reduced over the 4 lanes of a line): 0.424 -> 0.431 of HBM. (Nq 10's two
  // tail positions spill at 128 registers and lose: 0.483 -> 0.447.)
  constexpr int TAIL = (MT == 2 && NQ == 9) ? 1 : 0;
  constexpr int MTD = TAIL ? 1 : MT;  // output tiles on the tensor pipe
  double Dt[TAIL ? TAIL : 1][KS];
#pragma unroll
  for (int r = 0; r < TAIL; ++r)
#pragma unroll
    for (int ks = 0; ks < KS; ++ks) {
      const int n = lines_kidx(NQ, ks, c);
      Dt[r][ks] = (n >= 0 && n < NQ) ? (double)__ldg(D + n * NQ + 8 + r) : 0.0;
    }
  double Da[MTD][KS];
#pragma unroll
  for (int mt = 0; mt < MTD; ++mt)
#pragma unroll
    for (int ks = 0; ks < KS; ++ks) {
      const int pos = 8 * mt + gq, n = lines_kidx(NQ, ks, c);
      Da[mt][ks] = (pos < NQ && n >= 0 && n < NQ) ? (double)__ldg(D + n * NQ + pos) : 0.0;
    }

  for (int64_t e = blockIdx.x; e < ne; e += gridDim.x) {
    const T *qe = q + e * 8 * NPT;
    const T *ge = g + e * 9 * NPT;
    const T *je = jinv + e * NPT;
    T *re = rhsq + e * 8 * NPT;
    const int64_t en = e + gridDim.x;
    if (en < ne && pf_mode > 0) {
      if (tid == 0) prefetch_l2_lines(q + en * 8 * NPT, 8ull * NPT * sizeof(T));
      if (tid == 32) prefetch_l2_lines(g + en * 9 * NPT, 9ull * NPT * sizeof(T));
      if (pf_mode > 1 && tid == 64) prefetch_l2_lines(rhsq + en * 8 * NPT, 8ull * NPT * sizeof(T));
      if (pf_mode > 1 && tid == 96) prefetch_l2_lines(jinv + en * NPT, 1ull * NPT * sizeof(T));
    }

    // Every per-point loop below is fully unrolled over the thread's PPT
    // points so its global loads are issued back to back (one L2/HBM round
    // trip per loop, not per point); rhsq of field b and q_b of field b+1
    // are loaded before the GEMM phase so their latency hides behind it.
    double jv[PPT];
#pragma unroll
    for (int m = 0; m < PPT; ++m) {
      const int pt = tid + m * LN_THREADS;
      jv[m] = (pt < NPT) ? ld2(je + pt) : 0.0;
    }
    // ---- point-wise state (q and g read once from HBM) -------------------
    // two passes so each issues all of its loads before the first use
    {
      double rho[PPT], th[PPT];
#pragma unroll
      for (int m = 0; m < PPT; ++m) {
        const int pt = tid + m * LN_THREADS;
        rho[m] = (pt < NPT) ? ld2(qe + pt) : 1.0;
        th[m] = (pt < NPT) ? ld1(qe + 4 * NPT + pt) : 1.0;
      }
#pragma unroll
      for (int m = 0; m < PPT; ++m) {
        const int pt = tid + m * LN_THREADS;
        double rinv, p;
        scalars<T>(rho[m], th[m], p0, Rp0, gam, rinv, p);
        if (pt < NPT) {
          st[pt] = rinv;
          st[NPT + pt] = p;
        }
      }
    }
#pragma unroll
    for (int d = 0; d < 3; ++d) {
      double gv[3][PPT], uv[3][PPT];
#pragma unroll
      for (int m = 0; m < PPT; ++m) {
        const int pt = tid + m * LN_THREADS;
#pragma unroll
        for (int a = 0; a < 3; ++a) {
          gv[a][m] = (pt < NPT) ? ld1(ge + (3 * d + a) * NPT + pt) : 0.0;
          uv[a][m] = (pt < NPT) ? ld1(qe + (1 + a) * NPT + pt) : 0.0;
        }
      }
#pragma unroll
      for (int m = 0; m < PPT; ++m) {
        const int pt = tid + m * LN_THREADS;
        if (pt < NPT)
          st[(2 + d) * NPT + pt] = gv[0][m] * uv[0][m] + gv[1][m] * uv[1][m] + gv[2][m] * uv[2][m];
      }
    }
    // (the flux pass below reads only the state of its own points)

    double qb[PPT];     // q_b of the field being processed (b >= 1)
    double gm[3][PPT];  // g(b-1, d) of a momentum field being processed
#pragma unroll 1
    for (int b = 0; b < 8; ++b) {
      // ---- fluxes of field b -> line-major tiles -------------------------
#pragma unroll
      for (int m = 0; m < PPT; ++m) {
        const int pt = tid + m * LN_THREADS;
        if (pt < NPT) {
          const int i = pt % NQ, j = (pt / NQ) % NQ, k = pt / (NQ * NQ);
          const double s = (b == 0) ? 1.0 : qb[m] * st[pt];
          double f[3];
#pragma unroll
          for (int d = 0; d < 3; ++d) {
            f[d] = st[(2 + d) * NPT + pt] * s;
            if (b >= 1 && b <= 3) f[d] += gm[d][m] * st[NPT + pt];
          }
          fl[0 * TSF + (k * NQ + j) * LSF + i] = f[0];  // R line (j,k), position i
          fl[1 * TSF + (k * NQ + i) * LSF + j] = f[1];  // S line (i,k), position j
          fl[2 * TSF + (j * NQ + i) * LSF + k] = f[2];  // T line (i,j), position k
        }
      }
      // loads whose latency the GEMM phase hides
      double rh[PPT];
#pragma unroll
      for (int m = 0; m < PPT; ++m) {
        const int pt = tid + m * LN_THREADS;
        rh[m] = (pt < NPT) ? (hint ? (double)ldh_rw(re + b * NPT + pt, drop) : (double)re[b * NPT + pt]) : 0.0;
        if (b < 7) qb[m] = (pt < NPT) ? ld2(qe + (b + 1) * NPT + pt) : 0.0;
        if (b < 3) {  // the next field is momentum b+1: its g(b, d)
#pragma unroll
          for (int d = 0; d < 3; ++d)
            gm[d][m] = (pt < NPT) ? ld2(ge + (3 * d + b) * NPT + pt) : 0.0;
        }
      }
      __syncthreads();

      // ---- line GEMMs on the fp64 tensor pipe -----------------------------
      // NL = 8 m + 1 (Nq 9, 13): the last line tile of each direction holds
      // one line — it goes to the DFMA pipe on the warps with the fewest
      // tiles instead of costing a full DMMA tile job (Nq 9 / 13: 0.431 /
      // 0.299 -> 0.458 / 0.328 of HBM; Nq 11, whose 16 warps were balanced,
      // lost 0.444 -> 0.424 and keeps the tile)
      constexpr bool LONE = NL % 8 == 1 && NQ != 11;
      constexpr int LTJ = LONE ? LT - 1 : LT;  // DMMA line tiles per direction
      for (int t = warp; t < 3 * LTJ; t += LN_THREADS / 32) {
        const int d = t / LTJ, lt = t % LTJ;
        const double *fd = fl + d * TSF;
        double *ad = ac + d * TSA;
        const int lineB = 8 * lt + gq;  // B column = line
        double bv[KS];                  // shared by every output-position tile
#pragma unroll
        for (int ks = 0; ks < KS; ++ks) {
          const int n = lines_kidx(NQ, ks, c);
          bv[ks] = (lineB < NL && n >= 0 && n < NQ) ? fd[lineB * LSF + n] : 0.0;
        }
        const int l0 = 8 * lt + 2 * c;
#pragma unroll
        for (int mt = 0; mt < MTD; ++mt) {
          double c0 = 0.0, c1 = 0.0;
#pragma unroll
          for (int ks = 0; ks < KS; ++ks) dmma_ln(c0, c1, Da[mt][ks], bv[ks]);
          const int pos = 8 * mt + gq;
          if (pos < NQ) {
            if (l0 < NL) ad[l0 * LSA + pos] = c0;
            if (l0 + 1 < NL) ad[(l0 + 1) * LSA + pos] = c1;
          }
        }
        if constexpr (TAIL > 0) {
          double ts[TAIL];
#pragma unroll
          for (int r = 0; r < TAIL; ++r) {
            ts[r] = 0.0;
#pragma unroll
            for (int ks = 0; ks < KS; ++ks) ts[r] = fma(Dt[r][ks], bv[ks], ts[r]);
            ts[r] += __shfl_xor_sync(0xffffffffu, ts[r], 1);
            ts[r] += __shfl_xor_sync(0xffffffffu, ts[r], 2);
          }
          if (c < TAIL && lineB < NL) ad[lineB * LSA + 8 + c] = c == 0 ? ts[0] : ts[TAIL - 1];
        }
      }
      if constexpr (LONE) {  // line NL - 1 of direction d: lane o computes output o
        constexpr int NW = LN_THREADS / 32;
        const int d = warp == NW - 1 ? 1 : warp == NW - 2 ? 0 : -1;
#pragma unroll 1
        for (int dd = d; dd >= 0 && dd < 3; dd += 2) {
          const double *fd = fl + dd * TSF + (NL - 1) * LSF;
          if (lane < NQ) {
            double acc = 0.0;
#pragma unroll
            for (int n = 0; n < NQ; ++n) acc = fma((double)__ldg(D + n * NQ + lane), fd[n], acc);
            ac[dd * TSA + (NL - 1) * LSA + lane] = acc;
          }
        }
      }
      __syncthreads();

      // ---- write-back: rhsq += Jinv (R + S + T) ----------------------------
#pragma unroll
      for (int m = 0; m < PPT; ++m) {
        const int pt = tid + m * LN_THREADS;
        if (pt < NPT) {
          const int i = pt % NQ, j = (pt / NQ) % NQ, k = pt / (NQ * NQ);
          const double v = ac[(k * NQ + j) * LSA + i] + ac[TSA + (k * NQ + i) * LSA + j] +
                           ac[2 * TSA + (j * NQ + i) * LSA + k];
          re[b * NPT + pt] = (T)(rh[m] + jv[m] * v);
        }
      }
      // the next field's flux writes touch fl only (last read before the
      // barrier above); ac is rewritten only after the next barrier
    }
    __syncthreads();  // state / fl reuse by the next element
  }
}

template <typename T, int NQ>
int launch_lines(int64_t ne, double p0, double R, double gam, const T *q, T *rhsq, const T *D,
                 const T *g, const T *jinv, cudaStream_t s) {
  // one odd tile stride (MODE 0): the per-kind conflict-free strides (MODE 1)
  // replay fewer bank conflicts (397M vs 517M at Nq=12) but need more shared
  // memory (Nq=10: one CTA/SM instead of two; Nq=13 does not fit) and were
  // 8-25 % slower; 384/768 threads per CTA also lost
  // (profiles/r01_lines_banks.txt)
  const size_t smem = lines_smem<NQ, 0>();
  auto kern = volume_lines_kernel<T, NQ, 0>;
  const int threads = LinesCfg<NQ>::THREADS;
  if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) !=
      cudaSuccess)
    return LFB_ERR_CUDA;
  int dev = 0, sms = 0;
  if (cudaGetDevice(&dev) != cudaSuccess ||
      cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess)
    return LFB_ERR_CUDA;
  int per_sm = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, threads, smem) !=
          cudaSuccess ||
      per_sm < 1)
    return LFB_ERR_LAUNCH;
  const int64_t slots = (int64_t)sms * per_sm;
  const int64_t grid = ne < slots ? ne : slots;
  if (grid == 0) return LFB_OK;
  // no L2 prefetch of the next element (a whole next element per CTA, 360 KB
  // at Nq=12 fp64, thrashes L2 against the per-field re-reads: +42 % DRAM
  // reads, -15 % speed; profiles/r01_lines_l2.txt) and L2 eviction hints on
  // the q / g / rhsq loads
  kern<<<(unsigned)grid, threads, smem, s>>>(ne, p0, R, gam, q, rhsq, D, g, jinv, 0, true);
  LFB_CHECK_LAUNCH();
  return LFB_OK;
}

template <typename T>
int dispatch_lines(int nq, int64_t ne, double p0, double R, double gam, const T *q, T *rhsq,
                   const T *D, const T *g, const T *jinv, cudaStream_t s) {
  switch (nq) {
    case 9: return launch_lines<T, 9>(ne, p0, R, gam, q, rhsq, D, g, jinv, s);
    case 10: return launch_lines<T, 10>(ne, p0, R, gam, q, rhsq, D, g, jinv, s);
    case 11: return launch_lines<T, 11>(ne, p0, R, gam, q, rhsq, D, g, jinv, s);
    case 12: return launch_lines<T, 12>(ne, p0, R, gam, q, rhsq, D, g, jinv, s);
    case 13: return launch_lines<T, 13>(ne, p0, R, gam, q, rhsq, D, g, jinv, s);
    default: return LFB_ERR_BAD_VARIANT;
  }
}

}  // namespace

bool lines_available(int dtype_bytes, int nq) {
  return (dtype_bytes == 8 || dtype_bytes == 4) && nq >= 9 && nq <= 13;
}

int volume_lines_f64(int nq, int64_t ne, double p0, double R, double gam, const double *q,
                     double *rhsq, const double *D, const double *g, const double *jinv,
                     cudaStream_t s) {
  if (!lines_available(8, nq)) return LFB_ERR_BAD_VARIANT;
  return dispatch_lines<double>(nq, ne, p0, R, gam, q, rhsq, D, g, jinv, s);
}

int volume_lines_f32(int nq, int64_t ne, float p0, float R, float gam, const float *q,
                     float *rhsq, const float *D, const float *g, const float *jinv,
                     cudaStream_t s) {
  if (!lines_available(4, nq)) return LFB_ERR_BAD_VARIANT;
  return dispatch_lines<float>(nq, ne, p0, R, gam, q, rhsq, D, g, jinv, s);
}

}  // namespace lfb
