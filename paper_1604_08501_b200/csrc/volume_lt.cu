// LFB_VARIANT_LINES, fp64 storage, Nq 9..12 — "line-tile" kernel: the R
// derivative contracted on the fp64 tensor pipe from the point owner's own
// registers, S and T exchanged through swizzled shared tiles, ONE CTA
// barrier per field.
//
// Why this shape: at Nq >= 9 one element's q + g (99 KB at
// Nq=9, 235 KB at Nq=12) no longer fits the tc kernel's staged virtual-cube
// scheme, and the first `lines` kernel — all three directions as line GEMMs
// through shared memory, state in shared memory, two barriers per field —
// was latency-bound at 0.42-0.47 of HBM (profiles/r01_lines_nq12_f64.json:
// 31 % issue active, 34 % bank-conflict wavefronts).
//
// Decomposition (one element per CTA iteration, persistent grid, one CTA of
// W warps per SM):
//   * lines (j,k) are cut into tiles of 8; warp w owns R tile w: lane
//     (g = lane/4, c = lane%4) owns the points (i = c + 4t, line 8w+g),
//     t < KS = ceil(Nq/4) — stride-4 columns, so every global access of a
//     warp is 8 lines x 32 contiguous bytes (full sectors);
//   * R (contract i) is an m8n8k4 GEMM with M = the 8 lines, K = i in the
//     permuted order (c + 4t), N = output i: the A fragment (row g, k-col c
//     of step t) is exactly F_r at the lane's own point t, and the output
//     column permutation (col 2c+s of n-tile u -> i = c + 4(2u+s)) lands
//     every result on its owner — no data movement at all;
//   * S (contract j) and T (contract k) cross lines: the owners park F_s and
//     F_t of one field in two shared tiles X[n][line'] (n = the contracted
//     index, line' = (k,i) resp. (j,i) with i padded to LP = 4 KS), the
//     S/T tile owners run C[out][line'] = D(out,n) X[n][line'] as m8n8k4
//     GEMMs (A = D fragments in registers, B = 4 tile rows x 8 lines), and
//     write C back to two more tiles that the point owners read;
//   * tiles are double-buffered across fields, so one __syncthreads per
//     field separates "flux written" from "GEMM reads it", and the owners
//     combine field b-1 (rhsq += Jinv (R + S + T)) right after the barrier of
//     field b (9 barriers per element);
//   * row stride RS and an XOR swizzle of the 16-byte unit within each
//     128-byte row segment make the B-fragment reads, the C-fragment pair
//     writes and the owners' accesses bank-conflict-free for Nq 11, 12
//     (~13 % extra wavefronts at Nq 9, 10; modelled by tools/lt_banks.py).
// HBM traffic is the 272 B/pt minimum: q, g, Jinv read once from HBM (the
// per-field re-reads of q_b and g(b-1, .) hit L2), rhsq read and written
// once.

#include <stdint.h>

#include "lfb_common.cuh"
#include "lfb_math.cuh"
#include "lfb_tma.cuh"

#ifndef LT_RPW
#define LT_RPW 1
#endif
#ifndef LT_PF  // L2 prefetch of the next element's phase-1 inputs: 0 off,
#define LT_PF 2  // 1 at element start, 2 in region 6 (two fields ahead)
#endif
#ifndef LT_PF_REGION  // LT_PF = 2: the region whose end issues the prefetch
// (A/B after the stage-fed phase 1, profiles/r02b_lt_pf_ab.txt: regions 1..7
// -> 3 leads, Nq 12 / 11 0.623 / 0.496 at 6 -> 0.674 / 0.512)
#define LT_PF_REGION 3
#endif
#ifndef LT_P1S  // phase 1 reads q_1, q_4, g(0, .) from the field / g stages
#define LT_P1S 1
#endif
#ifndef LT_HINT  // L2 policies: phase-1 reads evict_last, stage re-reads evict_first
#define LT_HINT 0
#endif

namespace lfb {
namespace {

__device__ __forceinline__ void lt_dmma(double &d0, double &d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

template <int NQ, int RPW>
struct LtCfg {
  static constexpr int NPT = NQ * NQ * NQ;
  static constexpr int KS = (NQ + 3) / 4;            // own points per lane per tile = k-steps
  static constexpr int NTL = (KS + 1) / 2;           // R output n-tiles
  static constexpr int MT = (NQ + 7) / 8;            // S/T output m-tiles
  static constexpr int LP = 4 * KS;                  // S/T line' stride (i padded)
  static constexpr int LPJ = (NQ % 2) ? NQ + 1 : NQ; // R line stride in j (dummy j = NQ)
  static constexpr int NLR = NQ * LPJ;               // R lines incl. dummies
  static constexpr int RT = (NLR + 7) / 8;           // R tiles
  static constexpr int NT = (NQ * LP + 7) / 8;       // S/T line' tiles
  // RPW R tiles per warp (1: more warps; 2: more registers per thread)
  static constexpr int W = (RT + RPW - 1) / RPW;     // warps per CTA
  static constexpr int JOBS = 2 * NT;                // S and T line' tiles
  static constexpr int JPW = (JOBS + W - 1) / W;     // GEMM jobs per warp
  static constexpr int THREADS = 32 * W;
  // CTAs per SM the registers are budgeted for: one element per CTA, so the
  // small-Nq instances (4..8 warps) run several CTAs per SM
  static constexpr int MINB = NQ >= 9 ? 1 : NQ >= 7 ? 2 : 3;
  static constexpr int ROWS = 4 * KS;                // tile rows (rows >= NQ stay zero)
  // row stride (doubles): the line' range plus the largest row offset of
  // lt_pos, in whole 128-byte segments (bank model: tools/lt_banks.py)
  static constexpr int RS = (NT * 8 + 12 + 15) / 16 * 16;
  static constexpr int TILE = ROWS * RS;
  static_assert(RS >= NT * 8, "row holds every line' tile");
  // field stage slab: a 16-byte aligned superset of one Nq^3 slab
  static constexpr int GSLAB = (NPT + 3) & ~1;
  // 2 bufs x {fS, fT, cS, cT} tiles + 2 q stages + 1 g stage (3 slabs) +
  // 3 mbarriers
  // + the per-lane D fragment tables (R: NTL x KS, S/T: MT x KS values per lane)
  static constexpr int DTAB = (NTL + MT) * KS * 32;
  static constexpr size_t SMEM =
      sizeof(double) * (8 * (size_t)TILE + 5 * (size_t)GSLAB + DTAB + 3);
};

// position of X[n][x] in a tile: row n starts 8 (n&1) + 4 ((n>>1)&1) doubles
// into its 128-byte segment, so four consecutive rows (a B fragment, an
// owner access) and two consecutive rows of 16-byte pairs (a C fragment) hit
// distinct bank groups; linear in x, so a lane's own points are base + 4t
// field processed at pipeline position p: the momentum fields (which also
// need the g(b-1, .) stage) on positions 0, 2, 4, so one g stage suffices
__device__ __forceinline__ int lt_field(int p) {
  return (p & 1) ? (p == 7 ? 7 : 4 + (p >> 1)) : (p == 6 ? 0 : 1 + (p >> 1));
}

template <int NQ>
__device__ __forceinline__ int lt_pos(int n, int x) {
  return n * LtCfg<NQ, 1>::RS + 8 * (n & 1) + 4 * ((n >> 1) & 1) + x;
}

template <int NQ, int RPW>
__global__ void __launch_bounds__(LtCfg<NQ, RPW>::THREADS, LtCfg<NQ, RPW>::MINB)
    volume_lt_kernel(int64_t ne, double p0, double R, double gam, const double *__restrict__ q,
                     double *__restrict__ rhsq, const double *__restrict__ D,
                     const double *__restrict__ g, const double *__restrict__ jinv) {
  using C = LtCfg<NQ, RPW>;
  constexpr int NPT = C::NPT, KS = C::KS, NTL = C::NTL, MT = C::MT, LP = C::LP;
  constexpr int TILE = C::TILE, NT = C::NT, JPW = C::JPW, W = C::W, GSLAB = C::GSLAB;
  extern __shared__ __align__(16) double lt_sm[];
  // tile (buffer b&1, kind): 0 F_s, 1 F_t, 2 C_s, 3 C_t
  auto tile = [&](int buf, int kind) { return lt_sm + (buf * 4 + kind) * TILE; };
  // q stages [2][GSLAB] (the field at position p, bulk-copied two regions
  // ahead) and ONE g stage [3][GSLAB] (g(b-1, d) of the momentum fields,
  // which sit at positions 0, 2, 4 — lt_field — one region ahead)
  double *qst = lt_sm + 8 * TILE;
  double *gst = qst + 2 * GSLAB;
  // D fragments, one value per lane: brt[(u*KS + t)*32 + lane], adt[(mt*KS + t)*32 + lane]
  double *brt = gst + 3 * GSLAB, *adt = brt + NTL * KS * 32;
  uint64_t *fbar = reinterpret_cast<uint64_t *>(brt + C::DTAB);  // q0, q1, g

  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int gq = lane >> 2, c = lane & 3;
  const double Rp0 = R / p0;

  for (int x = tid; x < 8 * TILE; x += C::THREADS) lt_sm[x] = 0.0;
  if (tid == 0) {
    mbar_init(&fbar[0], 1);
    mbar_init(&fbar[1], 1);
    mbar_init(&fbar[2], 1);
    mbar_init_fence();
  }

  // ---- point ownership: R tile r = RPW w + m, line L = 8 r + g = (j, k),
  //      points i = c + 4t ---------------------------------------------------
  bool vt[RPW][KS];
  int pofs[RPW];
#pragma unroll
  for (int m = 0; m < RPW; ++m) {
    const int L = 8 * (RPW * w + m) + gq;
    const int jj = L % C::LPJ, kk = L / C::LPJ;
    const bool own = L < C::NLR && jj < NQ;
    pofs[m] = own ? kk * NQ * NQ + jj * NQ : 0;
#pragma unroll
    for (int t = 0; t < KS; ++t) vt[m][t] = own && c + 4 * t < NQ;
  }
  // smem positions of own point (m, t) in the S and T layouts: base + 4t
  int sS0[RPW], sT0[RPW];
#pragma unroll
  for (int m = 0; m < RPW; ++m) {
    const int L = 8 * (RPW * w + m) + gq, jj = L % C::LPJ, kk = L / C::LPJ;
    sS0[m] = lt_pos<NQ>(jj, kk * LP + c);
    sT0[m] = lt_pos<NQ>(kk, jj * LP + c);
  }
  auto posS = [&](int m, int t) { return sS0[m] + 4 * t; };
  auto posT = [&](int m, int t) { return sT0[m] + 4 * t; };
  // ---- D fragments (D[n*NQ + i] = D(i, n)) --------------------------------
  //   R: B[k-row c][n-col g] at step t = D(out = slot(u, g), n = c + 4t),
  //      slot(u, x) = c' + 4(2u + s') for x = 2c' + s';
  //   S/T: A[g][c] at step t, m-tile mt = D(out = 8 mt + g, n = 4t + c)
  //   (kept in shared memory: one LDS per use instead of 2 (NTL + MT) KS
  //   registers held through the kernel)
  if (w == 0) {
#pragma unroll
    for (int u = 0; u < NTL; ++u)
#pragma unroll
      for (int t = 0; t < KS; ++t) {
        const int out = (gq >> 1) + 4 * (2 * u + (gq & 1)), n = c + 4 * t;
        brt[(u * KS + t) * 32 + lane] = (out < NQ && n < NQ) ? __ldg(D + n * NQ + out) : 0.0;
      }
#pragma unroll
    for (int mt = 0; mt < MT; ++mt)
#pragma unroll
      for (int t = 0; t < KS; ++t) {
        const int out = 8 * mt + gq, n = 4 * t + c;
        adt[(mt * KS + t) * 32 + lane] = (out < NQ && n < NQ) ? __ldg(D + n * NQ + out) : 0.0;
      }
  }
  __syncthreads();

  // bulk copies (thread 0) of a slab's 16-byte aligned superset (the
  // launcher never hands this kernel an element whose superset would leave
  // the arrays)
  auto slab_bytes = [&](const double *a0) {
    const uintptr_t lo = reinterpret_cast<uintptr_t>(a0) & ~(uintptr_t)15;
    const uintptr_t hi = (reinterpret_cast<uintptr_t>(a0 + NPT) + 15) & ~(uintptr_t)15;
    return (uint32_t)(hi - lo);
  };
  auto slab_copy = [&](double *dst, const double *a0, uint64_t *bar) {
    const void *src = reinterpret_cast<const void *>(reinterpret_cast<uintptr_t>(a0) & ~(uintptr_t)15);
    if (LT_HINT)
      bulk_g2s_hint(dst, src, slab_bytes(a0), bar, l2_evict_first_policy());
    else
      bulk_g2s(dst, src, slab_bytes(a0), bar);
  };
  auto issue_q = [&](int64_t e, int p) {  // q of the field at position p -> q stage p & 1
    const double *a0 = q + (e * 8 + lt_field(p)) * NPT;
    mbar_expect_tx(&fbar[p & 1], slab_bytes(a0));
    slab_copy(qst + (p & 1) * GSLAB, a0, &fbar[p & 1]);
  };
  auto issue_g = [&](int64_t e, int b) {  // g(b-1, d), d = 0..2 -> the g stage
    uint32_t total = 0;
#pragma unroll
    for (int d = 0; d < 3; ++d) total += slab_bytes(g + (e * 9 + 3 * d + b - 1) * NPT);
    mbar_expect_tx(&fbar[2], total);
#pragma unroll
    for (int d = 0; d < 3; ++d) slab_copy(gst + d * GSLAB, g + (e * 9 + 3 * d + b - 1) * NPT, &fbar[2]);
  };
  // value o of a slab starting at global a0, from its stage copy st (the
  // copy starts at the 16-byte unit below a0; the launcher never hands this
  // kernel an element whose aligned superset would leave the arrays)
  auto staged = [](const double *a0, const double *st, int o) {
    const int sh = (NPT & 1) ? (int)((reinterpret_cast<uintptr_t>(a0) & 15) >> 3) : 0;
    return st[sh + o];
  };

  // ---- software pipeline over the stream of (element, field) pairs -------
  // Region f of element e (one CTA barrier at its end) does three
  // independent things, so one warp's instruction stream interleaves them:
  //   A  fluxes of field f -> F tiles [f&1], R contraction (registers);
  //   B  S/T line GEMMs of field f-1 (of the previous element for f = 0):
  //      F tiles [(f-1)&1] -> C tiles [(f-1)&1];
  //   C  combine of field f-2 (the previous element's fields 6, 7 for
  //      f = 0, 1): rhsq += Jinv (R + S + T) from C tiles [(f-2)&1].
  // Phase 1 of element e (its point-wise state) opens region 0 of e.
  // Buffer hazards are one barrier apart: F[f&1] is written in region f and
  // read in f+1, last read (field f-2) in f-1; C[(f-1)&1] is written in f and
  // read in f+1, last read (field f-3) in f-1. The stage of field f+2 is
  // issued right after the barrier of region f (its buffer was read in f).
  auto gemm_st = [&](int buf) {
#pragma unroll
    for (int jb = 0; jb < JPW; ++jb) {
      const int job = w + jb * W;
      if (job < 2 * NT) {
        const int kind = job >= NT, lt = kind ? job - NT : job;
        const double *X = tile(buf, kind);
        double *Co = tile(buf, 2 + kind);
        double bv[KS];
#pragma unroll
        for (int t = 0; t < KS; ++t) bv[t] = X[lt_pos<NQ>(4 * t + c, 8 * lt + gq)];
#pragma unroll
        for (int mt = 0; mt < MT; ++mt) {
          double c0 = 0.0, c1 = 0.0;
#pragma unroll
          for (int t = 0; t < KS; ++t) lt_dmma(c0, c1, adt[(mt * KS + t) * 32 + lane], bv[t]);
          if (8 * mt + gq < NQ)
            *reinterpret_cast<double2 *>(Co + lt_pos<NQ>(8 * mt + gq, 8 * lt + 2 * c)) =
                make_double2(c0, c1);
        }
      }
    }
  };
  // rhsq_f += Jinv (R + S + T) at the own points: part = rhsq_f + Jinv R_f
  auto combine = [&](int buf, double *rf, const double (&part)[RPW][KS],
                     const double (&jw)[RPW][KS]) {
    const double *pS = tile(buf, 2), *pT = tile(buf, 3);
#pragma unroll
    for (int m = 0; m < RPW; ++m)
#pragma unroll
      for (int t = 0; t < KS; ++t)
        if (vt[m][t])
          rf[pofs[m] + 4 * t] = fma(jw[m][t], pS[posS(m, t)] + pT[posT(m, t)], part[m][t]);
  };

  // phase-1 reads of values the field stages read again keep their L2 lines
  const uint64_t keep = LT_HINT ? l2_evict_last_policy() : 0;
  auto ld1 = [&](const double *p) { return LT_HINT ? ldg_hint(p, keep) : __ldg(p); };

  int64_t e = blockIdx.x;
  if (tid == 0 && e < ne) {
    issue_q(e, 0);
    issue_q(e, 1);
    issue_g(e, lt_field(0));
  }
  uint32_t gpar = 0;
  double part[2][RPW][KS];  // rhsq_f + Jinv R_f of fields f-1, f-2 (by f & 1)
  double rhn[RPW][KS];      // rhsq of the next field, loaded one region ahead
  if (e < ne) {
#pragma unroll
    for (int m = 0; m < RPW; ++m)
#pragma unroll
      for (int t = 0; t < KS; ++t)
        rhn[m][t] = vt[m][t] ? rhsq[(e * 8 + lt_field(0)) * NPT + c + pofs[m] + 4 * t] : 0.0;
  }
  double jvp[RPW][KS];      // Jinv of the previous element (its fields 6, 7)
  double *rep = nullptr;    // rhsq + c of the previous element
  for (; e < ne; e += gridDim.x) {
    const double *qe = q + e * 8 * NPT + c;
    const double *ge = g + e * 9 * NPT + c;
    double *re = rhsq + e * 8 * NPT + c;
    const int64_t en = e + gridDim.x;
    if (LT_PF == 1 && tid == 32 && en < ne) {
      // next element's phase-1 inputs into L2: rho, U, Theta, g, Jinv
      prefetch_l2_range(q + en * 8 * NPT, 5ull * NPT * sizeof(double));
      prefetch_l2_range(g + en * 9 * NPT, 9ull * NPT * sizeof(double));
      prefetch_l2_range(jinv + en * NPT, 1ull * NPT * sizeof(double));
    }

    // ---- phase 1: W_d = V_d / rho (V_d = sum_a g(a,d) U_a), p, Jinv ----------
    // every flux is then F_d,b = W_d q_b (+ g(b-1,d) p for b = 1..3); q_0 = rho
    // (LT_P1S: U_0 = q_1 and Theta = q_4 — the fields at positions 0, 1 —
    // and g(0, d) — the g stage of position 0 — are read from their stage
    // copies, 5 of the 14 phase-1 global loads per point)
    if (LT_P1S) {
      mbar_wait(&fbar[0], 0u);
      mbar_wait(&fbar[1], 0u);
      mbar_wait(&fbar[2], gpar);
    }

    double Wd[3][RPW][KS], pp[RPW][KS], jv[RPW][KS];
#pragma unroll
    for (int m = 0; m < RPW; ++m) {
      double rho[KS], th[KS], U[3][KS];
#pragma unroll
      for (int t = 0; t < KS; ++t) {
        const int o = pofs[m] + 4 * t;
        rho[t] = vt[m][t] ? ld1(qe + o) : 1.0;
        jv[m][t] = vt[m][t] ? __ldg(jinv + e * NPT + c + o) : 0.0;
        if (LT_P1S) {
          th[t] = vt[m][t] ? staged(q + (e * 8 + 4) * NPT, qst + GSLAB, o + c) : 1.0;
          U[0][t] = vt[m][t] ? staged(q + (e * 8 + 1) * NPT, qst, o + c) : 0.0;
        } else {
          th[t] = vt[m][t] ? __ldg(qe + 4 * NPT + o) : 1.0;
          U[0][t] = vt[m][t] ? ld1(qe + NPT + o) : 0.0;
        }
#pragma unroll
        for (int a = 1; a < 3; ++a) U[a][t] = vt[m][t] ? ld1(qe + (1 + a) * NPT + o) : 0.0;
      }
#pragma unroll
      for (int d = 0; d < 3; ++d) {
        double gv[3][KS];
#pragma unroll
        for (int t = 0; t < KS; ++t)
#pragma unroll
          for (int a = 0; a < 3; ++a)
            gv[a][t] = !vt[m][t] ? 0.0
                       : (LT_P1S && a == 0)
                           ? staged(g + (e * 9 + 3 * d) * NPT, gst + d * GSLAB, pofs[m] + c + 4 * t)
                           : ld1(ge + (3 * d + a) * NPT + pofs[m] + 4 * t);
#pragma unroll
        for (int t = 0; t < KS; ++t)
          Wd[d][m][t] = fma(gv[0][t], U[0][t], fma(gv[1][t], U[1][t], gv[2][t] * U[2][t]));
      }
#pragma unroll
      for (int t = 0; t < KS; ++t) {
        const double rinv = fast_rcp(rho[t]);
#pragma unroll
        for (int d = 0; d < 3; ++d) Wd[d][m][t] *= rinv;
        pp[m][t] = p0 * pos_pow(Rp0 * th[t], gam);
      }
    }

#pragma unroll
    for (int f = 0; f < 8; ++f) {
      // ---- A: fluxes of field f, R contraction ------------------------------
      const int b = lt_field(f);            // the field at position f
      const bool mom = b >= 1 && b <= 3;  // momentum field: pressure term g(b-1, d) p
      // rhsq of field f arrived during region f-1; issue field f+1's (the next
      // element's field 0 after f = 7) and pull field f+2's slab into L2
      double rh[RPW][KS];
      {
        const int bn = lt_field((f + 1) & 7);
        double *rnext = f < 7 ? re + bn * NPT : rhsq + (en * 8 + bn) * NPT + c;
        const bool have = f < 7 || en < ne;
#pragma unroll
        for (int m = 0; m < RPW; ++m)
#pragma unroll
          for (int t = 0; t < KS; ++t) {
            rh[m][t] = rhn[m][t];
            rhn[m][t] = (have && vt[m][t]) ? rnext[pofs[m] + 4 * t] : 0.0;
          }
        if (tid == 64) {
          if (f + 2 < 8)
            prefetch_l2_range(rhsq + (e * 8 + lt_field(f + 2)) * NPT, (uint64_t)NPT * sizeof(double));
          else if (en < ne)
            prefetch_l2_range(rhsq + (en * 8 + lt_field(f - 6)) * NPT, (uint64_t)NPT * sizeof(double));
        }
      }
      mbar_wait(&fbar[f & 1], (uint32_t)((f >> 1) & 1));  // 4 fills per buffer per element
      if (mom) {
        mbar_wait(&fbar[2], gpar);
        gpar ^= 1u;
      }
      double pnew[RPW][KS];  // part of field f (slot f & 1 still holds field f-2)
      {
        double *fS = tile(f & 1, 0), *fT = tile(f & 1, 1);
        const double *st = qst + (f & 1) * GSLAB;
        const double *qslab = q + (e * 8 + b) * NPT;
#pragma unroll
        for (int m = 0; m < RPW; ++m) {
          double Fr[KS];
#pragma unroll
          for (int t = 0; t < KS; ++t) {
            const int o = pofs[m] + c + 4 * t;  // point index in the slab
            const double qv = vt[m][t] ? staged(qslab, st, o) : 0.0;
            double fr = Wd[0][m][t] * qv, fs = Wd[1][m][t] * qv, ft = Wd[2][m][t] * qv;
            if (mom && vt[m][t]) {
              double gd[3];
#pragma unroll
              for (int d = 0; d < 3; ++d)
                gd[d] = staged(g + (e * 9 + 3 * d + b - 1) * NPT, gst + d * GSLAB, o);
              fr = fma(gd[0], pp[m][t], fr);
              fs = fma(gd[1], pp[m][t], fs);
              ft = fma(gd[2], pp[m][t], ft);
            }
            Fr[t] = vt[m][t] ? fr : 0.0;
            if (vt[m][t]) {
              fS[posS(m, t)] = fs;
              fT[posT(m, t)] = ft;
            }
          }
          double cr[NTL][2];
#pragma unroll
          for (int u = 0; u < NTL; ++u) {
            cr[u][0] = 0.0;
            cr[u][1] = 0.0;
#pragma unroll
            for (int t = 0; t < KS; ++t)
              lt_dmma(cr[u][0], cr[u][1], Fr[t], brt[(u * KS + t) * 32 + lane]);
          }
#pragma unroll
          for (int t = 0; t < KS; ++t)
            pnew[m][t] = fma(jv[m][t], cr[t >> 1][t & 1], rh[m][t]);
        }
      }
      // ---- B: S/T GEMMs of the previous field --------------------------------
      if (f >= 1 || rep != nullptr) gemm_st((f + 1) & 1);
      // ---- C: combine the field before that ---------------------------------
      if (f >= 2) combine(f & 1, re + lt_field(f - 2) * NPT, part[f & 1], jv);
      else if (rep != nullptr) combine(f & 1, rep + lt_field(6 + f) * NPT, part[f & 1], jvp);
#pragma unroll
      for (int m = 0; m < RPW; ++m)
#pragma unroll
        for (int t = 0; t < KS; ++t) part[f & 1][m][t] = pnew[m][t];
      if (LT_PF == 2 && f == LT_PF_REGION && tid == 32 && en < ne) {
        prefetch_l2_range(q + en * 8 * NPT, 5ull * NPT * sizeof(double));
        prefetch_l2_range(g + en * 9 * NPT, 9ull * NPT * sizeof(double));
        prefetch_l2_range(jinv + en * NPT, 1ull * NPT * sizeof(double));
      }
      __syncthreads();
      if (tid == 0) {  // q stage of position f+2 (or the next element's 0, 1), g stages
        fence_proxy_async();
        if (f + 2 < 8) issue_q(e, f + 2);
        else if (en < ne) issue_q(en, f - 6);
        if (f == 0 || f == 2) issue_g(e, lt_field(f + 2));
        else if (f == 4 && en < ne) issue_g(en, lt_field(0));
      }
    }
#pragma unroll
    for (int m = 0; m < RPW; ++m)
#pragma unroll
      for (int t = 0; t < KS; ++t) jvp[m][t] = jv[m][t];
    rep = re;
  }
  // ---- drain: GEMMs of the last field, combine of the last two ------------
  if (rep != nullptr) {
    gemm_st(1);
    combine(0, rep + lt_field(6) * NPT, part[0], jvp);
    __syncthreads();
    combine(1, rep + lt_field(7) * NPT, part[1], jvp);
  }
}

template <int NQ, int RPW>
int launch_lt(int64_t ne, double p0, double R, double gam, const double *q, double *rhsq,
              const double *D, const double *g, const double *jinv, cudaStream_t s) {
  using C = LtCfg<NQ, RPW>;
  auto kern = volume_lt_kernel<NQ, RPW>;
  if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::SMEM) !=
      cudaSuccess)
    return LFB_ERR_CUDA;
  int dev = 0, sms = 0;
  if (cudaGetDevice(&dev) != cudaSuccess ||
      cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess)
    return LFB_ERR_CUDA;
  int per_sm = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, C::THREADS, C::SMEM) !=
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

}  // namespace

bool lt32_available(int nq);
bool lt_available(int dtype_bytes, int nq) {
  return dtype_bytes == 8 ? (nq >= 5 && nq <= 12) : (dtype_bytes == 4 && lt32_available(nq));
}

int volume_col_f64(int, int64_t, double, double, double, const double *, double *,
                   const double *, const double *, const double *, cudaStream_t);

namespace {
int dispatch_lt(int nq, int64_t ne, double p0, double R, double gam, const double *q,
                double *rhsq, const double *D, const double *g, const double *jinv,
                cudaStream_t s) {
  switch (nq) {
    case 5: return launch_lt<5, LT_RPW>(ne, p0, R, gam, q, rhsq, D, g, jinv, s);
    case 6: return launch_lt<6, LT_RPW>(ne, p0, R, gam, q, rhsq, D, g, jinv, s);
    case 7: return launch_lt<7, LT_RPW>(ne, p0, R, gam, q, rhsq, D, g, jinv, s);
    case 8: return launch_lt<8, LT_RPW>(ne, p0, R, gam, q, rhsq, D, g, jinv, s);
    case 9: return launch_lt<9, LT_RPW>(ne, p0, R, gam, q, rhsq, D, g, jinv, s);
    case 10: return launch_lt<10, LT_RPW>(ne, p0, R, gam, q, rhsq, D, g, jinv, s);
    case 11: return launch_lt<11, LT_RPW>(ne, p0, R, gam, q, rhsq, D, g, jinv, s);
    case 12: return launch_lt<12, LT_RPW>(ne, p0, R, gam, q, rhsq, D, g, jinv, s);
    default: return LFB_ERR_BAD_VARIANT;
  }
}
}  // namespace

// The bulk copies need 16-byte aligned q / g (else: the column kernel). For
// odd Nq a slab is not a 16-byte multiple and the last element — whose
// aligned superset would leave the arrays — goes to the column kernel.
int volume_lt_f64(int nq, int64_t ne, double p0, double R, double gam, const double *q,
                  double *rhsq, const double *D, const double *g, const double *jinv,
                  cudaStream_t s) {
  if (!lt_available(8, nq)) return LFB_ERR_BAD_VARIANT;
  if ((reinterpret_cast<uintptr_t>(q) | reinterpret_cast<uintptr_t>(g)) & 15)
    return volume_col_f64(nq, ne, p0, R, gam, q, rhsq, D, g, jinv, s);
  const int64_t npt = (int64_t)nq * nq * nq;
  const int64_t n = ((npt * 8) % 16 && ne > 0) ? ne - 1 : ne;
  int rc = n > 0 ? dispatch_lt(nq, n, p0, R, gam, q, rhsq, D, g, jinv, s) : LFB_OK;
  if (rc != LFB_OK || n == ne) return rc;
  return volume_col_f64(nq, ne - n, p0, R, gam, q + n * 8 * npt, rhsq + n * 8 * npt, D,
                        g + n * 9 * npt, jinv + n * npt, s);
}

}  // namespace lfb
