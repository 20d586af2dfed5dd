// LFB_VARIANT_LT, fp32 storage, Nq 9..12 — the line-tile kernel on the TF32
// tensor path (mma.sync m16n8k8 .tf32, split products), two CTAs per SM.
//
// Same decomposition as the fp64 line-tile kernel (volume_lt.cu), re-cut for
// the m16n8k8 fragment:
//   * R tiles are 16 lines (j,k): lane (g, c) owns the points (i = c + 4t,
//     lines 16r + g and 16r + g + 8) — the A fragment's rows g, g+8 and its
//     k-columns c, c+4 of k-step s are exactly the lane's own points
//     t = 2s, 2s+1, and the n-tile column permutation (col 2c+s' of n-tile u
//     -> i = c + 4(2u+s')) returns every R result to its owner;
//   * S and T go through swizzled shared tiles X[n][line'] as
//     C[out][line'] = D(out, n) X[n][line'] with M = 16 outputs (one m-tile
//     covers Nq <= 16), K = n in steps of 8, N = 8 lines';
//   * fp32 accuracy on TF32 inputs: every product is split x = x_hi + x_lo
//     (x_hi = the top 19 bits, an ALU mask — no XU conversion), and
//     x_hi y_hi + x_lo y_hi + x_hi y_lo is accumulated in fp32 (3 MMAs; the
//     dropped x_lo y_lo is ~2^-22 relative);
//   * the point-wise physics runs in FP32 (rcp, exp2/log2 for p), as in the
//     fp32 column and tc32 kernels (observed parity ~3e-7, tolerance 1e-5);
//   * per field: fluxes + R | barrier | S/T GEMMs | barrier | write-back,
//     with single F/C tiles (two CTAs per SM provide the overlap that the
//     fp64 kernel gets from its software pipeline, at half the registers);
//     fields in the order 1 4 2 5 3 6 0 7 so the three momentum fields
//     (which also need g(b-1, .)) come every other field and share ONE g
//     stage loaded a field ahead;
//   * q_b slabs bulk-copied two regions ahead (2-stage ring), g(b-1, .)
//     slabs one region ahead, next element's phase-1 inputs L2-prefetched.
// Shared memory ~70 KB at Nq=12; two CTAs (two elements) per SM.

#include <stdint.h>

#include "lfb_common.cuh"
#include "lfb_tma.cuh"

namespace lfb {
namespace {

__device__ __forceinline__ void mma_tf32(float (&d)[4], const uint32_t (&a)[4],
                                         const uint32_t (&b)[2]) {
  asm volatile(
      "mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
      "{%8,%9}, {%0,%1,%2,%3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
}

// x = hi + lo, hi = x with the low 13 mantissa bits cleared (exact), lo = x - hi
__device__ __forceinline__ void split_tf32(float x, uint32_t &hi, uint32_t &lo) {
  hi = __float_as_uint(x) & 0xffffe000u;
  lo = __float_as_uint(x - __uint_as_float(hi));
}

template <int NQ>
struct Lt32Cfg {
  static constexpr int NPT = NQ * NQ * NQ;
  static constexpr int KS = (NQ + 3) / 4;            // own i-slots per lane and line
  static constexpr int NKS = (KS + 1) / 2;           // R k-steps (8 i per step) = R n-tiles
  static constexpr int SKS = (NQ + 7) / 8;           // S/T k-steps (8 n per step)
  static constexpr int LP = 4 * KS;                  // S/T line' stride (i padded)
  static constexpr int LPJ = (NQ % 2) ? NQ + 1 : NQ; // R line stride in j (dummy j = NQ)
  static constexpr int NLR = NQ * LPJ;               // R lines incl. dummies
  static constexpr int RT = (NLR + 15) / 16;         // R tiles (16 lines)
  static constexpr int NT = (NQ * LP + 7) / 8;       // S/T line' tiles
  static constexpr int W = RT;                       // warps per CTA
  static constexpr int JPW = (2 * NT + W - 1) / W;   // GEMM jobs per warp
  static constexpr int THREADS = 32 * W;
  static constexpr int MINB = W <= 6 ? 3 : 2;        // CTAs (elements) per SM
  // tile row stride (floats): the line' range plus the largest row offset,
  // rounded to whole 128-byte rows
  static constexpr int RS = (NT * 8 + 28 + 31) / 32 * 32;
  static constexpr int TILE = NQ * RS;
  static constexpr int SLAB = (NPT + 4 + 3) & ~3;    // stage slab: 16-byte aligned superset
  // D fragment tables (floats per lane): R B hi/lo [u][s][2], S/T A hi/lo [s][4]
  static constexpr int DR = NKS * NKS * 2, DA = SKS * 4;
  static constexpr int DTAB = 2 * (DR + DA) * 32;
  // 4 tiles {fS, fT, cS, cT} + 2 q stages + 1 g stage (3 slabs) + D tables
  // + 3 mbarriers
  static constexpr size_t SMEM =
      sizeof(float) * (4 * (size_t)TILE + 5 * (size_t)SLAB + DTAB) + 3 * sizeof(uint64_t);
  static_assert(KS <= 4 && SKS <= 2, "Nq <= 16");
};

// X[n][x]: each row starts at a row-dependent offset 8 (n&3) + 4 ((n>>2)&1)
// words into its 128-byte segment (so four consecutive rows — a B fragment —
// and eight consecutive rows — an owner access — hit distinct bank groups);
// linear in x, so a lane's own points are one base + 4t
template <int NQ>
__device__ __forceinline__ int lt32_pos(int n, int x) {
  return n * Lt32Cfg<NQ>::RS + 8 * (n & 3) + 4 * ((n >> 2) & 1) + x;
}

// field processed at pipeline position p: momentum fields on even positions
__device__ __forceinline__ int lt32_field(int p) {
  return (p & 1) ? (p == 7 ? 7 : 4 + (p >> 1)) : (p == 6 ? 0 : 1 + (p >> 1));
}

template <int NQ>
__global__ void __launch_bounds__(Lt32Cfg<NQ>::THREADS, Lt32Cfg<NQ>::MINB)
    volume_lt32_kernel(int64_t ne, float p0, float R, float gam, const float *__restrict__ q,
                       float *__restrict__ rhsq, const float *__restrict__ D,
                       const float *__restrict__ g, const float *__restrict__ jinv) {
  using C = Lt32Cfg<NQ>;
  constexpr int NPT = C::NPT, KS = C::KS, NKS = C::NKS, SKS = C::SKS, LP = C::LP;
  constexpr int TILE = C::TILE, NT = C::NT, JPW = C::JPW, W = C::W, SLAB = C::SLAB;
  extern __shared__ __align__(16) float l32_sm[];
  auto tile = [&](int buf, int kind) { return l32_sm + (buf * 4 + kind) * TILE; };
  float *qst = l32_sm + 4 * TILE;  // q stages [2][SLAB]
  float *gst = qst + 2 * SLAB;     // g stage [3][SLAB]
  float *drt = gst + 3 * SLAB;     // R B tables: hi [DR][32], lo [DR][32]
  float *dat = drt + 2 * C::DR * 32;  // S/T A tables: hi [DA][32], lo [DA][32]
  uint64_t *bars = reinterpret_cast<uint64_t *>(dat + 2 * C::DA * 32);  // q0, q1, g

  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int gq = lane >> 2, c = lane & 3;
  const float Rp0 = R / p0;

  for (int x = tid; x < 4 * TILE; x += C::THREADS) l32_sm[x] = 0.f;
  if (w == 0) {
    // R: B[k-row][n-col g] = D(out = slot(u, g), i = 8s + c (+4))
#pragma unroll
    for (int u = 0; u < NKS; ++u)
#pragma unroll
      for (int s = 0; s < NKS; ++s)
#pragma unroll
        for (int r = 0; r < 2; ++r) {
          const int out = 8 * u + (gq >> 1) + 4 * (gq & 1), i = 8 * s + c + 4 * r;
          const float v = (out < NQ && i < NQ) ? __ldg(D + i * NQ + out) : 0.f;
          uint32_t hi, lo;
          split_tf32(v, hi, lo);
          const int x = ((u * NKS + s) * 2 + r) * 32 + lane;
          drt[x] = __uint_as_float(hi);
          drt[C::DR * 32 + x] = __uint_as_float(lo);
        }
    // S/T: A[row][k-col] = D(out = g (+8), n = 8s + c (+4))
#pragma unroll
    for (int s = 0; s < SKS; ++s)
#pragma unroll
      for (int r = 0; r < 4; ++r) {
        const int out = gq + 8 * (r & 1), n = 8 * s + c + 4 * (r >> 1);
        const float v = (out < NQ && n < NQ) ? __ldg(D + n * NQ + out) : 0.f;
        uint32_t hi, lo;
        split_tf32(v, hi, lo);
        const int x = (s * 4 + r) * 32 + lane;
        dat[x] = __uint_as_float(hi);
        dat[C::DA * 32 + x] = __uint_as_float(lo);
      }
  }
  if (tid == 0) {
#pragma unroll
    for (int x = 0; x < 3; ++x) mbar_init(&bars[x], 1);
    mbar_init_fence();
  }

  // ---- point ownership: lines L = 16w + g + 8 rho, points i = c + 4t --------
  bool vt[2][KS];
  int pofs[2], jj[2], kk[2];
#pragma unroll
  for (int rho = 0; rho < 2; ++rho) {
    const int L = 16 * w + gq + 8 * rho;
    jj[rho] = L % C::LPJ;
    kk[rho] = L / C::LPJ;
    const bool own = L < C::NLR && jj[rho] < NQ;
    pofs[rho] = own ? kk[rho] * NQ * NQ + jj[rho] * NQ : 0;
#pragma unroll
    for (int t = 0; t < KS; ++t) vt[rho][t] = own && c + 4 * t < NQ;
  }
  const int sS0[2] = {lt32_pos<NQ>(jj[0], kk[0] * LP + c), lt32_pos<NQ>(jj[1], kk[1] * LP + c)};
  const int sT0[2] = {lt32_pos<NQ>(kk[0], jj[0] * LP + c), lt32_pos<NQ>(kk[1], jj[1] * LP + c)};
  auto posS = [&](int rho, int t) { return sS0[rho] + 4 * t; };
  auto posT = [&](int rho, int t) { return sT0[rho] + 4 * t; };
  __syncthreads();

  // ---- stages (thread 0) ---------------------------------------------------
  // a slab's 16-byte aligned superset (the launcher never hands this kernel
  // the last element of an array whose slabs are not 16-byte multiples, so
  // the superset stays inside the array)
  auto slab_bytes = [&](const float *a0) {
    const uintptr_t lo = reinterpret_cast<uintptr_t>(a0) & ~(uintptr_t)15;
    const uintptr_t hi = (reinterpret_cast<uintptr_t>(a0 + NPT) + 15) & ~(uintptr_t)15;
    return (uint32_t)(hi - lo);
  };
  auto slab_copy = [&](float *dst, const float *a0, uint64_t *bar) {
    bulk_g2s(dst, reinterpret_cast<const void *>(reinterpret_cast<uintptr_t>(a0) & ~(uintptr_t)15),
             slab_bytes(a0), bar);
  };
  auto issue_q = [&](int64_t e, int p) {  // q of the field at position p -> q stage p & 1
    const float *a0 = q + (e * 8 + lt32_field(p)) * NPT;
    mbar_expect_tx(&bars[p & 1], slab_bytes(a0));
    slab_copy(qst + (p & 1) * SLAB, a0, &bars[p & 1]);
  };
  auto issue_g = [&](int64_t e, int b) {  // g(b-1, d), d = 0..2 -> the g stage
    uint32_t total = 0;
#pragma unroll
    for (int d = 0; d < 3; ++d) total += slab_bytes(g + (e * 9 + 3 * d + b - 1) * NPT);
    mbar_expect_tx(&bars[2], total);
#pragma unroll
    for (int d = 0; d < 3; ++d) slab_copy(gst + d * SLAB, g + (e * 9 + 3 * d + b - 1) * NPT, &bars[2]);
  };

  auto gemm_st = [&](int buf) {
    // the D fragments once per field (not per job)
    uint32_t ah[SKS][4], al[SKS][4];
#pragma unroll
    for (int s = 0; s < SKS; ++s)
#pragma unroll
      for (int r = 0; r < 4; ++r) {
        ah[s][r] = __float_as_uint(dat[(s * 4 + r) * 32 + lane]);
        al[s][r] = __float_as_uint(dat[C::DA * 32 + (s * 4 + r) * 32 + lane]);
      }
#pragma unroll
    for (int jb = 0; jb < JPW; ++jb) {
      const int job = w + jb * W;
      if (job < 2 * NT) {
        const int kind = job >= NT, lt = kind ? job - NT : job;
        const float *X = tile(buf, kind);
        float *Co = tile(buf, 2 + kind);
        float acc[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
        for (int s = 0; s < SKS; ++s) {
          uint32_t bh[2], bl[2];
#pragma unroll
          for (int r = 0; r < 2; ++r) {
            const int n = 8 * s + c + 4 * r;
            const float v = n < NQ ? X[lt32_pos<NQ>(n, 8 * lt + gq)] : 0.f;
            split_tf32(v, bh[r], bl[r]);
          }
          mma_tf32(acc, ah[s], bh);
          mma_tf32(acc, al[s], bh);
          mma_tf32(acc, ah[s], bl);
        }
        if (gq < NQ)
          *reinterpret_cast<float2 *>(Co + lt32_pos<NQ>(gq, 8 * lt + 2 * c)) =
              make_float2(acc[0], acc[1]);
        if (gq + 8 < NQ)
          *reinterpret_cast<float2 *>(Co + lt32_pos<NQ>(gq + 8, 8 * lt + 2 * c)) =
              make_float2(acc[2], acc[3]);
      }
    }
  };
  int64_t e = blockIdx.x;
  if (tid == 0 && e < ne) {
    issue_q(e, 0);
    issue_q(e, 1);
    issue_g(e, lt32_field(0));
  }
  uint32_t gpar = 0;
  float rhn[2][KS];  // rhsq of the next field, loaded one field ahead
  if (e < ne) {
#pragma unroll
    for (int rho = 0; rho < 2; ++rho)
#pragma unroll
      for (int t = 0; t < KS; ++t)
        rhn[rho][t] = vt[rho][t] ? rhsq[(e * 8 + lt32_field(0)) * NPT + c + pofs[rho] + 4 * t]
                                 : 0.f;
  }
  for (; e < ne; e += gridDim.x) {
    const float *qe = q + e * 8 * NPT + c;
    const float *ge = g + e * 9 * NPT + c;
    float *re = rhsq + e * 8 * NPT + c;
    const int64_t en = e + gridDim.x;

    // ---- phase 1: W_d = V_d / rho, p, Jinv (FP32) ---------------------------
    // U_0 = q_1 and Theta = q_4 (the fields at positions 0, 1) and g(0, d)
    // (the g stage of position 0) come from their stage copies: 5 of the 14
    // global loads per point (the fp64 kernel's A/B: Nq 12 0.588 -> 0.624)
    mbar_wait(&bars[0], 0u);
    mbar_wait(&bars[1], 0u);
    mbar_wait(&bars[2], gpar);
    auto sh1 = [](const float *a0) { return (int)((reinterpret_cast<uintptr_t>(a0) & 15) >> 2); };
    const float *u0s = qst + sh1(q + (e * 8 + 1) * NPT) + c;
    const float *ths = qst + SLAB + sh1(q + (e * 8 + 4) * NPT) + c;
    const float *g0s[3];
#pragma unroll
    for (int d = 0; d < 3; ++d) g0s[d] = gst + d * SLAB + sh1(g + (e * 9 + 3 * d) * NPT) + c;
    float Wd[3][2][KS], pp[2][KS], jv[2][KS];
#pragma unroll
    for (int rho = 0; rho < 2; ++rho) {
#pragma unroll
      for (int t = 0; t < KS; ++t) {
        const int o = pofs[rho] + 4 * t;
        const bool v = vt[rho][t];
        const float rr = v ? __ldg(qe + o) : 1.f, th = v ? ths[o] : 1.f;
        float U[3], gv[9];
        U[0] = v ? u0s[o] : 0.f;
#pragma unroll
        for (int a = 1; a < 3; ++a) U[a] = v ? __ldg(qe + (1 + a) * NPT + o) : 0.f;
#pragma unroll
        for (int x = 0; x < 9; ++x) gv[x] = !v ? 0.f : (x % 3 == 0) ? g0s[x / 3][o] : __ldg(ge + x * NPT + o);
        jv[rho][t] = v ? __ldg(jinv + e * NPT + c + o) : 0.f;
        const float rinv = __frcp_rn(rr);
#pragma unroll
        for (int d = 0; d < 3; ++d)
          Wd[d][rho][t] =
              fmaf(gv[3 * d], U[0], fmaf(gv[3 * d + 1], U[1], gv[3 * d + 2] * U[2])) * rinv;
        pp[rho][t] = p0 * exp2f(gam * log2f(Rp0 * th));
      }
    }

    // ---- per field (in the order 1 4 2 5 3 6 0 7): fluxes + R | barrier |
    //      S/T GEMMs | barrier | rhsq += Jinv (R + S + T) -------------------
#pragma unroll 1
    for (int p = 0; p < 8; ++p) {
      const int b = lt32_field(p);
      const bool mom = b >= 1 && b <= 3;
      float part[2][KS];
      {
        const int bn = lt32_field((p + 1) & 7);
        const float *rnext = p < 7 ? re + bn * NPT : rhsq + (en * 8 + bn) * NPT + c;
        const bool have = p < 7 || en < ne;
#pragma unroll
        for (int rho = 0; rho < 2; ++rho)
#pragma unroll
          for (int t = 0; t < KS; ++t) {
            part[rho][t] = rhn[rho][t];
            rhn[rho][t] = (have && vt[rho][t]) ? rnext[pofs[rho] + 4 * t] : 0.f;
          }
      }
      mbar_wait(&bars[p & 1], (uint32_t)((p >> 1) & 1));
      if (mom) {
        mbar_wait(&bars[2], gpar);
        gpar ^= 1u;
      }
      {
        float *fS = tile(0, 0), *fT = tile(0, 1);
        const float *qs = qst + (p & 1) * SLAB;
        const float *qslab = q + (e * 8 + b) * NPT;
        uint32_t ahi[2][KS], alo[2][KS];
        // stage slab bases (the copies start at the 16-byte unit below each slab)
        auto shift = [](const float *a0) { return (int)((reinterpret_cast<uintptr_t>(a0) & 15) >> 2); };
        const float *qb0 = qs + shift(qslab) + c;
        const float *gb0[3];
#pragma unroll
        for (int d = 0; d < 3; ++d)
          gb0[d] = gst + d * SLAB + shift(g + (e * 9 + 3 * d + b - 1) * NPT) + c;
#pragma unroll
        for (int rho = 0; rho < 2; ++rho)
#pragma unroll
          for (int t = 0; t < KS; ++t) {
            const int o = pofs[rho] + 4 * t;
            const float qv = vt[rho][t] ? qb0[o] : 0.f;
            float fr = Wd[0][rho][t] * qv, fs = Wd[1][rho][t] * qv, ft = Wd[2][rho][t] * qv;
            if (mom && vt[rho][t]) {
              float gd[3];
#pragma unroll
              for (int d = 0; d < 3; ++d) gd[d] = gb0[d][o];
              fr = fmaf(gd[0], pp[rho][t], fr);
              fs = fmaf(gd[1], pp[rho][t], fs);
              ft = fmaf(gd[2], pp[rho][t], ft);
            }
            split_tf32(vt[rho][t] ? fr : 0.f, ahi[rho][t], alo[rho][t]);
            if (vt[rho][t]) {
              fS[posS(rho, t)] = fs;
              fT[posT(rho, t)] = ft;
            }
          }
        uint32_t brh[NKS][NKS][2], brl[NKS][NKS][2];
#pragma unroll
        for (int u = 0; u < NKS; ++u)
#pragma unroll
          for (int s = 0; s < NKS; ++s)
#pragma unroll
            for (int r = 0; r < 2; ++r) {
              const int x = ((u * NKS + s) * 2 + r) * 32 + lane;
              brh[u][s][r] = __float_as_uint(drt[x]);
              brl[u][s][r] = __float_as_uint(drt[C::DR * 32 + x]);
            }
#pragma unroll
        for (int u = 0; u < NKS; ++u) {
          float acc[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
          for (int s = 0; s < NKS; ++s) {
            // A[rows g, g+8][k-cols c, c+4] = own points t = 2s, 2s+1
            const int t0 = 2 * s, t1 = 2 * s + 1;
            uint32_t ah[4] = {ahi[0][t0], ahi[1][t0], t1 < KS ? ahi[0][t1] : 0u,
                              t1 < KS ? ahi[1][t1] : 0u};
            uint32_t al[4] = {alo[0][t0], alo[1][t0], t1 < KS ? alo[0][t1] : 0u,
                              t1 < KS ? alo[1][t1] : 0u};
            mma_tf32(acc, ah, brh[u][s]);
            mma_tf32(acc, al, brh[u][s]);
            mma_tf32(acc, ah, brl[u][s]);
          }
          // C: (row g, slot t = 2u), (g, 2u+1), (g+8, 2u), (g+8, 2u+1)
#pragma unroll
          for (int s2 = 0; s2 < 2; ++s2) {
            const int t = 2 * u + s2;
            if (t < KS) {
              part[0][t] = fmaf(jv[0][t], acc[s2], part[0][t]);
              part[1][t] = fmaf(jv[1][t], acc[2 + s2], part[1][t]);
            }
          }
        }
      }
      if (p == 6 && tid == 32 && en < ne) {  // next element's phase-1 inputs into L2
        prefetch_l2_range(q + en * 8 * NPT, 5ull * NPT * sizeof(float));
        prefetch_l2_range(g + en * 9 * NPT, 9ull * NPT * sizeof(float));
        prefetch_l2_range(jinv + en * NPT, 1ull * NPT * sizeof(float));
      }
      __syncthreads();  // F_s, F_t complete; every stage read of position p done
      if (tid == 0) {
        fence_proxy_async();
        if (p + 2 < 8) issue_q(e, p + 2);
        else if (en < ne) issue_q(en, p - 6);
        // g stage: momentum fields sit at positions 0, 2, 4
        if (p == 0 || p == 2) issue_g(e, lt32_field(p + 2));
        else if (p == 4 && en < ne) issue_g(en, lt32_field(0));
      }
      gemm_st(0);
      __syncthreads();  // C_s, C_t complete
      {
        const float *pS = tile(0, 2), *pT = tile(0, 3);
#pragma unroll
        for (int rho = 0; rho < 2; ++rho)
#pragma unroll
          for (int t = 0; t < KS; ++t)
            if (vt[rho][t])
              re[b * NPT + pofs[rho] + 4 * t] =
                  fmaf(jv[rho][t], pS[posS(rho, t)] + pT[posT(rho, t)], part[rho][t]);
      }
    }
  }
}

template <int NQ>
int launch_lt32(int64_t ne, float p0, float R, float gam, const float *q, float *rhsq,
                const float *D, const float *g, const float *jinv, cudaStream_t s) {
  using C = Lt32Cfg<NQ>;
  auto kern = volume_lt32_kernel<NQ>;
  if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::SMEM) !=
      cudaSuccess)
    return LFB_ERR_CUDA;
  int dev = 0, sms = 0, per_sm = 0;
  if (cudaGetDevice(&dev) != cudaSuccess ||
      cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess ||
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, C::THREADS, C::SMEM) !=
          cudaSuccess)
    return LFB_ERR_CUDA;
  if (per_sm < 1) return LFB_ERR_LAUNCH;
  const int64_t slots = (int64_t)sms * per_sm;
  const int64_t grid = ne < slots ? ne : slots;
  if (grid == 0) return LFB_OK;
  kern<<<(unsigned)grid, C::THREADS, C::SMEM, s>>>(ne, p0, R, gam, q, rhsq, D, g, jinv);
  LFB_CHECK_LAUNCH();
  return LFB_OK;
}

}  // namespace

bool lt32_available(int nq) { return nq >= 9 && nq <= 12; }
int volume_col_f32(int, int64_t, float, float, float, const float *, float *, const float *,
                   const float *, const float *, cudaStream_t);

namespace {
int dispatch_lt32(int nq, int64_t ne, float p0, float R, float gam, const float *q, float *rhsq,
                  const float *D, const float *g, const float *jinv, cudaStream_t s) {
  switch (nq) {
    case 9: return launch_lt32<9>(ne, p0, R, gam, q, rhsq, D, g, jinv, s);
    case 10: return launch_lt32<10>(ne, p0, R, gam, q, rhsq, D, g, jinv, s);
    case 11: return launch_lt32<11>(ne, p0, R, gam, q, rhsq, D, g, jinv, s);
    case 12: return launch_lt32<12>(ne, p0, R, gam, q, rhsq, D, g, jinv, s);
    default: return LFB_ERR_BAD_VARIANT;
  }
}
}  // namespace

// The bulk copies need 16-byte aligned q / g (else: the column kernel). When
// a slab is not a 16-byte multiple (odd Nq), the last element — whose
// aligned superset would leave the arrays — goes to the column kernel on the
// same stream.
int volume_lt_f32(int nq, int64_t ne, float p0, float R, float gam, const float *q, float *rhsq,
                  const float *D, const float *g, const float *jinv, cudaStream_t s) {
  if (!lt32_available(nq)) return LFB_ERR_BAD_VARIANT;
  if ((reinterpret_cast<uintptr_t>(q) | reinterpret_cast<uintptr_t>(g)) & 15)
    return volume_col_f32(nq, ne, p0, R, gam, q, rhsq, D, g, jinv, s);
  const int64_t npt = (int64_t)nq * nq * nq;
  const int64_t n = ((npt * 4) % 16 && ne > 0) ? ne - 1 : ne;
  int rc = n > 0 ? dispatch_lt32(nq, n, p0, R, gam, q, rhsq, D, g, jinv, s) : LFB_OK;
  if (rc != LFB_OK || n == ne) return rc;
  return volume_col_f32(nq, ne - n, p0, R, gam, q + n * 8 * npt, rhsq + n * 8 * npt, D,
                        g + n * 9 * npt, jinv + n * npt, s);
}

}  // namespace lfb
