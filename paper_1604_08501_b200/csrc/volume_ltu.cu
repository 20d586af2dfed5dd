// LFB_VARIANT_LTU, fp32 storage, Nq 9..11 — the three derivatives as
// tcgen05 (UMMA) GEMMs: operands staged in shared memory, accumulators in
// TMEM, issued by one elected thread (SASS: UTCHMMA / UTCBAR / LDTM).
//
// Why: the mma.sync line-tile kernel (volume_lt32.cu) is
// issue-bound at 19-30 warp-instructions per point — fragment loads, tf32
// splits and HMMAs in every warp. Here every direction d in {R, S, T} is ONE
// M=128 GEMM chain per field:
//     C_d[line][out] = sum_K A_d[line][K] B[out][K]
// with the Nq^2 <= 128 lines of the direction as M (R: (j,k), S: (i,k),
// T: (i,j)). fp32 accuracy on TF32 inputs: the owners split each flux
// x = x_hi + x_lo (top 19 bits by an ALU mask) and store both halves into ONE
// K-major operand row, x_hi at K = n and x_lo at K = 12 + n (K = 24, three
// K=8 steps). B is [D_hi | D_hi] in rows 0..15 and [D_lo | 0] in rows 16..31
// (N = 32), so columns o and 16 + o of the accumulator hold
// X_hi D_hi + X_lo D_hi and X_hi D_lo (the dropped X_lo D_lo is ~2^-22
// relative); the readers add them. A K=8 tf32 UMMA costs ~52 cycles for any
// N <= 64 (tools/scratch-measured), so folding the split into K and N halves
// the tensor time of the 18-UMMA hi/lo/hi formulation.
//
// Per element (one CTA, persistent grid, two CTAs per SM), per field in the
// order 1 4 2 5 3 6 0 7 (one g stage serves the momentum fields):
//   owners (P points per thread, strided — coalesced global accesses):
//     fluxes from the q / g stages -> split -> the three operand tiles (the
//     SWIZZLE_NONE canonical layout: 8-row x 16-byte core matrices,
//     K-adjacent ones 128 B apart, 8-row groups 768 B apart)
//   | barrier | warp 0, one elected lane: 9 UMMAs, a tcgen05.commit per
//   direction to its own mbarrier, then the next stage copies; warps 0..3
//   read R and T outputs 0..7, warps 4..7 S and T outputs 8..15 (a warp sees
//   the 32 TMEM lanes of quadrant w % 4) into line-major exchange tiles
//   | barrier | owners: rhsq += Jinv (R + S + T).
// q_b slabs are bulk-copied two fields ahead, g(b-1, .) one field ahead,
// the next element's phase-1 inputs L2-prefetched.
//
// Measured (profiles/r02_sweep_f32.jsonl): it leads the mma.sync line tiles
// at every Nq it covers and is the AUTO kernel at fp32 Nq 11; the column
// kernel keeps Nq 9, 10. A per-phase clock64 breakdown (-DLTU_TIMING) shows
// the field cost split between the flux stores (shared-memory bound: the
// K-major rows give each line only four banks), the UMMA chain and the
// TMEM readback.

#include <stdint.h>

#include "lfb_common.cuh"
#include "lfb_tma.cuh"
#ifdef LTU_TIMING
#include <stdio.h>
#define LTU_T(k) do { tt[k] = clock64(); } while (0)
#else
#define LTU_T(k) do { } while (0)
#endif

namespace lfb {
namespace {

__device__ __forceinline__ uint32_t ltu_split_hi(float x) { return __float_as_uint(x) & 0xffffe000u; }

// byte offset of element (row, k) of a K-major operand tile (K = 24 tf32):
// core matrices of 8 rows x 16 bytes; LBO = 128 (K-adjacent), SBO = 768
constexpr int LTU_K = 24;
constexpr int LTU_SBO = LTU_K / 4 * 128;
__device__ __forceinline__ int ltu_off(int row, int k) {
  return (row >> 3) * LTU_SBO + (k >> 2) * 128 + (row & 7) * 16 + (k & 3) * 4;
}

__device__ __forceinline__ bool ltu_elect_one() {
  uint32_t pred;
  asm volatile(
      "{\n .reg .pred P;\n elect.sync _|P, 0xffffffff;\n selp.b32 %0, 1, 0, P;\n}\n"
      : "=r"(pred));
  return pred != 0;
}

__device__ __forceinline__ void ltu_ld16(uint32_t (&v)[16], uint32_t taddr) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,"
      "%14,%15}, [%16];\n tcgen05.wait::ld.sync.aligned;"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
        "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]),
        "=r"(v[14]), "=r"(v[15])
      : "r"(taddr));
}

__device__ __forceinline__ void ltu_ld8(uint32_t (&v)[8], uint32_t taddr) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];\n"
      " tcgen05.wait::ld.sync.aligned;"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
        "=r"(v[7])
      : "r"(taddr));
}

__device__ __forceinline__ uint64_t ltu_desc(uint32_t saddr) {
  return (uint64_t)((saddr >> 4) & 0x3fff) | ((uint64_t)(128 >> 4) << 16) |
         ((uint64_t)(LTU_SBO >> 4) << 32) | ((uint64_t)1 << 46);  // version 1, SWIZZLE_NONE
}

// field processed at position p (momentum fields on even positions)
__device__ __forceinline__ int ltu_field(int p) {
  return (p & 1) ? (p == 7 ? 7 : 4 + (p >> 1)) : (p == 6 ? 0 : 1 + (p >> 1));
}

template <int NQ>
struct LtuCfg {
  static constexpr int NPT = NQ * NQ * NQ;
  static constexpr int NL = NQ * NQ;                // lines per direction (<= 128)
  // points per thread: Nq 9, 10 -> 8 warps; Nq 11 -> 7 warps (128 registers at
  // two CTAs per SM; warp 3 then also reads quadrant 3's second half)
  static constexpr int P = NQ == 9 ? 3 : NQ == 10 ? 4 : 6;
  static constexpr int THREADS = ((NPT + P - 1) / P + 31) / 32 * 32;
  static constexpr int CRS = 17;                    // exchange-tile row stride (odd)
  static constexpr int SLAB = (NPT + 4 + 3) & ~3;   // stage slab (16-byte aligned superset)
  static constexpr int AT = 128 * LTU_K;            // one operand tile (floats)
  static constexpr int BT = 32 * LTU_K;             // the B tile
  // A tiles [dir 3][hi, lo], B tiles [hi, lo] (16 x 16), exchange tiles
  // [dir 3][128][CRS], q stages [2], g stage [3]
  static constexpr size_t SMEM = sizeof(float) * (3 * (size_t)AT + BT +
                                                  3 * 128 * (size_t)CRS + 5 * (size_t)SLAB) +
                                 6 * sizeof(uint64_t) + 16;
  static_assert(NL <= 128, "one M=128 tile per direction");
  static constexpr int W = THREADS / 32;
  static_assert(W >= 4, "four TMEM reader warps");
};

template <int NQ>
__global__ void __launch_bounds__(LtuCfg<NQ>::THREADS, 2)
    volume_ltu_kernel(int64_t ne, float p0, float R, float gam, const float *__restrict__ q,
                      float *__restrict__ rhsq, const float *__restrict__ D,
                      const float *__restrict__ g, const float *__restrict__ jinv) {
  using C = LtuCfg<NQ>;
  constexpr int NPT = C::NPT, P = C::P, T = C::THREADS, AT = C::AT, CRS = C::CRS;
  constexpr int SLAB = C::SLAB, NQQ = NQ * NQ;
  extern __shared__ __align__(1024) float u_sm[];
  float *At = u_sm;                 // [dir][AT]
  float *Bt = At + 3 * AT;          // [BT]
  float *Xc = Bt + C::BT;           // [dir][128][CRS]
  float *qst = Xc + 3 * 128 * CRS;  // [2][SLAB]
  float *gst = qst + 2 * SLAB;      // [3][SLAB]
  uint64_t *bars = reinterpret_cast<uint64_t *>(gst + 3 * SLAB);  // q0, q1, g, mma R, S, T
  uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(bars + 6);

  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const float Rp0 = R / p0;
  char *const Ab = reinterpret_cast<char *>(At);

  for (int x = tid; x < 3 * AT + C::BT; x += T) u_sm[x] = 0.f;
  __syncthreads();
  // B = D^T hi / lo: B[row = out][k = n] = D(out, n)
  for (int x = tid; x < NQ * NQ; x += T) {
    const int out = x % NQ, n = x / NQ;
    const float v = __ldg(D + n * NQ + out);
    const uint32_t hi = ltu_split_hi(v);
    Bt[ltu_off(out, n) / 4] = __uint_as_float(hi);
    Bt[ltu_off(out, 12 + n) / 4] = __uint_as_float(hi);
    Bt[ltu_off(16 + out, n) / 4] = v - __uint_as_float(hi);
  }
  if (w == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tmem_slot)),
                 "r"(128));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
#pragma unroll
    for (int x = 0; x < 6; ++x) mbar_init(&bars[x], 1);
    mbar_init_fence();
  }
  fence_proxy_async();
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = *tmem_slot;

  // ---- own points p = tid + m T: offsets in the operand and exchange tiles --
  int pt[P];
  bool vp[P];
  int aR[P], aS[P], aT[P], xR[P], xS[P], xT[P];
#pragma unroll
  for (int m = 0; m < P; ++m) {
    const int p = tid + m * T;
    vp[m] = p < NPT;
    pt[m] = vp[m] ? p : 0;
    const int i = pt[m] % NQ, j = (pt[m] / NQ) % NQ, k = pt[m] / NQQ;
    aR[m] = ltu_off(k * NQ + j, i) / 4;  // R line (j,k), K index i
    aS[m] = ltu_off(k * NQ + i, j) / 4;  // S line (i,k), K index j
    aT[m] = ltu_off(j * NQ + i, k) / 4;  // T line (i,j), K index k
    xR[m] = (k * NQ + j) * CRS + i;      // exchange tiles: [line][out]
    xS[m] = (k * NQ + i) * CRS + j;
    xT[m] = (j * NQ + i) * CRS + k;
  }

  // ---- store rotation: in the warp-wide operand store s of direction d, lane
  // group g_d(lane) stores its point (s + g_d) mod P instead of point s — the
  // points of one store then come from several k-planes / lines, so fewer
  // lanes share a bank (a K-major row keeps a line's K values in four banks).
  // Bank model over the real patterns, wavefronts per field (hi stores; R+S+T):
  // Nq 9: 207 -> 153, Nq 10: 281 -> 182, Nq 11: 372 -> 247 (tools/ltu_banks.py).
  const int gR = NQ == 11 ? (lane >> 2) & 3 : (lane >> 1) & 3;
  const int gS = NQ == 9 ? lane >> 3 : 0;
  const int gT = lane >> 3;
  auto rot = [](int s, int gg) { return s + gg < P ? s + gg : s + gg - P; };
  auto pick_i = [](const int (&a)[P], int m) {
    int v = a[0];
#pragma unroll
    for (int x = 1; x < P; ++x) v = m == x ? a[x] : v;
    return v;
  };
  int oR[P], oS[P], oT[P];
  uint32_t vR = 0, vS = 0, vT = 0;
  {
    int vpi[P];
#pragma unroll
    for (int m = 0; m < P; ++m) vpi[m] = vp[m] ? 1 : 0;
#pragma unroll
    for (int x = 0; x < P; ++x) {
      oR[x] = pick_i(aR, rot(x, gR));
      oS[x] = pick_i(aS, rot(x, gS));
      oT[x] = pick_i(aT, rot(x, gT));
      vR |= (uint32_t)pick_i(vpi, rot(x, gR)) << x;
      vS |= (uint32_t)pick_i(vpi, rot(x, gS)) << x;
      vT |= (uint32_t)pick_i(vpi, rot(x, gT)) << x;
    }
  }
  auto store_split = [&](int d, int off, float v) {
    const uint32_t hi = ltu_split_hi(v);
    At[d * AT + off] = __uint_as_float(hi);
    At[d * AT + off + 96] = v - __uint_as_float(hi);  // K index 12 + n
  };

  // ---- stages (thread 0) ---------------------------------------------------
  auto slab_bytes = [&](const float *a0) {
    const uintptr_t lo = reinterpret_cast<uintptr_t>(a0) & ~(uintptr_t)15;
    const uintptr_t hi = (reinterpret_cast<uintptr_t>(a0 + NPT) + 15) & ~(uintptr_t)15;
    return (uint32_t)(hi - lo);
  };
  auto slab_copy = [&](float *dst, const float *a0, uint64_t *bar) {
    bulk_g2s(dst, reinterpret_cast<const void *>(reinterpret_cast<uintptr_t>(a0) & ~(uintptr_t)15),
             slab_bytes(a0), bar);
  };
  auto shift = [](const float *a0) { return (int)((reinterpret_cast<uintptr_t>(a0) & 15) >> 2); };
  auto issue_q = [&](int64_t e, int p) {
    const float *a0 = q + (e * 8 + ltu_field(p)) * NPT;
    mbar_expect_tx(&bars[p & 1], slab_bytes(a0));
    slab_copy(qst + (p & 1) * SLAB, a0, &bars[p & 1]);
  };
  auto issue_g = [&](int64_t e, int b) {
    uint32_t total = 0;
#pragma unroll
    for (int d = 0; d < 3; ++d) total += slab_bytes(g + (e * 9 + 3 * d + b - 1) * NPT);
    mbar_expect_tx(&bars[2], total);
#pragma unroll
    for (int d = 0; d < 3; ++d) slab_copy(gst + d * SLAB, g + (e * 9 + 3 * d + b - 1) * NPT, &bars[2]);
  };
  // instruction descriptor: D f32, A / B tf32, both K-major, N = 16, M = 128
  const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(32 >> 3) << 17) |
                         ((uint32_t)(128 >> 4) << 24);
  const uint32_t a_base = smem_u32(At), b_base = smem_u32(Bt);
  auto umma = [&](uint32_t dcol, uint32_t aaddr, uint32_t baddr, uint32_t acc) {
    asm volatile(
        "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem + dcol),
        "l"(ltu_desc(aaddr)), "l"(ltu_desc(baddr)), "r"(idesc), "r"(acc));
  };

  int64_t e = blockIdx.x;
#ifdef LTU_TIMING
  long long acc[10] = {0};
  const long long tstart = clock64();
#endif
  if (tid == 0 && e < ne) {
    issue_q(e, 0);
    issue_q(e, 1);
    issue_g(e, ltu_field(0));
  }
  uint32_t gpar = 0, mpar = 0;
  float rhn[P];
  if (e < ne) {
#pragma unroll
    for (int m = 0; m < P; ++m) rhn[m] = vp[m] ? rhsq[(e * 8 + ltu_field(0)) * NPT + pt[m]] : 0.f;
  }
  for (; e < ne; e += gridDim.x) {
    const float *qe = q + e * 8 * NPT;
    const float *ge = g + e * 9 * NPT;
    float *re = rhsq + e * 8 * NPT;
    const int64_t en = e + gridDim.x;

    // ---- phase 1: W_d = V_d / rho, p, Jinv (FP32) ---------------------------
    float Wd[3][P], pp[P], jv[P];
#pragma unroll
    for (int m = 0; m < P; ++m) {
      const int o = pt[m];
      const bool v = vp[m];
      const float rr = v ? __ldg(qe + o) : 1.f, th = v ? __ldg(qe + 4 * NPT + o) : 1.f;
      float U[3], gv[9];
#pragma unroll
      for (int a = 0; a < 3; ++a) U[a] = v ? __ldg(qe + (1 + a) * NPT + o) : 0.f;
#pragma unroll
      for (int x = 0; x < 9; ++x) gv[x] = v ? __ldg(ge + x * NPT + o) : 0.f;
      jv[m] = v ? __ldg(jinv + e * NPT + o) : 0.f;
      const float rinv = __frcp_rn(rr);
#pragma unroll
      for (int d = 0; d < 3; ++d)
        Wd[d][m] = fmaf(gv[3 * d], U[0], fmaf(gv[3 * d + 1], U[1], gv[3 * d + 2] * U[2])) * rinv;
      pp[m] = p0 * exp2f(gam * log2f(Rp0 * th));
    }

#pragma unroll 1
    for (int p = 0; p < 8; ++p) {
#ifdef LTU_TIMING
      long long tt[9] = {0};
      tt[3] = tt[4] = tt[5] = 0;
#endif
      LTU_T(0);
      const int b = ltu_field(p);
      const bool mom = b >= 1 && b <= 3;
      float part[P];
      {
        const int bn = ltu_field((p + 1) & 7);
        const float *rnext = p < 7 ? re + bn * NPT : rhsq + (en * 8 + bn) * NPT;
        const bool have = p < 7 || en < ne;
#pragma unroll
        for (int m = 0; m < P; ++m) {
          part[m] = rhn[m];
          rhn[m] = (have && vp[m]) ? rnext[pt[m]] : 0.f;
        }
      }
      mbar_wait(&bars[p & 1], (uint32_t)((p >> 1) & 1));
      if (mom) {
        mbar_wait(&bars[2], gpar);
        gpar ^= 1u;
      }
      LTU_T(1);
      // ---- fluxes -> split operand tiles -------------------------------------
      {
        const float *qs = qst + (p & 1) * SLAB + shift(q + (e * 8 + b) * NPT);
        const float *gs0 = gst + shift(g + (e * 9 + b - 1) * NPT);
        const float *gs1 = gst + SLAB + shift(g + (e * 9 + 3 + b - 1) * NPT);
        const float *gs2 = gst + 2 * SLAB + shift(g + (e * 9 + 6 + b - 1) * NPT);
        float fR[P], fS[P], fT[P];
#pragma unroll
        for (int m = 0; m < P; ++m) {
          const float qv = qs[pt[m]];
          fR[m] = Wd[0][m] * qv;
          fS[m] = Wd[1][m] * qv;
          fT[m] = Wd[2][m] * qv;
          if (mom) {
            fR[m] = fmaf(gs0[pt[m]], pp[m], fR[m]);
            fS[m] = fmaf(gs1[pt[m]], pp[m], fS[m]);
            fT[m] = fmaf(gs2[pt[m]], pp[m], fT[m]);
          }
        }
        auto pick_f = [](const float (&a)[P], int m) {
          float v = a[0];
#pragma unroll
          for (int x = 1; x < P; ++x) v = m == x ? a[x] : v;
          return v;
        };
#pragma unroll
        for (int x = 0; x < P; ++x) {
          if ((vR >> x) & 1) store_split(0, oR[x], pick_f(fR, rot(x, gR)));
          if ((vS >> x) & 1) store_split(1, oS[x], pick_f(fS, rot(x, gS)));
          if ((vT >> x) & 1) store_split(2, oT[x], pick_f(fT, rot(x, gT)));
        }
      }
      if (p == 6 && tid == 32 && en < ne) {  // next element's phase-1 inputs into L2
        prefetch_l2_range(q + en * 8 * NPT, 5ull * NPT * sizeof(float));
        prefetch_l2_range(g + en * 9 * NPT, 9ull * NPT * sizeof(float));
        prefetch_l2_range(jinv + en * NPT, 1ull * NPT * sizeof(float));
      }
      LTU_T(8);
      fence_proxy_async();  // operand stores -> visible to the tensor core
      __syncthreads();      // operands complete; stage reads of position p done
      LTU_T(2);
      if (w == 0) {  // one elected lane issues; each direction commits to its own barrier
        asm volatile("tcgen05.fence::after_thread_sync;");
        if (ltu_elect_one()) {
          const int dord[3] = {0, 1, 2};
#pragma unroll
          for (int x = 0; x < 3; ++x) {
            const int d = dord[x];
            const uint32_t ad = a_base + d * AT * 4;
#pragma unroll
            for (int ks = 0; ks < LTU_K / 8; ++ks) umma(32 * d, ad + ks * 256, b_base + ks * 256, ks > 0);
            asm volatile(
                "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                    smem_u32(&bars[3 + d])));
          }
          fence_proxy_async();
          if (p + 2 < 8) issue_q(e, p + 2);
          else if (en < ne) issue_q(en, p - 6);
          if (p == 0 || p == 2) issue_g(e, ltu_field(p + 2));
          else if (p == 4 && en < ne) issue_g(en, ltu_field(0));
        }
        __syncwarp();
        LTU_T(3);
      }
      // ---- TMEM -> exchange tiles: half h = 0 (R and T outputs 0..7) or 1 (S and
      // T outputs 8..15) of quadrant qd (TMEM lanes 32 qd.., readable by warps
      // with w % 4 == qd): warp qd takes half 0, warp 4 + qd half 1 — or, with
      // fewer than 8 warps, warp qd both
      auto read_half = [&](int qd, int h) {
        const int line = 32 * qd + lane;
        const uint32_t tq = tmem + ((uint32_t)(32 * qd) << 16);
        mbar_wait(&bars[3 + h], mpar);
        LTU_T(4);
        asm volatile("tcgen05.fence::after_thread_sync;");
        {  // columns o (X_hi D_hi + X_lo D_hi) and 16 + o (X_hi D_lo)
          uint32_t v[16], u[16];
          ltu_ld16(v, tq + 32 * h);
          ltu_ld16(u, tq + 32 * h + 16);
          if (line < C::NL) {
#pragma unroll
            for (int o = 0; o < NQ; ++o)
              Xc[(h * 128 + line) * CRS + o] = __uint_as_float(v[o]) + __uint_as_float(u[o]);
          }
        }
        mbar_wait(&bars[5], mpar);
        LTU_T(5);
        asm volatile("tcgen05.fence::after_thread_sync;");
        {
          const int o0 = 8 * h;
          uint32_t v[8], u[8];
          ltu_ld8(v, tq + 64 + o0);
          ltu_ld8(u, tq + 80 + o0);
          if (line < C::NL) {
#pragma unroll
            for (int o = 0; o < 8; ++o)
              if (o0 + o < NQ)
                Xc[(256 + line) * CRS + o0 + o] = __uint_as_float(v[o]) + __uint_as_float(u[o]);
          }
        }
      };
      if (w < 8) {
        read_half(w & 3, w >> 2);
        if (w < 4 && w + 4 >= C::W) read_half(w, 1);
        asm volatile("tcgen05.fence::before_thread_sync;");
      }
      mpar ^= 1u;
      __syncthreads();  // exchange tiles complete; the MMAs have read the operands
      LTU_T(6);
      // ---- rhsq_b += Jinv (R + S + T) ----------------------------------------------
#pragma unroll
      for (int m = 0; m < P; ++m)
        if (vp[m])
          re[b * NPT + pt[m]] =
              fmaf(jv[m], Xc[xR[m]] + Xc[128 * CRS + xS[m]] + Xc[256 * CRS + xT[m]], part[m]);
#ifdef LTU_TIMING
      LTU_T(7);
      if (tid == 0 || tid == 128) {
        acc[0] += tt[1] - tt[0]; acc[1] += tt[2] - tt[1];
        if (tid == 0) acc[2] += tt[3] - tt[2];
        acc[3] += tt[4] - tt[2]; acc[4] += tt[5] - tt[2]; acc[5] += tt[6] - tt[2];
        acc[6] += tt[7] - tt[6]; acc[7] += 1; acc[8] += tt[8] - tt[1];
      }
#endif
    }
  }
#ifdef LTU_TIMING
  if (blockIdx.x < 2 && (tid == 0 || tid == 128))
    printf("LTUT cta %d tid %d fields %lld total %lld per field: flux %lld q %lld bar1 %lld mma %lld r %lld t %lld bar2 %lld comb %lld\n",
           blockIdx.x, tid, acc[7], clock64() - tstart, acc[8] / acc[7], acc[0] / acc[7], acc[1] / acc[7], acc[2] / acc[7],
           acc[3] / acc[7], acc[4] / acc[7], acc[5] / acc[7], acc[6] / acc[7]);
#endif
  __syncthreads();
  if (w == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(128));
}

template <int NQ>
int launch_ltu(int64_t ne, float p0, float R, float gam, const float *q, float *rhsq,
               const float *D, const float *g, const float *jinv, cudaStream_t s) {
  using C = LtuCfg<NQ>;
  auto kern = volume_ltu_kernel<NQ>;
  if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::SMEM) !=
          cudaSuccess ||
      cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout,
                           (int)cudaSharedmemCarveoutMaxShared) != cudaSuccess)
    return LFB_ERR_CUDA;
  // residency from the shared-memory budget: the occupancy API reports one
  // CTA per SM for this kernel although two fit (the launch bounds guarantee
  // the registers for two)
  int dev = 0, sms = 0, smem_sm = 0, reserved = 0;
  if (cudaGetDevice(&dev) != cudaSuccess ||
      cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess ||
      cudaDeviceGetAttribute(&smem_sm, cudaDevAttrMaxSharedMemoryPerMultiprocessor, dev) !=
          cudaSuccess ||
      cudaDeviceGetAttribute(&reserved, cudaDevAttrReservedSharedMemoryPerBlock, dev) !=
          cudaSuccess)
    return LFB_ERR_CUDA;
  int per_sm = smem_sm / ((int)C::SMEM + reserved);
  if (per_sm < 1) return LFB_ERR_LAUNCH;
  if (per_sm > 2) per_sm = 2;  // 128 TMEM columns per CTA; the launch bounds cover two
  const int64_t slots = (int64_t)sms * per_sm;
  const int64_t grid = ne < slots ? ne : slots;
  if (grid == 0) return LFB_OK;
  kern<<<(unsigned)grid, C::THREADS, C::SMEM, s>>>(ne, p0, R, gam, q, rhsq, D, g, jinv);
  LFB_CHECK_LAUNCH();
  return LFB_OK;
}

int dispatch_ltu(int nq, int64_t ne, float p0, float R, float gam, const float *q, float *rhsq,
                 const float *D, const float *g, const float *jinv, cudaStream_t s) {
  switch (nq) {
    case 9: return launch_ltu<9>(ne, p0, R, gam, q, rhsq, D, g, jinv, s);
    case 10: return launch_ltu<10>(ne, p0, R, gam, q, rhsq, D, g, jinv, s);
    case 11: return launch_ltu<11>(ne, p0, R, gam, q, rhsq, D, g, jinv, s);
    default: return LFB_ERR_BAD_VARIANT;
  }
}

}  // namespace

bool ltu_available(int dtype_bytes, int nq) { return dtype_bytes == 4 && nq >= 9 && nq <= 11; }
int volume_col_f32(int, int64_t, float, float, float, const float *, float *, const float *,
                   const float *, const float *, cudaStream_t);

// 16-byte aligned q / g needed by the bulk copies (else: the column kernel);
// for odd Nq the last element goes to the column kernel (its slab superset
// would leave the arrays)
int volume_ltu_f32(int nq, int64_t ne, float p0, float R, float gam, const float *q, float *rhsq,
                   const float *D, const float *g, const float *jinv, cudaStream_t s) {
  if (!ltu_available(4, nq)) return LFB_ERR_BAD_VARIANT;
  if ((reinterpret_cast<uintptr_t>(q) | reinterpret_cast<uintptr_t>(g)) & 15)
    return volume_col_f32(nq, ne, p0, R, gam, q, rhsq, D, g, jinv, s);
  const int64_t npt = (int64_t)nq * nq * nq;
  const int64_t n = ((npt * 4) % 16 && ne > 0) ? ne - 1 : ne;
  int rc = n > 0 ? dispatch_ltu(nq, n, p0, R, gam, q, rhsq, D, g, jinv, s) : LFB_OK;
  if (rc != LFB_OK || n == ne) return rc;
  return volume_col_f32(nq, ne - n, p0, R, gam, q + n * 8 * npt, rhsq + n * 8 * npt, D,
                        g + n * 9 * npt, jinv + n * npt, s);
}

}  // namespace lfb
