// LFB_VARIANT_TC for fp32 storage — TMA-staged volume kernel with the three
// derivative contractions on the TF32 tensor path (mma.sync m16n8k8) at
// fp32 accuracy, point-wise physics in the FP32 pipe.
//
// Why (profiles/r01_tc_nq8_f32.json, profiles/r01_microbench_fp32.txt): the
// fp64-DMMA formulation of the fp32 variant spends half its cycles in the
// shared fp64/tensor-DP pipe plus 34 f32<->f64 conversions per point and
// stalls at 0.72 of HBM. mma.sync tf32 runs at 136 TFMA/s on B200 (7.4x the
// DMMA rate), so three-term split products cost less pipe time than one
// DMMA formulation, and every operand stays fp32.
//
// Accuracy: every operand x is split x = x_hi + x_lo (x_hi its top 19 bits,
// x_lo the fp32 remainder, read by the tensor core to 19 bits: |x - x_hi -
// x_lo| < 2^-20 |x|); the products x_hi y_hi + x_hi y_lo + x_lo y_hi
// (+ x_lo y_lo) accumulate in fp32 inside the tensor core: relative error
// ~1e-6 per term, inside the 1e-5 fp32 tolerance (tests/test_volume_gpu.py,
// observed ~2e-7).
//
// Fragments (g = lane/4, c = lane%4), m16n8k8 row.col:
//   A 16x8: a0 = A[g][c], a1 = A[g+8][c], a2 = A[g][c+4], a3 = A[g+8][c+4]
//   B 8x8:  b0 = B[c][g], b1 = B[c+4][g]
//   C 16x8: c0 = C[g][2c], c1 = C[g][2c+1], c2 = C[g+8][2c], c3 = C[g+8][2c+1]
// The decomposition is the fp64 tc kernel's (volume_tc.cu): warp w owns
// plane k = w, lane (g, c) owns the points (i = 2c+s, j = g, k = w), s=0,1,
// the K index c / c+4 is permuted to n = 2c / 2c+1 where the thread's own
// values are the operand. Rows 8..15 carry the lo halves, so ONE mma gives
// two split products:
//   R (contract i, own data as A):  A = [F_hi ; F_lo] (lines j), B = D_hi,
//                                   then B = D_lo          -> 2 mma
//   S (contract j, F_s transposed through a per-warp tile as B):
//                                   A = [D_hi ; D_lo], B = F_hi, then F_lo -> 2 mma
//   T (contract k, (i,k)-plane owners, F_t through the ft tile as B): same, 2 mma;
//                                   the T result goes back through tout.
// C rows 8..15 are added to rows 0..7 at write-back.
//
// Memory pipeline as the fp64 kernel: q, g of element n+NS streamed by
// cp.async.bulk into an NS-stage ring (mbarrier complete_tx), the next
// stage beyond the ring and the next rhsq/Jinv prefetched into L2.

#include <stdint.h>
#include <stdlib.h>

#include <type_traits>

#include "lfb_common.cuh"

namespace lfb {
int volume_fused_f32(int, int64_t, float, float, float, const float *, float *, const float *,
                     const float *, const float *, cudaStream_t);
int volume_basic_f32(int, int64_t, float, float, float, const float *, float *, const float *,
                     const float *, const float *, cudaStream_t);
int volume_col_f32(int, int64_t, float, float, float, const float *, float *, const float *,
                   const float *, const float *, cudaStream_t);
bool col_available(int dtype_bytes, int nq);

namespace {

constexpr int NPT8 = 512;
constexpr int WARPS = 8;
constexpr int THREADS = 32 * WARPS;
constexpr int STAGE = 17 * NPT8;  // floats: q (8 fields) + g (9)

__device__ __forceinline__ uint32_t saddr(const void *p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(saddr(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(saddr(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@!P1 bra WAIT_%=;\n"
      "}\n" ::"r"(saddr(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, uint32_t bytes,
                                         uint64_t *bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          saddr(dst)),
      "l"(src), "r"(bytes), "r"(saddr(bar))
      : "memory");
}
__device__ __forceinline__ void prefetch_l2(const void *p, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes) : "memory");
}
__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

__device__ __forceinline__ uint32_t tf32(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return r;
}
struct Split {
  uint32_t hi, lo;
};
// Once-per-kernel operands (D): round-to-nearest tf32 hi, tf32 lo.
__device__ __forceinline__ Split split_rn(float x) {
  const uint32_t h = tf32(x);
  return {h, tf32(x - __uint_as_float(h))};
}
// Per-field operands: cvt.rna.tf32 issues on the XU pipe (16 lanes/SM/clk,
// the measured bottleneck of a cvt-based split), so the hot split is
// hi = x with the 13 low mantissa bits cleared (ALU), lo = x - hi (exact in
// fp32; the tensor core reads its top 19 bits): |x - hi - tf32(lo)| < 2^-20 |x|.
__device__ __forceinline__ Split split(float x) {
  const uint32_t h = __float_as_uint(x) & 0xffffe000u;
  return {h, __float_as_uint(x - __uint_as_float(h))};
}

// C(16x8) += A(16x8) B(8x8), tf32 inputs, fp32 accumulate
__device__ __forceinline__ void mma(float (&c)[4], uint32_t a0, uint32_t a1, uint32_t a2,
                                    uint32_t a3, uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
      "{%8,%9}, {%0,%1,%2,%3};"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}

// shared tiles (floats), bank-conflict-free for the accesses below:
//   ft   [field][k][j][i], plane stride 72 (= 8 mod 32): pairs along i in,
//        single values (4 planes x 8 rows per warp) out;
//   tout [field][k][j][i], plane stride 72: pairs in from 4 planes, pairs out;
//   stile per warp [j][i], row stride 8: pairs in, single values out.
constexpr int FT_PS = 72, FT_FS = 8 * FT_PS;
constexpr int TO_PS = 72, TO_FS = 8 * TO_PS;
constexpr int ST_RS = 8, ST_SZ = 8 * ST_RS;

// packed Nq = 4 groups: per-element slabs 64 B apart in the stage (bank
// conflicts of the 2 KB slab stride otherwise; see volume_tc.cu)
constexpr int STAGE_ALLOC = STAGE + 16 * 16;

// NW = 8: the virtual Nq=8 cube. NW = SUB < 8 (zero-padded Nq = 5..7, the
// PLANE variant as in volume_tc.cu): one warp per real k-plane, stages sized
// for the real q + g slab (+ the g superset's 16-byte shift), F_t planes
// k >= SUB zeroed once, three CTAs per SM.
template <int NS, int SUB, int NW>
struct Smem32 {
  static constexpr int STAGE_N = NW == 8 ? STAGE_ALLOC : ((17 * SUB * SUB * SUB + 4 + 3) & ~3);
  float stage[NS][STAGE_N];
  float ft[8 * FT_FS];
  float tout[8 * TO_FS];
  float stile[NW][2][ST_SZ];
  unsigned long long bar[NS];
};

// NS = 2, NW = 8: 108 KB of shared memory -> two CTAs (16 warps) per SM
template <int NS, int SUB, int NW = WARPS>
__global__ void __launch_bounds__(32 * NW, NW == 8 ? (NS == 2 ? 2 : 1) : (SUB <= 6 ? 3 : 2))
    volume_tc32_kernel(int64_t ne, float p0, float R, float gam, const float *__restrict__ q,
                       float *__restrict__ rhsq, const float *__restrict__ D,
                       const float *__restrict__ g, const float *__restrict__ jinv) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  Smem32<NS, SUB, NW> &sm = *reinterpret_cast<Smem32<NS, SUB, NW> *>(smem_raw);
  if (NW < 8) {  // F_t planes k >= SUB have no owner warp: they stay zero
    for (int x = threadIdx.x; x < 8 * FT_FS; x += 32 * NW) sm.ft[x] = 0.f;
  }

  const int tid = threadIdx.x;
  const int lane = tid & 31, w = tid >> 5;
  const int gq = lane >> 2, c = lane & 3;
  const int64_t G = gridDim.x;
  const int64_t e0 = blockIdx.x;
  const int64_t nmine = (e0 < ne) ? (ne - 1 - e0) / G + 1 : 0;
  const float Rp0 = R / p0;

  // SUB = real Nq: 8 one element per group; 4 / 2 pack (8/SUB)^3 elements
  // into a virtual Nq=8 cube with blockdiag D; 5..7 zero-pad one element
  constexpr bool PAD = !(SUB == 8 || SUB == 4 || SUB == 2);
  // even padded Nq (6): a lane's two points are valid together and 8-byte
  // aligned -> one 8-byte access (as volume_tc.cu)
  constexpr bool PAIRS = PAD && SUB % 2 == 0;
  static_assert(SUB >= 2 && SUB <= 8, "virtual Nq=8 cube");
  constexpr int P = PAD ? 1 : 8 / SUB, NPTR = SUB * SUB * SUB;
  constexpr int SLABQ = PAD ? 8 * NPTR : 8 * NPT8;
  constexpr int SLABG = PAD ? 9 * NPTR : 9 * NPT8;
  constexpr int SLABJ = PAD ? NPTR : NPT8;
  const int ur = PAD ? 0 : (2 * c) / SUB + P * (gq / SUB) + P * P * (w / SUB);
  const int ptr = PAD ? (w * SUB + gq) * SUB + 2 * c
                      : ((w % SUB) * SUB + (gq % SUB)) * SUB + (2 * c) % SUB;
  const int qo = ur * 8 * NPTR + ptr;
  constexpr int EPAD = (SUB == 4) ? 16 : 0;  // floats
  constexpr int SQE = 8 * NPTR + EPAD, SGE = 9 * NPTR + EPAD;
  constexpr int SGOFF = (SUB == 4) ? 8 * SQE : SLABQ;
  const int sqo = (SUB == 4) ? ur * SQE + ptr : qo;
  const int go = (SUB == 4) ? ur * SGE + ptr : ur * 9 * NPTR + ptr;
  const int jo = ur * NPTR + ptr;
  bool vld[2];
#pragma unroll
  for (int s = 0; s < 2; ++s) vld[s] = !PAD || (2 * c + s < SUB && gq < SUB && w < SUB);
  // odd padded Nq: per-lane order of the two 4-byte stage reads of a point
  // pair, searched so both instructions are conflict-free (Nq 7; as
  // volume_tc.cu)
  const int sw = (PAD && !PAIRS && SUB == 7) ? (int)((0x38b4b11eu >> lane) & 1u) : 0;
  auto ld_stage = [&](const float *p, float dflt, float &a, float &b) {
    const bool v0 = vld[sw], v1 = vld[sw ^ 1];
    const float x0 = v0 ? p[sw] : dflt;
    const float x1 = v1 ? p[sw ^ 1] : dflt;
    a = sw ? x1 : x0;
    b = sw ? x0 : x1;
  };
  const int ftW = w * FT_PS + gq * 8 + 2 * c;
  const int toR = w * TO_PS + gq * 8 + 2 * c;
  const int toW = gq * TO_PS + w * 8 + 2 * c;
  int ftR[2];
#pragma unroll
  for (int t = 0; t < 2; ++t) ftR[t] = (c + 4 * t) * FT_PS + w * 8 + gq;
  auto Dv = [&](int iv, int nv) -> float {
    if (PAD) return (iv < SUB && nv < SUB) ? __ldg(D + nv * SUB + iv) : 0.0f;
    if (iv / SUB != nv / SUB) return 0.0f;
    return __ldg(D + (nv % SUB) * SUB + (iv % SUB));
  };
  // R: B[K = c + 4t -> n = 2c + t][col g = i] = D(i = g, n = 2c + t)
  // S, T: A[row g][K = c + 4t -> n = c + 4t] = D(g, c + 4t); rows 8..15 = lo
  Split Dr[2], Dst[2];
#pragma unroll
  for (int t = 0; t < 2; ++t) {
    Dr[t] = split_rn(Dv(gq, 2 * c + t));
    Dst[t] = split_rn(Dv(gq, c + 4 * t));
  }
  auto span16 = [](const float *p, size_t n, const float *&start, uint32_t &bytes) {
    const uintptr_t a = reinterpret_cast<uintptr_t>(p);
    const uintptr_t lo = a & ~(uintptr_t)15;
    const uintptr_t hi = (a + n * sizeof(float) + 15) & ~(uintptr_t)15;
    start = reinterpret_cast<const float *>(lo);
    bytes = (uint32_t)(hi - lo);
  };

  uint64_t *bars = reinterpret_cast<uint64_t *>(sm.bar);
  if (tid == 0) {
#pragma unroll
    for (int s = 0; s < NS; ++s) mbar_init(&bars[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  auto issue = [&](int64_t n) {
    const int s = (int)(n % NS);
    const int64_t e = e0 + n * G;
    const float *gs;
    uint32_t gb;
    span16(g + e * SLABG, SLABG, gs, gb);
    mbar_expect_tx(&bars[s], SLABQ * sizeof(float) + gb);
    if constexpr (SUB == 4) {
#pragma unroll 1
      for (int u = 0; u < 8; ++u) {
        bulk_g2s(sm.stage[s] + u * SQE, q + e * SLABQ + u * 8 * NPTR, 8 * NPTR * sizeof(float),
                 &bars[s]);
        bulk_g2s(sm.stage[s] + SGOFF + u * SGE, g + e * SLABG + u * 9 * NPTR,
                 9 * NPTR * sizeof(float), &bars[s]);
      }
    } else {
      bulk_g2s(sm.stage[s], q + e * SLABQ, SLABQ * sizeof(float), &bars[s]);
      bulk_g2s(sm.stage[s] + SLABQ, gs, gb, &bars[s]);
    }
  };
  if (tid == 0) {
    for (int64_t n = 0; n < NS && n < nmine; ++n) issue(n);
  }
  auto l2pf = [&](int64_t n) {
    const float *sp;
    uint32_t sb_;
    if (tid == 0 && n + NS < nmine) {
      const int64_t e = e0 + (n + NS) * G;
      prefetch_l2(q + e * SLABQ, SLABQ * sizeof(float));
      span16(g + e * SLABG, SLABG, sp, sb_);
      prefetch_l2(sp, sb_);
    }
    if (tid == 32 && n + 1 < nmine) {
      const int64_t e = e0 + (n + 1) * G;
      prefetch_l2(rhsq + e * SLABQ, SLABQ * sizeof(float));
      span16(jinv + e * SLABJ, SLABJ, sp, sb_);
      prefetch_l2(sp, sb_);
    }
  };

  for (int64_t n = 0; n < nmine; ++n) {
    const int st = (int)(n % NS);
    const uint32_t parity = (uint32_t)((n / NS) & 1);
    const int64_t e = e0 + n * G;
    const float *sq = sm.stage[st];
    const float *sg = sm.stage[st] + SGOFF +
                      (PAD ? (reinterpret_cast<uintptr_t>(g + e * SLABG) & 15) / sizeof(float) : 0);
    float *re = rhsq + e * SLABQ;

    float rh[8][2], jv[2];
#pragma unroll
    for (int b = 0; b < 8; ++b) {
      if (PAD && !PAIRS) {
        rh[b][0] = vld[0] ? re[qo + b * NPTR] : 0.0f;
        rh[b][1] = vld[1] ? re[qo + b * NPTR + 1] : 0.0f;
      } else if (PAIRS && !vld[0]) {
        rh[b][0] = rh[b][1] = 0.0f;
      } else {
        const float2 v = *reinterpret_cast<const float2 *>(re + qo + b * NPTR);
        rh[b][0] = v.x;
        rh[b][1] = v.y;
      }
    }
    if (PAD && !PAIRS) {
      jv[0] = vld[0] ? jinv[e * SLABJ + jo] : 0.0f;
      jv[1] = vld[1] ? jinv[e * SLABJ + jo + 1] : 0.0f;
    } else if (PAIRS && !vld[0]) {
      jv[0] = jv[1] = 0.0f;
    } else {
      const float2 v = __ldg(reinterpret_cast<const float2 *>(jinv + e * SLABJ + jo));
      jv[0] = v.x;
      jv[1] = v.y;
    }
    l2pf(n);

    mbar_wait(&bars[st], parity);

    // ---- phase 1: point-wise quantities (FP32 pipe) ----------------------
    float sb[8][2], V0[2], V1[2], pP[2], gr[3][2], gs[3][2];
    {
      float qv[8][2], gv[9][2];
#pragma unroll
      for (int f = 0; f < 8; ++f) {
        if (PAD && !PAIRS) {
          ld_stage(sq + sqo + f * NPTR, f == 0 ? 1.0f : 0.0f, qv[f][0], qv[f][1]);
        } else if (PAIRS && !vld[0]) {
          qv[f][0] = qv[f][1] = (f == 0 ? 1.0f : 0.0f);
        } else {
          const float2 v = *reinterpret_cast<const float2 *>(sq + sqo + f * NPTR);
          qv[f][0] = v.x;
          qv[f][1] = v.y;
        }
      }
#pragma unroll
      for (int x = 0; x < 9; ++x) {
        if (PAD && !PAIRS) {
          ld_stage(sg + go + x * NPTR, 0.0f, gv[x][0], gv[x][1]);
        } else if (PAIRS && !vld[0]) {
          gv[x][0] = gv[x][1] = 0.0f;
        } else {
          const float2 v = *reinterpret_cast<const float2 *>(sg + go + x * NPTR);
          gv[x][0] = v.x;
          gv[x][1] = v.y;
        }
      }
      float V2[2];
#pragma unroll
      for (int s = 0; s < 2; ++s) {
        const float rinv = __frcp_rn(qv[0][s]);
        pP[s] = p0 * exp2f(gam * __log2f(Rp0 * qv[4][s]));
#pragma unroll
        for (int b = 1; b < 8; ++b) sb[b][s] = qv[b][s] * rinv;
        V0[s] = gv[0][s] * qv[1][s] + gv[1][s] * qv[2][s] + gv[2][s] * qv[3][s];
        V1[s] = gv[3][s] * qv[1][s] + gv[4][s] * qv[2][s] + gv[5][s] * qv[3][s];
        V2[s] = gv[6][s] * qv[1][s] + gv[7][s] * qv[2][s] + gv[8][s] * qv[3][s];
#pragma unroll
        for (int a = 0; a < 3; ++a) {
          gr[a][s] = gv[a][s];
          gs[a][s] = gv[3 + a][s];
        }
      }
      *reinterpret_cast<float2 *>(sm.ft + ftW) = make_float2(V2[0], V2[1]);
#pragma unroll
      for (int b = 1; b < 8; ++b) {
        float f0 = V2[0] * sb[b][0], f1 = V2[1] * sb[b][1];
        if (b <= 3) {
          f0 = fmaf(gv[6 + (b - 1)][0], pP[0], f0);
          f1 = fmaf(gv[6 + (b - 1)][1], pP[1], f1);
        }
        *reinterpret_cast<float2 *>(sm.ft + b * FT_FS + ftW) = make_float2(f0, f1);
      }
    }
    __syncthreads();  // ft complete; every stage read of this element is done
    if (tid == 0 && n + NS < nmine) {
      fence_proxy_async();
      issue(n + NS);
    }
    // ---- phase 2: per field ------------------------------------------------
    float acc[8][2];
#pragma unroll
    for (int b = 0; b < 8; ++b) {
      float fr[2], fs[2];
#pragma unroll
      for (int s = 0; s < 2; ++s) {
        if (b == 0) {
          fr[s] = V0[s];
          fs[s] = V1[s];
        } else {
          fr[s] = V0[s] * sb[b][s];
          fs[s] = V1[s] * sb[b][s];
          if (b <= 3) {
            fr[s] = fmaf(gr[b - 1][s], pP[s], fr[s]);
            fs[s] = fmaf(gs[b - 1][s], pP[s], fs[s]);
          }
        }
      }
      float *stl = sm.stile[w][b & 1];
      *reinterpret_cast<float2 *>(stl + gq * ST_RS + 2 * c) = make_float2(fs[0], fs[1]);
      __syncwarp();
      Split fsT[2], ftQ[2], frs[2];
#pragma unroll
      for (int t = 0; t < 2; ++t) {
        fsT[t] = split(stl[(c + 4 * t) * ST_RS + gq]);
        ftQ[t] = split(sm.ft[b * FT_FS + ftR[t]]);
        frs[t] = split(fr[t]);
      }
      float a[4] = {0.f, 0.f, 0.f, 0.f}, tq[4] = {0.f, 0.f, 0.f, 0.f};
      // R: A = [F_r hi ; F_r lo] (own values), B = D_hi then D_lo
      mma(a, frs[0].hi, frs[0].lo, frs[1].hi, frs[1].lo, Dr[0].hi, Dr[1].hi);
      mma(a, frs[0].hi, frs[0].lo, frs[1].hi, frs[1].lo, Dr[0].lo, Dr[1].lo);
      // S: A = [D_hi ; D_lo], B = F_s^T hi then lo
      mma(a, Dst[0].hi, Dst[0].lo, Dst[1].hi, Dst[1].lo, fsT[0].hi, fsT[1].hi);
      mma(a, Dst[0].hi, Dst[0].lo, Dst[1].hi, Dst[1].lo, fsT[0].lo, fsT[1].lo);
      // T on the transposed (i,k)-plane j = w
      mma(tq, Dst[0].hi, Dst[0].lo, Dst[1].hi, Dst[1].lo, ftQ[0].hi, ftQ[1].hi);
      mma(tq, Dst[0].hi, Dst[0].lo, Dst[1].hi, Dst[1].lo, ftQ[0].lo, ftQ[1].lo);
      acc[b][0] = a[0] + a[2];
      acc[b][1] = a[1] + a[3];
      *reinterpret_cast<float2 *>(sm.tout + b * TO_FS + toW) =
          make_float2(tq[0] + tq[2], tq[1] + tq[3]);
    }
    __syncthreads();  // tout complete
#pragma unroll
    for (int b = 0; b < 8; ++b) {
      const float2 t = *reinterpret_cast<const float2 *>(sm.tout + b * TO_FS + toR);
      const float o0 = fmaf(jv[0], acc[b][0] + t.x, rh[b][0]);
      const float o1 = fmaf(jv[1], acc[b][1] + t.y, rh[b][1]);
      if (PAD && !PAIRS) {
        if (vld[0]) re[qo + b * NPTR] = o0;
        if (vld[1]) re[qo + b * NPTR + 1] = o1;
      } else if (!PAIRS || vld[0]) {
        *reinterpret_cast<float2 *>(re + qo + b * NPTR) = make_float2(o0, o1);
      }
    }
  }
}

template <int NS, int SUB>
int launch_tc32(int64_t ngroups, float p0, float R, float gam, const float *q, float *rhsq,
                const float *D, const float *g, const float *jinv, cudaStream_t stream) {
  constexpr bool PAD_ = !(SUB == 8 || SUB == 4 || SUB == 2);
  // PLANE for the zero-padded Nq (8 warps -> SUB warps: Nq 5 / 6 / 7 from
  // 0.33 / 0.50 / 0.72 to 0.48 / 0.61 / 0.74 of HBM, profiles/r02_tc_plane.txt)
  constexpr int NW = PAD_ ? SUB : WARPS;
  const size_t smem = sizeof(Smem32<NS, SUB, NW>);
  auto kern = volume_tc32_kernel<NS, SUB, NW>;
  constexpr int THREADS = 32 * NW;
  if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) !=
      cudaSuccess)
    return LFB_ERR_CUDA;
  int dev = 0, sms = 0, per_sm = 0;
  if (cudaGetDevice(&dev) != cudaSuccess ||
      cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess ||
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, THREADS, smem) !=
          cudaSuccess)
    return LFB_ERR_CUDA;
  if (per_sm < 1) return LFB_ERR_LAUNCH;
  const int64_t slots = (int64_t)sms * per_sm;
  const int64_t grid = ngroups < slots ? ngroups : slots;
  if (grid == 0) return LFB_OK;
  kern<<<(unsigned)grid, THREADS, smem, stream>>>(ngroups, p0, R, gam, q, rhsq, D, g, jinv);
  LFB_CHECK_LAUNCH();
  return LFB_OK;
}

}  // namespace

// fp32 storage, tensor-core path: full groups through the TF32 kernel, the
// leftover elements (packed Nq 4 / 2: < 8 / < 64; padded Nq: the last one,
// whose 16-byte superset copy could run past the arrays) through col/fused.
int volume_tc32_f32(int nq, int64_t ne, float p0, float R, float gam, const float *q,
                    float *rhsq, const float *D, const float *g, const float *jinv,
                    cudaStream_t s) {
  const bool pad = !(nq == 8 || nq == 4 || nq == 2);
  const int64_t pe = pad ? 1 : (int64_t)(8 / nq) * (8 / nq) * (8 / nq);
  const int64_t groups = pad ? (ne > 0 ? ne - 1 : 0) : ne / pe;
  const int64_t done = groups * pe, npt = (int64_t)nq * nq * nq;
  int rc = LFB_OK;
  if (groups > 0) {
    auto run = [&](auto ns) {
      constexpr int NS = decltype(ns)::value;
      switch (nq) {
        case 8: return launch_tc32<NS, 8>(groups, p0, R, gam, q, rhsq, D, g, jinv, s);
        case 7: return launch_tc32<NS, 7>(groups, p0, R, gam, q, rhsq, D, g, jinv, s);
        case 6: return launch_tc32<NS, 6>(groups, p0, R, gam, q, rhsq, D, g, jinv, s);
        case 5: return launch_tc32<NS, 5>(groups, p0, R, gam, q, rhsq, D, g, jinv, s);
        case 4: return launch_tc32<NS, 4>(groups, p0, R, gam, q, rhsq, D, g, jinv, s);
        case 2: return launch_tc32<NS, 2>(groups, p0, R, gam, q, rhsq, D, g, jinv, s);
        default: return (int)LFB_ERR_BAD_VARIANT;
      }
    };
    // 2-stage ring, two CTAs per SM (a 1-CTA 3-stage ring measured slower,
    // profiles/r01_ab_tc32.txt)
    rc = run(std::integral_constant<int, 2>{});
  }
  if (rc != LFB_OK || done == ne) return rc;
  return volume_col_f32(nq, ne - done, p0, R, gam, q + done * 8 * npt, rhsq + done * 8 * npt, D,
                        g + done * 9 * npt, jinv + done * npt, s);
}

}  // namespace lfb
