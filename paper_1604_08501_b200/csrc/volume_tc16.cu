// LFB_VARIANT_TC for fp32 storage at Nq = 9..16: the TF32 split-product
// scheme of volume_tc32.cu on virtual 16x16 planes.
//
// Why: above Nq = 8 the fp32 path ran on the column kernel (FFMA with line
// reads from shared memory, 0.36-0.44 of HBM at Nq 9-12, shared-memory
// bound). mma.sync m16n8k8 tiles a 16x16 plane exactly (M = 16 rows, two
// n8 tiles), and the K-permutation trick of the Nq=8 kernel still works:
// thread (g, c) owns the points (j = g + 8r, i = 8nt + 2c + s), r, nt, s in
// {0,1}, and its K slots {c, c+4} in k-step ks are mapped to n = 8ks + 2c and
// 8ks + 2c + 1 — its own columns — so the R contraction reads its A operand
// straight from registers. Planes are zero-padded to 16x16 (D zero outside
// [0,Nq)^2, padding points carry zero flux and are never written).
//
// Per element (one CTA of 16 warps per SM, persistent; warp w owns the
// (i,j)-plane k = w and the (i,k)-plane j = w, idle where w >= Nq):
//   phase 1: 1/rho, p, V_r, V_s, V_t of the 8 own points from global memory
//            (the element is L2-prefetched one iteration ahead);
//   per field b: fluxes of the own points (q_b, g(b,.) re-read from L1/L2);
//     R  A = F_r own (hi/lo split), B = D^T            -> 12 mma
//     S  F_s transposed through a per-warp 16x16 tile   -> 12 mma
//     T  F_t through the plane-major ft tile, contracted on the (i,k)-planes,
//        results back through tout                      -> 12 mma
//     two CTA barriers; rhsq_b += Jinv (R + S + T) at the own points.
// Three-term split products (x_hi y_hi + x_lo y_hi + x_hi y_lo), fp32
// accumulate: ~1e-6 relative per term (tolerance 1e-5).

#include <stdint.h>
#include <stdlib.h>

#include "lfb_common.cuh"

namespace lfb {
namespace {

constexpr int W16 = 16;                // warps per CTA
constexpr int T16 = 32 * W16;          // threads
// shared tiles (floats): row stride 24 (= 8 mod 32), plane stride 392
// (= 8 mod 32) -> the 64-bit own-point accesses and the 32-bit fragment
// reads of a warp hit distinct banks
constexpr int RS16 = 24;
constexpr int PS16 = 16 * RS16 + 8;
constexpr int TILE16 = 16 * PS16;      // one 16-plane tile (ft or tout)
constexpr int STILE16 = 16 * RS16;     // per-warp S tile

struct Smem16 {
  float ft[TILE16];
  float tout[TILE16];
  float stile[W16][STILE16];
};

__device__ __forceinline__ uint32_t tf32_rn(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return r;
}
struct Sp {
  uint32_t hi, lo;
};
__device__ __forceinline__ Sp split_rn16(float x) {
  const uint32_t h = tf32_rn(x);
  return {h, tf32_rn(x - __uint_as_float(h))};
}
// hot split: ALU only (see volume_tc32.cu)
__device__ __forceinline__ Sp split16(float x) {
  const uint32_t h = __float_as_uint(x) & 0xffffe000u;
  return {h, __float_as_uint(x - __uint_as_float(h))};
}
__device__ __forceinline__ void mma16(float (&c)[4], uint32_t a0, uint32_t a1, uint32_t a2,
                                      uint32_t a3, uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
      "{%8,%9}, {%0,%1,%2,%3};"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}
__device__ __forceinline__ void pf_l2(const void *p, uint64_t bytes) {
  uintptr_t lo = reinterpret_cast<uintptr_t>(p) & ~(uintptr_t)15;
  const uintptr_t hi = (reinterpret_cast<uintptr_t>(p) + bytes + 15) & ~(uintptr_t)15;
  while (lo < hi) {
    const uint32_t n = (uint32_t)((hi - lo) > 65536 ? 65536 : (hi - lo));
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(lo), "r"(n) : "memory");
    lo += n;
  }
}

template <int NQ>
__global__ void __launch_bounds__(T16, 1)
    volume_tc16_kernel(int64_t ne, float p0, float R, float gam, const float *__restrict__ q,
                       float *__restrict__ rhsq, const float *__restrict__ D,
                       const float *__restrict__ g, const float *__restrict__ jinv) {
  static_assert(NQ >= 9 && NQ <= 16, "virtual 16x16 planes");
  constexpr int NPT = NQ * NQ * NQ;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  Smem16 &sm = *reinterpret_cast<Smem16 *>(smem_raw);

  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int gq = lane >> 2, c = lane & 3;
  const float Rp0 = R / p0;
  const bool wact = w < NQ;  // plane k = w (and (i,k)-plane j = w) exists

  for (int t = tid; t < TILE16; t += T16) {  // padding planes / rows stay zero
    sm.ft[t] = 0.f;
    sm.tout[t] = 0.f;
  }
  // D fragments (D[n*NQ + i] = D(i, n)), zero outside [0, NQ)^2
  auto Dv = [&](int iv, int nv) -> float {
    return (iv < NQ && nv < NQ) ? __ldg(D + nv * NQ + iv) : 0.0f;
  };
  // R: B[slot][i_out] = D(i_out = 8nt + g, n = pi(ks, slot)), pi = 8ks + 2c (+1)
  Sp Br[2][2][2];  // [nt][ks][b0/b1]
  // S, T: A[row][slot] = D(row = g (+8), n = 8ks + c (+4))
  Sp Ast[2][4];    // [ks][a0..a3]
#pragma unroll
  for (int ks = 0; ks < 2; ++ks) {
#pragma unroll
    for (int nt = 0; nt < 2; ++nt) {
      Br[nt][ks][0] = split_rn16(Dv(8 * nt + gq, 8 * ks + 2 * c));
      Br[nt][ks][1] = split_rn16(Dv(8 * nt + gq, 8 * ks + 2 * c + 1));
    }
    Ast[ks][0] = split_rn16(Dv(gq, 8 * ks + c));
    Ast[ks][1] = split_rn16(Dv(gq + 8, 8 * ks + c));
    Ast[ks][2] = split_rn16(Dv(gq, 8 * ks + c + 4));
    Ast[ks][3] = split_rn16(Dv(gq + 8, 8 * ks + c + 4));
  }
  // own points p = 4r + 2nt + s: (i = 8nt + 2c + s, j = gq + 8r, k = w)
  bool vld[8];
  int off[8];
#pragma unroll
  for (int r = 0; r < 2; ++r)
#pragma unroll
    for (int nt = 0; nt < 2; ++nt)
#pragma unroll
      for (int s = 0; s < 2; ++s) {
        const int p = 4 * r + 2 * nt + s, i = 8 * nt + 2 * c + s, j = gq + 8 * r;
        vld[p] = wact && i < NQ && j < NQ;
        off[p] = vld[p] ? (w * NQ + j) * NQ + i : 0;
      }
  __syncthreads();

  float *const stl = sm.stile[w];
  for (int64_t e = blockIdx.x; e < ne; e += gridDim.x) {
    const float *qe = q + e * 8 * NPT;
    const float *ge = g + e * 9 * NPT;
    const float *je = jinv + e * NPT;
    float *re = rhsq + e * 8 * NPT;
    const int64_t en = e + gridDim.x;
    if (en < ne) {
      if (tid == 0) pf_l2(q + en * 8 * NPT, 8ull * NPT * sizeof(float));
      if (tid == 32) pf_l2(g + en * 9 * NPT, 9ull * NPT * sizeof(float));
      if (tid == 64) pf_l2(rhsq + en * 8 * NPT, 8ull * NPT * sizeof(float));
      if (tid == 96) pf_l2(jinv + en * NPT, 1ull * NPT * sizeof(float));
    }
    // ---- phase 1: point-wise state of the own points --------------------
    float rinv[8], pr[8], V[3][8], jv[8];
#pragma unroll
    for (int p = 0; p < 8; ++p) {
      const int o = off[p];
      const bool ok = vld[p];
      const float rho = ok ? __ldg(qe + o) : 1.f;
      const float u1 = ok ? __ldg(qe + NPT + o) : 0.f, u2 = ok ? __ldg(qe + 2 * NPT + o) : 0.f,
                  u3 = ok ? __ldg(qe + 3 * NPT + o) : 0.f;
      const float th = ok ? __ldg(qe + 4 * NPT + o) : 1.f;
      jv[p] = ok ? __ldg(je + o) : 0.f;
      float gg[9];
#pragma unroll
      for (int x = 0; x < 9; ++x) gg[x] = ok ? __ldg(ge + x * NPT + o) : 0.f;
      rinv[p] = __frcp_rn(rho);
      pr[p] = p0 * exp2f(gam * __log2f(Rp0 * th));
#pragma unroll
      for (int d = 0; d < 3; ++d) V[d][p] = gg[3 * d] * u1 + gg[3 * d + 1] * u2 + gg[3 * d + 2] * u3;
    }

    // fields fully unrolled: b is a compile-time constant in every body, so
    // the momentum-only g loads and the b == 0 special case cost nothing
    // elsewhere; even Nq: the own pairs (s = 0, 1) are 8-byte loads
    auto ld_own = [&](const float *base, float (&out)[8]) {
#pragma unroll
      for (int rn = 0; rn < 4; ++rn) {
        const int p = 2 * rn;
        if constexpr (NQ % 2 == 0) {
          const float2 v = vld[p] ? __ldg(reinterpret_cast<const float2 *>(base + off[p]))
                                  : make_float2(0.f, 0.f);
          out[p] = v.x;
          out[p + 1] = v.y;
        } else {
          out[p] = vld[p] ? __ldg(base + off[p]) : 0.f;
          out[p + 1] = vld[p + 1] ? __ldg(base + off[p + 1]) : 0.f;
        }
      }
    };
#pragma unroll
    for (int b = 0; b < 8; ++b) {
      float rh[8], qb[8], gm[3][8];
#pragma unroll
      for (int p = 0; p < 8; ++p) {
        rh[p] = vld[p] ? re[b * NPT + off[p]] : 0.f;
        qb[p] = 0.f;
        gm[0][p] = gm[1][p] = gm[2][p] = 0.f;
      }
      if (b > 0) ld_own(qe + b * NPT, qb);
      if (b >= 1 && b <= 3) {
#pragma unroll
        for (int d = 0; d < 3; ++d) ld_own(ge + (3 * d + b - 1) * NPT, gm[d]);
      }
      // fluxes of the own points; F_t -> ft, F_s -> the warp's S tile (pairs
      // along i: 64-bit stores, conflict-free with the 24-float row stride)
      float fr[8];
#pragma unroll
      for (int r = 0; r < 2; ++r)
#pragma unroll
        for (int nt = 0; nt < 2; ++nt) {
          float fs2[2], ft2[2];
#pragma unroll
          for (int s = 0; s < 2; ++s) {
            const int p = 4 * r + 2 * nt + s;
            const float sc = (b == 0) ? 1.f : qb[p] * rinv[p];
            float f[3];
#pragma unroll
            for (int d = 0; d < 3; ++d) f[d] = fmaf(gm[d][p], pr[p], V[d][p] * sc);
            if (!vld[p]) f[0] = f[1] = f[2] = 0.f;
            fr[p] = f[0];
            fs2[s] = f[1];
            ft2[s] = f[2];
          }
          const int jj = gq + 8 * r, ii = 8 * nt + 2 * c;
          *reinterpret_cast<float2 *>(stl + jj * RS16 + ii) = make_float2(fs2[0], fs2[1]);
          if (wact)
            *reinterpret_cast<float2 *>(sm.ft + w * PS16 + jj * RS16 + ii) =
                make_float2(ft2[0], ft2[1]);
        }
      __syncwarp();
      // R (A = own F_r) and S (B = F_s transposed) into one accumulator per n-tile
      float acc[2][4] = {{0.f, 0.f, 0.f, 0.f}, {0.f, 0.f, 0.f, 0.f}};
      if (wact) {
#pragma unroll
        for (int ks = 0; ks < 2; ++ks) {
          // own points of n-tile ks: (r, s) -> A rows g / g+8, slots c / c+4
          const Sp a0 = split16(fr[0 + 2 * ks]), a1 = split16(fr[4 + 2 * ks]),
                   a2 = split16(fr[1 + 2 * ks]), a3 = split16(fr[5 + 2 * ks]);
#pragma unroll
          for (int nt = 0; nt < 2; ++nt) {
            mma16(acc[nt], a0.hi, a1.hi, a2.hi, a3.hi, Br[nt][ks][0].hi, Br[nt][ks][1].hi);
            mma16(acc[nt], a0.lo, a1.lo, a2.lo, a3.lo, Br[nt][ks][0].hi, Br[nt][ks][1].hi);
            mma16(acc[nt], a0.hi, a1.hi, a2.hi, a3.hi, Br[nt][ks][0].lo, Br[nt][ks][1].lo);
            // S: B[n][i] = F_s(i = 8nt + g, j = n = 8ks + c (+4)) = stile[n][i]
            const Sp b0 = split16(stl[(8 * ks + c) * RS16 + 8 * nt + gq]);
            const Sp b1 = split16(stl[(8 * ks + c + 4) * RS16 + 8 * nt + gq]);
            mma16(acc[nt], Ast[ks][0].hi, Ast[ks][1].hi, Ast[ks][2].hi, Ast[ks][3].hi, b0.hi,
                  b1.hi);
            mma16(acc[nt], Ast[ks][0].hi, Ast[ks][1].hi, Ast[ks][2].hi, Ast[ks][3].hi, b0.lo,
                  b1.lo);
            mma16(acc[nt], Ast[ks][0].lo, Ast[ks][1].lo, Ast[ks][2].lo, Ast[ks][3].lo, b0.hi,
                  b1.hi);
          }
        }
      }
      __syncthreads();  // ft complete
      if (wact) {  // T on the (i,k)-plane j = w: C[k][i] = sum_n D(k,n) F_t(i, w, n)
#pragma unroll
        for (int nt = 0; nt < 2; ++nt) {
          float tq[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
          for (int ks = 0; ks < 2; ++ks) {
            const Sp b0 = split16(sm.ft[(8 * ks + c) * PS16 + w * RS16 + 8 * nt + gq]);
            const Sp b1 = split16(sm.ft[(8 * ks + c + 4) * PS16 + w * RS16 + 8 * nt + gq]);
            mma16(tq, Ast[ks][0].hi, Ast[ks][1].hi, Ast[ks][2].hi, Ast[ks][3].hi, b0.hi, b1.hi);
            mma16(tq, Ast[ks][0].hi, Ast[ks][1].hi, Ast[ks][2].hi, Ast[ks][3].hi, b0.lo, b1.lo);
            mma16(tq, Ast[ks][0].lo, Ast[ks][1].lo, Ast[ks][2].lo, Ast[ks][3].lo, b0.hi, b1.hi);
          }
          // C rows k = g / g+8, cols i = 8nt + 2c (+1) of plane j = w
          *reinterpret_cast<float2 *>(sm.tout + gq * PS16 + w * RS16 + 8 * nt + 2 * c) =
              make_float2(tq[0], tq[1]);
          *reinterpret_cast<float2 *>(sm.tout + (gq + 8) * PS16 + w * RS16 + 8 * nt + 2 * c) =
              make_float2(tq[2], tq[3]);
        }
      }
      __syncthreads();  // tout complete
#pragma unroll
      for (int r = 0; r < 2; ++r)
#pragma unroll
        for (int nt = 0; nt < 2; ++nt) {
          const int jj = gq + 8 * r, ii = 8 * nt + 2 * c;
          const float2 tv = wact ? *reinterpret_cast<const float2 *>(sm.tout + w * PS16 +
                                                                    jj * RS16 + ii)
                                 : make_float2(0.f, 0.f);
#pragma unroll
          for (int s = 0; s < 2; ++s) {
            const int p = 4 * r + 2 * nt + s;
            if (vld[p])
              re[b * NPT + off[p]] = fmaf(jv[p], acc[nt][2 * r + s] + (s ? tv.y : tv.x), rh[p]);
          }
        }
    }
  }
}

template <int NQ>
int launch_tc16(int64_t ne, float p0, float R, float gam, const float *q, float *rhsq,
                const float *D, const float *g, const float *jinv, cudaStream_t s) {
  const size_t smem = sizeof(Smem16);
  auto kern = volume_tc16_kernel<NQ>;
  if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) !=
      cudaSuccess)
    return LFB_ERR_CUDA;
  int dev = 0, sms = 0, per_sm = 0;
  if (cudaGetDevice(&dev) != cudaSuccess ||
      cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess ||
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, T16, smem) != cudaSuccess)
    return LFB_ERR_CUDA;
  if (per_sm < 1) return LFB_ERR_LAUNCH;
  const int64_t slots = (int64_t)sms * per_sm;
  const int64_t grid = ne < slots ? ne : slots;
  if (grid == 0) return LFB_OK;
  kern<<<(unsigned)grid, T16, smem, s>>>(ne, p0, R, gam, q, rhsq, D, g, jinv);
  LFB_CHECK_LAUNCH();
  return LFB_OK;
}

}  // namespace

bool tc16_available(int nq) { return nq >= 9 && nq <= 16; }

int volume_tc16_f32(int nq, int64_t ne, float p0, float R, float gam, const float *q,
                    float *rhsq, const float *D, const float *g, const float *jinv,
                    cudaStream_t s) {
  switch (nq) {
    case 9: return launch_tc16<9>(ne, p0, R, gam, q, rhsq, D, g, jinv, s);
    case 10: return launch_tc16<10>(ne, p0, R, gam, q, rhsq, D, g, jinv, s);
    case 11: return launch_tc16<11>(ne, p0, R, gam, q, rhsq, D, g, jinv, s);
    case 12: return launch_tc16<12>(ne, p0, R, gam, q, rhsq, D, g, jinv, s);
    case 13: return launch_tc16<13>(ne, p0, R, gam, q, rhsq, D, g, jinv, s);
    case 14: return launch_tc16<14>(ne, p0, R, gam, q, rhsq, D, g, jinv, s);
    case 15: return launch_tc16<15>(ne, p0, R, gam, q, rhsq, D, g, jinv, s);
    case 16: return launch_tc16<16>(ne, p0, R, gam, q, rhsq, D, g, jinv, s);
    default: return LFB_ERR_BAD_VARIANT;
  }
}

}  // namespace lfb
