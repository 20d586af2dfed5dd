// LFB_VARIANT_TC — Nq = 8 (and 2, 4 packed / 5..7 padded into a virtual
// Nq=8 cube): TMA-staged, DMMA-contracted volume kernel, fp64 storage.
//
// fp32 storage takes the TF32 split-product kernel of volume_tc32.cu (the
// first fp32 variant — this kernel with fp64 arithmetic on f32 storage —
// reached 34 GDOF/s vs 47; it was removed after that A/B).
//
// Why this shape (numbers from tools/microbench.cu on
// B200): the fp64 tensor pipe (DMMA m8n8k4) has the same throughput as the
// DFMA pipe (18.3 vs 18.4 TFMA/s) and shares it, so tensor cores do not add
// flops here — they remove instructions, registers and shared-memory
// traffic: one DMMA is 256 FMAs whose operand exchange happens inside the
// tensor core, and the Nq = 8 derivative is exactly an 8x8x8 product
// (two m8n8k4 k-steps).
//
// Work decomposition, one element per CTA iteration (persistent grid, one
// CTA of 8 warps per SM):
//   * warp w owns the (i,j)-plane k = w; lane (g = lane/4, c = lane%4) owns
//     the points P_s = (i=g, j=c+4s, k=w), s = 0,1 — the DMMA C-fragment
//     (row g, col 2c+s) with the column permutation pi(2c+s) = c+4s;
//   * S (contract j): A = F_s at the thread's own points (k-index permuted
//     the same way), B = D — no data movement;
//   * R (contract i): B = F_r transposed in the plane — an 8x8 per-warp
//     shared tile;
//   * T (contract k) crosses planes, so each warp also owns the
//     (i,k)-plane j = w ("transposed" points Q_s = (i=g, j=w, k=c+4s)):
//     every thread evaluates F_t of all 8 fields at its own points once per
//     element and parks them in a padded shared tile; the transposed-plane
//     owners contract them by DMMA and hand the T result back to the
//     (i,j)-plane owners through a second shared tile.
//   * q and g of element e+2G are streamed into a shared stage by
//     cp.async.bulk (TMA) with an mbarrier while element e computes; the
//     stage is released right after phase 1, so the copy overlaps almost
//     two element-times of compute. rhsq and Jinv of the NEXT element are
//     prefetched into registers.
// Traffic is exactly the 272 B/pt minimum: every q, g, Jinv, rhsq value is
// read once and rhsq written once.

#include <stdlib.h>

#include "lfb_common.cuh"
#include "lfb_math.cuh"


namespace lfb {

int volume_basic_f64(int, int64_t, double, double, double, const double *, double *,
                     const double *, const double *, const double *, cudaStream_t);
int volume_fused_f64(int, int64_t, double, double, double, const double *, double *,
                     const double *, const double *, const double *, cudaStream_t);
bool fused_available(int dtype_bytes, int nq);
int volume_tc32_f32(int, int64_t, float, float, float, const float *, float *, const float *,
                    const float *, const float *, cudaStream_t);
int volume_tc16_f32(int, int64_t, float, float, float, const float *, float *, const float *,
                    const float *, const float *, cudaStream_t);

namespace {

#ifdef LFB_EXPERIMENTS
// test library only: which barrier-deletion mutant launch_tc runs (0 = none)
int g_tc_mutant = 0;
#endif

constexpr int TC_NQ = 8;
constexpr int TC_NPT = 512;
constexpr int TC_WARPS = 8;
constexpr int TC_THREADS = 32 * TC_WARPS;
constexpr int TC_STAGE = 17 * TC_NPT;  // values: q (8 fields) + g (9)
// packed Nq = 4 groups keep their 8 elements' slabs 64 B apart in the stage
// (one bulk copy per slab): unpadded, the 4 KB / 2 KB slab stride put the
// two elements a half-warp touches on the same banks (4-way conflicts)
template <typename T>
constexpr int tc_stage_alloc() { return TC_STAGE + 16 * 64 / (int)sizeof(T); }

__device__ __forceinline__ uint32_t smem_addr(const void *p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count)
               : "memory");
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)),
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
      "}\n" ::"r"(smem_addr(bar)),
      "r"(parity)
      : "memory");
}

__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, uint32_t bytes,
                                         uint64_t *bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_addr(dst)),
      "l"(src), "r"(bytes), "r"(smem_addr(bar))
      : "memory");
}

__device__ __forceinline__ void prefetch_l2(const void *p, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes) : "memory");
}

__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

// D += A * B on one m8n8k4 fp64 tile (A row-major 8x4, B col-major 4x8).
__device__ __forceinline__ void dmma(double &d0, double &d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

// A pair of adjacent values (the thread's two points) in storage type T.
template <typename T>
struct Pair;
template <>
struct Pair<double> {
  using V = double2;
};
template <>
struct Pair<float> {
  using V = float2;
};

template <typename T>
__device__ __forceinline__ void ld_pair(const T *p, double &a, double &b) {
  const typename Pair<T>::V v = *reinterpret_cast<const typename Pair<T>::V *>(p);
  a = (double)v.x;
  b = (double)v.y;
}
template <typename T>
__device__ __forceinline__ void ldg_pair(const T *p, double &a, double &b) {
  const typename Pair<T>::V v = __ldg(reinterpret_cast<const typename Pair<T>::V *>(p));
  a = (double)v.x;
  b = (double)v.y;
}
template <typename T>
__device__ __forceinline__ void st_pair(T *p, double a, double b) {
  typename Pair<T>::V v;
  v.x = (T)a;
  v.y = (T)b;
  *reinterpret_cast<typename Pair<T>::V *>(p) = v;
}

// Shared tiles (doubles), laid out so every access below is conflict-free
// per half-warp (64-bit accesses are served 16 lanes at a time, 128-bit ones
// 8 lanes at a time):
//   ft [field][k][j][i], k-plane stride 68: F_t written as 16-byte pairs
//      along i in one plane, read by the (i,k)-plane owners 4 k-planes x 4 i
//      at a time (plane offsets 544 B = 32 B mod 128: distinct bank groups);
//   tout [field][k][j][i], k-plane stride 72 (576 B = 64 B mod 128): T
//      results written as pairs from 4 k-planes, read back within one plane;
//   stile per-warp [j][i], row stride 12 (96 B): the in-plane S transpose.
constexpr int FT_PS = 68, FT_FS = 8 * FT_PS;
constexpr int TO_PS = 72, TO_FS = 8 * TO_PS;
constexpr int ST_SZ = 72;
// row r of the per-warp F_s transpose tile (8 rows x 8 doubles): the 16-byte
// pair stores (rows gq, 2a / 2a+1 per quarter-warp) and the transposed 8-byte
// reads (rows c + 4t, column gq per half-warp) are both conflict-free with
// these row starts (a plain stride of 12 made the stores 2-way)
__device__ __forceinline__ int st_row(int r) {
  return 8 * r + 4 * (((r >> 1) & 1) + ((r >> 2) & 1));
}

// NW < 8 (zero-padded Nq, one warp per real k-plane): stages hold the real
// q + g slab only (+ the g superset's 16-byte shift)
template <typename T, int NS, int SUB, int NW>
struct TcSmem {
  static constexpr int STAGE =
      NW == 8 ? tc_stage_alloc<T>() : ((17 * SUB * SUB * SUB + 2 + 1) & ~1);
  T stage[NS][STAGE];
  double ft[8 * FT_FS];
  double tout[8 * TO_FS];
  double stile[NW][2][ST_SZ];
  unsigned long long bar[NS];
};

// 1/rho and p = p0 (R Theta / p0)^gam of one point. fp32 storage
// (tolerance 1e-5): both in the FP32 pipe (MUFU rcp/lg2/ex2, ~5e-7
// relative); the fluxes and the contractions stay fp64.
template <typename T>
__device__ __forceinline__ void point_scalars(double rho, double th, double p0, double Rp0,
                                              double gam, double &rinv, double &p) {
  if constexpr (sizeof(T) == 4) {
    rinv = (double)__frcp_rn((float)rho);
    p = p0 * (double)exp2f((float)gam * log2f((float)Rp0 * (float)th));
  } else {
    rinv = fast_rcp(rho);
    p = p0 * pos_pow(Rp0 * th, gam);
  }
}

__device__ __forceinline__ void sts2(double *p, double a, double b) {
  *reinterpret_cast<double2 *>(p) = make_double2(a, b);
}

// Phase 2 walks the fields one at a time: F_s transposed through a
// per-warp tile (__syncwarp only), T results exchanged through tout, 2 CTA
// barriers per element. (An all-fields-at-once variant with an element-wide
// F_s tile and 4 barriers measured 3% slower: profiles/r01_ab_perfield.txt.)
// SUB = the real Nq. SUB = 8: one element per iteration. SUB = 4 or 2: a
// "virtual" Nq=8 element packs P^3 real elements (P = 8/SUB) — virtual point
// (i + SUB a, j + SUB b, k + SUB c) is point (i,j,k) of real element
// a + P b + P^2 c of the group — and the virtual D is blockdiag(D, ..., D),
// so the Nq=8 contraction machinery computes P^3 independent elements.
// A group of P^3 consecutive elements is the same 8*512 / 9*512 value slab
// as one Nq=8 element, so the TMA and prefetch code is unchanged; only the
// thread's own-point offsets inside the slab differ. `ne` counts groups.
// MUT != 0 builds a barrier-deletion mutant for the race-detector test (only
// in the test library, -DLFB_EXPERIMENTS)
// (tests/test_mutants.py; cf. the reference's barrier-deletion mutation test,
// pkg/tests/test_acceptance.py:191-219): 1 drops the F_t barrier, 2 the
// T-out barrier, 3 the per-warp S-tile __syncwarp.
template <typename T, int NS, int SUB, int MUT = 0, int NW = TC_WARPS>
__global__ void __launch_bounds__(32 * NW, 1)
    volume_tc_kernel(int64_t ne, double p0, double R, double gam, const T *__restrict__ q,
                     T *__restrict__ rhsq, const T *__restrict__ D, const T *__restrict__ g,
                     const T *__restrict__ jinv) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  TcSmem<T, NS, SUB, NW> &sm = *reinterpret_cast<TcSmem<T, NS, SUB, NW> *>(smem_raw);
  if (NW < 8) {  // F_t planes k >= SUB have no owner warp: they stay zero
    for (int x = threadIdx.x; x < 8 * FT_FS; x += 32 * NW) sm.ft[x] = 0.0;
  }

  const int tid = threadIdx.x;
  const int lane = tid & 31, w = tid >> 5;
  const int gq = lane >> 2, c = lane & 3;
  const int64_t G = gridDim.x;
  const int64_t e0 = blockIdx.x;
  const int64_t nmine = (e0 < ne) ? (ne - 1 - e0) / G + 1 : 0;
  const double Rp0 = R / p0;

  // Own points P_s = (i = 2c+s, j = g, k = w): the DMMA C-fragment (row g = j,
  // cols 2c+s = i) of the warp's (i,j)-plane; an adjacent pair in memory.
  // PAD (Nq = 5, 6, 7): one real element zero-padded into the virtual Nq=8
  // cube; virtual points with a coordinate >= Nq carry zero flux and D is
  // zero outside [0,Nq)^2, so they neither contribute nor get written.
  constexpr bool PAD = !(SUB == 8 || SUB == 4 || SUB == 2);
  static_assert(SUB >= 2 && SUB <= 8, "virtual Nq=8 cube");
  constexpr int P = PAD ? 1 : 8 / SUB, NPTR = SUB * SUB * SUB;
  constexpr int SLABQ = PAD ? 8 * NPTR : 8 * TC_NPT;  // values per group: q, rhsq
  constexpr int SLABG = PAD ? 9 * NPTR : 9 * TC_NPT;  // g
  constexpr int SLABJ = PAD ? NPTR : TC_NPT;          // Jinv
  // own pair (virtual i = 2c, 2c+1; j = g; k = w) inside the group's slabs
  const int ur = PAD ? 0 : (2 * c) / SUB + P * (gq / SUB) + P * P * (w / SUB);  // real element
  const int ptr = PAD ? (w * SUB + gq) * SUB + 2 * c
                      : ((w % SUB) * SUB + (gq % SUB)) * SUB + (2 * c) % SUB;     // real point
  const int qo = ur * 8 * NPTR + ptr;  // q / rhsq field 0; fields stride NPTR
  // stage layout: SUB = 4 -> per-element slabs padded by EPAD values
  constexpr int EPAD = (SUB == 4) ? 64 / (int)sizeof(T) : 0;
  constexpr int SQE = 8 * NPTR + EPAD, SGE = 9 * NPTR + EPAD;
  constexpr int SGOFF = (SUB == 4) ? 8 * SQE : SLABQ;  // g section of the stage
  const int sqo = (SUB == 4) ? ur * SQE + ptr : qo;    // own pair in the stage: q
  const int go = (SUB == 4) ? ur * SGE + ptr : ur * 9 * NPTR + ptr;  // and g
  const int jo = ur * NPTR + ptr;      // Jinv
  bool vld[2];
#pragma unroll
  for (int s = 0; s < 2; ++s) vld[s] = !PAD || (2 * c + s < SUB && gq < SUB && w < SUB);
  const int ftW = w * FT_PS + gq * 8 + 2 * c;          // own pair in ft
  const int toR = w * TO_PS + gq * 8 + 2 * c;          // own pair in tout
  const int toW = gq * TO_PS + w * 8 + 2 * c;          // T result (k=g, j=w, i=2c..)
  int ftR[2];
#pragma unroll
  for (int t = 0; t < 2; ++t) {
    ftR[t] = (c + 4 * t) * FT_PS + w * 8 + gq;         // F_t(i=g, j=w, k=c+4t)
  }
  // D fragments (D[n*8 + i] = D(i, n)):
  //   R: B[c][g] = D(i=g, n=2c+t);  S and T: A[g][c] = D(g, n=c+4t)
  // (virtual D = blockdiag of the real D for SUB < 8)
  auto Dv = [&](int iv, int nv) -> double {
    if (PAD) return (iv < SUB && nv < SUB) ? (double)__ldg(D + nv * SUB + iv) : 0.0;
    if (iv / SUB != nv / SUB) return 0.0;
    return (double)__ldg(D + (nv % SUB) * SUB + (iv % SUB));
  };
  // 16-byte aligned superset of element e's g slab (PAD: 9 Nq^3 values need
  // not be a multiple of 16 bytes); returns the copy start and byte count
  auto gspan = [&](int64_t e, const T *&start, uint32_t &bytes) {
    const uintptr_t a = reinterpret_cast<uintptr_t>(g + e * SLABG);
    const uintptr_t lo = a & ~(uintptr_t)15;
    const uintptr_t hi = (a + SLABG * sizeof(T) + 15) & ~(uintptr_t)15;
    start = reinterpret_cast<const T *>(lo);
    bytes = (uint32_t)(hi - lo);
  };
  auto jspan = [&](int64_t e, const T *&start, uint32_t &bytes) {
    const uintptr_t a = reinterpret_cast<uintptr_t>(jinv + e * SLABJ);
    const uintptr_t lo = a & ~(uintptr_t)15;
    const uintptr_t hi = (a + SLABJ * sizeof(T) + 15) & ~(uintptr_t)15;
    start = reinterpret_cast<const T *>(lo);
    bytes = (uint32_t)(hi - lo);
  };
  double Dr[2], Dst[2];
#pragma unroll
  for (int t = 0; t < 2; ++t) {
    Dr[t] = Dv(gq, 2 * c + t);
    Dst[t] = Dv(gq, c + 4 * t);
  }

  uint64_t *bars = reinterpret_cast<uint64_t *>(sm.bar);
  if (tid == 0) {
#pragma unroll
    for (int s = 0; s < NS; ++s) mbar_init(&bars[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  auto issue = [&](int64_t n) {  // element index n (in this CTA's sequence) -> stage n % NS
    const int s = (int)(n % NS);
    const int64_t e = e0 + n * G;
    const T *gs;
    uint32_t gb;
    gspan(e, gs, gb);
    mbar_expect_tx(&bars[s], SLABQ * sizeof(T) + gb);
    if constexpr (SUB == 4) {
#pragma unroll 1
      for (int u = 0; u < 8; ++u) {
        bulk_g2s(sm.stage[s] + u * SQE, q + e * SLABQ + u * 8 * NPTR, 8 * NPTR * sizeof(T),
                 &bars[s]);
        bulk_g2s(sm.stage[s] + SGOFF + u * SGE, g + e * SLABG + u * 9 * NPTR,
                 9 * NPTR * sizeof(T), &bars[s]);
      }
    } else {
      bulk_g2s(sm.stage[s], q + e * SLABQ, SLABQ * sizeof(T), &bars[s]);
      bulk_g2s(sm.stage[s] + SLABQ, gs, gb, &bars[s]);
    }
  };
  if (tid == 0) {
    for (int64_t n = 0; n < NS && n < nmine; ++n) issue(n);
  }
  // L2 prefetch (cp.async.bulk.prefetch.L2) of the stage one beyond the
  // shared ring and of the next element's rhsq / Jinv: ~1 element per CTA
  // (~20 MB chip-wide at fp64) in flight ahead of the TMA copies (a longer
  // distance measured no better, profiles/r01_ab_tc_prefetch.txt)
  auto l2pf = [&](int64_t n) {
    if (tid == 0 && n + NS < nmine) {
      const int64_t e = e0 + (n + NS) * G;
      const T *gs;
      uint32_t gb;
      gspan(e, gs, gb);
      prefetch_l2(q + e * SLABQ, SLABQ * sizeof(T));
      prefetch_l2(gs, gb);
    }
    if (tid == 32 && n + 1 < nmine) {
      const int64_t e = e0 + (n + 1) * G;
      const T *js;
      uint32_t jb;
      jspan(e, js, jb);
      prefetch_l2(rhsq + e * SLABQ, SLABQ * sizeof(T));
      prefetch_l2(js, jb);
    }
  };

  for (int64_t n = 0; n < nmine; ++n) {
    const int st = (int)(n % NS);
    const uint32_t parity = (uint32_t)((n / NS) & 1);
    const int64_t e = e0 + n * G;
    const T *sq = sm.stage[st];
    const T *sg = sm.stage[st] + SGOFF +
                  (PAD ? (reinterpret_cast<uintptr_t>(g + e * SLABG) & 15) / sizeof(T) : 0);
    T *re = rhsq + e * SLABQ;

    // rhsq / Jinv of this element: only needed at write-back, so the latency
    // hides behind the element's compute (and the lines are L2-prefetched)
    double rh[8][2], jv[2];
#pragma unroll
    for (int b = 0; b < 8; ++b) {
      if (PAD) {
        rh[b][0] = vld[0] ? (double)re[qo + b * NPTR] : 0.0;
        rh[b][1] = vld[1] ? (double)re[qo + b * NPTR + 1] : 0.0;
      } else {
        ld_pair(re + qo + b * NPTR, rh[b][0], rh[b][1]);
      }
    }
    if (PAD) {
      jv[0] = vld[0] ? (double)jinv[e * SLABJ + jo] : 0.0;
      jv[1] = vld[1] ? (double)jinv[e * SLABJ + jo + 1] : 0.0;
    } else {
      ldg_pair(jinv + e * SLABJ + jo, jv[0], jv[1]);
    }
    l2pf(n);

    mbar_wait(&bars[st], parity);

    // ---- phase 1: point-wise quantities of the thread's two points ------
    double sb[8][2], V0[2], V1[2], pP[2], gr[3][2], gs[3][2];
    {
      double qv[8][2], gv[9][2];
#pragma unroll
      for (int f = 0; f < 8; ++f) {
        if (PAD) {  // padding points: rho = 1, everything else 0 -> zero flux
          qv[f][0] = vld[0] ? (double)sq[sqo + f * NPTR] : (f == 0 ? 1.0 : 0.0);
          qv[f][1] = vld[1] ? (double)sq[sqo + f * NPTR + 1] : (f == 0 ? 1.0 : 0.0);
        } else {
          ld_pair(sq + sqo + f * NPTR, qv[f][0], qv[f][1]);
        }
      }
#pragma unroll
      for (int x = 0; x < 9; ++x) {
        if (PAD) {
          gv[x][0] = vld[0] ? (double)sg[go + x * NPTR] : 0.0;
          gv[x][1] = vld[1] ? (double)sg[go + x * NPTR + 1] : 0.0;
        } else {
          ld_pair(sg + go + x * NPTR, gv[x][0], gv[x][1]);
        }
      }
      double V2[2];
#pragma unroll
      for (int s = 0; s < 2; ++s) {
        double rinv;
        point_scalars<T>(qv[0][s], qv[4][s], p0, Rp0, gam, rinv, pP[s]);
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
      sts2(sm.ft + ftW, V2[0], V2[1]);
#pragma unroll
      for (int b = 1; b < 8; ++b) {
        double f0 = V2[0] * sb[b][0], f1 = V2[1] * sb[b][1];
        if (b <= 3) {
          f0 += gv[6 + (b - 1)][0] * pP[0];
          f1 += gv[6 + (b - 1)][1] * pP[1];
        }
        sts2(sm.ft + b * FT_FS + ftW, f0, f1);
      }
    }
    if (MUT != 1) __syncthreads();  // ft complete; every stage read of this element is done
    if (tid == 0 && n + NS < nmine) {
      fence_proxy_async();
      issue(n + NS);
    }
    // ---- phase 2: per field ----------------------------------------------
    double acc[8][2];
#pragma unroll
    for (int b = 0; b < 8; ++b) {
      double fr[2], fs[2];
#pragma unroll
      for (int s = 0; s < 2; ++s) {
        if (b == 0) {
          fr[s] = V0[s];
          fs[s] = V1[s];
        } else {
          fr[s] = V0[s] * sb[b][s];
          fs[s] = V1[s] * sb[b][s];
          if (b <= 3) {
            fr[s] += gr[b - 1][s] * pP[s];
            fs[s] += gs[b - 1][s] * pP[s];
          }
        }
      }
      double *stl = sm.stile[w][b & 1];
      sts2(stl + st_row(gq) + 2 * c, fs[0], fs[1]);
      if (MUT != 3) __syncwarp();
      double fsT[2], ftQ[2];
#pragma unroll
      for (int t = 0; t < 2; ++t) {
        fsT[t] = stl[st_row(c + 4 * t) + gq];
        ftQ[t] = sm.ft[b * FT_FS + ftR[t]];
      }
      double a0 = 0.0, a1 = 0.0, q0 = 0.0, q1 = 0.0;
#pragma unroll
      for (int t = 0; t < 2; ++t) {
        dmma(a0, a1, fr[t], Dr[t]);
        dmma(a0, a1, Dst[t], fsT[t]);
        dmma(q0, q1, Dst[t], ftQ[t]);
      }
      acc[b][0] = a0;
      acc[b][1] = a1;
      sts2(sm.tout + b * TO_FS + toW, q0, q1);
    }
    if (MUT != 2) __syncthreads();  // tout complete
#pragma unroll
    for (int b = 0; b < 8; ++b) {
      const double2 t = *reinterpret_cast<const double2 *>(sm.tout + b * TO_FS + toR);
      const double o0 = rh[b][0] + jv[0] * (acc[b][0] + t.x);
      const double o1 = rh[b][1] + jv[1] * (acc[b][1] + t.y);
      if (PAD) {
        if (vld[0]) re[qo + b * NPTR] = (T)o0;
        if (vld[1]) re[qo + b * NPTR + 1] = (T)o1;
      } else {
        st_pair(re + qo + b * NPTR, o0, o1);
      }
    }
  }
}

// ---------------------------------------------------------------------------
// LEAN schedule: two CTAs per SM (<= 128 registers, ~102 KB shared each).
// One stage per CTA; after phase 1 the dead stage holds the per-warp S tiles
// and a per-field double-buffered T-out tile, and every field is written
// back as soon as its T result is exchanged (no 8-field register state).
// The next element's TMA is issued when the element is done (its bytes are
// already L2-prefetched); the co-resident CTA computes meanwhile.
//
// PLANE variant (NW = SUB < 8 warps, zero-padded Nq = 5..7): only the SUB
// real k-planes get a warp (the 8 - SUB all-padding planes of the virtual
// cube issued DMMAs on zeros), the stage holds just the element's real
// q + g slab, the padding planes of the F_t tile are zeroed once, and
// several such CTAs share an SM (MINB).
constexpr int LEAN_TOUT = 0;                    // doubles into the stage: tout[2][TO_FS]
constexpr int LEAN_STILE = 2 * TO_FS;           // stile[NW warps][ST_SZ]

template <typename T, int SUB, int NW>
struct TcLeanCfg {
  static constexpr bool PAD = !(SUB == 8 || SUB == 4 || SUB == 2);
  // NW = 8: the virtual-cube stage; NW < 8: the real slab (+ the g superset's
  // 16-byte shift), at least as large as the tout / stile aliases
  static constexpr int REAL = (17 * SUB * SUB * SUB + 2 + 1) & ~1;
  static constexpr int ALIAS = (LEAN_STILE + NW * ST_SZ) * (int)(sizeof(double) / sizeof(T));
  static constexpr int STAGE = NW == 8 ? TC_STAGE : (REAL > ALIAS ? REAL : ALIAS);
  static constexpr int MINB = NW == 8 ? 2 : (SUB == 5 ? 3 : 2);
  // NW < 8, Nq <= 6: a 2-stage ring — element n+1's copy is issued when
  // element n starts (its stage was element n-1's, free after n-1's last
  // barrier); at Nq = 7 two stages would leave one CTA per SM
  static constexpr int NSTG = (NW < 8 && SUB <= 6) ? 2 : 1;  // Nq=7: 2 stages -> 1 CTA/SM
  // NW < 8 with one stage (Nq = 7): the S and T-out tiles get their own
  // space, so the stage is dead right after phase 1 and the next element's
  // copy is issued then, not after the write-back (0.77 -> 0.82 of HBM; at
  // Nq 5, 6 own tiles with 1 or 2 stages measured no better than the ring,
  // profiles/r02_tc_plane.txt)
  static constexpr bool OWN_TILES = NW < 8 && NSTG == 1;
  static_assert(NW == 8 || PAD, "plane variant is for the zero-padded Nq");
  static_assert(LEAN_STILE + NW * ST_SZ <= STAGE * (int)sizeof(T) / (int)sizeof(double),
                "aliases fit in the stage");
};

template <typename T, int SUB, int NW>
struct TcSmemLean {
  T stage[TcLeanCfg<T, SUB, NW>::NSTG][TcLeanCfg<T, SUB, NW>::STAGE];
  double tiles[TcLeanCfg<T, SUB, NW>::OWN_TILES ? LEAN_STILE + NW * ST_SZ : 2];  // (keeps ft 16-byte aligned)
  double ft[8 * FT_FS];
  unsigned long long bar[TcLeanCfg<T, SUB, NW>::NSTG];
};

template <typename T, int SUB, int NW = TC_WARPS>
__global__ void __launch_bounds__(32 * NW, (TcLeanCfg<T, SUB, NW>::MINB))
    volume_tc_lean_kernel(int64_t ne, double p0, double R, double gam, const T *__restrict__ q,
                          T *__restrict__ rhsq, const T *__restrict__ D,
                          const T *__restrict__ g, const T *__restrict__ jinv) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  TcSmemLean<T, SUB, NW> &sm = *reinterpret_cast<TcSmemLean<T, SUB, NW> *>(smem_raw);
  constexpr int NSTG = TcLeanCfg<T, SUB, NW>::NSTG;
  constexpr bool OWN_TILES = TcLeanCfg<T, SUB, NW>::OWN_TILES;
  if (NW < 8) {  // F_t planes k >= SUB have no owner warp: they stay zero
    for (int x = threadIdx.x; x < 8 * FT_FS; x += 32 * NW) sm.ft[x] = 0.0;
  }

  const int tid = threadIdx.x;
  const int lane = tid & 31, w = tid >> 5;
  const int gq = lane >> 2, c = lane & 3;
  const int64_t G = gridDim.x;
  const int64_t e0 = blockIdx.x;
  const int64_t nmine = (e0 < ne) ? (ne - 1 - e0) / G + 1 : 0;
  const double Rp0 = R / p0;

  constexpr bool PAD = !(SUB == 8 || SUB == 4 || SUB == 2);
  // even padded Nq (6): a lane's two points are valid together and 16-byte
  // aligned, so they move as one 16-byte access (the separate 8-byte stage
  // reads were 2-3-way bank conflicted)
  constexpr bool PAIRS = PAD && SUB % 2 == 0;
  constexpr int P = PAD ? 1 : 8 / SUB, NPTR = SUB * SUB * SUB;
  constexpr int SLABQ = PAD ? 8 * NPTR : 8 * TC_NPT;
  constexpr int SLABG = PAD ? 9 * NPTR : 9 * TC_NPT;
  constexpr int SLABJ = PAD ? NPTR : TC_NPT;
  const int ur = PAD ? 0 : (2 * c) / SUB + P * (gq / SUB) + P * P * (w / SUB);
  const int ptr = PAD ? (w * SUB + gq) * SUB + 2 * c
                      : ((w % SUB) * SUB + (gq % SUB)) * SUB + (2 * c) % SUB;
  const int qo = ur * 8 * NPTR + ptr;
  const int go = ur * 9 * NPTR + ptr;
  const int jo = ur * NPTR + ptr;
  bool vld[2];
#pragma unroll
  for (int s = 0; s < 2; ++s) vld[s] = !PAD || (2 * c + s < SUB && gq < SUB && w < SUB);
  // odd padded Nq: the two 8-byte stage reads of a lane's point pair go out
  // in a per-lane order (bit = point 2c+1 first) chosen by exhaustive search
  // so that both instructions are conflict-free (Nq 7: 2-way -> none; Nq 5
  // is conflict-free either way); a uniform shift (plane, field, g offset)
  // does not change the bank pattern, so one mask serves every read
  const int sw = (PAD && !PAIRS && SUB == 7) ? (int)((0x70873u >> lane) & 1u) : 0;
  auto ld_stage = [&](const T *p, double dflt, double &a, double &b) {
    const bool v0 = vld[sw], v1 = vld[sw ^ 1];
    const double x0 = v0 ? (double)p[sw] : dflt;
    const double x1 = v1 ? (double)p[sw ^ 1] : dflt;
    a = sw ? x1 : x0;
    b = sw ? x0 : x1;
  };
  const int ftW = w * FT_PS + gq * 8 + 2 * c;
  const int toR = w * TO_PS + gq * 8 + 2 * c;
  const int toW = gq * TO_PS + w * 8 + 2 * c;
  int ftR[2];
#pragma unroll
  for (int t = 0; t < 2; ++t) ftR[t] = (c + 4 * t) * FT_PS + w * 8 + gq;
  auto Dv = [&](int iv, int nv) -> double {
    if (PAD) return (iv < SUB && nv < SUB) ? (double)__ldg(D + nv * SUB + iv) : 0.0;
    if (iv / SUB != nv / SUB) return 0.0;
    return (double)__ldg(D + (nv % SUB) * SUB + (iv % SUB));
  };
  double Dr[2], Dst[2];
#pragma unroll
  for (int t = 0; t < 2; ++t) {
    Dr[t] = Dv(gq, 2 * c + t);
    Dst[t] = Dv(gq, c + 4 * t);
  }
  auto span16 = [](const T *p, size_t n, const T *&start, uint32_t &bytes) {
    const uintptr_t a = reinterpret_cast<uintptr_t>(p);
    const uintptr_t lo = a & ~(uintptr_t)15;
    const uintptr_t hi = (a + n * sizeof(T) + 15) & ~(uintptr_t)15;
    start = reinterpret_cast<const T *>(lo);
    bytes = (uint32_t)(hi - lo);
  };

  uint64_t *bars = reinterpret_cast<uint64_t *>(sm.bar);
  if (tid == 0) {
#pragma unroll
    for (int x = 0; x < NSTG; ++x) mbar_init(&bars[x], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  auto issue = [&](int64_t n) {
    const int64_t e = e0 + n * G;
    const int st = (int)(n % NSTG);
    const T *gs;
    uint32_t gb;
    span16(g + e * SLABG, SLABG, gs, gb);
    mbar_expect_tx(&bars[st], SLABQ * sizeof(T) + gb);
    bulk_g2s(sm.stage[st], q + e * SLABQ, SLABQ * sizeof(T), &bars[st]);
    bulk_g2s(sm.stage[st] + SLABQ, gs, gb, &bars[st]);
  };
  if (tid == 0 && nmine > 0) issue(0);

  for (int64_t n = 0; n < nmine; ++n) {
    const int64_t e = e0 + n * G;
    const int st = (int)(n % NSTG);
    double *const alias = OWN_TILES ? sm.tiles : reinterpret_cast<double *>(sm.stage[st]);
    if (NSTG == 2 && tid == 0 && n + 1 < nmine) {
      fence_proxy_async();  // the other stage's last reads were before the previous barrier
      issue(n + 1);
    }
    // L2 prefetch of the next element (NSTG = 1: its q / g TMA is issued at
    // the end of this one; NSTG = 2: already issued above)
    if (n + 1 < nmine) {
      const int64_t en = e + G;
      const T *sp;
      uint32_t sb_;
      if (NSTG == 1 && !OWN_TILES && tid == 0) {
        prefetch_l2(q + en * SLABQ, SLABQ * sizeof(T));
        span16(g + en * SLABG, SLABG, sp, sb_);
        prefetch_l2(sp, sb_);
      } else if (tid == 32) {
        prefetch_l2(rhsq + en * SLABQ, SLABQ * sizeof(T));
        span16(jinv + en * SLABJ, SLABJ, sp, sb_);
        prefetch_l2(sp, sb_);
      }
    }
    const T *sq = sm.stage[st];
    const T *sg = sm.stage[st] + SLABQ +
                  (PAD ? (reinterpret_cast<uintptr_t>(g + e * SLABG) & 15) / sizeof(T) : 0);
    T *re = rhsq + e * SLABQ;
    double jv[2];
    if (PAD && !PAIRS) {
      jv[0] = vld[0] ? (double)jinv[e * SLABJ + jo] : 0.0;
      jv[1] = vld[1] ? (double)jinv[e * SLABJ + jo + 1] : 0.0;
    } else if (PAIRS && !vld[0]) {
      jv[0] = jv[1] = 0.0;
    } else {
      ldg_pair(jinv + e * SLABJ + jo, jv[0], jv[1]);
    }

    mbar_wait(&bars[st], (uint32_t)((n / NSTG) & 1));

    // ---- phase 1 (as in the 1-CTA kernel) ----------------------------------
    double sb[8][2], V0[2], V1[2], pP[2], gr[3][2], gs[3][2];
    {
      double qv[8][2], gv[9][2];
#pragma unroll
      for (int f = 0; f < 8; ++f) {
        if (PAD && !PAIRS) {
          ld_stage(sq + qo + f * NPTR, f == 0 ? 1.0 : 0.0, qv[f][0], qv[f][1]);
        } else if (PAIRS && !vld[0]) {
          qv[f][0] = qv[f][1] = (f == 0 ? 1.0 : 0.0);
        } else {
          ld_pair(sq + qo + f * NPTR, qv[f][0], qv[f][1]);
        }
      }
#pragma unroll
      for (int x = 0; x < 9; ++x) {
        if (PAD && !PAIRS) {
          ld_stage(sg + go + x * NPTR, 0.0, gv[x][0], gv[x][1]);
        } else if (PAIRS && !vld[0]) {
          gv[x][0] = gv[x][1] = 0.0;
        } else {
          ld_pair(sg + go + x * NPTR, gv[x][0], gv[x][1]);
        }
      }
      double V2[2];
#pragma unroll
      for (int s = 0; s < 2; ++s) {
        double rinv;
        point_scalars<T>(qv[0][s], qv[4][s], p0, Rp0, gam, rinv, pP[s]);
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
      sts2(sm.ft + ftW, V2[0], V2[1]);
#pragma unroll
      for (int b = 1; b < 8; ++b) {
        double f0 = V2[0] * sb[b][0], f1 = V2[1] * sb[b][1];
        if (b <= 3) {
          f0 += gv[6 + (b - 1)][0] * pP[0];
          f1 += gv[6 + (b - 1)][1] * pP[1];
        }
        sts2(sm.ft + b * FT_FS + ftW, f0, f1);
      }
    }
    __syncthreads();  // ft complete; the stage is dead -> S and T-out tiles live in it
    if (OWN_TILES && tid == 0 && n + 1 < nmine) {  // (or have their own space)
      fence_proxy_async();
      issue(n + 1);
    }

    // ---- phase 2: per field, written back as soon as T is exchanged ------
    // (rhsq of field b+1 is loaded while field b computes)
    auto ld_rh = [&](int b, double &r0, double &r1) {
      if (PAD && !PAIRS) {
        r0 = vld[0] ? (double)re[qo + b * NPTR] : 0.0;
        r1 = vld[1] ? (double)re[qo + b * NPTR + 1] : 0.0;
      } else if (PAIRS && !vld[0]) {
        r0 = r1 = 0.0;
      } else {
        ld_pair(re + qo + b * NPTR, r0, r1);
      }
    };
    double rn0, rn1;
    ld_rh(0, rn0, rn1);
#pragma unroll
    for (int b = 0; b < 8; ++b) {
      const double rh0 = rn0, rh1 = rn1;
      if (b < 7) ld_rh(b + 1, rn0, rn1);
      double fr[2], fs[2];
#pragma unroll
      for (int s = 0; s < 2; ++s) {
        if (b == 0) {
          fr[s] = V0[s];
          fs[s] = V1[s];
        } else {
          fr[s] = V0[s] * sb[b][s];
          fs[s] = V1[s] * sb[b][s];
          if (b <= 3) {
            fr[s] += gr[b - 1][s] * pP[s];
            fs[s] += gs[b - 1][s] * pP[s];
          }
        }
      }
      double *stl = alias + LEAN_STILE + w * ST_SZ;
      if (b > 0) __syncwarp();  // previous field's transposed reads are done
      sts2(stl + st_row(gq) + 2 * c, fs[0], fs[1]);
      __syncwarp();
      double fsT[2], ftQ[2];
#pragma unroll
      for (int t = 0; t < 2; ++t) {
        fsT[t] = stl[st_row(c + 4 * t) + gq];
        ftQ[t] = sm.ft[b * FT_FS + ftR[t]];
      }
      double a0 = 0.0, a1 = 0.0, q0 = 0.0, q1 = 0.0;
#pragma unroll
      for (int t = 0; t < 2; ++t) {
        dmma(a0, a1, fr[t], Dr[t]);
        dmma(a0, a1, Dst[t], fsT[t]);
        dmma(q0, q1, Dst[t], ftQ[t]);
      }
      double *tout = alias + LEAN_TOUT + (b & 1) * TO_FS;
      sts2(tout + toW, q0, q1);
      __syncthreads();  // this field's T results are complete
      const double2 t = *reinterpret_cast<const double2 *>(tout + toR);
      const double o0 = rh0 + jv[0] * (a0 + t.x);
      const double o1 = rh1 + jv[1] * (a1 + t.y);
      if (PAD && !PAIRS) {
        if (vld[0]) re[qo + b * NPTR] = (T)o0;
        if (vld[1]) re[qo + b * NPTR + 1] = (T)o1;
      } else if (!PAIRS || vld[0]) {
        st_pair(re + qo + b * NPTR, o0, o1);
      }
    }
    __syncthreads();  // every alias read done: the stage may be refilled
    if (NSTG == 1 && !OWN_TILES && tid == 0 && n + 1 < nmine) {
      fence_proxy_async();
      issue(n + 1);
    }
  }
}

template <typename T, int SUB, int NW = TC_WARPS>
int launch_tc_lean(int64_t ngroups, double p0, double R, double gam, const T *q, T *rhsq,
                   const T *D, const T *g, const T *jinv, cudaStream_t stream) {
  const size_t smem = sizeof(TcSmemLean<T, SUB, NW>);
  auto kern = volume_tc_lean_kernel<T, SUB, NW>;
  if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) !=
      cudaSuccess)
    return LFB_ERR_CUDA;
  int dev = 0, sms = 0, per_sm = 0;
  if (cudaGetDevice(&dev) != cudaSuccess ||
      cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess ||
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, 32 * NW, smem) !=
          cudaSuccess)
    return LFB_ERR_CUDA;
  if (per_sm < 1) return LFB_ERR_LAUNCH;
  const int64_t slots = (int64_t)sms * per_sm;
  const int64_t grid = ngroups < slots ? ngroups : slots;
  if (grid == 0) return LFB_OK;
  kern<<<(unsigned)grid, 32 * NW, smem, stream>>>(ngroups, p0, R, gam, q, rhsq, D, g, jinv);
  LFB_CHECK_LAUNCH();
  return LFB_OK;
}

template <typename T, int NS, int SUB>
int launch_tc(int64_t ngroups, double p0, double R, double gam, const T *q, T *rhsq,
              const T *D, const T *g, const T *jinv, cudaStream_t stream) {
  // Schedule choice from the A/B on this pool (profiles/r01_ab_lean.txt):
  // the 2-CTA LEAN schedule wins for the zero-padded Nq = 5..7 (+8..10 %);
  // the 1-CTA ring wins for Nq = 8 (+8 %) and the packed Nq = 4, 2. (Two
  // further 2-CTA schedules for Nq=8 — q staged, g from L2; q and g staged,
  // T-out in the dead stage — lost to the ring, profiles/r01_ab_qstage.txt,
  // r01_ab_qg.txt, and were removed.)
  // Zero-padded Nq = 5..7: the LEAN schedule with one warp per real
  // k-plane (PLANE variant; vs 8 warps: Nq=5 0.49 / 0.34, Nq=6 0.62 / 0.51,
  // Nq=7 0.72 / 0.70 of HBM; the 1-CTA ring with SUB warps: 0.31 / 0.51 /
  // 0.67 — profiles/r02_tc_plane.txt)
  constexpr bool PAD_ = !(SUB == 8 || SUB == 4 || SUB == 2);
  if constexpr (PAD_) {
    return launch_tc_lean<T, SUB, SUB>(ngroups, p0, R, gam, q, rhsq, D, g, jinv, stream);
  } else {
    constexpr int NW = TC_WARPS;
    const size_t smem = sizeof(TcSmem<T, NS, SUB, NW>);
    auto kern = volume_tc_kernel<T, NS, SUB, 0, NW>;
#ifdef LFB_EXPERIMENTS
    // barrier-deletion mutants for the race-detector test (tests/test_mutants.py),
    // built only into the test library liblfb_volume_mutants.so
    if constexpr (SUB == 8) {
      if (g_tc_mutant == 1) kern = volume_tc_kernel<T, NS, SUB, 1>;
      if (g_tc_mutant == 2) kern = volume_tc_kernel<T, NS, SUB, 2>;
      if (g_tc_mutant == 3) kern = volume_tc_kernel<T, NS, SUB, 3>;
    }
#endif
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) !=
        cudaSuccess)
      return LFB_ERR_CUDA;
    int dev = 0, sms = 0;
    if (cudaGetDevice(&dev) != cudaSuccess ||
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess)
      return LFB_ERR_CUDA;
    const int64_t grid = ngroups < sms ? ngroups : sms;
    if (grid == 0) return LFB_OK;
    kern<<<(unsigned)grid, 32 * NW, smem, stream>>>(ngroups, p0, R, gam, q, rhsq, D, g, jinv);
    LFB_CHECK_LAUNCH();
    return LFB_OK;
  }
}

template <typename T>
int tail_launch(int nq, int64_t ne, T p0, T R, T gam, const T *q, T *rhsq, const T *D,
                const T *g, const T *jinv, cudaStream_t s);

template <>
int tail_launch<double>(int nq, int64_t ne, double p0, double R, double gam, const double *q,
                        double *rhsq, const double *D, const double *g, const double *jinv,
                        cudaStream_t s) {
  return fused_available(8, nq) ? volume_fused_f64(nq, ne, p0, R, gam, q, rhsq, D, g, jinv, s)
                                : volume_basic_f64(nq, ne, p0, R, gam, q, rhsq, D, g, jinv, s);
}


// Full groups of P^3 elements go through the packed tensor-core kernel; the
// < P^3 leftover elements (Nq = 4: < 8, Nq = 2: < 64) take the fused/basic
// kernel on the same stream.
template <typename T, int NS>
int dispatch_tc(int nq, int64_t ne, T p0, T R, T gam, const T *q, T *rhsq, const T *D,
                const T *g, const T *jinv, cudaStream_t s) {
  const bool pad = !(nq == 8 || nq == 4 || nq == 2);
  const int64_t pe = pad ? 1 : (int64_t)(8 / nq) * (8 / nq) * (8 / nq);
  // PAD: the last element goes to the tail kernel, so no 16-byte superset
  // copy of a g / Jinv slab can run past the end of the arrays
  const int64_t groups = pad ? (ne > 0 ? ne - 1 : 0) : ne / pe;
  const int64_t done = groups * pe, npt = (int64_t)nq * nq * nq;
  int rc = LFB_OK;
  if (groups > 0) {
    if (nq == 8) rc = launch_tc<T, NS, 8>(groups, p0, R, gam, q, rhsq, D, g, jinv, s);
    else if (nq == 7) rc = launch_tc<T, NS, 7>(groups, p0, R, gam, q, rhsq, D, g, jinv, s);
    else if (nq == 6) rc = launch_tc<T, NS, 6>(groups, p0, R, gam, q, rhsq, D, g, jinv, s);
    else if (nq == 5) rc = launch_tc<T, NS, 5>(groups, p0, R, gam, q, rhsq, D, g, jinv, s);
    else if (nq == 4) rc = launch_tc<T, NS, 4>(groups, p0, R, gam, q, rhsq, D, g, jinv, s);
    else rc = launch_tc<T, NS, 2>(groups, p0, R, gam, q, rhsq, D, g, jinv, s);
  }
  if (rc != LFB_OK || done == ne) return rc;
  return tail_launch<T>(nq, ne - done, p0, R, gam, q + done * 8 * npt, rhsq + done * 8 * npt,
                        D, g + done * 9 * npt, jinv + done * npt, s);
}

}  // namespace

#ifdef LFB_EXPERIMENTS
extern "C" __attribute__((visibility("default"))) void lfb_test_set_tc_mutant(int m) {
  g_tc_mutant = m;
}
#endif

bool tc16_available(int nq);

// fp64: Nq 2, 4..8 (virtual Nq=8 cube); fp32 also 9..16 (volume_tc16.cu)
bool tc_available(int dtype_bytes, int nq) {
  if (dtype_bytes == 4 && tc16_available(nq)) return true;
  return (dtype_bytes == 8 || dtype_bytes == 4) && nq >= 2 && nq <= 8 && nq != 3;
}

// bulk copies need 16-byte aligned q and g element slabs; the paired
// accesses need rhsq / Jinv aligned to two elements
bool tc_aligned(int dtype_bytes, const void *q, const void *rhsq, const void *g,
                const void *jinv) {
  const uintptr_t pair = 2 * (uintptr_t)dtype_bytes - 1;
  return (((reinterpret_cast<uintptr_t>(q) | reinterpret_cast<uintptr_t>(g)) & 15) == 0) &&
         (((reinterpret_cast<uintptr_t>(rhsq) | reinterpret_cast<uintptr_t>(jinv)) & pair) == 0);
}

int volume_tc_f64(int nq, int64_t ne, double p0, double R, double gam, const double *q,
                  double *rhsq, const double *D, const double *g, const double *jinv,
                  cudaStream_t s) {
  if (!tc_available(8, nq)) return LFB_ERR_BAD_VARIANT;
  if (!tc_aligned(8, q, rhsq, g, jinv)) return LFB_ERR_MISALIGNED;
  return dispatch_tc<double, 2>(nq, ne, p0, R, gam, q, rhsq, D, g, jinv, s);
}

int volume_tc_f32(int nq, int64_t ne, float p0, float R, float gam, const float *q,
                  float *rhsq, const float *D, const float *g, const float *jinv,
                  cudaStream_t s) {
  if (!tc_available(4, nq)) return LFB_ERR_BAD_VARIANT;
  if (tc16_available(nq)) {  // 16x16-plane TF32 kernel: paired accesses need 8-byte
    // alignment for even Nq (element alignment is all validate() guarantees)
    const uintptr_t a = reinterpret_cast<uintptr_t>(q) | reinterpret_cast<uintptr_t>(rhsq) |
                        reinterpret_cast<uintptr_t>(g) | reinterpret_cast<uintptr_t>(jinv);
    if ((nq % 2) == 0 && (a & 7)) return LFB_ERR_MISALIGNED;
    return volume_tc16_f32(nq, ne, p0, R, gam, q, rhsq, D, g, jinv, s);
  }
  if (!tc_aligned(4, q, rhsq, g, jinv)) return LFB_ERR_MISALIGNED;
  // fp32 storage: the TF32 split-product kernel (volume_tc32.cu)
  return volume_tc32_f32(nq, ne, p0, R, gam, q, rhsq, D, g, jinv, s);
}

}  // namespace lfb
