// Reduced-instruction fp64 math for the volume kernels.
//
// The equation of state p = p0 (R Theta / p0)^gamma (
// lf/bench/reference.py:21) costs ~100 FP64-pipe instructions per point with
// CUDA's correctly-rounded pow() — about a third of the kernel's fp64 work
// at Nq = 8. pos_pow() evaluates x^y = exp(y ln x) with
//   ln: x = 2^e m, m in [1/sqrt2, sqrt2), ln m = 2 atanh(u), u = (m-1)/(m+1),
//       odd series in u to u^19 (|u| <= 0.1716: truncation < 3e-17);
//   exp: n = rint(t / ln2), r = t - n ln2 (two-part ln2), Taylor to r^13
//       (|r| <= 0.347: truncation < 5e-18), scaled by 2^n via the exponent;
// ~41 FP64 ops, relative error <= ~4e-16 (1 + |y ln x|) — far inside the
// 1e-12 parity bound (tests/test_volume_gpu.py; tools/check_fastmath.cu
// measures it against long-double powl on the host).
// Inputs outside (normal positive x, |y ln x| < 700) take CUDA's pow().
#pragma once

#include <math.h>
#include <stdint.h>
#include <string.h>

#ifndef LFB_HD
#define LFB_HD __host__ __device__ __forceinline__
#endif

namespace lfb {

LFB_HD int64_t dbits(double x) {
#ifdef __CUDA_ARCH__
  return __double_as_longlong(x);
#else
  int64_t b;
  memcpy(&b, &x, 8);
  return b;
#endif
}

LFB_HD double bitsd(int64_t b) {
#ifdef __CUDA_ARCH__
  return __longlong_as_double(b);
#else
  double x;
  memcpy(&x, &b, 8);
  return x;
#endif
}

// 1/d to ~1 ulp: hardware seed (MUFU.RCP64H) + two Newton steps.
LFB_HD double fast_rcp(double d) {
#ifdef __CUDA_ARCH__
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(d));
#else
  double r = (double)(1.0f / (float)d);
#endif
  double e = fma(-d, r, 1.0);
  r = fma(r, e, r);
  e = fma(-d, r, 1.0);
  r = fma(r, e, r);
  return r;
}

LFB_HD double pos_pow(double x, double y) {
  const int64_t bx = dbits(x);
  const int64_t ex_raw = (bx >> 52) & 0x7ff;
  if (x <= 0.0 || ex_raw == 0 || ex_raw == 0x7ff) return pow(x, y);
  // x = 2^e * m with m in [1/sqrt2, sqrt2)
  int64_t e = ex_raw - 1023;
  int64_t mb = (bx & 0x000fffffffffffffLL) | 0x3ff0000000000000LL;  // m in [1, 2)
  if (mb > 0x3ff6a09e667f3bcdLL) {                                  // m > sqrt2
    mb -= 0x0010000000000000LL;                                     // m /= 2
    e += 1;
  }
  const double m = bitsd(mb);
  const double f = m - 1.0;
  const double u = f * fast_rcp(2.0 + f);
  const double v = u * u;
  double s = 1.0 / 19.0;
  s = fma(s, v, 1.0 / 17.0);
  s = fma(s, v, 1.0 / 15.0);
  s = fma(s, v, 1.0 / 13.0);
  s = fma(s, v, 1.0 / 11.0);
  s = fma(s, v, 1.0 / 9.0);
  s = fma(s, v, 1.0 / 7.0);
  s = fma(s, v, 1.0 / 5.0);
  s = fma(s, v, 1.0 / 3.0);
  // ln m = 2u (1 + v s) = 2u + 2u v s
  const double twou = u + u;
  const double lnm_lo = twou * v * s;  // small correction term
  const double LN2_HI = 6.93147180369123816490e-01;
  const double LN2_LO = 1.90821492927058770002e-10;
  const double fe = (double)e;
  // t = y * (e ln2 + ln m), kept as hi + lo for the exp reduction
  const double lnx_hi = fma(fe, LN2_HI, twou);
  const double lnx_lo = fma(fe, LN2_LO, lnm_lo);
  const double lnx = lnx_hi + lnx_lo;
  const double t = y * lnx;
  if (!(fabs(t) < 700.0)) return pow(x, y);
  const double t_lo = fma(y, lnx, -t) + y * ((lnx_hi - lnx) + lnx_lo);
  // exp(t + t_lo)
  const double INV_LN2 = 1.44269504088896338700e+00;
  const double SHIFT = 6755399441055744.0;  // 1.5 * 2^52
  const double kk = fma(t, INV_LN2, SHIFT);
  const double n = kk - SHIFT;
  double r = fma(-n, LN2_HI, t);
  r = fma(-n, LN2_LO, r) + t_lo;
  double p = 1.0 / 6227020800.0;  // 1/13!
  p = fma(p, r, 1.0 / 479001600.0);
  p = fma(p, r, 1.0 / 39916800.0);
  p = fma(p, r, 1.0 / 3628800.0);
  p = fma(p, r, 1.0 / 362880.0);
  p = fma(p, r, 1.0 / 40320.0);
  p = fma(p, r, 1.0 / 5040.0);
  p = fma(p, r, 1.0 / 720.0);
  p = fma(p, r, 1.0 / 120.0);
  p = fma(p, r, 1.0 / 24.0);
  p = fma(p, r, 1.0 / 6.0);
  p = fma(p, r, 0.5);
  p = fma(p, r, 1.0);
  p = fma(p, r, 1.0);
  const int64_t ni = (int64_t)n;
  return p * bitsd((ni + 1023) << 52);
}

}  // namespace lfb
