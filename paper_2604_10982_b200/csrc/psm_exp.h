// psm_exp.h — the one libm function on the render hot path, restated so that
// the CUDA kernels and the CPU oracle produce the same bits.
//
// The reference evaluates alpha = o * std::exp(-0.5 * (u*u + v*v)) with glibc
// `exp` (proj/src/raster.cpp:390, :175). glibc picks an FMA or non-FMA variant
// at load time (ifunc), so its last bit already depends on the host CPU, and
// CUDA's device `exp` is a third implementation. Every decision the renderer
// makes (alpha >= alpha_min, T < t_min, Top-K order by weight) is taken on
// this value, so bit-exact parity needs one exp evaluated identically on both
// sides. This one uses only IEEE-754 double add/mul and explicit fused
// multiply-adds (fma is correctly rounded on x86-64 and on sm_100a), in a fixed
// order, so host and device results are identical by construction.
//
// Algorithm: exp(x) = 2^k * exp(r), k = rint(x / ln2), r = x - k*ln2 with a
// two-term (Cody–Waite) ln2; exp(r) by the degree-13 Taylor polynomial in
// Horner/FMA form (|r| <= 0.347, truncation < 5e-18 relative). Measured error
// against glibc: tests/test_oracle_kat.py::test_psm_exp_vs_glibc (<= 1 ulp).
//
// Compile with contraction disabled (host: -ffp-contract=off; device:
// --fmad=false) so the non-fused products below are not fused behind our back.
#ifndef PSM_EXP_H
#define PSM_EXP_H

#include <stdint.h>

#if defined(__CUDACC__)
#define PSM_HD __host__ __device__ __forceinline__
#else
#define PSM_HD static inline
#include <math.h>
#include <string.h>
#endif

PSM_HD double psm_bits_to_double(uint64_t b) {
#if defined(__CUDA_ARCH__)
  return __longlong_as_double(static_cast<long long>(b));
#else
  double d;
  memcpy(&d, &b, sizeof d);
  return d;
#endif
}

PSM_HD double psm_fma(double a, double b, double c) {
#if defined(__CUDA_ARCH__)
  return __fma_rn(a, b, c);
#else
  return fma(a, b, c);
#endif
}

PSM_HD double psm_exp(double x) {
  if (x != x) return x + x;                       // NaN propagates
  if (x > 709.782712893384) return 1.0 / 0.0;     // overflow -> +inf
  if (x < -745.1332191019412) return 0.0;         // below half the smallest subnormal
  const double kLog2e = 1.4426950408889634;
  const double kShift = 6755399441055744.0;       // 1.5 * 2^52: add/sub rounds to integer (ties-even)
  const double kLn2Hi = 0.6931471803691238;       // 0x3fe62e42fee00000, k*kLn2Hi exact for |k| < 2^11
  const double kLn2Lo = 1.9082149292705877e-10;
  double t = x * kLog2e;
  double kd = t + kShift;
  kd = kd - kShift;
  const int k = static_cast<int>(kd);
  double r = psm_fma(-kd, kLn2Hi, x);
  r = psm_fma(-kd, kLn2Lo, r);
  double p = 1.6059043836821613e-10;              // 1/13!
  p = psm_fma(p, r, 2.08767569878681e-09);        // 1/12!
  p = psm_fma(p, r, 2.505210838544172e-08);       // 1/11!
  p = psm_fma(p, r, 2.755731922398589e-07);       // 1/10!
  p = psm_fma(p, r, 2.7557319223985893e-06);      // 1/9!
  p = psm_fma(p, r, 2.48015873015873e-05);        // 1/8!
  p = psm_fma(p, r, 0.0001984126984126984);       // 1/7!
  p = psm_fma(p, r, 0.001388888888888889);        // 1/6!
  p = psm_fma(p, r, 0.008333333333333333);        // 1/5!
  p = psm_fma(p, r, 0.041666666666666664);        // 1/4!
  p = psm_fma(p, r, 0.16666666666666666);         // 1/3!
  p = psm_fma(p, r, 0.5);                         // 1/2!
  p = psm_fma(p, r, 1.0);                         // 1/1!
  p = psm_fma(p, r, 1.0);                         // 1/0!
  if (k > 1023) {  // only reachable for x within ~0.35 of the overflow bound
    return (p * 2.0) * psm_bits_to_double(static_cast<uint64_t>(k - 1 + 1023) << 52);
  }
  if (k >= -1021) {
    return p * psm_bits_to_double(static_cast<uint64_t>(k + 1023) << 52);
  }
  // subnormal result: scale in two exact-then-rounded steps
  return (p * psm_bits_to_double(static_cast<uint64_t>(k + 1023 + 64) << 52)) *
         psm_bits_to_double(static_cast<uint64_t>(1023 - 64) << 52);
}

#endif  // PSM_EXP_H
