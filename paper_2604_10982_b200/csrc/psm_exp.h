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

// exp(r) coefficients 1/n!, n = 13 .. 0 (Horner order). On the device they live in
// the constant bank so each DFMA takes its coefficient as a c[] operand instead of
// re-materialising a 64-bit immediate; the values (hence the bits) are identical.
#define PSM_EXP_COEFFS                                                                     \
  {1.6059043836821613e-10, 2.08767569878681e-09, 2.505210838544172e-08,                    \
   2.755731922398589e-07, 2.7557319223985893e-06, 2.48015873015873e-05,                    \
   0.0001984126984126984, 0.001388888888888889, 0.008333333333333333,                      \
   0.041666666666666664, 0.16666666666666666, 0.5, 1.0, 1.0}
#if defined(__CUDACC__)
static __constant__ double psm_exp_c_dev[14] = PSM_EXP_COEFFS;
#endif
static const double psm_exp_c_host[14] = PSM_EXP_COEFFS;

// exp(r) for the reduced argument r, times 2^k, k = rint(x / ln2). Shared tail of
// psm_exp and psm_exp_nonpos.
PSM_HD double psm_exp_core(double x, double t) {
  const double kShift = 6755399441055744.0;       // 1.5 * 2^52: add/sub rounds to integer (ties-even)
  const double kLn2Hi = 0.6931471803691238;       // 0x3fe62e42fee00000, k*kLn2Hi exact for |k| < 2^11
  const double kLn2Lo = 1.9082149292705877e-10;
  const double ks = t + kShift;
  const double kd = ks - kShift;
  // k from the low mantissa bits of ks (two's complement of k): no float->int conversion
#if defined(__CUDA_ARCH__)
  const int k = __double2loint(ks);
  const double* c = psm_exp_c_dev;
#else
  uint64_t ksb;
  memcpy(&ksb, &ks, sizeof ksb);
  const int k = (int)(uint32_t)(ksb & 0xffffffffu);
  const double* c = psm_exp_c_host;
#endif
  double r = psm_fma(-kd, kLn2Hi, x);
  r = psm_fma(-kd, kLn2Lo, r);
  double p = c[0];
#if defined(__CUDA_ARCH__)
#pragma unroll
#endif
  for (int i = 1; i < 14; ++i) p = psm_fma(p, r, c[i]);
  if (k > 1023) {  // only reachable for x within ~0.35 of the overflow bound
    return (p * 2.0) * psm_bits_to_double((uint64_t)(k - 1 + 1023) << 52);
  }
  if (k >= -1021) {
    return p * psm_bits_to_double((uint64_t)(k + 1023) << 52);
  }
  // subnormal result: scale in two exact-then-rounded steps
  return (p * psm_bits_to_double((uint64_t)(k + 1023 + 64) << 52)) *
         psm_bits_to_double((uint64_t)(1023 - 64) << 52);
}

PSM_HD double psm_exp(double x) {
  if (x != x) return x + x;                       // NaN propagates
  if (x > 709.782712893384) return 1.0 / 0.0;     // overflow -> +inf
  if (x < -745.1332191019412) return 0.0;         // below half the smallest subnormal
  return psm_exp_core(x, x * 1.4426950408889634);
}

// psm_exp restricted to x <= 0 or NaN (the alpha argument -0.5 (u^2 + v^2)):
// same bits as psm_exp there, without the overflow branch.
PSM_HD double psm_exp_nonpos(double x) {
  if (!(x >= -745.1332191019412)) return x != x ? x + x : 0.0;
  return psm_exp_core(x, x * 1.4426950408889634);
}

#endif  // PSM_EXP_H
