// psm_exp.h — the one libm function on the render hot path, restated so that
// the CUDA kernels, the CPU oracle and the reference's own glibc produce the
// same bits.
//
// The reference evaluates alpha = o * std::exp(-0.5 * (u*u + v*v)) with glibc
// `exp` (proj/src/raster.cpp:390, :175). Every decision the renderer makes
// (alpha >= alpha_min, T < t_min, Top-K order by weight) is taken on that value,
// so bit-exact parity needs one exp evaluated identically everywhere.
//
// glibc >= 2.28 implements exp with the optimized-routines algorithm
// (sysdeps/ieee754/dbl-64/e_exp.c + e_exp_data.c; third-party dependency of the
// reference, not vendored in /root/reference): exp(x) = 2^(k/128) * exp(r),
// k = rint(x * 128/ln2), r = x - k ln2/128 (two-term ln2), 2^(k/128) from a
// 128-entry table {tail, scale bits}, exp(r) - 1 by a degree-5 polynomial,
// result scale + scale * tmp. On x86-64 hosts with FMA+AVX2 (this image and the
// GPU boxes) the ifunc selects the -mfma build (__exp_fma); the operation
// order below is that build's, read off the image's libm.so.6 disassembly
// (fused: kd, both r steps, the three polynomial combinations, the final
// scale + scale*tmp; k < 0 special case unfused as compiled). The constants are
// the published e_exp_data.c values; the table is regenerated from its
// definition by gen_exp_table.py. tests/test_oracle_kat.py::test_psm_exp_is_glibc_exp
// checks bit equality with the host glibc exp on millions of arguments.
//
// Only IEEE-754 add/mul and explicit fused multiply-adds are used (fma is
// correctly rounded on x86-64 and on sm_100a). Compile with contraction off
// (host: -ffp-contract=off; device: --fmad=false) so nothing else is fused.
#ifndef PSM_EXP_H
#define PSM_EXP_H

#include <stdint.h>

#include "psm_exp_table.h"

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

PSM_HD uint64_t psm_double_to_bits(double d) {
#if defined(__CUDA_ARCH__)
  return static_cast<uint64_t>(__double_as_longlong(d));
#else
  uint64_t b;
  memcpy(&b, &d, sizeof b);
  return b;
#endif
}

PSM_HD double psm_fma(double a, double b, double c) {
#if defined(__CUDA_ARCH__)
  return __fma_rn(a, b, c);
#else
  return fma(a, b, c);
#endif
}

// {tail_i, bits(2^(i/128)) - (i << 45)}, i = 0..127 (2 KB; L1-resident on the device)
#if defined(__CUDACC__)
static __device__ const uint64_t psm_exp_tab_dev[256] = PSM_EXP_TABLE_INIT;
#endif
static const uint64_t psm_exp_tab_host[256] = PSM_EXP_TABLE_INIT;

PSM_HD void psm_exp_tab(const uint64_t* tab, uint64_t idx, double* tail, uint64_t* sbits_hi) {
#if defined(__CUDA_ARCH__)
  const ulonglong2 e = reinterpret_cast<const ulonglong2*>(tab)[idx >> 1];
  *tail = psm_bits_to_double(e.x);
  *sbits_hi = e.y;
#else
  *tail = psm_bits_to_double(tab[idx]);
  *sbits_hi = tab[idx + 1];
#endif
}

// e_exp.c specialcase(): |x| in [512, 1024) where the scale leaves the normal range.
PSM_HD double psm_exp_special(double tmp, uint64_t sbits, uint64_t ki) {
  if ((ki & 0x80000000u) == 0) {  // k > 0: scale down by 2^1009, result may overflow
    sbits -= 1009ull << 52;
    const double scale = psm_bits_to_double(sbits);
    return 0x1p1009 * psm_fma(scale, tmp, scale);
  }
  // k < 0: the result may be subnormal; round it once (unfused, as compiled)
  sbits += 1022ull << 52;
  const double scale = psm_bits_to_double(sbits);
  const double st = scale * tmp;
  double y = scale + st;
  if (y < 1.0) {
    double lo = scale - y + st;
    const double hi = 1.0 + y;
    lo = 1.0 - hi + y + lo;
    y = (lo + hi) - 1.0;
    if (y == 0.0) y = 0.0;
  }
  return 0x1p-1022 * y;
}

// Device: the polynomial / reduction constants live in the constant bank, so the
// fp64 instructions take them as c[] operands instead of re-materialising each
// 64-bit immediate into registers on every call.
#if defined(__CUDACC__)
static __constant__ double psm_exp_kc[8] = {0x1.71547652b82fep7, 0x1.8p52, -0x1.62e42fefa0000p-8,
                                            -0x1.cf79abc9e3b3ap-47, 0x1.ffffffffffdbdp-2, 0x1.555555555543cp-3,
                                            0x1.55555cf172b91p-5, 0x1.1111167a4d017p-7};
#endif
#if defined(__CUDA_ARCH__)
#define PSM_EXPK(i, lit) psm_exp_kc[i]
#else
#define PSM_EXPK(i, lit) (lit)
#endif

// `tab` is the 256-word table (psm_exp_tab_dev, a shared-memory copy of it, or the host array).
PSM_HD double psm_exp_t(double x, const uint64_t* tab) {
  const double kInvLn2N = PSM_EXPK(0, 0x1.71547652b82fep7);  // 128 / ln2
  const double kShift = 0x1.8p52;
  const double kNegLn2HiN = PSM_EXPK(2, -0x1.62e42fefa0000p-8);
  const double kNegLn2LoN = PSM_EXPK(3, -0x1.cf79abc9e3b3ap-47);
  const double C2 = PSM_EXPK(4, 0x1.ffffffffffdbdp-2), C3 = PSM_EXPK(5, 0x1.555555555543cp-3);
  const double C4 = PSM_EXPK(6, 0x1.55555cf172b91p-5), C5 = PSM_EXPK(7, 0x1.1111167a4d017p-7);
  const uint64_t ix = psm_double_to_bits(x);
  uint32_t abstop = static_cast<uint32_t>(ix >> 52) & 0x7ffu;
  if (abstop - 0x3c9u >= 0x3fu) {                      // |x| < 2^-54, |x| >= 512, inf or nan
    if (static_cast<int32_t>(abstop - 0x3c9u) < 0) return 1.0 + x;  // tiny: rounds to 1
    if (abstop >= 0x409u) {                            // |x| >= 1024
      if (ix == 0xfff0000000000000ull) return 0.0;     // -inf
      if (abstop >= 0x7ffu) return 1.0 + x;            // +inf or nan
      return (ix >> 63) ? 0.0 : psm_bits_to_double(0x7ff0000000000000ull);  // underflow to +0 / overflow to +inf
    }
    abstop = 0;                                        // 512 <= |x| < 1024: special-cased below
  }
  double kd = psm_fma(x, kInvLn2N, kShift);
  const uint64_t ki = psm_double_to_bits(kd);
  kd = kd - kShift;
  double r = psm_fma(kd, kNegLn2HiN, x);
  r = psm_fma(kd, kNegLn2LoN, r);
  const uint64_t idx = 2 * (ki % 128);
  const uint64_t top = ki << 45;
  double tail;
  uint64_t sbits;
  psm_exp_tab(tab, idx, &tail, &sbits);
  sbits += top;
  const double r2 = r * r;
  const double a = psm_fma(r, C3, C2);
  const double t1 = psm_fma(a, r2, r + tail);
  const double b = psm_fma(r, C5, C4);
  const double r4 = r2 * r2;
  const double tmp = psm_fma(r4, b, t1);
  if (abstop == 0) return psm_exp_special(tmp, sbits, ki);
  const double scale = psm_bits_to_double(sbits);
  return psm_fma(scale, tmp, scale);
}

// The common case of psm_exp_t (2^-54 <= |x| < 512) without its range branches, so
// that two independent evaluations can be interleaved; psm_exp_t(x) == psm_exp_main(x)
// whenever psm_exp_main_ok(x).
PSM_HD bool psm_exp_main_ok(double x) {
  const uint32_t abstop = static_cast<uint32_t>(psm_double_to_bits(x) >> 52) & 0x7ffu;
  return abstop - 0x3c9u < 0x3fu;
}
PSM_HD double psm_exp_main(double x, const uint64_t* tab) {
  const double kInvLn2N = PSM_EXPK(0, 0x1.71547652b82fep7);
  const double kShift = 0x1.8p52;
  const double kNegLn2HiN = PSM_EXPK(2, -0x1.62e42fefa0000p-8);
  const double kNegLn2LoN = PSM_EXPK(3, -0x1.cf79abc9e3b3ap-47);
  const double C2 = PSM_EXPK(4, 0x1.ffffffffffdbdp-2), C3 = PSM_EXPK(5, 0x1.555555555543cp-3);
  const double C4 = PSM_EXPK(6, 0x1.55555cf172b91p-5), C5 = PSM_EXPK(7, 0x1.1111167a4d017p-7);
  double kd = psm_fma(x, kInvLn2N, kShift);
  const uint64_t ki = psm_double_to_bits(kd);
  kd = kd - kShift;
  double r = psm_fma(kd, kNegLn2HiN, x);
  r = psm_fma(kd, kNegLn2LoN, r);
  double tail;
  uint64_t sbits;
  psm_exp_tab(tab, 2 * (ki % 128), &tail, &sbits);
  sbits += ki << 45;
  const double r2 = r * r;
  const double t1 = psm_fma(psm_fma(r, C3, C2), r2, r + tail);
  const double tmp = psm_fma(r2 * r2, psm_fma(r, C5, C4), t1);
  const double scale = psm_bits_to_double(sbits);
  return psm_fma(scale, tmp, scale);
}

PSM_HD double psm_exp(double x) {
#if defined(__CUDA_ARCH__)
  return psm_exp_t(x, psm_exp_tab_dev);
#else
  return psm_exp_t(x, psm_exp_tab_host);
#endif
}

#endif  // PSM_EXP_H
