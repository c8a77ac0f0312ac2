// Natural log in float64 for the float64-accumulator scatter-add (fusion.py:177's
// np.log of a clipped probability product), table-driven: ~20 instructions against
// the ~40 of the libdevice log, within 1 ulp (tests/test_gpu_fuse_kernels.py checks it
// against NumPy over random and edge-case arguments).
//
// x = 2^k * z with z in [0.6875, 1.375): the bits of x minus those of 0.6875 give k
// (the exponent field) and an 8-bit interval index i (tools/gen_log_table.py).  With
// invc ~ 1/c for the interval's centre c, r = z * invc - 1 is formed by one fma, so it
// is the correctly rounded value of the exact r (|r| < 0.0040), and
//   log(x) = k ln2 + logc + log1p(r),  logc = -log(invc),
// log1p(r) = r + r^2 * Q(r) with the Taylor polynomial to r^7 / 7 (truncation below
// 2^-59 relative; 128 intervals needed r^9 / 9).  The two intervals around z = 1 use c = 1 exactly (invc = 1, logc = 0),
// so for x near 1 the result is r + r^2 Q(r) with r = z - 1 exact: no cancellation.
// Zero, negative, subnormal, infinite and NaN arguments take the libdevice log.
#pragma once
#include "log_f64_table.h"

namespace tfb_log {

#ifndef TFB_LOG_SLOW_NOINLINE
#define TFB_LOG_SLOW_NOINLINE 1
#endif
// the rare arguments' libdevice log, kept out of line so the call sites stay small
// (the scatter-add inlines several log_f64 per piece; inlined, the libdevice body made
// instruction fetch its top stall)
#if TFB_LOG_SLOW_NOINLINE
__device__ __noinline__ double log_slow(double x) { return log(x); }
#else
__device__ __forceinline__ double log_slow(double x) { return log(x); }
#endif

__device__ __forceinline__ double log_f64(double x, const double2 *__restrict__ tab) {
  const unsigned long long ix = (unsigned long long)__double_as_longlong(x);
  // positive normal and finite: 0x0010... <= ix < 0x7ff0...
  if (ix - 0x0010000000000000ULL >= 0x7fe0000000000000ULL) return log_slow(x);
  const unsigned long long tmp = ix - 0x3FE6000000000000ULL;
  const int i = (int)((tmp >> (52 - kLogBits)) & ((1u << kLogBits) - 1u));
  const long long k = (long long)tmp >> 52;
  const double z = __longlong_as_double((long long)(ix - (tmp & 0xFFF0000000000000ULL)));
  const double2 t = tab[i];  // {invc, logc}
  const double r = __fma_rn(z, t.x, -1.0);
  const double kd = (double)k;
  // w = k ln2_hi + logc (k * ln2_hi exact); hi + lo = w + r exactly (|w| >= |r| whenever w != 0)
  const double w = __fma_rn(kd, kLn2Hi, t.y);
  const double hi = __dadd_rn(w, r);
  const double lo = __fma_rn(kd, kLn2Lo, __dadd_rn(__dsub_rn(w, hi), r));
  double q = 1.0 / 7.0;
  q = __fma_rn(q, r, -1.0 / 6.0);
  q = __fma_rn(q, r, 1.0 / 5.0);
  q = __fma_rn(q, r, -1.0 / 4.0);
  q = __fma_rn(q, r, 1.0 / 3.0);
  q = __fma_rn(q, r, -0.5);
  const double r2 = __dmul_rn(r, r);
  return __dadd_rn(hi, __fma_rn(r2, q, lo));
}

}  // namespace tfb_log
