// Bit-exact restatement of glibc 2.39's x86-64 FMA variants of log() and exp()
// (__log_fma / __exp_fma, the ARM optimized-routines algorithms in
// sysdeps/ieee754/dbl-64/e_log.c and e_exp.c built with -mfma -mavx2).
//
// Why: the reference interpolates in log-log space with CPython math.log /
// math.exp (/root/reference/pkg/src/llmconf/perfdb.py:505, 535-536), i.e. with
// glibc.  CUDA's own log/exp differ from glibc in the last bit for a fraction
// of inputs, which is enough to reorder rows and flip Pareto ties
// (SURVEY.md §7 "Hard parts").  The operation order below (which products are
// fused) was read from the disassembly of this image's libm.so.6 and is
// verified bit-for-bit against the host libm by tests/test_libm_parity.py
// (host compile of this header) and tests/test_gpu_parity.py (device).
//
// Compile with contraction OFF (nvcc --fmad=false, gcc -ffp-contract=off):
// every fma() below is explicit and every other product must round.
#pragma once
#include <stdint.h>
#include <math.h>
#include <string.h>
#include "glibc_libm_tables.h"

#if defined(__CUDACC__)
#define LC_HD __host__ __device__ __forceinline__
#else
#define LC_HD static inline
#endif

namespace glibc {

LC_HD uint64_t as_u64(double x) {
#if defined(__CUDA_ARCH__)
  return (uint64_t)__double_as_longlong(x);
#else
  uint64_t u; memcpy(&u, &x, 8); return u;
#endif
}

LC_HD double as_f64(uint64_t u) {
#if defined(__CUDA_ARCH__)
  return __longlong_as_double((long long)u);
#else
  double x; memcpy(&x, &u, 8); return x;
#endif
}

// Natural log for the inputs the search produces: integers >= 2 (grid
// coordinates strictly between two axis values, which are >= 1).  Any
// positive normal x outside [0x1.ep-1, 0x1.1090p0) takes this same main path;
// x == 1 returns +0 like glibc.  The near-1 polynomial path is not restated
// (unreachable for integer coordinates) and returns NaN so misuse is loud.
// `tab` = 256 doubles {invc_i, logc_i} (GLIBC_LOG_TAB_INIT).
LC_HD double log_fma(double x, const double* tab) {
  const uint64_t ix = as_u64(x);
  if (ix == 0x3ff0000000000000ull) return 0.0;
  if (ix - 0x3fee000000000000ull < 0x3090000000000ull) return NAN;  // near-1 path
  const uint32_t top = (uint32_t)(ix >> 48);
  if (top - 0x0010u >= 0x7ff0u - 0x0010u) return NAN;  // <=0, subnormal, inf, nan
  const uint64_t tmp = ix - 0x3fe6000000000000ull;
  const int i = (int)((tmp >> 45) & 127);
  const int k = (int)((int64_t)tmp >> 52);
  const uint64_t iz = ix - (tmp & 0xfff0000000000000ull);
  const double invc = tab[2 * i];
  const double logc = tab[2 * i + 1];
  const double z = as_f64(iz);
  const double kd = (double)k;
  const double w = fma(kd, GLIBC_LOG_LN2HI, logc);
  const double r = fma(z, invc, -1.0);
  const double p12 = fma(r, GLIBC_LOG_A2, GLIBC_LOG_A1);
  const double hi = w + r;
  const double r2 = r * r;
  double lo = (w - hi) + r;
  lo = fma(kd, GLIBC_LOG_LN2LO, lo);
  const double r3 = r * r2;
  const double p34 = fma(r, GLIBC_LOG_A4, GLIBC_LOG_A3);
  const double lo2 = fma(r2, GLIBC_LOG_A0, lo);
  const double p = fma(p34, r2, p12);
  const double y = fma(r3, p, lo2);
  return y + hi;
}

// exp(x) for all finite and infinite x.  `tab` = 256 uint64 (GLIBC_EXP_TAB_INIT).
LC_HD double exp_fma(double x, const uint64_t* tab) {
  const uint64_t ix = as_u64(x);
  uint32_t abstop = (uint32_t)(ix >> 52) & 0x7ff;
  if (abstop - 0x3c9u >= 0x3fu) {
    if ((int32_t)(abstop - 0x3c9u) < 0) return 1.0 + x;  // |x| < 2^-54
    if (abstop >= 0x409u) {                                // |x| >= 1024
      if (ix == 0xfff0000000000000ull) return 0.0;
      if (abstop >= 0x7ffu) return 1.0 + x;
      return (ix >> 63) ? 0.0 : INFINITY;
    }
    abstop = 0;  // large |x|: scale may overflow, handled below
  }
  double kd = fma(x, GLIBC_EXP_INVLN2N, GLIBC_EXP_SHIFT);
  const uint64_t ki = as_u64(kd);
  kd = kd - GLIBC_EXP_SHIFT;
  double r = fma(kd, GLIBC_EXP_NEGLN2HIN, x);
  r = fma(kd, GLIBC_EXP_NEGLN2LON, r);
  const int idx = 2 * (int)(ki & 127);
  const uint64_t top = ki << 45;
  const double p23 = fma(r, GLIBC_EXP_C3, GLIBC_EXP_C2);
  const double tail = as_f64(tab[idx]);
  const double tr = r + tail;
  uint64_t sbits = tab[idx + 1] + top;
  const double r2 = r * r;
  const double p45 = fma(r, GLIBC_EXP_C5, GLIBC_EXP_C4);
  const double a = fma(p23, r2, tr);
  const double r4 = r2 * r2;
  const double tmp = fma(r4, p45, a);
  if (abstop == 0) {
    if ((ki & 0x80000000ull) == 0) {
      sbits -= 1009ull << 52;
      const double scale = as_f64(sbits);
      return 0x1p1009 * fma(scale, tmp, scale);
    }
    sbits += 1022ull << 52;
    const double scale = as_f64(sbits);
    const double st = scale * tmp;
    double y = scale + st;
    if (y < 1.0) {
      double lo = (scale - y) + st;
      const double hi = 1.0 + y;
      lo = ((1.0 - hi) + y) + lo;
      y = (lo + hi) - 1.0;
      if (y == 0.0) y = 0.0;
    }
    return 0x1p-1022 * y;
  }
  const double scale = as_f64(sbits);
  return fma(scale, tmp, scale);
}

}  // namespace glibc
