// Exact (correctly rounded) division by constants on the hot loops, cheaper than
// the general double-division sequence.  Host-compilable: tests/native/div_check.cpp
// compares it with IEEE division.  Compile with contraction off (every fma explicit).
#pragma once
#include <math.h>
#include "glibc_libm.cuh"  // LC_HD

namespace lc {

// x / 1000.0 correctly rounded (the reference's `lat * repeat / 1000.0`,
// estimator.py:93), without the general double-division sequence: q0 = RN(x * y')
// with y' = RN(1/1000), two Newton corrections through the exact fma remainder.
// After the first, q1 is within one ulp of x/1000; Markstein's theorem (y' the
// correctly rounded reciprocal, q faithful) then makes RN(q1 + r1 y') the correctly
// rounded quotient.  Outside [2^-1000, 2^1000] (zero, tiny, huge, inf, NaN) the plain
// division runs.  Checked against IEEE division on 4e8 random operands offline
// and ~5e7 in
// tests/test_libm_parity.py::test_div1000_is_correctly_rounded.
LC_HD double div1000(double x) {
  constexpr double kInv = 1.0 / 1000.0;
  const double ax = fabs(x);
  if (!(ax >= 0x1p-1000 && ax <= 0x1p1000)) return x / 1000.0;
  const double q0 = x * kInv;
  const double r0 = fma(-q0, 1000.0, x);
  const double q1 = fma(r0, kInv, q0);
  const double r1 = fma(-q1, 1000.0, x);
  return fma(r1, kInv, q1);
}

}  // namespace lc
