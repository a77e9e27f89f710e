// Portable binary64 log / cos used by the normal draw on BOTH sides of the
// parity boundary (CUDA kernels and the CPU oracle's "portable" mode).
//
// Why this file exists: the reference draws normals as
//   sqrt(-2 log u1) * cos(2 pi u2)                 (rng.hpp:43-49)
// with glibc's log/cos, whose last bits depend on the host ISA (the survey
// measured 0.066% of normals differing between glibc's FMA and non-FMA
// ifunc variants).  No device libm can reproduce glibc bit
// for bit, so both the GPU and the oracle evaluate log/cos with the
// algorithms below, written only in IEEE-754 +,-,*,/ (no FMA, no tables).
// Identical inputs therefore give identical bits on x86 (built with
// -ffp-contract=off) and on sm_100a (built with --fmad=false).
//
// Algorithms: the classic argument-reduction + minimax-polynomial schemes
// (Cody-Waite reduction by pi/2 in three 33-bit pieces; log via
// s = f/(2+f) and an odd series in s).  The coefficients are the published
// minimax coefficients of those schemes.  Accuracy is < 1 ulp; agreement
// with glibc is measured by tests/test_oracle.py::test_portable_vs_glibc.
#pragma once

#include <stdint.h>

#if defined(__CUDACC__)
#define PUMP_HD __host__ __device__ __forceinline__
#else
#define PUMP_HD inline
#endif

namespace pump_pm {

PUMP_HD uint64_t dbits(double x) {
#if defined(__CUDA_ARCH__)
  return static_cast<uint64_t>(__double_as_longlong(x));
#else
  union { double d; uint64_t u; } c;
  c.d = x;
  return c.u;
#endif
}

PUMP_HD double bitsd(uint64_t u) {
#if defined(__CUDA_ARCH__)
  return __longlong_as_double(static_cast<long long>(u));
#else
  union { double d; uint64_t u; } c;
  c.u = u;
  return c.d;
#endif
}

// Natural log for positive normal x (the normal draw only ever passes
// u in [2^-53, 1]).
PUMP_HD double plog(double x) {
  const double ln2_hi = 6.93147180369123816490e-01;
  const double ln2_lo = 1.90821492927058770002e-10;
  const double Lg1 = 6.666666666666735130e-01;
  const double Lg2 = 3.999999999940941908e-01;
  const double Lg3 = 2.857142874366239149e-01;
  const double Lg4 = 2.222219843214978396e-01;
  const double Lg5 = 1.818357216161805012e-01;
  const double Lg6 = 1.531383769920937332e-01;
  const double Lg7 = 1.479819860511658591e-01;

  uint64_t b = dbits(x);
  int32_t hx = static_cast<int32_t>(b >> 32);
  int32_t k = ((hx >> 20) & 0x7ff) - 1023;
  hx &= 0x000fffff;
  // mantissa above ~sqrt(2): use m/2 and k+1 so f = m-1 is in [-0.293, 0.414]
  int32_t i = (hx + 0x95f64) & 0x100000;
  uint64_t mb = (static_cast<uint64_t>(static_cast<uint32_t>(hx | (i ^ 0x3ff00000))) << 32) |
                (b & 0xffffffffull);
  k += (i >> 20);
  double m = bitsd(mb);
  double f = m - 1.0;
  double s = f / (2.0 + f);
  double dk = static_cast<double>(k);
  double z = s * s;
  double w = z * z;
  double t1 = w * (Lg2 + w * (Lg4 + w * Lg6));
  double t2 = z * (Lg1 + w * (Lg3 + w * (Lg5 + w * Lg7)));
  double R = t2 + t1;
  double hfsq = 0.5 * f * f;
  return dk * ln2_hi - ((hfsq - (s * (hfsq + R) + dk * ln2_lo)) - f);
}

// cos kernel on [-pi/4, pi/4]; y is the tail of the reduced argument.
PUMP_HD double kcos(double x, double y) {
  const double C1 = 4.16666666666666019037e-02;
  const double C2 = -1.38888888888741095749e-03;
  const double C3 = 2.48015872894767294178e-05;
  const double C4 = -2.75573143513906633035e-07;
  const double C5 = 2.08757232129817482790e-09;
  const double C6 = -1.13596475577881948265e-11;
  double z = x * x;
  double r = z * (C1 + z * (C2 + z * (C3 + z * (C4 + z * (C5 + z * C6)))));
  uint32_t ix = static_cast<uint32_t>(dbits(x) >> 32) & 0x7fffffffu;
  if (ix < 0x3FD33333u) return 1.0 - (0.5 * z - (z * r - x * y));  // |x| < 0.3
  double qx;
  if (ix > 0x3fe90000u)
    qx = 0.28125;
  else
    qx = bitsd(static_cast<uint64_t>(ix - 0x00200000u) << 32);  // x/4, low word 0
  double hz = 0.5 * z - qx;
  double a = 1.0 - qx;
  return a - (hz - (z * r - x * y));
}

// sin kernel on [-pi/4, pi/4] with tail y.
PUMP_HD double ksin(double x, double y) {
  const double S1 = -1.66666666666666324348e-01;
  const double S2 = 8.33333333332248946124e-03;
  const double S3 = -1.98412698298579493134e-04;
  const double S4 = 2.75573137070700676789e-06;
  const double S5 = -2.50507602534068634195e-08;
  const double S6 = 1.58969099521155010221e-10;
  double z = x * x;
  double v = z * x;
  double r = S2 + z * (S3 + z * (S4 + z * (S5 + z * S6)));
  return x - ((z * (0.5 * y - v * r) - y) - v * S1);
}

// cos(x) for x in [0, 2*pi + 1] (the normal draw passes fl(2 pi u), u in (0,1]).
PUMP_HD double pcos(double x) {
  const double invpio2 = 6.36619772367581382433e-01;
  const double pio2_1 = 1.57079632673412561417e+00;
  const double pio2_2 = 6.07710050630396597660e-11;
  const double pio2_2t = 2.02226624879595063154e-21;
  const double pio2_3 = 2.02226624871116645580e-21;
  const double pio2_3t = 8.47842766036889956997e-32;
  int n = static_cast<int>(x * invpio2 + 0.5);
  double fn = static_cast<double>(n);
  double r = x - fn * pio2_1;  // exact for n <= 4
  double t = r;
  double w = fn * pio2_2;
  r = t - w;
  w = fn * pio2_2t - ((t - r) - w);
  t = r;
  w = fn * pio2_3;
  r = t - w;
  w = fn * pio2_3t - ((t - r) - w);
  double y0 = r - w;
  double y1 = (r - y0) - w;
  double c = kcos(y0, y1);
  double s = ksin(y0, y1);
  switch (n & 3) {
    case 0: return c;
    case 1: return -s;
    case 2: return -c;
    default: return s;
  }
}

}  // namespace pump_pm
