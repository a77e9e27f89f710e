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

// Coefficient table.  On the device it lives in the constant bank so the
// FP64 instructions take the coefficients as c[][] operands (as literals
// each one cost two uniform-register moves per use).  Same values, same
// bits on both sides.
#define PUMP_PM_TABLE                                                                                     \
  {                                                                                                     \
    6.93147180369123816490e-01, 1.90821492927058770002e-10, /* 0-1 ln2_hi, ln2_lo */                   \
        6.666666666666735130e-01, 3.999999999940941908e-01, 2.857142874366239149e-01,                   \
        2.222219843214978396e-01, 1.818357216161805012e-01, 1.531383769920937332e-01,                   \
        1.479819860511658591e-01, /* 2-8 Lg1..Lg7 */                                                    \
        4.16666666666666019037e-02, -1.38888888888741095749e-03, 2.48015872894767294178e-05,            \
        -2.75573143513906633035e-07, 2.08757232129817482790e-09, -1.13596475577881948265e-11,           \
        /* 9-14 C1..C6 */                                                                               \
        -1.66666666666666324348e-01, 8.33333333332248946124e-03, -1.98412698298579493134e-04,           \
        2.75573137070700676789e-06, -2.50507602534068634195e-08, 1.58969099521155010221e-10,            \
        /* 15-20 S1..S6 */                                                                              \
        6.36619772367581382433e-01, 1.57079632673412561417e+00, 6.07710050630396597660e-11,             \
        2.02226624879595063154e-21, 2.02226624871116645580e-21, 8.47842766036889956997e-32              \
        /* 21-26 invpio2, pio2_1, pio2_2, pio2_2t, pio2_3, pio2_3t */                                   \
  }
#if defined(__CUDA_ARCH__)
static __constant__ double kPmTab[27] = PUMP_PM_TABLE;
#else
static constexpr double kPmTab[27] = PUMP_PM_TABLE;
#endif
#undef PUMP_PM_TABLE
enum : int { kLn2Hi = 0, kLn2Lo, kLg1, kLg2, kLg3, kLg4, kLg5, kLg6, kLg7, kC1, kC2, kC3, kC4, kC5, kC6,
             kS1, kS2, kS3, kS4, kS5, kS6, kInvPio2, kPio2_1, kPio2_2, kPio2_2t, kPio2_3, kPio2_3t };

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
  const double* K = kPmTab;
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
  double t1 = w * (K[kLg2] + w * (K[kLg4] + w * K[kLg6]));
  double t2 = z * (K[kLg1] + w * (K[kLg3] + w * (K[kLg5] + w * K[kLg7])));
  double R = t2 + t1;
  double hfsq = 0.5 * f * f;
  return dk * K[kLn2Hi] - ((hfsq - (s * (hfsq + R) + dk * K[kLn2Lo])) - f);
}

// cos kernel on [-pi/4, pi/4]; y is the tail of the reduced argument.
PUMP_HD double kcos(double x, double y) {
  const double* K = kPmTab;
  double z = x * x;
  double r = z * (K[kC1] + z * (K[kC2] + z * (K[kC3] + z * (K[kC4] + z * (K[kC5] + z * K[kC6])))));
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
  const double* K = kPmTab;
  double z = x * x;
  double v = z * x;
  double r = K[kS2] + z * (K[kS3] + z * (K[kS4] + z * (K[kS5] + z * K[kS6])));
  return x - ((z * (0.5 * y - v * r) - y) - v * K[kS1]);
}

// Argument reduction by pi/2 (three-piece Cody-Waite): x = n pi/2 + (y0 + y1).
PUMP_HD int rem_pio2(double x, double& y0, double& y1) {
  const double* K = kPmTab;
  int n = static_cast<int>(x * K[kInvPio2] + 0.5);
  double fn = static_cast<double>(n);
  double r = x - fn * K[kPio2_1];  // exact for n <= 4
  double t = r;
  double w = fn * K[kPio2_2];
  r = t - w;
  w = fn * K[kPio2_2t] - ((t - r) - w);
  t = r;
  w = fn * K[kPio2_3];
  r = t - w;
  w = fn * K[kPio2_3t] - ((t - r) - w);
  y0 = r - w;
  y1 = (r - y0) - w;
  return n;
}

// cos(x), definition form: both kernels, quadrant select.
PUMP_HD double pcos_ref(double x) {
  double y0, y1;
  const int n = rem_pio2(x, y0, y1);
  double c = kcos(y0, y1);
  double s = ksin(y0, y1);
  switch (n & 3) {
    case 0: return c;
    case 1: return -s;
    case 2: return -c;
    default: return s;
  }
}

// cos(x) for x in [0, 2*pi + 1] (the normal draw passes fl(2 pi u), u in (0,1]).
// Bit-identical to pcos_ref (tests/cpp/test_pmath.cpp) but evaluates only
// the kernel the quadrant needs: the Horner steps C6..C2 / S6..S2 have the
// same shape, so they run once on selected coefficients; each IEEE
// operation sees the operands pcos_ref's chosen kernel gives it.
PUMP_HD double pcos(double x) {
  const double* K = kPmTab;
  double y0, y1;
  const int n = rem_pio2(x, y0, y1);
  const bool odd = (n & 1) != 0;  // sin kernel
  const double z = y0 * y0;
  double h = odd ? K[kS6] : K[kC6];
  h = (odd ? K[kS5] : K[kC5]) + z * h;
  h = (odd ? K[kS4] : K[kC4]) + z * h;
  h = (odd ? K[kS3] : K[kC3]) + z * h;
  h = (odd ? K[kS2] : K[kC2]) + z * h;
  double res;
  if (odd) {
    const double v = z * y0;
    res = y0 - ((z * (0.5 * y1 - v * h) - y1) - v * K[kS1]);
  } else {
    const double r = z * (K[kC1] + z * h);
    const uint32_t ix = static_cast<uint32_t>(dbits(y0) >> 32) & 0x7fffffffu;
    if (ix < 0x3FD33333u) {
      res = 1.0 - (0.5 * z - (z * r - y0 * y1));
    } else {
      const double qx = ix > 0x3fe90000u ? 0.28125 : bitsd(static_cast<uint64_t>(ix - 0x00200000u) << 32);
      const double hz = 0.5 * z - qx;
      const double a = 1.0 - qx;
      res = a - (hz - (z * r - y0 * y1));
    }
  }
  return ((n + 1) & 2) ? -res : res;
}

}  // namespace pump_pm
