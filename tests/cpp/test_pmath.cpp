// pcos (single-kernel evaluation) must equal pcos_ref (both kernels +
// quadrant switch) bit for bit on the normal draw's whole input range.
// Built with -ffp-contract=off like the oracle.  Usage: test_pmath [n]
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <initializer_list>

#include "../../paper_1607_06886_b200/csrc/common/pmath.h"

static uint64_t mix(uint64_t x) {
  x += 0x9e3779b97f4a7c15ull;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
  return x ^ (x >> 31);
}

int main(int argc, char** argv) {
  const long n = argc > 1 ? std::atol(argv[1]) : 20000000;
  const double two_pi = 6.283185307179586;
  long bad = 0, checked = 0;
  auto check = [&](double x) {
    ++checked;
    const double a = pump_pm::pcos(x), b = pump_pm::pcos_ref(x);
    if (pump_pm::dbits(a) != pump_pm::dbits(b)) {
      if (bad < 10) std::printf("mismatch x=%.17g pcos=%.17g ref=%.17g\n", x, a, b);
      ++bad;
    }
  };
  for (long i = 0; i < n; ++i) {
    const double u = static_cast<double>((mix(static_cast<uint64_t>(i)) >> 11) + 1) * 0x1.0p-53;  // (0, 1]
    check(two_pi * u);
  }
  // quadrant edges and the kcos branch points (|y0| = 0.3, 0.78125)
  for (int q = 0; q <= 4; ++q)
    for (double d : {0.0, 0.3, -0.3, 0.78125, -0.78125, 0.785398, -0.785398})
      for (int s = -64; s <= 64; ++s) check(std::nextafter(q * 1.5707963267948966 + d, 10.0) + s * 1e-16 * (1 + q));
  check(two_pi);
  check(0x1.0p-53 * two_pi);
  std::printf("%ld checked, %ld mismatches\n", checked, bad);
  return bad ? 1 : 0;
}
