// pmath.h plog / pcos against correctly rounded references (libquadmath,
// 113-bit) and against glibc on the normal draw's input sets: u in (0, 1] on
// the 2^-53 grid for log, fl(2 pi u) for cos, plus the draw itself.  Built
// with -ffp-contract=off like the oracle.  Prints the rates; exit 1 if plog /
// pcos are not correctly rounded on more than 1e-6 of the inputs.
// Usage: test_pmath [n]
#include <quadmath.h>

#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>

#include "../../paper_1607_06886_b200/csrc/common/pmath.h"

static uint64_t mix(uint64_t x) {
  x += 0x9e3779b97f4a7c15ull;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
  return x ^ (x >> 31);
}
static uint64_t bits(double x) { return pump_pm::dbits(x); }

int main(int argc, char** argv) {
  const long n = argc > 1 ? std::atol(argv[1]) : 2000000;
  const double two_pi = 2.0 * 3.14159265358979323846;
  long log_cr_bad = 0, cos_cr_bad = 0, log_glibc = 0, cos_glibc = 0, normal_glibc = 0, glibc_log_cr = 0,
       glibc_cos_cr = 0, checked = 0;
  auto one = [&](double u1, double u2) {
    ++checked;
    const double l = pump_pm::plog(u1), lq = static_cast<double>(logq(static_cast<__float128>(u1)));
    const double x2 = two_pi * u2;
    const double c = pump_pm::pcos(x2), cq = static_cast<double>(cosq(static_cast<__float128>(x2)));
    if (bits(l) != bits(lq)) {
      if (log_cr_bad < 5) std::printf("log not CR: u=%a got %a want %a\n", u1, l, lq);
      ++log_cr_bad;
    }
    if (bits(c) != bits(cq)) {
      if (cos_cr_bad < 5) std::printf("cos not CR: x=%a got %a want %a\n", x2, c, cq);
      ++cos_cr_bad;
    }
    const double lg = std::log(u1), cg = std::cos(x2);
    log_glibc += bits(l) == bits(lg);
    cos_glibc += bits(c) == bits(cg);
    glibc_log_cr += bits(lg) == bits(lq);
    glibc_cos_cr += bits(cg) == bits(cq);
    normal_glibc += bits(std::sqrt(-2.0 * l) * c) == bits(std::sqrt(-2.0 * lg) * cg);
  };
  for (long i = 0; i < n; ++i) {
    const double u1 = static_cast<double>((mix(2 * static_cast<uint64_t>(i)) >> 11) + 1) * 0x1.0p-53;
    const double u2 = static_cast<double>((mix(2 * static_cast<uint64_t>(i) + 1) >> 11) + 1) * 0x1.0p-53;
    one(u1, u2);
  }
  // edges: u near 1 and tiny, quadrant boundaries of 2 pi u
  for (long k = 1; k <= 4096; ++k) {
    one(1.0 - k * 0x1.0p-53, k * 0x1.0p-53);
    one(k * 0x1.0p-53, 0.25 - k * 0x1.0p-53);
    one(0.5 + k * 0x1.0p-53, 0.5 + k * 0x1.0p-53);
    one(0.75 - k * 0x1.0p-53, 0.75 - k * 0x1.0p-53);
    one(0.999 + k * 0x1.0p-53, 1.0 - k * 0x1.0p-53);
  }
  std::printf("%ld checked: log not CR %ld, cos not CR %ld | equal to glibc: log %.6f%% cos %.6f%% normal %.6f%% "
              "| glibc CR: log %.6f%% cos %.6f%%\n",
              checked, log_cr_bad, cos_cr_bad, 100.0 * log_glibc / checked, 100.0 * cos_glibc / checked,
              100.0 * normal_glibc / checked, 100.0 * glibc_log_cr / checked, 100.0 * glibc_cos_cr / checked);
  return (log_cr_bad + cos_cr_bad) * 1e6 > checked ? 1 : 0;
}
