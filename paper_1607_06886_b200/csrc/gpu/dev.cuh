// Device building blocks shared by the sm_100a kernels.
//
// Bit-exactness contract: this translation unit is
// compiled with --fmad=false, every reduction is sequential from +0.0 in the
// reference's order, divisions and square roots are IEEE (correctly rounded),
// and log/cos come from csrc/common/pmath.h (shared with the CPU oracle).
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

#include "../common/pmath.h"

namespace pumpg {

constexpr uint64_t kPhi = 0x9e3779b97f4a7c15ULL;
constexpr uint64_t kProcess = 1ull << 20;      // rng.hpp:52-56
constexpr uint64_t kMeasurement = 2ull << 20;
constexpr double kTwoPi = 2.0 * 3.14159265358979323846;

// splitmix64 finalizer (rng.hpp:8-15)
__device__ __forceinline__ uint64_t mix64(uint64_t x) {
  x ^= x >> 30;
  x *= 0xbf58476d1ce4e5b9ULL;
  x ^= x >> 27;
  x *= 0x94d049bb133111ebULL;
  x ^= x >> 31;
  return x;
}

// counter_hash(seed, a, b, c) = mix(prefix(seed, a, b) + c) with
// prefix = mix(mix(mix(seed + phi) + a) + b)  (rng.hpp:20-29).  Splitting
// out the prefix lets one (particle, timestep) key serve all its channels.
__device__ __forceinline__ uint64_t hash_prefix2(uint64_t seed_a /* mix(mix(seed+phi)+a) */, uint64_t b) {
  return mix64(seed_a + b);
}
__device__ __forceinline__ uint64_t hash_seed_a(uint64_t seed, uint64_t a) {
  return mix64(mix64(seed + kPhi) + a);
}
__device__ __forceinline__ double to_unit(uint64_t x) {  // rng.hpp:32-34
  return (static_cast<double>(x >> 11) + 1.0) * 0x1p-53;
}
// normal(seed, a, b, ch) given prefix = mix(mix(mix(seed+phi)+a)+b)  (rng.hpp:43-49)
__device__ __forceinline__ double normal_from_prefix(uint64_t prefix, uint64_t ch) {
  double u1 = to_unit(mix64(prefix + 2 * ch));
  double u2 = to_unit(mix64(prefix + 2 * ch + 1));
  return sqrt(-2.0 * pump_pm::plog(u1)) * pump_pm::pcos(kTwoPi * u2);
}

// Closed-loop matrices as a kernel parameter (constant bank), compile-time
// dims so every gemv is fully unrolled with constant-bank operands.
template <int D, int DW>
struct LoopP {
  double F[4 * D * D];
  double Gv[2 * D * D];
  double Gw[2 * D * DW];
  double Sv[D * D];
  double Sw[DW * DW];
  double S0[D * D];
  double C[DW * D];
};

// Eigen gemv row: c = 0; c = c + M_ij x_j (j ascending)
template <int N>
__device__ __forceinline__ double row_dot(const double* row, const double* x) {
  double c = 0.0;
#pragma unroll
  for (int j = 0; j < N; ++j) c = c + row[j] * x[j];
  return c;
}

// z <- ((F z) + Gv (Sv nv)) + Gw (Sw nw)   (lti.hpp:287, cp.hpp:254)
template <int D, int DW>
__device__ __forceinline__ void cl_step(const LoopP<D, DW>& L, double (&z)[2 * D], const double (&nv)[D],
                                        const double (&nw)[DW]) {
  double t1[D], t2[DW], zn[2 * D];
#pragma unroll
  for (int r = 0; r < D; ++r) t1[r] = row_dot<D>(L.Sv + r * D, nv);
#pragma unroll
  for (int r = 0; r < DW; ++r) t2[r] = row_dot<DW>(L.Sw + r * DW, nw);
#pragma unroll
  for (int r = 0; r < 2 * D; ++r) {
    double a = row_dot<2 * D>(L.F + r * 2 * D, z);
    double b = row_dot<D>(L.Gv + r * D, t1);
    double c = row_dot<DW>(L.Gw + r * DW, t2);
    zn[r] = (a + b) + c;
  }
#pragma unroll
  for (int r = 0; r < 2 * D; ++r) z[r] = zn[r];
}

__host__ __device__ __forceinline__ int __builtin_ctzll_hd(uint64_t x) {
#if defined(__CUDA_ARCH__)
  return __ffsll(static_cast<long long>(x)) - 1;
#else
  return __builtin_ctzll(x);
#endif
}

// Reciprocal to within a few ulps (not correctly rounded): MUFU seed + two
// Newton steps.  Only for values that carry their own error margin (the lazy
// cubic's 1e-12 S, the filter multipliers' rounding-down factor), never for
// a value the reference computes.  x > 0, finite, normal.
__host__ __device__ __forceinline__ double rcp_approx(double x) {
#if defined(__CUDA_ARCH__)
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
  double e = fma(-x, r, 1.0);
  r = fma(r, e, r);
  e = fma(-x, r, 1.0);
  return fma(r, e, r);
#else
  return 1.0 / x;
#endif
}

// ----------------------------------------------------------- geometry
// closed AABB containment (geom.hpp:19-23)
template <int DW>
__host__ __device__ __forceinline__ bool box_contains(const double* lo, const double* hi, const double* p) {
  bool in = true;
#pragma unroll
  for (int k = 0; k < DW; ++k) in = in && !(p[k] < lo[k] || p[k] > hi[k]);
  return in;
}

// Workspace with obstacles stored SoA-by-box: lo[o*DW+k], hi[o*DW+k].
struct WorldD {
  int n_obs;
  const double* lo;  // obstacles
  const double* hi;
  double blo[6], bhi[6];  // bounds
};

template <int DW>
__host__ __device__ __forceinline__ bool point_free(const WorldD& w, const double* y) {  // geom.hpp:56-61
  if (!box_contains<DW>(w.blo, w.bhi, y)) return false;
  for (int o = 0; o < w.n_obs; ++o)
    if (box_contains<DW>(w.lo + o * DW, w.hi + o * DW, y)) return false;
  return true;
}

// slab test, closed box (geom.hpp:64-80)
template <int DW>
__host__ __device__ __forceinline__ bool segment_hits(const double* p0, const double* p1, const double* lo, const double* hi) {
  double tmin = 0.0, tmax = 1.0;
#pragma unroll
  for (int k = 0; k < DW; ++k) {
    double d = p1[k] - p0[k];
    if ((d < 0 ? -d : d) < 1e-300) {
      if (p0[k] < lo[k] || p0[k] > hi[k]) return false;
      continue;
    }
    double t0 = (lo[k] - p0[k]) / d;
    double t1 = (hi[k] - p0[k]) / d;
    if (t0 > t1) {
      double s = t0;
      t0 = t1;
      t1 = s;
    }
    tmin = (tmin < t0) ? t0 : tmin;  // std::max(tmin, t0)
    tmax = (t1 < tmax) ? t1 : tmax;  // std::min(tmax, t1)
    if (tmin > tmax) return false;
  }
  return true;
}

// Conservative separation test: true only if, on some axis, both points lie
// outside the closed box by more than a relative margin of 1e-9.  Then the
// reference slab test (segment_hits) provably returns false — the entry
// parameter rounds to > 1 (or the exit parameter to < 0) — and point_free
// cannot find either point (or any point interpolated between them) inside
// the box.  So skipping such boxes never changes a collision decision.
template <int DW>
__host__ __device__ __forceinline__ bool box_separated(const double* p0, const double* p1, const double* lo,
                                                       const double* hi) {
  bool sep = false;
#pragma unroll
  for (int k = 0; k < DW; ++k) {
    const double a = p0[k] < p1[k] ? p0[k] : p1[k];
    const double b = p0[k] < p1[k] ? p1[k] : p0[k];
    const double m = 1e-9 * (1.0 + (lo[k] < 0 ? -lo[k] : lo[k]) + (hi[k] < 0 ? -hi[k] : hi[k]) + (a < 0 ? -a : a) +
                             (b < 0 ? -b : b));
    sep = sep || (b < lo[k] - m) || (a > hi[k] + m);
  }
  return sep;
}

template <int DW>
__host__ __device__ __forceinline__ bool segment_collides(const WorldD& w, const double* p0, const double* p1) {
  for (int o = 0; o < w.n_obs; ++o) {
    if (box_separated<DW>(p0, p1, w.lo + o * DW, w.hi + o * DW)) continue;  // cannot hit (see above)
    if (segment_hits<DW>(p0, p1, w.lo + o * DW, w.hi + o * DW)) return true;
  }
  return false;
}

template <int N>
__host__ __device__ __forceinline__ double sqnorm(const double* x) {
  double s = 0.0;
#pragma unroll
  for (int k = 0; k < N; ++k) s = s + x[k] * x[k];
  return s;
}

// ---------------------------------------------------------------- steer
// Motion polynomial per axis (steer.hpp:37-51)
template <int DW>
struct MotionD {
  double p0[DW], v0[DW], p1[DW], v1[DW], a[DW], j[DW];
  double tau;
};

template <int DW>
__host__ __device__ __forceinline__ void motion_pos(const MotionD<DW>& m, double s, double* out) {
  if (s <= 0) {
#pragma unroll
    for (int k = 0; k < DW; ++k) out[k] = m.p0[k];
    return;
  }
  if (s >= m.tau) {
#pragma unroll
    for (int k = 0; k < DW; ++k) out[k] = m.p1[k];
    return;
  }
#pragma unroll
  for (int k = 0; k < DW; ++k) out[k] = m.p0[k] + m.v0[k] * s + m.a[k] * s * s / 2 + m.j[k] * s * s * s / 6;
}

template <int DW>
__host__ __device__ __forceinline__ void motion_state(const MotionD<DW>& m, double s, double* pos, double* vel) {
  if (s <= 0) {
#pragma unroll
    for (int k = 0; k < DW; ++k) {
      pos[k] = m.p0[k];
      vel[k] = m.v0[k];
    }
    return;
  }
  if (s >= m.tau) {
#pragma unroll
    for (int k = 0; k < DW; ++k) {
      pos[k] = m.p1[k];
      vel[k] = m.v1[k];
    }
    return;
  }
#pragma unroll
  for (int k = 0; k < DW; ++k) {
    pos[k] = m.p0[k] + m.v0[k] * s + m.a[k] * s * s / 2 + m.j[k] * s * s * s / 6;
    vel[k] = m.v0[k] + m.a[k] * s + m.j[k] * s * s / 2;
  }
}

// c(tau) (steer.hpp:84-94)
template <int DW>
__host__ __device__ __forceinline__ double steer_cost(const double* ap, const double* av, const double* bp, const double* bv,
                                             double tau) {
  double c = tau;
#pragma unroll
  for (int k = 0; k < DW; ++k) {
    double dp = bp[k] - ap[k] - av[k] * tau;
    double dv = bv[k] - av[k];
    c += 12 * dp * dp / (tau * tau * tau) - 12 * dp * dv / (tau * tau) + 4 * dv * dv / tau;
  }
  return c;
}

// Conservative bounding box of a motion's positions on [0, tau]: the cubic
// per axis attains its extremes at s = 0, s = tau or a root of its
// derivative; the box is widened by a relative margin (1e-6 of the term
// magnitudes) that dwarfs every rounding error of the evaluated positions.
template <int DW>
__host__ __device__ __forceinline__ void motion_bbox(const MotionD<DW>& m, double* bl, double* bh) {
  const double tau = m.tau;
#pragma unroll
  for (int k = 0; k < DW; ++k) {
    const double p0 = m.p0[k], v0 = m.v0[k], a = m.a[k], j = m.j[k];
    double lo = p0 < m.p1[k] ? p0 : m.p1[k], hi = p0 < m.p1[k] ? m.p1[k] : p0;
    auto at = [&](double s) { return p0 + v0 * s + a * s * s / 2 + j * s * s * s / 6; };
    const double pt = at(tau);
    lo = pt < lo ? pt : lo;
    hi = pt > hi ? pt : hi;
    // p'(s) = v0 + a s + j s^2 / 2
    double r[2];
    int nr = 0;
    const double aj = j < 0 ? -j : j, aa = a < 0 ? -a : a;
    if (aj > 1e-300) {
      const double disc = a * a - 2.0 * j * v0;
      if (disc >= 0) {
        const double sq = sqrt(disc);
        r[nr++] = (-a + sq) / j;
        r[nr++] = (-a - sq) / j;
      } else if (disc > -1e-12 * (a * a + (2.0 * j * v0 < 0 ? -2.0 * j * v0 : 2.0 * j * v0))) {
        r[nr++] = -a / j;  // near-double root
      }
    } else if (aa > 1e-300) {
      r[nr++] = -v0 / a;
    }
    for (int x = 0; x < nr; ++x) {
      if (r[x] > 0 && r[x] < tau) {
        const double pr = at(r[x]);
        lo = pr < lo ? pr : lo;
        hi = pr > hi ? pr : hi;
      }
    }
    const double mag = 1.0 + (p0 < 0 ? -p0 : p0) + (v0 < 0 ? -v0 : v0) * tau + aa * tau * tau / 2 + aj * tau * tau * tau / 6 +
                       (m.p1[k] < 0 ? -m.p1[k] : m.p1[k]);
    bl[k] = lo - 1e-6 * mag;
    bh[k] = hi + 1e-6 * mag;
  }
}

// motion_collides (geom.hpp:96-123): adaptive midpoint bisection until the
// chord is <= eps_cc (or the span < 1e-9 s), exact segment test at leaves.
// Iterative DFS over (t0, t1) spans; endpoints are recomputed with the same
// polynomial so they carry the same bits the reference stores.  The result
// is an OR over a fixed tree of tests, so traversal order cannot change it.
//
// Culling (exact-preserving): every tested point lies on the motion and
// every tested segment joins two such points, so all of them lie in the
// motion's (widened) bounding box.  Obstacles separated from that box can
// neither contain a tested point nor be hit by a tested segment, and if the
// box is strictly inside the workspace bounds no bounds test can fail; when
// nothing remains the answer is "no collision" without subdividing.
//
// Span pruning (exact-preserving, same argument one level down): every point
// tested inside a span [t0, t1] and every leaf segment below it lies within
// the chord box of (p(t0), p(t1)) widened per axis by the interpolation error
// bound (t1 - t0)^2 / 8 * max|p''| (p'' = a + j s is linear, so its maximum
// is at an end) plus the rounding margin of motion_bbox.  A span whose box
// is inside the workspace and separated from every candidate obstacle holds
// no failing test, so its subtree is skipped.
// The culling state of one motion: its widened bounding box strictly inside
// the workspace bounds (no bounds test can fail) and the obstacles not
// separated from the box (the only ones any point on the motion, or any
// segment between such points, can touch).
constexpr int kCullWords = 4;
constexpr int kCullList = 64;  // candidate index list when there are more boxes than bitmask bits
// LIST = 0: bitmask only (<= 64 kCullWords boxes; more boxes are all tested);
// LIST = kCullList: an index list of up to LIST candidates for larger worlds
template <int LIST>
struct MotionCullT {
  bool inside, masked, any;
  int nlist;  // -1: candidates in the bitmask; else list[0..nlist)
  uint64_t cand[kCullWords];
  uint16_t list[LIST > 0 ? LIST : 1];
};
using MotionCull = MotionCullT<0>;

// f(o) for every candidate box o (ascending); true as soon as one f is true
template <int LIST, class F>
__host__ __device__ __forceinline__ bool cull_any(const MotionCullT<LIST>& c, F f) {
  if (LIST == 0 || c.nlist < 0) {
    for (int q = 0; q < kCullWords; ++q)
      for (uint64_t x = c.cand[q]; x; x &= x - 1)
        if (f(q * 64 + __builtin_ctzll_hd(x))) return true;
    return false;
  }
  for (int i = 0; i < c.nlist; ++i)
    if (f(static_cast<int>(c.list[i]))) return true;
  return false;
}

template <int DW, int LIST = 0>
__host__ __device__ inline MotionCullT<LIST> motion_cull(const MotionD<DW>& m, const WorldD& w) {
  MotionCullT<LIST> c;
  double bl[DW], bh[DW];
  motion_bbox<DW>(m, bl, bh);
  c.inside = true;
#pragma unroll
  for (int k = 0; k < DW; ++k) c.inside = c.inside && bl[k] > w.blo[k] && bh[k] < w.bhi[k];
  for (int q = 0; q < kCullWords; ++q) c.cand[q] = 0;
  c.nlist = w.n_obs <= 64 * kCullWords ? -1 : 0;
  c.masked = true;
  c.any = false;
  for (int o = 0; o < w.n_obs; ++o) {
    bool sep = false;
#pragma unroll
    for (int k = 0; k < DW; ++k) sep = sep || (bh[k] < w.lo[o * DW + k]) || (bl[k] > w.hi[o * DW + k]);
    if (sep) continue;
    c.any = true;
    if (c.nlist < 0) {
      c.cand[o >> 6] |= 1ull << (o & 63);
    } else if (c.nlist < LIST) {
      c.list[c.nlist++] = static_cast<uint16_t>(o);
    } else {
      c.masked = false;  // too many candidates: test every box
      break;
    }
  }
  return c;
}

// point_free (geom.hpp:56-61) for a point on the motion `c` was computed for
template <int DW, int LIST>
__host__ __device__ inline bool point_free_culled(const WorldD& w, const MotionCullT<LIST>& c, const double* p) {
  if (!c.inside && !box_contains<DW>(w.blo, w.bhi, p)) return false;
  if (!c.masked) {
    for (int o = 0; o < w.n_obs; ++o)
      if (box_contains<DW>(w.lo + o * DW, w.hi + o * DW, p)) return false;
    return true;
  }
  return !cull_any(c, [&](int o) { return box_contains<DW>(w.lo + o * DW, w.hi + o * DW, p); });
}

template <int DW, int LIST = 0>
__host__ __device__ inline bool motion_collides(const MotionD<DW>& m, const WorldD& w, double eps_cc,
                                                const MotionCullT<LIST>* pre = nullptr) {
  MotionCullT<LIST> own;
  if (!pre) own = motion_cull<DW, LIST>(m, w);
  const MotionCullT<LIST>& cull = pre ? *pre : own;
  const bool inside = cull.inside, masked = cull.masked, any = cull.any;
  if (inside && !any) return false;
  auto free_pt = [&](const double* p) {
    if (!inside && !box_contains<DW>(w.blo, w.bhi, p)) return false;
    if (!masked) {
      for (int o = 0; o < w.n_obs; ++o)
        if (box_contains<DW>(w.lo + o * DW, w.hi + o * DW, p)) return false;
      return true;
    }
    return !cull_any(cull, [&](int o) { return box_contains<DW>(w.lo + o * DW, w.hi + o * DW, p); });
  };
  auto seg_hit = [&](const double* a, const double* b) {
    if (!masked) return segment_collides<DW>(w, a, b);
    return cull_any(cull, [&](int o) { return segment_hits<DW>(a, b, w.lo + o * DW, w.hi + o * DW); });
  };
  double p0[DW], p1[DW];
  motion_pos<DW>(m, 0.0, p0);
  if (!free_pt(p0)) return true;
  if (m.tau <= 0) return false;
  motion_pos<DW>(m, m.tau, p1);
  if (!free_pt(p1)) return true;
  double marg[DW];
#pragma unroll
  for (int k = 0; k < DW; ++k) {
    const double p0k = m.p0[k], v0 = m.v0[k], a = m.a[k], j = m.j[k], tau = m.tau;
    marg[k] = 1e-6 * (1.0 + (p0k < 0 ? -p0k : p0k) + (v0 < 0 ? -v0 : v0) * tau + (a < 0 ? -a : a) * tau * tau / 2 +
                      (j < 0 ? -j : j) * tau * tau * tau / 6 + (m.p1[k] < 0 ? -m.p1[k] : m.p1[k]));
  }
  auto span_clear = [&](double t0, double t1, const double* q0, const double* q1) {
    if (!masked) return false;
    const double h = t1 - t0;
    double sl[DW], sh[DW];
#pragma unroll
    for (int k = 0; k < DW; ++k) {
      const double d0 = m.a[k] + m.j[k] * t0, d1 = m.a[k] + m.j[k] * t1;
      const double ad0 = d0 < 0 ? -d0 : d0, ad1 = d1 < 0 ? -d1 : d1;
      const double dev = 0.125 * h * h * (ad0 > ad1 ? ad0 : ad1) + marg[k];
      sl[k] = (q0[k] < q1[k] ? q0[k] : q1[k]) - dev;
      sh[k] = (q0[k] < q1[k] ? q1[k] : q0[k]) + dev;
      if (!inside && !(sl[k] > w.blo[k] && sh[k] < w.bhi[k])) return false;
    }
    return !cull_any(cull, [&](int o) {
      bool sep = false;
#pragma unroll
      for (int k = 0; k < DW; ++k) sep = sep || (sh[k] < w.lo[o * DW + k]) || (sl[k] > w.hi[o * DW + k]);
      return !sep;
    });
  };
  double st1[64];  // right siblings' ends (their starts are implied, see the pop)
  int sp = 0;
  double t0 = 0.0, t1 = m.tau;
  while (true) {
    double diff[DW];
#pragma unroll
    for (int k = 0; k < DW; ++k) diff[k] = p1[k] - p0[k];
    bool span_done = span_clear(t0, t1, p0, p1);
    if (!span_done && (sqrt(sqnorm<DW>(diff)) <= eps_cc || t1 - t0 < 1e-9)) {
      if (seg_hit(p0, p1)) return true;
      span_done = true;
    }
    if (span_done) {
      if (sp == 0) return false;
      --sp;
      t0 = t1;
      t1 = st1[sp];
      // depth-first, left to right: the popped span starts where the span just
      // finished ended (t0 == the old t1), so p(t0) is the old p1, bit for bit
#pragma unroll
      for (int k = 0; k < DW; ++k) p0[k] = p1[k];
      motion_pos<DW>(m, t1, p1);
      continue;
    }
    const double tm = 0.5 * (t0 + t1);
    double pm[DW];
    motion_pos<DW>(m, tm, pm);
    if (!free_pt(pm)) return true;
    if (sp >= 64) return true;  // unreachable: depth is bounded by t1 - t0 >= 1e-9
    st1[sp] = t1;
    ++sp;
    t1 = tm;
#pragma unroll
    for (int k = 0; k < DW; ++k) p1[k] = pm[k];
  }
}

// Lower bound of the connection cost (graph build filters).  With
// dp0 = pb - pa, vbar = (va + vb) / 2 and dv = vb - va the cost is,
// identically (steer.hpp:84-94 rewritten),
//   c(tau) = tau + 12 q(tau) / tau^3 + D / tau,
//   q(tau) = |dp0 - vbar tau|^2 = A - 2 B tau + C tau^2,  D = |dv|^2,
// so on [tl, th]:  c >= tl + 12 min_[tl,th] q / th^3 + D / th.  The quadratic's
// minimum is exact (vertex B / C or an end); the rounding margin
// 1e-12 (A + 2|B| th + C th^2) dwarfs its evaluation error, and the caller's
// threshold carries its own relative margin over r_n.
struct PairLb {
  double A, B, C, D, ts;  // ts = B / C (vertex), or -1 when C == 0
};

template <int DW>
__host__ __device__ __forceinline__ PairLb pair_lb(const double* ap, const double* av, const double* bp,
                                                   const double* bv) {
  PairLb p{0.0, 0.0, 0.0, 0.0, -1.0};
#pragma unroll
  for (int k = 0; k < DW; ++k) {
    const double dp = bp[k] - ap[k], vb = 0.5 * (av[k] + bv[k]), dv = bv[k] - av[k];
    p.A += dp * dp;
    p.B += dp * vb;
    p.C += vb * vb;
    p.D += dv * dv;
  }
  if (p.C > 0) p.ts = p.B / p.C;
  return p;
}

// c3 = 12 / th^3 and c1 = 1 / th, both rounded down (the caller's grid).
__host__ __device__ __forceinline__ bool interval_clears(const PairLb& p, double tl, double th, double c3, double c1,
                                                         double thr) {
  const double ql = p.A - 2.0 * p.B * tl + p.C * tl * tl, qh = p.A - 2.0 * p.B * th + p.C * th * th;
  double qm = ql < qh ? ql : qh;
  if (p.ts > tl && p.ts < th) qm = p.A - p.B * p.ts;
  const double ab = p.B < 0 ? -p.B : p.B;
  qm -= 1e-12 * (p.A + 2.0 * ab * th + p.C * th * th);
  if (qm < 0) qm = 0;
  return (tl + c3 * qm + c1 * p.D) * (1.0 - 1e-12) >= thr;
}

// connect() without the motion coefficients: returns ok; tau, cost out.
// With kReject (graph build only) a pair is abandoned after the 64-point scan
// when the cost's lower bound on the golden-section bracket [lo, hi] clears
// reject_thr on all 16 sub-intervals: the returned tau lies in that bracket,
// so its cost would be >= r_n and graph.hpp:72 would drop the pair anyway.
constexpr double kLazyErr = 1e-12;
template <int DW, bool kReject = false>
__host__ __device__ inline bool connect_dev(const double* ap, const double* av, const double* bp, const double* bv, double tau_max,
                            double ratio, double& tau_out, double& cost_out, double reject_thr = 0.0) {
  bool same = true;
#pragma unroll
  for (int k = 0; k < DW; ++k) same = same && (ap[k] == bp[k]) && (av[k] == bv[k]);
  if (same) {
    tau_out = 0.0;
    cost_out = 0.0;
    return true;
  }
  // Lazy exact evaluation (exact-preserving).  With P = bp - ap, V = av and
  // dv = bv - av the cost is, identically, the cubic in u = 1/tau
  //   c = tau + 12 A u^3 + (-24 B - 12 E) u^2 + (12 C + 12 F + 4 D) u
  // (A = |P|^2, B = P.V, C = |V|^2, E = P.dv, F = V.dv, D = |dv|^2).  Its
  // value, computed without divisions, differs from the reference's
  // evaluation (steer_cost) by far less than err = 1e-12 * S, S the sum of the
  // absolute values of every constituent term: the reference's evaluation errs
  // by <~3e-15 S (dp's rounding is bounded by the |P|, |V| tau terms of S; ~10
  // roundings of partial sums <= S), the cubic by as much plus its u error
  // (rcp_approx: a few ulps; the scan's product chain: <~1.5e-14, i.e.
  // <~5e-14 S through u^3), so the margin is >= 15x.  A comparison the
  // reference makes is decided from the cubic when the two intervals
  // [c - err, c + err] are disjoint, and from steer_cost otherwise, so every
  // decision (scan argmin, golden-section branch) and every returned value is
  // the reference's.
  double cA = 0, cB = 0, cC = 0, cE = 0, cF = 0, cD = 0, aB = 0, aE = 0, aF = 0;
#pragma unroll
  for (int k = 0; k < DW; ++k) {
    const double P = bp[k] - ap[k], V = av[k], dv = bv[k] - av[k];
    cA += P * P;
    cB += P * V;
    cC += V * V;
    cE += P * dv;
    cF += V * dv;
    cD += dv * dv;
    aB += (P < 0 ? -P : P) * (V < 0 ? -V : V);
    aE += (P < 0 ? -P : P) * (dv < 0 ? -dv : dv);
    aF += (V < 0 ? -V : V) * (dv < 0 ? -dv : dv);
  }
  const double k3 = 12.0 * cA, k2 = -24.0 * cB - 12.0 * cE, k1 = 12.0 * cC + 12.0 * cF + 4.0 * cD;
  const double s3 = 12.0 * cA, s2 = 24.0 * aB + 12.0 * aE, s1 = 12.0 * cC + 12.0 * aF + 4.0 * cD;
  struct Lazy {
    double tau, approx, err, exact;
    bool known;
  };
  // u = 1/t only needs a few ulps: its error moves the cubic by <~1e-13 S
  auto lazy_u = [&](double t, double u) {
    Lazy z;
    z.tau = t;
    z.approx = t + ((k3 * u + k2) * u + k1) * u;
    z.err = kLazyErr * (t + ((s3 * u + s2) * u + s1) * u);
    z.known = false;
    return z;
  };
  auto lazy = [&](double t) { return lazy_u(t, rcp_approx(t)); };
  auto exact = [&](Lazy& z) {
    if (!z.known) {
      z.exact = steer_cost<DW>(ap, av, bp, bv, z.tau);
      z.known = true;
    }
    return z.exact;
  };
  auto less = [&](Lazy& a, Lazy& b) {  // the reference's `f(a) < f(b)`
    if (a.approx + a.err < b.approx - b.err) return true;
    if (a.approx - a.err > b.approx + b.err) return false;
    return exact(a) < exact(b);
  };
  const double tau_lo = tau_max * 1e-7;
  // scan: an upper bound of the minimum from the cubic, then exact costs only
  // where the cubic cannot rule the point out, in index order with the
  // reference's strict update (the first index attaining the minimum)
  // u runs down its own product chain (<= 2 ulps per step: <~1.5e-14 after
  // 64), tau keeps the reference's chain exactly
  double m_hi = __builtin_inf();
  const double u_lo = 1.0 / tau_lo, u_r = 1.0 / ratio;
  {
    double tau = tau_lo, u = u_lo;
    for (int i = 0; i < 64; ++i) {
      if (i > 0) {
        tau *= ratio;
        u *= u_r;
      }
      const Lazy z = lazy_u(tau, u);
      const double h = z.approx + z.err;
      m_hi = h < m_hi ? h : m_hi;
    }
  }
  double best_tau = tau_lo, best_c = __builtin_inf();
  int best_idx = 0;
  {
    double tau = tau_lo, u = u_lo;
    for (int i = 0; i < 64; ++i) {
      if (i > 0) {
        tau *= ratio;
        u *= u_r;
      }
      Lazy z = lazy_u(tau, u);
      if (z.approx - z.err > m_hi) continue;  // above the minimum
      const double c = exact(z);
      if (c < best_c) {
        best_c = c;
        best_tau = tau;
        best_idx = i;
      }
    }
  }
  double lo = best_tau / (best_idx > 0 ? ratio : 1.0);
  double hi = best_tau * ratio;
  hi = (tau_max < hi) ? tau_max : hi;  // std::min(best_tau * ratio, tau_max)
  if constexpr (kReject) {
    const PairLb plb = pair_lb<DW>(ap, av, bp, bv);
    constexpr int kParts = 16;
    bool clears = lo > 0;
    double t_hi = hi;
    for (int p = kParts - 1; p >= 0 && clears; --p) {
      const double t_lo = p == 0 ? lo : lo + (hi - lo) * (static_cast<double>(p) / kParts);
      // multipliers rounded down by far more than rcp_approx's few ulps
      const double r = rcp_approx(t_hi) * (1.0 - 1e-13);
      const double c3 = 12.0 * (r * r * r) * (1.0 - 1e-13), c1 = r;
      clears = interval_clears(plb, t_lo, t_hi, c3, c1, reject_thr);
      t_hi = t_lo;
    }
    if (clears) return false;
  }
  const double gr = 0.5 * (sqrt(5.0) - 1.0);
  double x1 = hi - gr * (hi - lo), x2 = lo + gr * (hi - lo);
  Lazy f1 = lazy(x1), f2 = lazy(x2);
  while (hi - lo > 1e-9 * hi) {
    if (less(f1, f2)) {
      hi = x2;
      x2 = x1;
      f2 = f1;
      x1 = hi - gr * (hi - lo);
      f1 = lazy(x1);
    } else {
      lo = x1;
      x1 = x2;
      f1 = f2;
      x2 = lo + gr * (hi - lo);
      f2 = lazy(x2);
    }
  }
  tau_out = 0.5 * (lo + hi);
  cost_out = steer_cost<DW>(ap, av, bp, bv, tau_out);
  if (best_idx == 63 && tau_out > 0.999 * tau_max) {
    const double eps = 1e-6 * tau_max;
    if (steer_cost<DW>(ap, av, bp, bv, tau_max) <= steer_cost<DW>(ap, av, bp, bv, tau_max - eps)) return false;
  }
  return true;
}

// fixed_time_coeffs (steer.hpp:63-79): acc0, jerk
template <int DW>
__host__ __device__ __forceinline__ void coeffs_dev(const double* ap, const double* av, const double* bp, const double* bv,
                                           double tau, double* acc0, double* jerk) {
#pragma unroll
  for (int k = 0; k < DW; ++k) {
    const double dp = bp[k] - ap[k] - av[k] * tau;
    const double dv = bv[k] - av[k];
    acc0[k] = 6 * dp / (tau * tau) - 2 * dv / tau;
    jerk[k] = -12 * dp / (tau * tau * tau) + 6 * dv / (tau * tau);
  }
}

// local_convex_region (geom.hpp:189-225) for a free waypoint y with nominal
// velocity yd: repeatedly take the nearest unpruned obstacle point (first
// strict minimum of |clamp(y) - y|^2), prune every box whose 2^dw corners lie
// beyond its half-space (tolerance 1e-12 (1 + d.d)), and project the
// direction by the velocity (project_halfspace, geom.hpp:163-183, eps 1e-6).
// Writes the half-spaces when a != nullptr; returns their count, or -1 when
// the pruning loop fails (the reference's runtime_error).  <= 4096 boxes.
//
// The prune test "every corner c has d.(c - y) >= dd - tol" is evaluated on
// the single corner that minimizes each term: fl(d_k (c_k - y_k)) is monotone
// in c_k and rounded addition is monotone, so that corner's computed dot is
// <= every corner's computed dot, and it is itself one of the corners: the
// test is decided exactly by it (1 dot instead of 2^dw).  kWords bounds the
// pruned bitmap (1 word keeps it in a register for <= 32 boxes).
template <int DW, int kWords = 128>
__host__ __device__ inline int convex_region(const WorldD& ws, const double* y, const double* yd, double* a_out,
                                             double* b_out, uint8_t* fb_out, int a_stride = DW, int b_stride = 1,
                                             int out_cap = 1 << 30) {
  uint32_t pruned[kWords];
  const int nw = (ws.n_obs + 31) / 32;
  for (int q = 0; q < nw; ++q) pruned[q] = 0u;
  int count = 0;
  for (int iter = 0; iter < ws.n_obs; ++iter) {
    int best = -1;
    double best_sq = __builtin_inf();
    double d[DW];
    for (int o = 0; o < ws.n_obs; ++o) {
      if ((pruned[o >> 5] >> (o & 31)) & 1u) continue;
      double cand[DW];
#pragma unroll
      for (int k = 0; k < DW; ++k) {
        double c = y[k] < ws.lo[o * DW + k] ? ws.lo[o * DW + k] : y[k];  // max(y, lo)
        c = ws.hi[o * DW + k] < c ? ws.hi[o * DW + k] : c;               // min(., hi)
        cand[k] = c - y[k];
      }
      const double sq = sqnorm<DW>(cand);
      if (sq < best_sq) {
        best_sq = sq;
        best = o;
#pragma unroll
        for (int k = 0; k < DW; ++k) d[k] = cand[k];
      }
    }
    if (best < 0) break;
    const double dd = sqnorm<DW>(d);
    const double tol = 1e-12 * (1.0 + dd);
    bool any = false;
    for (int o = 0; o < ws.n_obs; ++o) {
      if ((pruned[o >> 5] >> (o & 31)) & 1u) continue;
      double dot = 0;
#pragma unroll
      for (int k = 0; k < DW; ++k) {
        const double tl = d[k] * (ws.lo[o * DW + k] - y[k]), th = d[k] * (ws.hi[o * DW + k] - y[k]);
        dot += tl < th ? tl : th;
      }
      const bool inside = !(dot < dd - tol);
      if (inside) {
        pruned[o >> 5] |= 1u << (o & 31);
        any = true;
      }
    }
    if (!any) return -1;
    if (a_out && count < out_cap) {  // (past out_cap only the count is kept)
      double a[DW];
      bool fb = false;
      const double vn = sqrt(sqnorm<DW>(yd));
      if (vn < 1e-6) {
        fb = true;
      } else {
        double dy = 0.0;
#pragma unroll
        for (int k = 0; k < DW; ++k) dy = dy + d[k] * yd[k];
        const double coef = dy / sqnorm<DW>(yd);
#pragma unroll
        for (int k = 0; k < DW; ++k) a[k] = d[k] - coef * yd[k];
        if (sqrt(sqnorm<DW>(a)) < 1e-6 * sqrt(sqnorm<DW>(d))) fb = true;
      }
      if (fb) {
#pragma unroll
        for (int k = 0; k < DW; ++k) a[k] = d[k];
      }
#pragma unroll
      for (int k = 0; k < DW; ++k) a_out[count * a_stride + k] = a[k];
      b_out[count * b_stride] = sqnorm<DW>(a);
      fb_out[count] = fb ? 1 : 0;
    }
    ++count;
  }
  return count;
}

// convex_region for <= 32 boxes with the per-box squared distances kept (in
// shared memory, stride sq_stride); one pass per iteration.  Identical output to convex_region:
//  - |clamp(y) - y|^2 of a box does not depend on the iteration, so it is
//    computed once; the next iteration's nearest box (first strict minimum
//    among the boxes still unpruned) is tracked inside the prune pass, which
//    visits the boxes in index order with the same strict comparison.
//  - the prune test's minimizing corner is chosen by the sign of d_k (lo for
//    d_k >= 0, hi otherwise).  For d_k != 0 that is the corner min(tl, th)
//    picks (monotone rounding); for d_k = +-0 both terms are +-0, and a zero
//    term of either sign leaves the sum from +0 unchanged, so the dot is the
//    same number.
template <int DW>
__device__ __forceinline__ int convex_region_fused(const WorldD& ws, const double* y, const double* yd, double* sq,
                                                   int sq_stride, double* a_out, double* b_out, uint8_t* fb_out,
                                                   unsigned& n_clamp, unsigned& n_prune) {
  n_clamp += ws.n_obs;
  int best = -1;
  double best_sq = __builtin_inf();
  for (int o = 0; o < ws.n_obs; ++o) {
    double cand[DW];
#pragma unroll
    for (int k = 0; k < DW; ++k) {
      double c = y[k] < ws.lo[o * DW + k] ? ws.lo[o * DW + k] : y[k];
      c = ws.hi[o * DW + k] < c ? ws.hi[o * DW + k] : c;
      cand[k] = c - y[k];
    }
    const double q = sqnorm<DW>(cand);
    sq[o * sq_stride] = q;
    if (q < best_sq) {
      best_sq = q;
      best = o;
    }
  }
  uint32_t pruned = 0u;  // <= 32 boxes
  int count = 0;
  while (best >= 0) {
    double d[DW];
#pragma unroll
    for (int k = 0; k < DW; ++k) {
      double c = y[k] < ws.lo[best * DW + k] ? ws.lo[best * DW + k] : y[k];
      c = ws.hi[best * DW + k] < c ? ws.hi[best * DW + k] : c;
      d[k] = c - y[k];
    }
    const double dd = sqnorm<DW>(d);
    const double lim = dd - 1e-12 * (1.0 + dd);
    bool any = false;
    int nb = -1;
    double nsq = __builtin_inf();
    const double* cp[DW];  // the minimizing corner's coordinate array per axis
#pragma unroll
    for (int k = 0; k < DW; ++k) cp[k] = (d[k] >= 0 ? ws.lo : ws.hi) + k;
    const uint32_t all = ws.n_obs >= 32 ? ~0u : ((1u << ws.n_obs) - 1u);
    for (uint32_t rest = all & ~pruned; rest; rest &= rest - 1) {  // unpruned boxes, ascending
      const int o = __builtin_ctzll_hd(rest);
      ++n_prune;
      double dot = 0;
#pragma unroll
      for (int k = 0; k < DW; ++k) dot += d[k] * (cp[k][o * DW] - y[k]);
      if (!(dot < lim)) {
        pruned |= 1u << o;
        any = true;
      } else {
        const double q = sq[o * sq_stride];
        if (q < nsq) {
          nsq = q;
          nb = o;
        }
      }
    }
    if (!any) return -1;
    double a[DW];
    bool fb = false;
    const double vn = sqrt(sqnorm<DW>(yd));
    if (vn < 1e-6) {
      fb = true;
    } else {
      double dy = 0.0;
#pragma unroll
      for (int k = 0; k < DW; ++k) dy = dy + d[k] * yd[k];
      const double coef = dy / sqnorm<DW>(yd);
#pragma unroll
      for (int k = 0; k < DW; ++k) a[k] = d[k] - coef * yd[k];
      if (sqrt(sqnorm<DW>(a)) < 1e-6 * sqrt(sqnorm<DW>(d))) fb = true;
    }
    if (fb) {
#pragma unroll
      for (int k = 0; k < DW; ++k) a[k] = d[k];
    }
#pragma unroll
    for (int k = 0; k < DW; ++k) a_out[count * DW + k] = a[k];
    b_out[count] = sqnorm<DW>(a);
    fb_out[count] = fb ? 1 : 0;
    ++count;
    best = nb;
  }
  return count;
}

// convex_region for any number of boxes (<= 32 * kW) with no per-box storage:
// the fused scheme above (one pass per iteration over the still-unpruned
// boxes, ascending, pruning with the half-space of this iteration and
// tracking the first strict minimum of |clamp(y) - y|^2 among the boxes that
// survive it), with the squared distance recomputed on the fly instead of
// kept, so forests of hundreds of boxes need neither shared memory per
// waypoint nor a pass over pruned boxes.  Each iteration prunes at least one
// box (else -1, the reference's no-progress throw), so the reference's
// n_obs-iteration cap never binds before every box is pruned.  Output
// identical to convex_region (the same distance and prune expressions; the
// minimizing-corner choice is the one convex_region_fused documents).
template <int DW>
__host__ __device__ __forceinline__ double clamp_sq(const WorldD& ws, int o, const double* y) {
  double cand[DW];
#pragma unroll
  for (int k = 0; k < DW; ++k) {
    double c = y[k] < ws.lo[o * DW + k] ? ws.lo[o * DW + k] : y[k];
    c = ws.hi[o * DW + k] < c ? ws.hi[o * DW + k] : c;
    cand[k] = c - y[k];
  }
  return sqnorm<DW>(cand);
}

//
// The counters report the work of the reference's loop (geom.hpp:189-225): a
// distance per unpruned box per nearest search, a prune test per unpruned box
// per iteration.
//
// lbs (optional, per warp): lbs[o] <= a lower bound of box o's squared
// distance to every waypoint of the warp, shrunk by 2e-9 relative and rounded
// down to binary32 (a float compared as a double: exact), and ub >=
// the squared distance from any of them to its nearest box.  A box with
// lbs[o] > ub (first search) or lbs[o] > the best squared distance found so
// far (later searches) has a computed |clamp(y) - y|^2 strictly larger than
// the current best (the margin covers every rounding on both sides), so it
// can neither win nor tie and its distance is not evaluated.
//
// BoxOrder (optional, per warp, with lbs): the boxes in 32 buckets of
// ascending lbs (a monotone bucket map, so every bound of a later bucket is
// >= every bound of an earlier one), each bucket's smallest bound.  The
// nearest searches then visit the boxes bucket by bucket and stop at the
// first bucket whose smallest bound exceeds the best distance so far; ties
// are broken by the lower box index explicitly, so the winner is the
// reference's first strict minimum in index order.
#ifndef PUMP_BUCKET_NEAR
#define PUMP_BUCKET_NEAR 0
#endif
constexpr bool kBucketNear = PUMP_BUCKET_NEAR;  // bucketed later searches: measured slower (they visit pruned boxes)
struct BoxOrder {
  const uint16_t* order;  // n_obs box indices, bucket-major
  const int* start;       // 33 bucket offsets into order
  const float* bmin;      // 32 smallest bounds (+inf: empty)
};

template <int DW, int kW>
__device__ __forceinline__ int convex_region_scan(const WorldD& ws, const double* y, const double* yd, double* a_out,
                                                  double* b_out, uint8_t* fb_out, int a_stride, int b_stride,
                                                  int out_cap, unsigned& n_clamp, unsigned& n_prune,
                                                  const float* lbs = nullptr, double ub = 0.0,
                                                  const BoxOrder* bo = nullptr) {
  n_clamp += ws.n_obs;
  int best = -1;
  double best_sq = __builtin_inf();
  if (bo) {
    for (int bk = 0; bk < 32; ++bk) {
      const int s0 = bo->start[bk], s1 = bo->start[bk + 1];
      if (s0 == s1) continue;
      if (bo->bmin[bk] > (best_sq < ub ? best_sq : ub)) break;
      for (int x = s0; x < s1; ++x) {
        const int o = bo->order[x];
        if (lbs[o] > (best_sq < ub ? best_sq : ub)) continue;
        const double q = clamp_sq<DW>(ws, o, y);
        if (q < best_sq || (q == best_sq && o < best)) {
          best_sq = q;
          best = o;
        }
      }
    }
  } else {
    for (int o = 0; o < ws.n_obs; ++o) {
      if (lbs && lbs[o] > ub) continue;  // warp-uniform
      const double q = clamp_sq<DW>(ws, o, y);
      if (q < best_sq) {
        best_sq = q;
        best = o;
      }
    }
  }
  uint32_t pruned[kW];
  for (int q = 0; q < (ws.n_obs + 31) / 32; ++q) {  // (only the words in use)
    const int lo = 32 * q;
    pruned[q] = ws.n_obs >= lo + 32 ? 0u : ~((1u << (ws.n_obs - lo)) - 1u);
  }
  int count = 0;
  while (best >= 0) {
    double d[DW];
#pragma unroll
    for (int k = 0; k < DW; ++k) {
      double c = y[k] < ws.lo[best * DW + k] ? ws.lo[best * DW + k] : y[k];
      c = ws.hi[best * DW + k] < c ? ws.hi[best * DW + k] : c;
      d[k] = c - y[k];
    }
    const double dd = sqnorm<DW>(d);
    const double lim = dd - 1e-12 * (1.0 + dd);
    bool any = false;
    int nb = -1;
    double nsq = __builtin_inf();
    const double* cp[DW];
#pragma unroll
    for (int k = 0; k < DW; ++k) cp[k] = (d[k] >= 0 ? ws.lo : ws.hi) + k;
    // prune pass, then the nearest search over the survivors: two loops
    // with no data-dependent branch inside (a warp's lanes prune different
    // boxes; one fused loop ran both paths on every trip)
    auto prune_word = [&](int q) {
      uint32_t kill = 0u;
      n_prune += __popc(~pruned[q]);
      for (uint32_t rest = ~pruned[q]; rest; rest &= rest - 1) {
        const int b = __builtin_ctzll_hd(rest);
        const int o = 32 * q + b;
        double dot = 0;
#pragma unroll
        for (int k = 0; k < DW; ++k) dot += d[k] * (cp[k][o * DW] - y[k]);
        kill |= (dot < lim ? 0u : 1u) << b;
      }
      pruned[q] |= kill;
      any = any || kill != 0u;
    };
    auto near_word = [&](int q) {
      n_clamp += __popc(~pruned[q]);
      for (uint32_t rest = ~pruned[q]; rest; rest &= rest - 1) {
        const int o = 32 * q + __builtin_ctzll_hd(rest);
        if (lbs && lbs[o] > nsq) continue;
        const double sq = clamp_sq<DW>(ws, o, y);
        nb = sq < nsq ? o : nb;
        nsq = sq < nsq ? sq : nsq;
      }
    };
    // one copy of each loop (the words in local memory): unrolled over 8
    // register words the kernel measured slower (2.04 vs 1.93 ms forest,
    // instruction-cache pressure)
    const int nw = (ws.n_obs + 31) / 32;
    for (int q = 0; q < nw; ++q) prune_word(q);
    if (kBucketNear && bo) {
      for (int q = 0; q < nw; ++q) n_clamp += __popc(~pruned[q]);
      for (int bk = 0; bk < 32; ++bk) {
        const int s0 = bo->start[bk], s1 = bo->start[bk + 1];
        if (s0 == s1) continue;
        if (bo->bmin[bk] > nsq) break;
        for (int x = s0; x < s1; ++x) {
          const int o = bo->order[x];
          if ((pruned[o >> 5] >> (o & 31)) & 1u) continue;
          if (lbs[o] > nsq) continue;
          const double sq = clamp_sq<DW>(ws, o, y);
          if (sq < nsq || (sq == nsq && o < nb)) {
            nb = o;
            nsq = sq;
          }
        }
      }
    } else {
      for (int q = 0; q < nw; ++q) near_word(q);
    }
    if (!any) return -1;
    if (count < out_cap) {
      double a[DW];
      bool fb = false;
      const double vn = sqrt(sqnorm<DW>(yd));
      if (vn < 1e-6) {
        fb = true;
      } else {
        double dy = 0.0;
#pragma unroll
        for (int k = 0; k < DW; ++k) dy = dy + d[k] * yd[k];
        const double coef = dy / sqnorm<DW>(yd);
#pragma unroll
        for (int k = 0; k < DW; ++k) a[k] = d[k] - coef * yd[k];
        if (sqrt(sqnorm<DW>(a)) < 1e-6 * sqrt(sqnorm<DW>(d))) fb = true;
      }
      if (fb) {
#pragma unroll
        for (int k = 0; k < DW; ++k) a[k] = d[k];
      }
#pragma unroll
      for (int k = 0; k < DW; ++k) a_out[count * a_stride + k] = a[k];
      b_out[count * b_stride] = sqnorm<DW>(a);
      fb_out[count] = fb ? 1 : 0;
    }
    ++count;
    best = nb;
  }
  return count;
}

// One (trajectory, step) row of the MC table path's candidate lists (a warp):
// the box of the step's nominal points y1 (and y0, the previous step's) widened
// by the table's largest deviations maxdev[t] (maxdev[t - 1]), the obstacles
// (widened by their margin) it meets listed in ascending order, up to kStepCap
// (more: nl = -1), and skip = the box lies strictly inside the bounds and meets
// no obstacle (no rollout of the table can hit in this step).  CAP = kStepCap.
template <int DW, int CAP>
__device__ __forceinline__ void mc_step_row(const WorldD& w, const double* y1, const double* y0,
                                            const unsigned long long* __restrict__ maxdev, int t, int64_t row,
                                            int lane, uint16_t* __restrict__ g_list, int32_t* __restrict__ g_nl,
                                            uint8_t* __restrict__ g_skip) {
  double bl[DW], bh[DW];
  bool inside = true;
#pragma unroll
  for (int k = 0; k < DW; ++k) {
    const double m1 = __longlong_as_double(static_cast<long long>(maxdev[t * DW + k]));
    double lo = y1[k] - m1, hi = y1[k] + m1;
    if (y0) {
      const double m0 = __longlong_as_double(static_cast<long long>(maxdev[(t - 1) * DW + k]));
      const double lo0 = y0[k] - m0, hi0 = y0[k] + m0;
      lo = lo0 < lo ? lo0 : lo;
      hi = hi0 > hi ? hi0 : hi;
    }
    const double mg = 1e-12 * (1.0 + (lo < 0 ? -lo : lo) + (hi < 0 ? -hi : hi));
    bl[k] = lo - mg;
    bh[k] = hi + mg;
    inside = inside && bl[k] > w.blo[k] && bh[k] < w.bhi[k];
  }
  int nl = 0;
  for (int o0 = 0; o0 < w.n_obs; o0 += 32) {
    const int o = o0 + lane;
    bool meet = false;
    if (o < w.n_obs) {
      bool sep = false;
#pragma unroll
      for (int k = 0; k < DW; ++k) {
        const double bl_o = w.blo[k] < 0 ? -w.blo[k] : w.blo[k], bh_o = w.bhi[k] < 0 ? -w.bhi[k] : w.bhi[k];
        const double lo = w.lo[o * DW + k], hi = w.hi[o * DW + k];
        const double M = 1e-9 * (1.0 + (lo < 0 ? -lo : lo) + (hi < 0 ? -hi : hi) + 2.0 * (bl_o > bh_o ? bl_o : bh_o));
        sep = sep || (bh[k] < lo - M) || (bl[k] > hi + M);
      }
      meet = !sep;
    }
    const unsigned bal = __ballot_sync(0xffffffffu, meet);
    const int at = nl + __popc(bal & ((1u << lane) - 1u));
    if (meet && at < CAP) g_list[row * CAP + at] = static_cast<uint16_t>(o);
    nl += __popc(bal);
  }
  if (nl > CAP) nl = -1;
  if (lane == 0) {
    g_nl[row] = nl;
    g_skip[row] = (inside && nl == 0) ? 1 : 0;
  }
}

// obstacle boxes staged in shared memory (block-wide; returns the view on them)
template <int DW>
__device__ __forceinline__ WorldD stage_world(const WorldD& w, double* smem) {
  double* lo = smem;
  double* hi = smem + w.n_obs * DW;
  for (int x = threadIdx.x; x < w.n_obs * DW; x += blockDim.x) {
    lo[x] = w.lo[x];
    hi[x] = w.hi[x];
  }
  __syncthreads();
  WorldD s = w;
  s.lo = lo;
  s.hi = hi;
  return s;
}

}  // namespace pumpg
