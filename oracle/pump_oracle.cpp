// ORACLE — TEST INFRASTRUCTURE ONLY (see pump_oracle.hpp header).
// CPU restatement of the PUMP reference hot path; built -O3 -std=c++20
// -ffp-contract=off like the reference's own -O3/no -march build.
#include "pump_oracle.hpp"

#include <algorithm>
#include <atomic>
#include <bit>
#include <chrono>
#include <cmath>
#include <exception>
#include <limits>
#include <mutex>
#include <stdexcept>
#include <thread>

#include "../paper_1607_06886_b200/csrc/common/pmath.h"

namespace oracle {

static std::atomic<int> g_mode{kPortable};
void set_normal_mode(int mode) { g_mode.store(mode); }
int normal_mode() { return g_mode.load(); }

// ------------------------------------------------------------ rng.hpp:8-56
std::uint64_t mix64(std::uint64_t x) {
  x ^= x >> 30;
  x *= 0xbf58476d1ce4e5b9ULL;
  x ^= x >> 27;
  x *= 0x94d049bb133111ebULL;
  x ^= x >> 31;
  return x;
}

std::uint64_t counter_hash(std::uint64_t seed, std::uint64_t a, std::uint64_t b, std::uint64_t c) {
  std::uint64_t h = mix64(seed + 0x9e3779b97f4a7c15ULL);  // rng.hpp:24
  h = mix64(h + a);
  h = mix64(h + b);
  return mix64(h + c);
}

double to_unit(std::uint64_t x) { return (static_cast<double>(x >> 11) + 1.0) * 0x1p-53; }  // rng.hpp:32-34

double uniform(std::uint64_t seed, std::uint64_t a, std::uint64_t b, std::uint64_t c) {
  return to_unit(counter_hash(seed, a, b, c));
}

// rng.hpp:43-49: Box-Muller on channels 2c and 2c+1.
double normal(std::uint64_t seed, std::uint64_t a, std::uint64_t b, std::uint64_t channel) {
  double u1 = to_unit(counter_hash(seed, a, b, 2 * channel));
  double u2 = to_unit(counter_hash(seed, a, b, 2 * channel + 1));
  const double two_pi = 2.0 * 3.14159265358979323846;
  if (g_mode.load(std::memory_order_relaxed) == kGlibc) return std::sqrt(-2.0 * std::log(u1)) * std::cos(two_pi * u2);
  return std::sqrt(-2.0 * pump_pm::plog(u1)) * pump_pm::pcos(two_pi * u2);
}

// parallel.hpp:15-43: chunked fork/join, first exception rethrown.
void parallel_for(std::size_t n, int workers, const std::function<void(std::size_t, std::size_t)>& chunk) {
  if (n == 0) return;
  if (workers < 1) workers = 1;
  std::size_t w = std::min<std::size_t>(workers, n);
  if (w <= 1) {
    chunk(0, n);
    return;
  }
  std::vector<std::thread> pool;
  std::exception_ptr err;
  std::mutex mu;
  std::size_t base = n / w, rem = n % w, lo = 0;
  for (std::size_t i = 0; i < w; ++i) {
    std::size_t hi = lo + base + (i < rem ? 1 : 0);
    pool.emplace_back([&, lo, hi] {
      try {
        chunk(lo, hi);
      } catch (...) {
        std::lock_guard<std::mutex> g(mu);
        if (!err) err = std::current_exception();
      }
    });
    lo = hi;
  }
  for (auto& t : pool) t.join();
  if (err) std::rethrow_exception(err);
}

// ----------------------------------------------------- small ordered math
// Eigen gemv row: c = 0; c = c + M_ij x_j, j ascending.
static inline double row_dot(const double* row, const double* x, int n) {
  double c = 0.0;
  for (int j = 0; j < n; ++j) c = c + row[j] * x[j];
  return c;
}
// y = M x for an r x n row-major block with leading dimension ld.
static inline void gemv(const double* M, int r, int n, int ld, const double* x, double* y) {
  for (int i = 0; i < r; ++i) y[i] = row_dot(M + static_cast<std::size_t>(i) * ld, x, n);
}
// sequential squaredNorm / dot for dw <= 3 (Eigen redux)
static inline double sqn(const double* x, int n) {
  double s = 0.0;
  for (int k = 0; k < n; ++k) s = s + x[k] * x[k];
  return s;
}
static inline double dotn(const double* x, const double* y, int n) {
  double s = 0.0;
  for (int k = 0; k < n; ++k) s = s + x[k] * y[k];
  return s;
}

// closed-loop step z <- F z + Gv (Sv nv) + Gw (Sw nw)   (lti.hpp:287, cp.hpp:254)
static inline void cl_step(const Loop& cl, double* z, const double* nv, const double* nw, double* tmp) {
  const int d = cl.d, dw = cl.dw, nz = 2 * d;
  double t1[12], t2[6];
  gemv(cl.Sv.data(), d, d, d, nv, t1);
  gemv(cl.Sw.data(), dw, dw, dw, nw, t2);
  for (int r = 0; r < nz; ++r) {
    double a = row_dot(cl.F.data() + static_cast<std::size_t>(r) * nz, z, nz);
    double b = row_dot(cl.Gv.data() + static_cast<std::size_t>(r) * d, t1, d);
    double c = row_dot(cl.Gw.data() + static_cast<std::size_t>(r) * dw, t2, dw);
    tmp[r] = (a + b) + c;
  }
  for (int r = 0; r < nz; ++r) z[r] = tmp[r];
}

// ------------------------------------------------- lti.hpp:257-292 (bank)
Bank presample_bank(const Loop& cl, int t_max, int n, std::uint64_t seed, int workers) {
  if (n < 1) throw std::invalid_argument("presample_bank: need at least one particle");
  if (t_max < 1) throw std::invalid_argument("presample_bank: horizon must be at least 1");
  const int d = cl.d, dw = cl.dw;
  Bank bank;
  bank.n = n;
  bank.horizon = t_max;
  bank.dw = dw;
  bank.seed = seed;
  bank.dy.assign(static_cast<std::size_t>(t_max + 1) * n * dw, 0.0);
  parallel_for(n, workers, [&](std::size_t lo, std::size_t hi) {
    double z[24], tmp[24], nv[12], nw[6], y[6];
    for (std::size_t i = lo; i < hi; ++i) {
      for (int k = 0; k < d; ++k) nv[k] = normal(seed, i, 0, kInitial + k);
      gemv(cl.S0.data(), d, d, d, nv, z);  // z.head(d) = S0 nv
      for (int k = d; k < 2 * d; ++k) z[k] = 0.0;
      for (int t = 0;; ++t) {
        gemv(cl.C.data(), dw, d, d, z, y);  // y = C z.head(d)
        double* slot = bank.dy.data() + (static_cast<std::size_t>(t) * n + i) * dw;
        for (int k = 0; k < dw; ++k) slot[k] = y[k];
        if (t == t_max) break;
        for (int k = 0; k < d; ++k) nv[k] = normal(seed, i, t, kProcess + k);
        for (int k = 0; k < dw; ++k) nw[k] = normal(seed, i, t + 1, kMeasurement + k);
        cl_step(cl, z, nv, nw, tmp);
      }
    }
  });
  return bank;
}

// --------------------------------------------------------- steer.hpp:63-212
double steer_cost(const St& a, const St& b, double tau) {  // steer.hpp:84-94
  double c = tau;
  const int n = static_cast<int>(a.p.size());
  for (int k = 0; k < n; ++k) {
    double dp = b.p[k] - a.p[k] - a.v[k] * tau;
    double dv = b.v[k] - a.v[k];
    c += 12 * dp * dp / (tau * tau * tau) - 12 * dp * dv / (tau * tau) + 4 * dv * dv / tau;
  }
  return c;
}

static void coeffs(const St& a, const St& b, double tau, Vec& acc0, Vec& jerk, double& effort) {  // :63-79
  const int n = static_cast<int>(a.p.size());
  acc0.assign(n, 0.0);
  jerk.assign(n, 0.0);
  effort = 0;
  for (int k = 0; k < n; ++k) {
    double dp = b.p[k] - a.p[k] - a.v[k] * tau;
    double dv = b.v[k] - a.v[k];
    acc0[k] = 6 * dp / (tau * tau) - 2 * dv / tau;
    jerk[k] = -12 * dp / (tau * tau * tau) + 6 * dv / (tau * tau);
    effort += 12 * dp * dp / (tau * tau * tau) - 12 * dp * dv / (tau * tau) + 4 * dv * dv / tau;
  }
}

Mot fixed_time_connect(const St& a, const St& b, double tau) {  // :97-107
  Mot m;
  m.from = a;
  m.to = b;
  m.tau = tau;
  m.ok = true;
  double effort;
  coeffs(a, b, tau, m.acc0, m.jerk, effort);
  m.cost = tau + effort;
  return m;
}

double scan_ratio(double tau_max) {  // steer.hpp:130-133
  const double tau_lo = tau_max * 1e-7;
  return std::pow(tau_max / tau_lo, 1.0 / (64 - 1));
}

Mot connect(const St& a, const St& b, double tau_max, double ratio) {  // steer.hpp:111-182
  if (a.p.size() != b.p.size()) throw std::invalid_argument("connect: dimension mismatch");
  Mot m;
  m.from = a;
  m.to = b;
  const int n = static_cast<int>(a.p.size());
  bool same = true;
  for (int k = 0; k < n; ++k)
    if (a.p[k] != b.p[k] || a.v[k] != b.v[k]) same = false;
  if (same) {
    m.ok = true;
    m.tau = 0;
    m.cost = 0;
    m.acc0.assign(n, 0.0);
    m.jerk.assign(n, 0.0);
    return m;
  }
  const int kScan = 64;
  const double tau_lo = tau_max * 1e-7;
  double best_tau = tau_lo, best_c = steer_cost(a, b, tau_lo);
  int best_idx = 0;
  double tau = tau_lo;
  for (int i = 1; i < kScan; ++i) {
    tau *= ratio;
    double c = steer_cost(a, b, tau);
    if (c < best_c) {
      best_c = c;
      best_tau = tau;
      best_idx = i;
    }
  }
  double lo = best_tau / (best_idx > 0 ? ratio : 1.0);
  double hi = std::min(best_tau * ratio, tau_max);
  const double gr = 0.5 * (std::sqrt(5.0) - 1.0);
  double x1 = hi - gr * (hi - lo), x2 = lo + gr * (hi - lo);
  double f1 = steer_cost(a, b, x1), f2 = steer_cost(a, b, x2);
  while (hi - lo > 1e-9 * hi) {
    if (f1 < f2) {
      hi = x2;
      x2 = x1;
      f2 = f1;
      x1 = hi - gr * (hi - lo);
      f1 = steer_cost(a, b, x1);
    } else {
      lo = x1;
      x1 = x2;
      f1 = f2;
      x2 = lo + gr * (hi - lo);
      f2 = steer_cost(a, b, x2);
    }
  }
  m.tau = 0.5 * (lo + hi);
  m.cost = steer_cost(a, b, m.tau);
  if (best_idx == kScan - 1 && m.tau > 0.999 * tau_max) {
    double eps = 1e-6 * tau_max;
    if (steer_cost(a, b, tau_max) <= steer_cost(a, b, tau_max - eps)) {
      m.ok = false;
      return m;
    }
  }
  double effort;
  coeffs(a, b, m.tau, m.acc0, m.jerk, effort);
  m.ok = true;
  return m;
}

St state_at(const Mot& m, double s) {  // steer.hpp:37-51
  if (s <= 0) return m.from;
  if (s >= m.tau) return m.to;
  const int n = static_cast<int>(m.from.p.size());
  St o;
  o.p.resize(n);
  o.v.resize(n);
  for (int k = 0; k < n; ++k) {
    double p0 = m.from.p[k], v0 = m.from.v[k], a = m.acc0[k], j = m.jerk[k];
    o.p[k] = p0 + v0 * s + a * s * s / 2 + j * s * s * s / 6;
    o.v[k] = v0 + a * s + j * s * s / 2;
  }
  return o;
}

Vec control_at(const Mot& m, double s) {  // steer.hpp:53-57
  const int n = static_cast<int>(m.from.p.size());
  if (m.tau <= 0) return Vec(n, 0.0);
  s = std::clamp(s, 0.0, m.tau);
  Vec u(n);
  for (int k = 0; k < n; ++k) u[k] = m.acc0[k] + m.jerk[k] * s;
  return u;
}

std::vector<Wp> waypoints(const Mot& m, double dt) {  // steer.hpp:192-212
  if (dt <= 0) throw std::invalid_argument("motion_waypoints: dt must be positive");
  std::vector<Wp> out;
  const int n = static_cast<int>(m.from.p.size());
  if (m.tau <= 0) {
    out.push_back({0.0, m.from, Vec(n, 0.0)});
    return out;
  }
  int k = static_cast<int>(std::floor(m.tau / dt + 1e-9));
  double rem = m.tau - k * dt;
  for (int i = 0; i <= k; ++i) {
    double t = i * dt;
    out.push_back({t, state_at(m, t), control_at(m, t)});
  }
  if (rem > 1e-9) {
    out.push_back({m.tau, m.to, control_at(m, m.tau)});
  } else {
    out.back().t = m.tau;
    out.back().s = m.to;
  }
  return out;
}

// ----------------------------------------------------------- geom.hpp:13-225
static inline bool box_contains(const double* lo, const double* hi, const double* p, int dw) {  // :19-23
  for (int k = 0; k < dw; ++k)
    if (p[k] < lo[k] || p[k] > hi[k]) return false;
  return true;
}

bool point_free(const World& w, const double* y) {  // :56-61
  if (!box_contains(w.blo.data(), w.bhi.data(), y, w.dw)) return false;
  for (int o = 0; o < w.n_obs; ++o)
    if (box_contains(w.olo.data() + o * w.dw, w.ohi.data() + o * w.dw, y, w.dw)) return false;
  return true;
}

bool segment_hits(const double* p0, const double* p1, const double* lo, const double* hi, int dw) {  // :64-80
  double tmin = 0.0, tmax = 1.0;
  for (int k = 0; k < dw; ++k) {
    double d = p1[k] - p0[k];
    if (std::abs(d) < 1e-300) {
      if (p0[k] < lo[k] || p0[k] > hi[k]) return false;
      continue;
    }
    double t0 = (lo[k] - p0[k]) / d;
    double t1 = (hi[k] - p0[k]) / d;
    if (t0 > t1) std::swap(t0, t1);
    tmin = std::max(tmin, t0);
    tmax = std::min(tmax, t1);
    if (tmin > tmax) return false;
  }
  return true;
}

bool segment_collides(const World& w, const double* p0, const double* p1) {  // :84-88
  for (int o = 0; o < w.n_obs; ++o)
    if (segment_hits(p0, p1, w.olo.data() + o * w.dw, w.ohi.data() + o * w.dw, w.dw)) return true;
  return false;
}

bool motion_collides(const World& w, const Mot& m, double eps_cc) {  // :96-123
  if (!m.ok) return true;
  const int dw = w.dw;
  Vec p0 = state_at(m, 0).p;
  if (!point_free(w, p0.data())) return true;
  if (m.tau <= 0) return false;
  Vec pT = state_at(m, m.tau).p;
  if (!point_free(w, pT.data())) return true;
  struct Span {
    double t0, t1;
    Vec a, b;
  };
  std::vector<Span> stack;
  stack.push_back({0.0, m.tau, p0, pT});
  while (!stack.empty()) {
    Span s = std::move(stack.back());
    stack.pop_back();
    double diff[6];
    for (int k = 0; k < dw; ++k) diff[k] = s.b[k] - s.a[k];
    if (std::sqrt(sqn(diff, dw)) <= eps_cc || s.t1 - s.t0 < 1e-9) {
      if (segment_collides(w, s.a.data(), s.b.data())) return true;
      continue;
    }
    double tm = 0.5 * (s.t0 + s.t1);
    Vec pm = state_at(m, tm).p;
    if (!point_free(w, pm.data())) return true;
    stack.push_back({s.t0, tm, s.a, pm});
    stack.push_back({tm, s.t1, std::move(pm), s.b});
  }
  return false;
}

Hs project_halfspace(const Vec& d, const Vec& ydot) {  // :163-183 (eps_v = eps_a = 1e-6)
  const int n = static_cast<int>(d.size());
  Hs h;
  double vn = std::sqrt(sqn(ydot.data(), n));
  if (vn < 1e-6) {
    h.a = d;
    h.b = sqn(d.data(), n);
    h.fallback = true;
    return h;
  }
  double coef = dotn(d.data(), ydot.data(), n) / sqn(ydot.data(), n);
  Vec a(n);
  for (int k = 0; k < n; ++k) a[k] = d[k] - coef * ydot[k];
  if (std::sqrt(sqn(a.data(), n)) < 1e-6 * std::sqrt(sqn(d.data(), n))) {
    h.a = d;
    h.b = sqn(d.data(), n);
    h.fallback = true;
    return h;
  }
  h.a = a;
  h.b = sqn(a.data(), n);
  return h;
}

Region local_convex_region(const World& w, const Vec& y, const Vec& ydot) {  // :189-225
  if (!point_free(w, y.data())) throw std::invalid_argument("local_convex_region: waypoint is in collision");
  const int dw = w.dw;
  Region reg;
  reg.center = y;
  std::vector<char> pruned(w.n_obs, 0);
  for (int iter = 0; iter < w.n_obs; ++iter) {
    // nearest_obstacle_vector (:128-142): first strict minimum of |clamp(y)-y|^2
    int best = -1;
    double best_sq = std::numeric_limits<double>::infinity();
    double dvec[6], cand[6];
    for (int o = 0; o < w.n_obs; ++o) {
      if (pruned[o]) continue;
      const double* lo = w.olo.data() + o * dw;
      const double* hi = w.ohi.data() + o * dw;
      for (int k = 0; k < dw; ++k) {
        double c = std::max(y[k], lo[k]);
        c = std::min(c, hi[k]);
        cand[k] = c - y[k];
      }
      double sq = sqn(cand, dw);
      if (sq < best_sq) {
        best_sq = sq;
        best = o;
        for (int k = 0; k < dw; ++k) dvec[k] = cand[k];
      }
    }
    if (best < 0) break;
    double dd = sqn(dvec, dw);
    double tol = 1e-12 * (1.0 + dd);
    bool any = false;
    for (int o = 0; o < w.n_obs; ++o) {
      if (pruned[o]) continue;
      const double* lo = w.olo.data() + o * dw;
      const double* hi = w.ohi.data() + o * dw;
      bool inside = true;
      for (unsigned corner = 0; corner < (1u << dw) && inside; ++corner) {
        double dot = 0;
        for (int k = 0; k < dw; ++k) {
          double c = (corner >> k) & 1 ? hi[k] : lo[k];
          dot += dvec[k] * (c - y[k]);
        }
        if (dot < dd - tol) inside = false;
      }
      if (inside) {
        pruned[o] = 1;
        any = true;
      }
    }
    if (!any) throw std::runtime_error("local_convex_region: pruning loop failed to make progress");
    reg.hs.push_back(project_halfspace(Vec(dvec, dvec + dw), ydot));
  }
  return reg;
}

// ------------------------------------------------------------ cp.hpp:20-43
Mask Mask::full(int n) {
  Mask m;
  m.n = n;
  m.w.assign((n + 63) / 64, ~0ULL);
  if (n % 64) m.w.back() = (1ULL << (n % 64)) - 1;
  return m;
}
int Mask::popcount() const {
  int c = 0;
  for (auto x : w) c += std::popcount(x);
  return c;
}
double Mask::cp() const { return 1.0 - static_cast<double>(popcount()) / n; }

// cp.hpp:180-208
std::pair<Mask, double> hsmc_extend(const Mask& mask, const Bank& bank,
                                    const std::vector<std::pair<int, const Region*>>& steps) {
  Mask out = mask;
  const int dw = bank.dw;
  for (const auto& [t, region] : steps) {
    if (t < 0 || t > bank.horizon) throw std::out_of_range("hsmc_extend: plan exceeds bank horizon");
    if (!region || region->hs.empty()) continue;
    const double* row = bank.dy.data() + static_cast<std::size_t>(t) * bank.n * dw;
    for (const auto& h : region->hs) {
      for (std::size_t wi = 0; wi < out.w.size(); ++wi) {
        std::uint64_t word = out.w[wi];
        while (word) {
          int bit = std::countr_zero(word);
          word &= word - 1;
          const double* p = row + (wi * 64 + bit) * static_cast<std::size_t>(dw);
          double s = 0;
          for (int k = 0; k < dw; ++k) s += h.a[k] * p[k];
          if (s > h.b) out.w[wi] &= ~(1ULL << bit);
        }
      }
    }
  }
  return {out, out.cp()};
}

// cp.hpp:214-268 — returns the number of colliding rollouts in [r0, r1)
long mc_hits(const std::vector<Vec>& y_nom, const Loop& cl, const World& w, long r0, long r1, std::uint64_t seed,
             double eps_cc, int workers, std::vector<char>* flags) {
  if (y_nom.empty()) throw std::invalid_argument("mc_certify: empty trajectory");
  const int d = cl.d, dw = cl.dw;
  const int T = static_cast<int>(y_nom.size()) - 1;
  const long n = r1 - r0;
  std::vector<char> hit(std::max(0L, n), 0);
  parallel_for(std::max(0L, n), workers, [&](std::size_t lo, std::size_t hi) {
    double z[24], tmp[24], nv[12], nw[6], y[6], prev[6], p0[6], p1[6], cz[6];
    for (std::size_t li = lo; li < hi; ++li) {
      const std::uint64_t i = static_cast<std::uint64_t>(r0) + li;
      for (int k = 0; k < d; ++k) nv[k] = normal(seed, i, 0, kInitial + k);
      gemv(cl.S0.data(), d, d, d, nv, z);
      for (int k = d; k < 2 * d; ++k) z[k] = 0.0;
      bool collided = false;
      for (int t = 0; t <= T && !collided; ++t) {
        gemv(cl.C.data(), dw, d, d, z, cz);
        for (int k = 0; k < dw; ++k) y[k] = y_nom[t][k] + cz[k];
        if (!point_free(w, y)) {
          collided = true;
          break;
        }
        if (t > 0) {
          double diff[6];
          for (int k = 0; k < dw; ++k) diff[k] = y[k] - prev[k];
          double len = std::sqrt(sqn(diff, dw));
          int segs = std::max(1, static_cast<int>(std::ceil(len / std::max(eps_cc, 1e-12))));
          for (int k = 0; k < dw; ++k) p0[k] = prev[k];
          for (int s2 = 1; s2 <= segs && !collided; ++s2) {
            double f = static_cast<double>(s2) / segs;
            for (int k = 0; k < dw; ++k) p1[k] = prev[k] + (y[k] - prev[k]) * f;
            if (!point_free(w, p1) || segment_collides(w, p0, p1)) collided = true;
            for (int k = 0; k < dw; ++k) p0[k] = p1[k];
          }
        }
        for (int k = 0; k < dw; ++k) prev[k] = y[k];
        if (t < T) {
          for (int k = 0; k < d; ++k) nv[k] = normal(seed, i, t, kProcess + k);
          for (int k = 0; k < dw; ++k) nw[k] = normal(seed, i, t + 1, kMeasurement + k);
          cl_step(cl, z, nv, nw, tmp);
        }
      }
      hit[li] = collided ? 1 : 0;
    }
  });
  long n_hit = 0;
  for (char h : hit) n_hit += h;
  if (flags) *flags = std::move(hit);
  return n_hit;
}

// ------------------------------------------------------------ sample.hpp
double halton(std::uint64_t index, int base) {  // :12-20
  double f = 1.0, r = 0.0;
  while (index > 0) {
    f /= base;
    r += f * (index % base);
    index /= base;
  }
  return r;
}

bool goal_contains(const Goal& g, const St& s) {  // :26-28
  const int n = static_cast<int>(s.p.size());
  return box_contains(g.lo.data(), g.hi.data(), s.p.data(), n) && std::sqrt(sqn(s.v.data(), n)) <= g.max_speed;
}

static const int kPrimes[] = {2, 3, 5, 7, 11, 13, 17, 19, 23, 29, 31, 37};

static St halton_state(std::uint64_t index, const double* lo, const double* hi, int dw, double max_speed) {  // :35-48
  St s;
  s.p.resize(dw);
  s.v.resize(dw);
  for (int k = 0; k < dw; ++k) {
    double u = halton(index, kPrimes[k]);
    s.p[k] = lo[k] + u * (hi[k] - lo[k]);
    double v = halton(index, kPrimes[dw + k]);
    s.v[k] = -max_speed + v * 2 * max_speed;
  }
  return s;
}

std::vector<St> sample_free(int n, const World& w, double max_speed, const Goal& goal) {  // :56-89
  if (n < 1) throw std::invalid_argument("sample_free: n must be at least 1");
  std::vector<St> out;
  bool have_goal = false;
  std::uint64_t index = 1;
  while (static_cast<int>(out.size()) < n) {
    St s = halton_state(index++, w.blo.data(), w.bhi.data(), w.dw, max_speed);
    if (!point_free(w, s.p.data())) continue;
    have_goal = have_goal || goal_contains(goal, s);
    out.push_back(std::move(s));
  }
  if (!have_goal) {
    St c;
    c.p.resize(w.dw);
    c.v.assign(w.dw, 0.0);
    for (int k = 0; k < w.dw; ++k) c.p[k] = 0.5 * (goal.lo[k] + goal.hi[k]);
    if (point_free(w, c.p.data())) {
      out.push_back(std::move(c));
    } else {
      bool placed = false;
      for (std::uint64_t gi = 1; gi <= 100000 && !placed; ++gi) {
        St s = halton_state(gi, goal.lo.data(), goal.hi.data(), w.dw, goal.max_speed);
        if (std::sqrt(sqn(s.v.data(), w.dw)) > goal.max_speed) continue;
        if (!point_free(w, s.p.data())) continue;
        out.push_back(std::move(s));
        placed = true;
      }
      if (!placed) throw std::runtime_error("sample_free: goal region appears entirely in collision");
    }
  }
  return out;
}

// ------------------------------------------------------------ graph.hpp:50-95
Graph build_graph(std::vector<St> nodes, const World& w, const Goal& goal, double r_n, double dt, double eps_cc,
                  double tau_max, int workers) {
  if (r_n <= 0) throw std::invalid_argument("build_graph: r_n must be positive");
  Graph g;
  g.nodes = std::move(nodes);
  g.r_n = r_n;
  g.dt = dt;
  const int n = static_cast<int>(g.nodes.size());
  const int dw = w.dw;
  g.adj.resize(n);
  for (int i = 0; i < n; ++i)
    if (goal_contains(goal, g.nodes[i])) g.goal_nodes.push_back(i);
  const double ratio = scan_ratio(tau_max);
  parallel_for(n, workers, [&](std::size_t lo, std::size_t hi) {
    for (std::size_t v = lo; v < hi; ++v) {
      const St& a = g.nodes[v];
      for (int u = 0; u < n; ++u) {
        if (u == static_cast<int>(v)) continue;
        const St& b = g.nodes[u];
        double dvel[6];
        for (int k = 0; k < dw; ++k) dvel[k] = b.v[k] - a.v[k];
        if (2.0 * std::sqrt(sqn(dvel, dw)) >= r_n) continue;
        Mot m = connect(a, b, tau_max, ratio);
        if (!m.ok || m.cost >= r_n || m.tau <= 0) continue;
        if (motion_collides(w, m, eps_cc)) continue;
        auto wps = waypoints(m, dt);
        Edge e;
        e.to = u;
        e.n_steps = static_cast<int>(wps.size()) - 1;
        bool valid = true;
        for (std::size_t j = 1; j < wps.size(); ++j) {
          if (!point_free(w, wps[j].s.p.data())) {
            valid = false;
            break;
          }
          e.regions.push_back(local_convex_region(w, wps[j].s.p, wps[j].s.v));
        }
        if (!valid) continue;
        e.m = std::move(m);
        g.adj[v].push_back(std::move(e));
      }
    }
  });
  return g;
}

// ------------------------------------------------------ planner.hpp:74-267
static inline bool dominates(double dc, double dcp, double c, double cp) { return c > dc && cp >= dcp; }  // :58-60

ExResult explore(const Graph& g, const Bank& bank, const ExParams& prm, const Hook& hook) {
  ExResult res;
  const int n = static_cast<int>(g.nodes.size());
  res.pareto.assign(n, {});
  std::vector<char> is_goal(n, 0);
  for (int v : g.goal_nodes) is_goal[v] = 1;
  const double width = prm.lambda * prm.r_n;
  std::vector<std::vector<int>> buckets;
  auto push_open = [&](int id, double cost) {  // :85-92
    int b = std::max(0, static_cast<int>(std::ceil(cost / width - 1e-12)));
    if (b >= static_cast<int>(buckets.size())) buckets.resize(b + 1);
    buckets[b].push_back(id);
  };
  double best_goal = std::numeric_limits<double>::infinity();
  auto note_goal = [&](const Plan& p) {  // :95-98
    if (is_goal[p.head] && p.cp < prm.alpha_min) best_goal = std::min(best_goal, p.cost);
  };
  res.plans.push_back({0, -1, 0.0, 0.0, 0, Mask::full(bank.n)});
  res.pareto[0].push_back(0);
  push_open(0, 0.0);
  note_goal(res.plans[0]);

  struct Cand {
    int source, head;
    double cost, cp;
    int t_end;
    Mask mask;
    bool keep;
  };
  std::vector<int> group{0};
  std::vector<char> is_open{0};
  long open_count = 1;
  int i = 0;
  buckets[0].clear();

  while (true) {
    if (!group.empty() && !std::isinf(best_goal)) {  // :126-133
      double mg = std::numeric_limits<double>::infinity();
      for (int id : group) mg = std::min(mg, res.plans[id].cost);
      if (best_goal <= mg) {
        res.termination = "goal_below_alpha_min";
        break;
      }
    }
    if (group.empty() && open_count == 0) {  // :134-138
      res.termination = std::isinf(best_goal) ? "frontier_exhausted" : "goal_below_alpha_min";
      break;
    }
    if (!group.empty()) {
      res.rounds++;
      std::vector<std::pair<int, int>> tasks;  // (plan, edge index)   :143-150
      for (int id : group)
        for (std::size_t e = 0; e < g.adj[res.plans[id].head].size(); ++e) tasks.push_back({id, static_cast<int>(e)});
      res.partial_plans += static_cast<long>(tasks.size());
      std::vector<Cand> cands(tasks.size());
      parallel_for(tasks.size(), prm.workers, [&](std::size_t lo, std::size_t hi) {  // :154-177
        std::vector<std::pair<int, const Region*>> steps;
        for (std::size_t ti = lo; ti < hi; ++ti) {
          const Plan& p = res.plans[tasks[ti].first];
          const Edge& e = g.adj[p.head][tasks[ti].second];
          Cand& c = cands[ti];
          c.source = tasks[ti].first;
          c.head = e.to;
          c.cost = p.cost + e.m.cost;
          c.t_end = p.t_end + e.n_steps;
          if (c.t_end > bank.horizon) {
            c.keep = false;
            c.cp = 2.0;
            continue;
          }
          steps.clear();
          for (int j = 0; j < e.n_steps; ++j) steps.push_back({p.t_end + j + 1, &e.regions[j]});
          auto [mask, cp] = hsmc_extend(p.mask, bank, steps);
          c.mask = std::move(mask);
          c.cp = cp;
          c.keep = cp < prm.alpha_max;
        }
      });
      const int first_fresh = static_cast<int>(res.plans.size());  // :180-196
      std::vector<int> fresh;
      for (auto& c : cands) {
        if (!c.keep) {
          if (c.cp > 1.5)
            res.discarded_horizon++;
          else
            res.discarded_cp++;
          continue;
        }
        int id = static_cast<int>(res.plans.size());
        res.plans.push_back({c.head, c.source, c.cost, c.cp, c.t_end, std::move(c.mask)});
        res.pareto[c.head].push_back(id);
        is_open.push_back(0);
        fresh.push_back(id);
        note_goal(res.plans[id]);
      }
      std::vector<char> drop(fresh.size(), 0);  // :200-211
      for (std::size_t fi = 0; fi < fresh.size(); ++fi) {
        const Plan& q = res.plans[fresh[fi]];
        for (int other : res.pareto[q.head]) {
          if (other == fresh[fi]) continue;
          const Plan& p = res.plans[other];
          if (dominates(p.cost, p.cp, q.cost, q.cp)) {
            drop[fi] = 1;
            break;
          }
        }
      }
      for (std::size_t fi = 0; fi < fresh.size(); ++fi) {  // :212-242
        auto& set = res.pareto[res.plans[fresh[fi]].head];
        if (drop[fi]) {
          set.erase(std::find(set.begin(), set.end(), fresh[fi]));
          res.removed_dominated++;
          continue;
        }
        const Plan& q = res.plans[fresh[fi]];
        for (std::size_t k = 0; k < set.size();) {
          int other = set[k];
          const Plan& p = res.plans[other];
          if (other < first_fresh && other != 0 && dominates(q.cost, q.cp, p.cost, p.cp)) {
            if (is_open[other]) {
              is_open[other] = 0;
              open_count--;
            }
            set.erase(set.begin() + k);
            res.removed_dominated++;
          } else {
            ++k;
          }
        }
        push_open(fresh[fi], q.cost);
        is_open[fresh[fi]] = 1;
        open_count++;
      }
      open_count -= static_cast<long>(group.size());
      if (hook) hook(res.rounds, res, group);
    }
    i++;  // :250-261
    group.clear();
    int limit = std::min(i, static_cast<int>(buckets.size()) - 1);
    for (int b = 0; b <= limit; ++b) {
      for (int id : buckets[b]) {
        if (!is_open[id]) continue;
        is_open[id] = 0;
        group.push_back(id);
      }
      buckets[b].clear();
    }
    if (group.empty() && open_count > 0) continue;
  }
  for (int v : g.goal_nodes)
    for (int id : res.pareto[v]) res.goal_plans.push_back(id);
  return res;
}

// ---------------------------------------------------- planner.hpp:270-330
std::vector<int> plan_path(const ExResult& r, int id) {
  std::vector<int> path;
  for (int x = id; x != -1; x = r.plans[x].parent) path.push_back(r.plans[x].head);
  std::reverse(path.begin(), path.end());
  return path;
}

std::vector<Wp> path_trajectory(const Graph& g, const std::vector<int>& path, double dt) {  // :292-315
  std::vector<Wp> traj;
  double offset = 0;
  for (std::size_t j = 0; j + 1 < path.size(); ++j) {
    const Edge* edge = nullptr;
    for (const auto& e : g.adj[path[j]])
      if (e.to == path[j + 1]) {
        edge = &e;
        break;
      }
    if (!edge) throw std::logic_error("path_trajectory: missing edge");
    auto wps = waypoints(edge->m, dt);
    for (std::size_t k = (j == 0 ? 0 : 1); k < wps.size(); ++k) {
      Wp wp = wps[k];
      wp.t += offset;
      traj.push_back(std::move(wp));
    }
    offset += edge->m.tau;
  }
  if (path.size() == 1) {
    const St& s = g.nodes[path[0]];
    traj.push_back({0.0, s, Vec(s.p.size(), 0.0)});
  }
  return traj;
}

double trajectory_cost(const std::vector<Wp>& traj) {  // :319-330
  double c = traj.empty() ? 0 : traj.back().t;
  for (std::size_t j = 0; j + 1 < traj.size(); ++j) {
    const auto& w0 = traj[j];
    const auto& w1 = traj[j + 1];
    const int n = static_cast<int>(w0.u.size());
    double h = w1.t - w0.t;
    double um[6];
    for (int k = 0; k < n; ++k) um[k] = 0.5 * (w0.u[k] + w1.u[k]);
    c += h / 6.0 * (sqn(w0.u.data(), n) + 4.0 * sqn(um, n) + sqn(w1.u.data(), n));
  }
  return c;
}

// ------------------------------------------------------------ pump.hpp
Selection bisect_select(const std::vector<int>& ids, const std::function<double(int)>& mc, double alpha) {  // :23-51
  Selection out;
  const int n = static_cast<int>(ids.size());
  if (n == 0) return out;
  std::vector<double> memo(n, -1.0);
  auto eval = [&](int m) {
    if (memo[m - 1] < 0) {
      memo[m - 1] = mc(ids[m - 1]);
      out.evals.push_back({ids[m - 1], memo[m - 1]});
    }
    return memo[m - 1];
  };
  int l = 1, u = n;
  while (l < u) {
    int m = (l + u + 1) / 2;
    if (eval(m) > alpha)
      u = m - 1;
    else
      l = m;
  }
  if (eval(l) > alpha) return out;
  out.success = true;
  out.plan_id = ids[l - 1];
  out.mc = memo[l - 1];
  return out;
}

bool nominal_free(const World& w, const std::vector<Wp>& traj, double eps_cc) {  // :64-75
  for (const auto& p : traj)
    if (!point_free(w, p.s.p.data())) return false;
  for (std::size_t j = 0; j + 1 < traj.size(); ++j) {
    double h = traj[j + 1].t - traj[j].t;
    if (h <= 0) continue;
    Mot seg = fixed_time_connect(traj[j].s, traj[j + 1].s, h);
    if (motion_collides(w, seg, eps_cc)) return false;
  }
  return true;
}

static std::vector<Vec> positions(const std::vector<Wp>& t) {
  std::vector<Vec> out;
  out.reserve(t.size());
  for (const auto& p : t) out.push_back(p.s.p);
  return out;
}

Smooth smooth(const std::vector<Wp>& plan, double plan_mc, double alpha, const Loop& cl, const World& w, int n_mc,
              std::uint64_t seed, double eps_cc, int workers) {  // :84-146
  Smooth best;
  best.traj = plan;
  best.cost = trajectory_cost(plan);
  best.mc = plan_mc;
  best.s = 0;
  if (plan.size() < 2) return best;
  const double total = plan.back().t;
  Mot opt = fixed_time_connect(plan.front().s, plan.back().s, total);
  const int n = static_cast<int>(plan.front().s.p.size());
  auto blend = [&](double s) {
    std::vector<Wp> t;
    t.reserve(plan.size());
    for (const auto& wp : plan) {
      Wp b;
      b.t = wp.t;
      St o = state_at(opt, wp.t);
      Vec ou = control_at(opt, wp.t);
      b.s.p.resize(n);
      b.s.v.resize(n);
      b.u.resize(n);
      for (int k = 0; k < n; ++k) {
        b.s.p[k] = (1 - s) * wp.s.p[k] + s * o.p[k];
        b.s.v[k] = (1 - s) * wp.s.v[k] + s * o.v[k];
        b.u[k] = (1 - s) * wp.u[k] + s * ou[k];
      }
      t.push_back(std::move(b));
    }
    return t;
  };
  auto certify = [&](const std::vector<Wp>& t, double& mc_out) {
    if (!nominal_free(w, t, eps_cc)) return false;
    mc_out = static_cast<double>(mc_hits(positions(t), cl, w, 0, n_mc, seed, eps_cc, workers)) / n_mc;
    return mc_out <= alpha;
  };
  auto accept = [&](double s, const std::vector<Wp>& t, double mc) {
    best.traj = t;
    best.cost = trajectory_cost(t);
    best.mc = mc;
    best.s = s;
  };
  {
    auto t = blend(1.0);
    double mc;
    if (certify(t, mc)) {
      accept(1.0, t, mc);
      return best;
    }
  }
  double lo = 0, hi = 1;
  for (int it = 0; it < 10; ++it) {
    double mid = 0.5 * (lo + hi);
    auto t = blend(mid);
    double mc;
    if (certify(t, mc)) {
      accept(mid, t, mc);
      lo = mid;
    } else {
      hi = mid;
    }
  }
  return best;
}

PumpOut run_pump(const PumpIn& in, int workers, const Graph* prebuilt) {  // pump.hpp:170-263
  using clk = std::chrono::steady_clock;
  auto secs = [](clk::time_point a, clk::time_point b) { return std::chrono::duration<double>(b - a).count(); };
  PumpOut res;
  auto t0 = clk::now();
  Graph local;
  const Graph* graph = prebuilt;
  if (!graph) {
    std::vector<St> nodes;
    nodes.push_back(in.x_init);
    for (auto& s : sample_free(in.samples, in.w, in.max_speed, in.goal)) nodes.push_back(std::move(s));
    local = build_graph(std::move(nodes), in.w, in.goal, in.r_n, in.dt, in.eps_cc, in.tau_max, workers);
    graph = &local;
  }
  auto t1 = clk::now();
  res.build_graph_seconds = secs(t0, t1);
  for (const auto& a : graph->adj) res.n_edges += static_cast<long>(a.size());

  Bank bank = presample_bank(in.cl, in.bank_horizon, in.particles, in.seed_bank, workers);
  ExParams ep;
  ep.alpha_min = in.alpha / in.eta;
  ep.alpha_max = std::min(1.0, in.eta * in.alpha);
  ep.lambda = in.lambda;
  ep.r_n = in.r_n;
  ep.workers = workers;
  ExResult ex = explore(*graph, bank, ep);
  auto t2 = clk::now();
  res.explore_seconds = secs(t1, t2);
  res.partial_plans = ex.partial_plans;
  res.termination = ex.termination;
  res.n_plans = static_cast<long>(ex.plans.size());

  // pump.hpp:212-235: global goal front, ascending cost / strictly falling cp_hat
  std::vector<int> sorted = ex.goal_plans;
  std::stable_sort(sorted.begin(), sorted.end(), [&](int a, int b) {
    const Plan& pa = ex.plans[a];
    const Plan& pb = ex.plans[b];
    if (pa.cost != pb.cost) return pa.cost < pb.cost;
    if (pa.cp != pb.cp) return pa.cp < pb.cp;
    return a < b;
  });
  std::vector<int> front;
  double min_cp = std::numeric_limits<double>::infinity();
  for (int id : sorted)
    if (ex.plans[id].cp < min_cp) {
      front.push_back(id);
      min_cp = ex.plans[id].cp;
    }
  for (int id : front) res.pareto.push_back({ex.plans[id].cost, ex.plans[id].cp});
  sorted.assign(front.rbegin(), front.rend());

  auto mc_of = [&](int id) {
    auto t = path_trajectory(*graph, plan_path(ex, id), in.dt);
    return static_cast<double>(mc_hits(positions(t), in.cl, in.w, 0, in.mc_samples, in.seed_mc, in.eps_cc, workers)) /
           in.mc_samples;
  };
  Selection sel = bisect_select(sorted, mc_of, in.alpha);
  res.mc_evals = sel.evals;
  if (!sel.success) {
    res.selection_seconds = secs(t2, clk::now());
    return res;
  }
  res.path = plan_path(ex, sel.plan_id);
  res.cp_hat = ex.plans[sel.plan_id].cp;
  auto plan_traj = path_trajectory(*graph, res.path, in.dt);
  res.pre_smoothing_cost = ex.plans[sel.plan_id].cost;
  Smooth sm = smooth(plan_traj, sel.mc, in.alpha, in.cl, in.w, in.mc_samples, in.seed_mc, in.eps_cc, workers);
  res.traj = std::move(sm.traj);
  res.cost = sm.cost;
  res.certified_cp = sm.mc;
  res.smoothing_s = sm.s;
  res.success = true;
  res.selection_seconds = secs(t2, clk::now());
  return res;
}

// ================================================================ rrt.hpp
// Accumulated cost of the prefix [0, s] of a motion (steer.hpp:214-225).
double motion_partial_cost(const Mot& m, double s) {
  if (s <= 0) return 0;
  s = std::min(s, m.tau);
  double c = s;
  for (std::size_t k = 0; k < m.acc0.size(); ++k) {
    const double a = m.acc0[k], j = m.jerk[k];
    c += a * a * s + a * j * s * s + j * j * s * s * s / 3;
  }
  return c;
}

// Prefix of a motion cut so its accumulated cost equals target_cost (:228-243).
Mot truncate_motion(const Mot& m, double target_cost) {
  if (!m.ok || m.cost <= target_cost) return m;
  double lo = 0, hi = m.tau;
  for (int it = 0; it < 60; ++it) {
    const double mid = 0.5 * (lo + hi);
    if (motion_partial_cost(m, mid) < target_cost)
      lo = mid;
    else
      hi = mid;
  }
  Mot out = m;
  out.tau = 0.5 * (lo + hi);
  out.to = state_at(m, out.tau);
  out.cost = motion_partial_cost(m, out.tau);
  return out;
}

namespace {
St rrt_sample(const RrtIn& in, std::uint64_t seed, std::uint64_t trial, std::uint64_t iter) {  // rrt.hpp:27-44
  const int dw = in.p.w.dw;
  St st;
  st.p.resize(dw);
  st.v.resize(dw);
  const double bias = uniform(seed, trial, iter, 0);
  const bool g = bias < in.goal_bias;
  const double* lo = g ? in.p.goal.lo.data() : in.p.w.blo.data();
  const double* hi = g ? in.p.goal.hi.data() : in.p.w.bhi.data();
  const double vmax = g ? in.p.goal.max_speed : in.p.max_speed;
  for (int k = 0; k < dw; ++k) {
    const double u = uniform(seed, trial, iter, 1 + k);
    st.p[k] = lo[k] + u * (hi[k] - lo[k]);
    const double v = uniform(seed, trial, iter, 1 + dw + k);
    st.v[k] = -vmax + v * 2 * vmax;
  }
  return st;
}

double sqn_diff(const Vec& a, const Vec& b) {  // Eigen squaredNorm of a - b: sequential from +0
  double s = 0;
  for (std::size_t k = 0; k < a.size(); ++k) {
    const double d = a[k] - b[k];
    s += d * d;
  }
  return s;
}
}  // namespace

// Goal-biased kinodynamic RRT, repeated independent trials (rrt.hpp:50-147).
RrtOut repeated_rrt(const RrtIn& in, int trials, double alpha, int n_mc, int workers) {
  if (trials < 1) throw std::invalid_argument("repeated_rrt: trials must be at least 1");
  const PumpIn& P = in.p;
  const int dw = P.w.dw;
  const double ratio = scan_ratio(P.tau_max);
  struct Node {
    St s;
    int parent = -1;
    Mot incoming;
  };
  struct Outcome {
    bool reached = false;
    std::vector<Wp> traj;
    double cost = 0;
  };
  std::vector<Outcome> outcomes(trials);
  parallel_for(trials, workers, [&](std::size_t lo, std::size_t hi) {
    for (std::size_t trial = lo; trial < hi; ++trial) {
      std::vector<Node> tree;
      tree.push_back({P.x_init, -1, {}});
      for (int iter = 0; iter < in.max_iterations; ++iter) {
        const St target = rrt_sample(in, in.seed_rrt, trial, iter);
        if (!point_free(P.w, target.p.data())) continue;
        int nearest = -1;
        double best_d = std::numeric_limits<double>::infinity();
        for (int ni = 0; ni < static_cast<int>(tree.size()); ++ni) {
          const double dist = sqn_diff(tree[ni].s.p, target.p) + sqn_diff(tree[ni].s.v, target.v);
          if (dist < best_d) {
            best_d = dist;
            nearest = ni;
          }
        }
        const Mot toward = connect(tree[nearest].s, target, P.tau_max, ratio);
        if (!toward.ok || toward.tau <= 0) continue;
        const Mot step = truncate_motion(toward, P.r_n);
        if (step.tau <= 0) continue;
        if (motion_collides(P.w, step, P.eps_cc)) continue;
        tree.push_back({step.to, nearest, step});
        if (goal_contains(P.goal, tree.back().s)) {
          std::vector<int> chain;
          for (int id = static_cast<int>(tree.size()) - 1; id != -1; id = tree[id].parent) chain.push_back(id);
          std::reverse(chain.begin(), chain.end());
          std::vector<Wp> traj;
          double offset = 0;
          for (std::size_t j = 0; j < chain.size(); ++j) {
            if (j == 0) {
              traj.push_back({0.0, tree[chain[0]].s, Vec(dw, 0.0)});
              continue;
            }
            auto wps = waypoints(tree[chain[j]].incoming, P.dt);
            for (std::size_t k = 1; k < wps.size(); ++k) {
              Wp wp = wps[k];
              wp.t += offset;
              traj.push_back(std::move(wp));
            }
            offset += tree[chain[j]].incoming.tau;
          }
          outcomes[trial].reached = true;
          outcomes[trial].cost = trajectory_cost(traj);
          outcomes[trial].traj = std::move(traj);
          break;
        }
      }
    }
  });
  RrtOut res;
  std::vector<int> reached;
  for (int t = 0; t < trials; ++t)
    if (outcomes[t].reached) reached.push_back(t);
  res.trials_reaching_goal = static_cast<int>(reached.size());
  std::stable_sort(reached.begin(), reached.end(),
                   [&](int a, int b) { return outcomes[a].cost < outcomes[b].cost; });
  for (int t : reached) {
    res.certification_attempts++;
    std::vector<Vec> pos;
    for (const auto& w : outcomes[t].traj) pos.push_back(w.s.p);
    const double mc = static_cast<double>(mc_hits(pos, P.cl, P.w, 0, n_mc, P.seed_mc, P.eps_cc, workers)) / n_mc;
    if (mc <= alpha) {
      res.success = true;
      res.traj = std::move(outcomes[t].traj);
      res.cost = outcomes[t].cost;
      res.certified_cp = mc;
      break;
    }
  }
  return res;
}

}  // namespace oracle
