// Drop-in C++ API of the PUMP reference (namespace pump, the public surface
// of /root/reference/proj/include/pump/*.hpp) implemented over the C ABI of
// libpump_gpu.so (include/pump_gpu.h).  The per-topic headers next to this
// file (rng.hpp, lti.hpp, steer.hpp, geom.hpp, cp.hpp, sample.hpp, graph.hpp,
// planner.hpp, pump.hpp, scenario.hpp, report.hpp, parallel.hpp) keep the
// reference's include paths; all of them include this file.
//
// Build: g++ -std=c++20 -I<repo>/include [-I<repo>/include/compat when Eigen
// is absent] -I<nlohmann dir> app.cpp -L<repo>/paper_1607_06886_b200
// -lpump_gpu.  Hot loops run on the GPU of the
// thread's default context (device $PUMP_DEVICE, default 0); there is no CPU
// fallback.
//
// Differences from the reference, all documented in INTEGRATION.md:
//  - rng::normal uses the portable log/cos (pmath.h) the GPU kernels use, so
//    host draws equal device draws; rng::normal_glibc is the literal one.
//  - explore() does not support a RoundHook (throws std::logic_error).
#pragma once

#include <Eigen/Dense>
#include <unsupported/Eigen/MatrixFunctions>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstdlib>
#include <deque>
#include <exception>
#include <fstream>
#include <functional>
#include <limits>
#include <memory>
#include <stdexcept>
#include <string>
#include <thread>
#include <utility>
#include <vector>

#include "../../paper_1607_06886_b200/csrc/common/pmath.h"
#include "../../paper_1607_06886_b200/csrc/host/scenario.hpp"
#include "../pump_gpu.h"

namespace pump {

using Eigen::MatrixXd;
using Eigen::VectorXd;
using nlohmann::json;

// ======================================================== errors / context
using ScenarioError = pumpb::ScenarioError;

namespace detail {

[[noreturn]] inline void raise(int rc) {
  const std::string msg = pump_last_error();
  switch (rc) {
    case PUMP_E_INVALID_ARGUMENT: throw std::invalid_argument(msg);
    case PUMP_E_OUT_OF_RANGE: throw std::out_of_range(msg);
    case PUMP_E_SCENARIO: throw ScenarioError(msg);
    case PUMP_E_LOGIC: throw std::logic_error(msg);
    default: throw std::runtime_error(msg);
  }
}
inline void check(int rc) {
  if (rc != PUMP_OK) raise(rc);
}

struct Context {
  pump_ctx* h = nullptr;
  Context() {
    const char* e = std::getenv("PUMP_DEVICE");
    check(pump_ctx_create(e ? std::atoi(e) : 0, &h));
  }
  ~Context() { pump_ctx_destroy(h); }
};
inline pump_ctx* ctx() {
  thread_local Context c;
  return c.h;
}

inline std::vector<double> row_major(const MatrixXd& m) {
  std::vector<double> o(static_cast<size_t>(m.rows() * m.cols()));
  for (Eigen::Index i = 0; i < m.rows(); ++i)
    for (Eigen::Index j = 0; j < m.cols(); ++j) o[static_cast<size_t>(i * m.cols() + j)] = m(i, j);
  return o;
}
inline MatrixXd from_row_major(const double* p, int r, int c) {
  MatrixXd m(r, c);
  for (int i = 0; i < r; ++i)
    for (int j = 0; j < c; ++j) m(i, j) = p[i * c + j];
  return m;
}
inline pumpb::la::Mat to_la(const MatrixXd& m) {
  pumpb::la::Mat o(static_cast<int>(m.rows()), static_cast<int>(m.cols()));
  for (Eigen::Index i = 0; i < m.rows(); ++i)
    for (Eigen::Index j = 0; j < m.cols(); ++j) o(static_cast<int>(i), static_cast<int>(j)) = m(i, j);
  return o;
}
inline MatrixXd from_la(const pumpb::la::Mat& m) {
  MatrixXd o(m.r, m.c);
  for (int i = 0; i < m.r; ++i)
    for (int j = 0; j < m.c; ++j) o(i, j) = m(i, j);
  return o;
}
inline VectorXd vec(const double* p, int n) {
  VectorXd v(n);
  for (int i = 0; i < n; ++i) v[i] = p[i];
  return v;
}
inline std::vector<double> std_vec(const VectorXd& v) {
  std::vector<double> o(static_cast<size_t>(v.size()));
  for (Eigen::Index i = 0; i < v.size(); ++i) o[static_cast<size_t>(i)] = v[i];
  return o;
}

}  // namespace detail

// =============================================================== rng.hpp
namespace rng {
inline std::uint64_t mix64(std::uint64_t x) {  // rng.hpp:8-15
  x ^= x >> 30;
  x *= 0xbf58476d1ce4e5b9ULL;
  x ^= x >> 27;
  x *= 0x94d049bb133111ebULL;
  return x ^ (x >> 31);
}
inline std::uint64_t counter_hash(std::uint64_t seed, std::uint64_t a, std::uint64_t b, std::uint64_t c) {
  std::uint64_t h = mix64(seed + 0x9e3779b97f4a7c15ULL);
  h = mix64(h + a);
  h = mix64(h + b);
  return mix64(h + c);
}
inline double to_unit(std::uint64_t x) { return (static_cast<double>(x >> 11) + 1.0) * 0x1p-53; }
inline double uniform(std::uint64_t seed, std::uint64_t a, std::uint64_t b, std::uint64_t c) {
  return to_unit(counter_hash(seed, a, b, c));
}
// the draw the GPU kernels make (portable log/cos, csrc/common/pmath.h)
inline double normal(std::uint64_t seed, std::uint64_t a, std::uint64_t b, std::uint64_t channel) {
  const double u1 = to_unit(counter_hash(seed, a, b, 2 * channel));
  const double u2 = to_unit(counter_hash(seed, a, b, 2 * channel + 1));
  return std::sqrt(-2.0 * pump_pm::plog(u1)) * pump_pm::pcos(2.0 * 3.14159265358979323846 * u2);
}
// the reference's draw with the host libm (rng.hpp:43-49)
inline double normal_glibc(std::uint64_t seed, std::uint64_t a, std::uint64_t b, std::uint64_t channel) {
  const double u1 = to_unit(counter_hash(seed, a, b, 2 * channel));
  const double u2 = to_unit(counter_hash(seed, a, b, 2 * channel + 1));
  return std::sqrt(-2.0 * std::log(u1)) * std::cos(2.0 * 3.14159265358979323846 * u2);
}
enum Stream : std::uint64_t { kInitial = 0, kProcess = 1 << 20, kMeasurement = 2 << 20 };
}  // namespace rng

// ========================================================== parallel.hpp
// Host helper with the reference's contract (parallel.hpp:15-43): chunked
// fork/join over [0, n), first worker exception rethrown.
inline void parallel_for(std::size_t n, int workers, const std::function<void(std::size_t, std::size_t)>& chunk) {
  if (n == 0) return;
  const std::size_t w = std::min<std::size_t>(std::max(1, workers), n);
  if (w <= 1) return chunk(0, n);
  std::vector<std::thread> pool;
  std::exception_ptr err;
  std::mutex mu;
  std::size_t base = n / w, rem = n % w, lo = 0;
  for (std::size_t i = 0; i < w; ++i) {
    const std::size_t hi = lo + base + (i < rem ? 1 : 0);
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

// =============================================================== lti.hpp
struct ContinuousModel {
  MatrixXd A, B, C, V, W;
  int state_dim() const { return static_cast<int>(A.rows()); }
  int input_dim() const { return static_cast<int>(B.cols()); }
  int output_dim() const { return static_cast<int>(C.rows()); }
};
struct DiscreteModel {
  MatrixXd A, B, C, V, W;
  double dt = 0;
  int state_dim() const { return static_cast<int>(A.rows()); }
  int input_dim() const { return static_cast<int>(B.cols()); }
  int output_dim() const { return static_cast<int>(C.rows()); }
};
struct LqgWeights {
  MatrixXd Q, R, F;
};
struct GainSchedule {
  MatrixXd L, K, sigma0;
};
struct ClosedLoopDynamics {
  MatrixXd F, Gv, Gw, Sv, Sw, S0, C;
  int d = 0, dw = 0;
};

namespace detail {
inline pumpb::DiscreteModel to_b(const DiscreteModel& m) {
  pumpb::DiscreteModel o;
  o.A = to_la(m.A);
  o.B = to_la(m.B);
  o.C = to_la(m.C);
  o.V = to_la(m.V);
  o.W = to_la(m.W);
  o.dt = m.dt;
  return o;
}
inline DiscreteModel from_b(const pumpb::DiscreteModel& m) {
  return {from_la(m.A), from_la(m.B), from_la(m.C), from_la(m.V), from_la(m.W), m.dt};
}
inline ClosedLoopDynamics from_b(const pumpb::ClosedLoop& c) {
  ClosedLoopDynamics o;
  o.F = from_la(c.F);
  o.Gv = from_la(c.Gv);
  o.Gw = from_la(c.Gw);
  o.Sv = from_la(c.Sv);
  o.Sw = from_la(c.Sw);
  o.S0 = from_la(c.S0);
  o.C = from_la(c.C);
  o.d = c.d;
  o.dw = c.dw;
  return o;
}
// row-major storage kept alive next to the POD view
struct LoopView {
  std::vector<double> F, Gv, Gw, Sv, Sw, S0, C;
  pump_closed_loop v{};
  explicit LoopView(const ClosedLoopDynamics& cl)
      : F(row_major(cl.F)), Gv(row_major(cl.Gv)), Gw(row_major(cl.Gw)), Sv(row_major(cl.Sv)),
        Sw(row_major(cl.Sw)), S0(row_major(cl.S0)), C(row_major(cl.C)) {
    v = {cl.d, cl.dw, F.data(), Gv.data(), Gw.data(), Sv.data(), Sw.data(), S0.data(), C.data()};
  }
};
}  // namespace detail

inline DiscreteModel discretize(const ContinuousModel& cm, double dt) {  // lti.hpp:75-109
  pumpb::ContinuousModel c{detail::to_la(cm.A), detail::to_la(cm.B), detail::to_la(cm.C), detail::to_la(cm.V),
                           detail::to_la(cm.W)};
  return detail::from_b(pumpb::discretize(c, dt));
}
inline GainSchedule lqg_synthesize(const DiscreteModel& dm, const LqgWeights& w, const MatrixXd& sigma0) {
  pumpb::LqgWeights lw{detail::to_la(w.Q), detail::to_la(w.R), detail::to_la(w.F)};
  pumpb::GainSchedule g = pumpb::lqg_synthesize(detail::to_b(dm), lw, detail::to_la(sigma0));
  return {detail::from_la(g.L), detail::from_la(g.K), detail::from_la(g.sigma0)};
}
inline ClosedLoopDynamics closed_loop(const DiscreteModel& dm, const GainSchedule& gs, const MatrixXd& sigma0) {
  pumpb::GainSchedule g{detail::to_la(gs.L), detail::to_la(gs.K), detail::to_la(gs.sigma0)};
  return detail::from_b(pumpb::closed_loop(detail::to_b(dm), g, detail::to_la(sigma0)));
}
inline std::vector<MatrixXd> propagate_covariances(const DiscreteModel& dm, const GainSchedule& gs,
                                                   const MatrixXd& sigma0, int T) {
  pumpb::GainSchedule g{detail::to_la(gs.L), detail::to_la(gs.K), detail::to_la(gs.sigma0)};
  auto v = pumpb::propagate_covariances(pumpb::closed_loop(detail::to_b(dm), g, detail::to_la(sigma0)),
                                        detail::to_la(sigma0), T);
  std::vector<MatrixXd> o;
  for (const auto& m : v) o.push_back(detail::from_la(m));
  return o;
}

struct DeviationBank {  // lti.hpp:244-255
  int n_particles = 0, horizon = 0, dw = 0;
  std::uint64_t seed = 0;
  std::vector<double> dy;
  const double* at(int t) const { return dy.data() + static_cast<std::size_t>(t) * n_particles * dw; }
  double entry(int i, int t, int k) const { return dy[(static_cast<std::size_t>(t) * n_particles + i) * dw + k]; }
};

// presample_bank (lti.hpp:257-292) on the GPU; workers is accepted for
// signature compatibility (host threads are not used).
inline DeviationBank presample_bank(const DiscreteModel& dm, const GainSchedule& gs, const MatrixXd& sigma0,
                                    int t_max, int n, std::uint64_t seed, int workers = 1) {
  (void)workers;
  if (n < 1) throw std::invalid_argument("presample_bank: need at least one particle");
  if (t_max < 1) throw std::invalid_argument("presample_bank: horizon must be at least 1");
  ClosedLoopDynamics cl = closed_loop(dm, gs, sigma0);
  detail::LoopView lv(cl);
  DeviationBank b;
  b.n_particles = n;
  b.horizon = t_max;
  b.dw = cl.dw;
  b.seed = seed;
  b.dy.assign(static_cast<std::size_t>(t_max + 1) * n * cl.dw, 0.0);
  detail::check(pump_presample_bank(detail::ctx(), &lv.v, t_max, n, seed, b.dy.data()));
  return b;
}

// ============================================================= steer.hpp
struct State {
  VectorXd position, velocity;
  int dim() const { return static_cast<int>(position.size()); }
  static State make(std::initializer_list<double> p, std::initializer_list<double> v) {
    State s;
    s.position = detail::vec(std::data(p), static_cast<int>(p.size()));
    s.velocity = detail::vec(std::data(v), static_cast<int>(v.size()));
    return s;
  }
};

struct Motion {
  State from, to;
  double tau = 0, cost = 0;
  bool ok = false;
  VectorXd acc0, jerk;
  State state_at(double s) const {  // steer.hpp:37-51
    if (s <= 0) return from;
    if (s >= tau) return to;
    const int n = from.dim();
    State o;
    o.position = VectorXd(n);
    o.velocity = VectorXd(n);
    for (int k = 0; k < n; ++k) {
      const double p0 = from.position[k], v0 = from.velocity[k], a = acc0[k], j = jerk[k];
      o.position[k] = p0 + v0 * s + a * s * s / 2 + j * s * s * s / 6;
      o.velocity[k] = v0 + a * s + j * s * s / 2;
    }
    return o;
  }
  VectorXd control_at(double s) const {
    if (tau <= 0) return VectorXd::Zero(from.dim());
    s = std::clamp(s, 0.0, tau);
    VectorXd u(from.dim());
    for (int k = 0; k < from.dim(); ++k) u[k] = acc0[k] + jerk[k] * s;
    return u;
  }
};

inline double steer_cost(const State& a, const State& b, double tau) {
  return pump_steer_cost(a.dim(), a.position.data(), a.velocity.data(), b.position.data(), b.velocity.data(), tau);
}
inline Motion fixed_time_connect(const State& a, const State& b, double tau) {
  Motion m;
  m.from = a;
  m.to = b;
  m.tau = tau;
  m.ok = true;
  m.acc0 = VectorXd(a.dim());
  m.jerk = VectorXd(a.dim());
  detail::check(pump_fixed_time_connect(a.dim(), a.position.data(), a.velocity.data(), b.position.data(),
                                        b.velocity.data(), tau, &m.cost, m.acc0.data(), m.jerk.data()));
  return m;
}
inline Motion connect(const State& a, const State& b, double tau_max) {
  if (a.dim() != b.dim()) throw std::invalid_argument("connect: dimension mismatch");
  Motion m;
  m.from = a;
  m.to = b;
  m.acc0 = VectorXd::Zero(a.dim());
  m.jerk = VectorXd::Zero(a.dim());
  double out[3];
  detail::check(pump_connect(a.dim(), a.position.data(), a.velocity.data(), b.position.data(), b.velocity.data(),
                             tau_max, out, m.acc0.data(), m.jerk.data()));
  m.ok = out[0] != 0;
  m.tau = out[1];
  m.cost = out[2];
  return m;
}

struct Waypoint {
  double t = 0;
  State state;
  VectorXd control;
};
inline std::vector<Waypoint> motion_waypoints(const Motion& m, double dt) {  // steer.hpp:192-212
  if (dt <= 0) throw std::invalid_argument("motion_waypoints: dt must be positive");
  const int dw = m.from.dim();
  const int n = pump_waypoints(dw, m.from.position.data(), m.from.velocity.data(), m.to.position.data(),
                               m.to.velocity.data(), m.tau, m.acc0.data(), m.jerk.data(), dt, 0, nullptr, nullptr,
                               nullptr, nullptr);
  std::vector<double> t(n), p(static_cast<size_t>(n) * dw), v(p.size()), u(p.size());
  pump_waypoints(dw, m.from.position.data(), m.from.velocity.data(), m.to.position.data(), m.to.velocity.data(),
                 m.tau, m.acc0.data(), m.jerk.data(), dt, n, t.data(), p.data(), v.data(), u.data());
  std::vector<Waypoint> out(n);
  for (int i = 0; i < n; ++i) {
    out[i].t = t[i];
    out[i].state.position = detail::vec(p.data() + i * dw, dw);
    out[i].state.velocity = detail::vec(v.data() + i * dw, dw);
    out[i].control = detail::vec(u.data() + i * dw, dw);
  }
  return out;
}

// ============================================================== geom.hpp
struct Aabb {
  VectorXd lo, hi;
  int dim() const { return static_cast<int>(lo.size()); }
  bool contains(const VectorXd& p) const {
    for (int k = 0; k < dim(); ++k)
      if (p[k] < lo[k] || p[k] > hi[k]) return false;
    return true;
  }
  VectorXd clamp(const VectorXd& p) const { return p.cwiseMax(lo).cwiseMin(hi); }
  double shortest_edge() const { return (hi - lo).minCoeff(); }
  static Aabb make(std::initializer_list<double> l, std::initializer_list<double> h) {
    return {detail::vec(std::data(l), static_cast<int>(l.size())), detail::vec(std::data(h), static_cast<int>(h.size()))};
  }
};

struct Workspace {
  Aabb bounds;
  std::vector<Aabb> obstacles;
  int dim() const { return bounds.dim(); }
  double min_obstacle_edge() const {
    double e = bounds.shortest_edge();
    for (const auto& o : obstacles) e = std::min(e, o.shortest_edge());
    return e;
  }
};

namespace detail {
struct WsView {
  std::vector<double> blo, bhi, lo, hi;
  pump_workspace v{};
  explicit WsView(const Workspace& w) : blo(std_vec(w.bounds.lo)), bhi(std_vec(w.bounds.hi)) {
    for (const auto& o : w.obstacles) {
      auto a = std_vec(o.lo), b = std_vec(o.hi);
      lo.insert(lo.end(), a.begin(), a.end());
      hi.insert(hi.end(), b.begin(), b.end());
    }
    v = {w.dim(), static_cast<int32_t>(w.obstacles.size()), blo.data(), bhi.data(), lo.data(), hi.data()};
  }
};
}  // namespace detail

inline bool point_free(const Workspace& w, const VectorXd& y) {
  detail::WsView v(w);
  return pump_point_free(&v.v, y.data()) != 0;
}
inline bool segment_hits_aabb(const VectorXd& p0, const VectorXd& p1, const Aabb& box) {
  return pump_segment_hits_aabb(box.dim(), p0.data(), p1.data(), box.lo.data(), box.hi.data()) != 0;
}
inline bool motion_collides(const Workspace& w, const Motion& m, double eps_cc) {
  if (!m.ok) return true;
  detail::WsView v(w);
  int32_t hit = 0;
  detail::check(pump_motion_collides(&v.v, m.from.position.data(), m.from.velocity.data(), m.to.position.data(),
                                     m.to.velocity.data(), m.tau, m.acc0.data(), m.jerk.data(), eps_cc, &hit));
  return hit != 0;
}

struct HalfSpace {
  VectorXd a;
  double b = 0;
  bool fallback = false;
};
struct ConvexRegion {
  VectorXd center;
  std::vector<HalfSpace> halfspaces;
};
inline ConvexRegion local_convex_region(const Workspace& w, const VectorXd& y_nom, const VectorXd& ydot) {
  detail::WsView v(w);
  const int cap = static_cast<int>(w.obstacles.size()) + 1, dw = w.dim();
  std::vector<double> a(static_cast<size_t>(cap) * dw), b(cap);
  std::vector<uint8_t> fb(cap);
  int32_t n = 0;
  detail::check(pump_local_convex_region(&v.v, y_nom.data(), ydot.data(), cap, a.data(), b.data(), fb.data(), &n));
  ConvexRegion r;
  r.center = y_nom;
  for (int i = 0; i < n; ++i) r.halfspaces.push_back({detail::vec(a.data() + i * dw, dw), b[i], fb[i] != 0});
  return r;
}

// =============================================================== cp.hpp
struct ParticleMask {  // cp.hpp:20-43
  int n = 0;
  std::vector<std::uint64_t> words;
  static ParticleMask full(int n_particles) {
    ParticleMask m;
    m.n = n_particles;
    m.words.assign((n_particles + 63) / 64, ~0ULL);
    if (n_particles % 64) m.words.back() = (1ULL << (n_particles % 64)) - 1;
    return m;
  }
  bool alive(int i) const { return (words[i / 64] >> (i % 64)) & 1; }
  void kill(int i) { words[i / 64] &= ~(1ULL << (i % 64)); }
  int popcount() const {
    int c = 0;
    for (auto w : words) c += __builtin_popcountll(w);
    return c;
  }
  double cp() const { return 1.0 - static_cast<double>(popcount()) / n; }
};

struct CpEstimate {
  double value = 0;
  std::string method;
  int samples = 0;
};

struct HsmcStep {
  int t = 0;
  const ConvexRegion* region = nullptr;
};

namespace detail {
inline void ensure_bank(const DeviationBank& bank) {
  // the context keeps one resident bank; re-upload only when it changes
  thread_local const void* last = nullptr;
  thread_local std::size_t last_size = 0;
  thread_local std::uint64_t last_first = 0;
  std::uint64_t first = 0;
  if (!bank.dy.empty()) std::memcpy(&first, bank.dy.data(), 8);
  if (last != bank.dy.data() || last_size != bank.dy.size() || first != last_first) {
    check(pump_bank_upload(ctx(), bank.n_particles, bank.horizon, bank.dw, bank.dy.data()));
    last = bank.dy.data();
    last_size = bank.dy.size();
    last_first = first;
  }
}
}  // namespace detail

// hsmc_extend (cp.hpp:180-208) on the GPU
inline std::pair<ParticleMask, double> hsmc_extend(const ParticleMask& mask, const DeviationBank& bank,
                                                   const std::vector<HsmcStep>& steps) {
  detail::ensure_bank(bank);
  std::vector<int64_t> step_off{0, static_cast<int64_t>(steps.size())}, hs_off{0};
  std::vector<int32_t> step_t;
  std::vector<double> a, b;
  for (const auto& s : steps) {
    step_t.push_back(s.t);
    if (s.region)
      for (const auto& h : s.region->halfspaces) {
        for (int k = 0; k < bank.dw; ++k) a.push_back(h.a[k]);
        b.push_back(h.b);
      }
    hs_off.push_back(static_cast<int64_t>(b.size()));
  }
  a.push_back(0);
  b.push_back(0);
  step_t.push_back(0);
  ParticleMask out = mask;
  int32_t pop = 0;
  detail::check(pump_hsmc_extend_batch(detail::ctx(), 1, static_cast<int32_t>(mask.words.size()), mask.words.data(),
                                       step_off.data(), step_t.data(), hs_off.data(), a.data(), b.data(),
                                       out.words.data(), &pop));
  return {out, out.cp()};
}

// mc_certify (cp.hpp:214-268) on the GPU
inline CpEstimate mc_certify(const std::vector<VectorXd>& y_nom, const ClosedLoopDynamics& cl, const Workspace& w,
                             int n_mc, std::uint64_t seed, double eps_cc, int workers = 1) {
  (void)workers;
  if (n_mc < 1) throw std::invalid_argument("mc_certify: need at least one rollout");
  if (y_nom.empty()) throw std::invalid_argument("mc_certify: empty trajectory");
  detail::LoopView lv(cl);
  detail::WsView wv(w);
  std::vector<double> y;
  for (const auto& p : y_nom)
    for (int k = 0; k < cl.dw; ++k) y.push_back(p[k]);
  CpEstimate e;
  detail::check(pump_mc_certify(detail::ctx(), &lv.v, &wv.v, static_cast<int32_t>(y_nom.size()), y.data(), n_mc,
                                seed, eps_cc, &e.value));
  e.method = "mc";
  e.samples = n_mc;
  return e;
}

// ============================================================ sample.hpp
inline double halton(std::uint64_t index, int base) {
  double f = 1.0, r = 0.0;
  while (index > 0) {
    f /= base;
    r += f * (index % base);
    index /= base;
  }
  return r;
}
struct GoalRegion {
  Aabb box;
  double max_speed = 0;
  bool contains(const State& s) const { return box.contains(s.position) && s.velocity.norm() <= max_speed; }
};
inline std::vector<State> sample_free(int n, const Workspace& w, double max_speed, const GoalRegion& goal) {
  detail::WsView v(w);
  auto glo = detail::std_vec(goal.box.lo), ghi = detail::std_vec(goal.box.hi);
  pump_goal g{glo.data(), ghi.data(), goal.max_speed};
  const int dw = w.dim(), cap = n + 1;
  std::vector<double> p(static_cast<size_t>(cap) * dw), vel(p.size());
  int32_t got = 0;
  detail::check(pump_sample_free(n, &v.v, max_speed, &g, cap, p.data(), vel.data(), &got));
  std::vector<State> out(got);
  for (int i = 0; i < got; ++i) {
    out[i].position = detail::vec(p.data() + i * dw, dw);
    out[i].velocity = detail::vec(vel.data() + i * dw, dw);
  }
  return out;
}

// ============================================================= graph.hpp
struct Edge {
  int to = -1;
  Motion motion;
  int n_steps = 0;
  std::vector<ConvexRegion> regions;
};
struct SampleGraph {
  std::vector<State> nodes;
  std::vector<std::vector<Edge>> adj;
  std::vector<int> goal_nodes;
  double r_n = 0, dt = 0;
  std::size_t edge_count() const {
    std::size_t c = 0;
    for (const auto& a : adj) c += a.size();
    return c;
  }
};
inline double suggested_connection_radius(int n, int dw, const Workspace& w, double max_speed) {  // graph.hpp:41-48
  const double diag = (w.bounds.hi - w.bounds.lo).norm();
  const double travel = diag / std::max(max_speed, 1e-9);
  const double frac = std::pow(std::log(static_cast<double>(n) + 1.0) / (n + 1.0), 1.0 / (2.0 * dw));
  return 4.0 * travel * frac;
}

namespace detail {
struct GraphArrays {
  pump_graph_view v{};
  std::vector<double> pos, vel, cost, tau, acc0, jerk, ha, hb;
  std::vector<int64_t> row_ptr, wp_off, hs_off;
  std::vector<int32_t> to, nsteps, goal;
  std::vector<uint8_t> fb;
  void point() {
    v.node_pos = pos.data();
    v.node_vel = vel.data();
    v.row_ptr = row_ptr.data();
    v.edge_to = to.data();
    v.edge_cost = cost.data();
    v.edge_tau = tau.data();
    v.edge_acc0 = acc0.data();
    v.edge_jerk = jerk.data();
    v.edge_nsteps = nsteps.data();
    v.edge_wp_off = wp_off.data();
    v.wp_hs_off = hs_off.data();
    v.hs_a = ha.data();
    v.hs_b = hb.data();
    v.hs_fallback = fb.data();
    v.goal_nodes = goal.data();
  }
  void size_from(const pump_graph_view& c) {
    v = c;
    const size_t n = c.n_nodes, dw = c.dw, E = c.n_edges, W = c.n_waypoints, H = c.n_halfspaces;
    pos.assign(n * dw + 1, 0);
    vel.assign(n * dw + 1, 0);
    row_ptr.assign(n + 1, 0);
    to.assign(E + 1, 0);
    cost.assign(E + 1, 0);
    tau.assign(E + 1, 0);
    acc0.assign(E * dw + 1, 0);
    jerk.assign(E * dw + 1, 0);
    nsteps.assign(E + 1, 0);
    wp_off.assign(E + 1, 0);
    hs_off.assign(W + 1, 0);
    ha.assign(H * dw + 1, 0);
    hb.assign(H + 1, 0);
    fb.assign(H + 1, 0);
    goal.assign(c.n_goal + 1, 0);
    point();
  }
};

inline SampleGraph to_graph(const GraphArrays& g) {
  SampleGraph G;
  const int n = g.v.n_nodes, dw = g.v.dw;
  G.r_n = g.v.r_n;
  G.dt = g.v.dt;
  for (int i = 0; i < n; ++i) G.nodes.push_back({vec(g.pos.data() + i * dw, dw), vec(g.vel.data() + i * dw, dw)});
  G.adj.resize(n);
  for (int v = 0; v < n; ++v)
    for (int64_t e = g.row_ptr[v]; e < g.row_ptr[v + 1]; ++e) {
      Edge ed;
      ed.to = g.to[e];
      ed.motion.from = G.nodes[v];
      ed.motion.to = G.nodes[ed.to];
      ed.motion.tau = g.tau[e];
      ed.motion.cost = g.cost[e];
      ed.motion.ok = true;
      ed.motion.acc0 = vec(g.acc0.data() + e * dw, dw);
      ed.motion.jerk = vec(g.jerk.data() + e * dw, dw);
      ed.n_steps = g.nsteps[e];
      auto wps = motion_waypoints(ed.motion, G.dt);
      for (int64_t w = g.wp_off[e]; w < g.wp_off[e] + ed.n_steps; ++w) {
        ConvexRegion r;
        r.center = wps[static_cast<size_t>(w - g.wp_off[e] + 1)].state.position;
        for (int64_t h = g.hs_off[w]; h < g.hs_off[w + 1]; ++h)
          r.halfspaces.push_back({vec(g.ha.data() + h * dw, dw), g.hb[h], g.fb[h] != 0});
        ed.regions.push_back(std::move(r));
      }
      G.adj[v].push_back(std::move(ed));
    }
  G.goal_nodes.assign(g.goal.begin(), g.goal.begin() + g.v.n_goal);
  return G;
}

inline GraphArrays from_graph(const SampleGraph& G) {
  GraphArrays g;
  const int n = static_cast<int>(G.nodes.size()), dw = n ? G.nodes[0].dim() : 0;
  for (const auto& s : G.nodes) {
    for (int k = 0; k < dw; ++k) {
      g.pos.push_back(s.position[k]);
      g.vel.push_back(s.velocity[k]);
    }
  }
  g.row_ptr.push_back(0);
  g.wp_off.push_back(0);
  g.hs_off.push_back(0);
  for (const auto& row : G.adj) {
    for (const auto& e : row) {
      g.to.push_back(e.to);
      g.cost.push_back(e.motion.cost);
      g.tau.push_back(e.motion.tau);
      for (int k = 0; k < dw; ++k) {
        g.acc0.push_back(e.motion.acc0[k]);
        g.jerk.push_back(e.motion.jerk[k]);
      }
      g.nsteps.push_back(e.n_steps);
      for (const auto& r : e.regions) {
        for (const auto& h : r.halfspaces) {
          for (int k = 0; k < dw; ++k) g.ha.push_back(h.a[k]);
          g.hb.push_back(h.b);
          g.fb.push_back(h.fallback ? 1 : 0);
        }
        g.hs_off.push_back(static_cast<int64_t>(g.hb.size()));
      }
      g.wp_off.push_back(static_cast<int64_t>(g.hs_off.size() - 1));
    }
    g.row_ptr.push_back(static_cast<int64_t>(g.to.size()));
  }
  g.goal.assign(G.goal_nodes.begin(), G.goal_nodes.end());
  const int64_t E = static_cast<int64_t>(g.to.size()), W = static_cast<int64_t>(g.hs_off.size() - 1),
                H = static_cast<int64_t>(g.hb.size());
  for (auto* vv : {&g.pos, &g.vel, &g.cost, &g.tau, &g.acc0, &g.jerk, &g.ha, &g.hb}) vv->push_back(0);
  g.to.push_back(0);
  g.nsteps.push_back(0);
  g.fb.push_back(0);
  g.goal.push_back(0);
  g.point();
  g.v.n_nodes = n;
  g.v.dw = dw;
  g.v.n_edges = E;
  g.v.n_waypoints = W;
  g.v.n_halfspaces = H;
  g.v.n_goal = static_cast<int32_t>(G.goal_nodes.size());
  g.v.r_n = G.r_n;
  g.v.dt = G.dt;
  return g;
}

struct GraphHandle {
  pump_graph* h = nullptr;
  ~GraphHandle() {
    if (h) pump_graph_free(h);
  }
};
}  // namespace detail

// build_graph (graph.hpp:50-95) on the GPU, materialized on the host
inline SampleGraph build_graph(std::vector<State> nodes, const Workspace& w, const GoalRegion& goal, double r_n,
                               double dt, double eps_cc, double tau_max, int workers = 1) {
  (void)workers;
  if (r_n <= 0) throw std::invalid_argument("build_graph: r_n must be positive");
  const int n = static_cast<int>(nodes.size()), dw = w.dim();
  std::vector<double> pos, vel;
  for (const auto& s : nodes)
    for (int k = 0; k < dw; ++k) {
      pos.push_back(s.position[k]);
      vel.push_back(s.velocity[k]);
    }
  detail::WsView wv(w);
  auto glo = detail::std_vec(goal.box.lo), ghi = detail::std_vec(goal.box.hi);
  pump_goal g{glo.data(), ghi.data(), goal.max_speed};
  detail::GraphHandle gh;
  detail::check(pump_build_graph(detail::ctx(), n, dw, pos.data(), vel.data(), &wv.v, &g, r_n, dt, eps_cc, tau_max,
                                 &gh.h));
  pump_graph_view c{};
  detail::check(pump_graph_counts(gh.h, &c));
  detail::GraphArrays ga;
  ga.size_from(c);
  detail::check(pump_graph_export(gh.h, &ga.v));
  return detail::to_graph(ga);
}

// =========================================================== planner.hpp
struct PlanRec {
  int head = 0, parent = -1;
  double cost = 0, cp_hat = 0;
  int t_end = 0;
  ParticleMask mask;
};
struct ExploreParams {
  double alpha_min = 0, alpha_max = 1, lambda = 0.5, r_n = 1;
  int workers = 1;
};
struct ExploreStats {
  long partial_plans = 0;
  int rounds = 0;
  long discarded_cp = 0, removed_dominated = 0, discarded_horizon = 0;
  std::string termination;
};
struct ExploreResult {
  std::deque<PlanRec> plans;
  std::vector<std::vector<int>> pareto;
  std::vector<int> goal_plans;
  ExploreStats stats;
};
using RoundHook = std::function<void(int round, const ExploreResult& state, const std::vector<int>& expanded)>;

namespace detail {
inline bool dominates(double dom_cost, double dom_cp, double cost, double cp) {  // planner.hpp:58-60
  return cost > dom_cost && cp >= dom_cp;
}
}  // namespace detail

namespace detail {
// an explore handle's state as the reference's ExploreResult
inline ExploreResult materialize(const pump_explore* eh, int n_particles) {
  pump_explore_view v{};
  check(pump_explore_counts(eh, &v));
  std::vector<int32_t> head(v.n_plans + 1), parent(v.n_plans + 1), t_end(v.n_plans + 1), pids(v.n_pareto + 1),
      goal(v.n_goal_plans + 1);
  std::vector<double> cost(v.n_plans + 1), cp(v.n_plans + 1);
  std::vector<uint64_t> masks(static_cast<size_t>(v.n_plans) * v.n_words + 1);
  std::vector<int64_t> pptr(v.n_nodes + 1);
  v.head = head.data();
  v.parent = parent.data();
  v.cost = cost.data();
  v.cp_hat = cp.data();
  v.t_end = t_end.data();
  v.masks = masks.data();
  v.pareto_ptr = pptr.data();
  v.pareto_ids = pids.data();
  v.goal_plans = goal.data();
  check(pump_explore_export(eh, &v));
  ExploreResult r;
  for (int64_t i = 0; i < v.n_plans; ++i) {
    PlanRec p2{head[i], parent[i], cost[i], cp[i], t_end[i], {}};
    p2.mask.n = n_particles;
    p2.mask.words.assign(masks.begin() + i * v.n_words, masks.begin() + (i + 1) * v.n_words);
    r.plans.push_back(std::move(p2));
  }
  r.pareto.resize(v.n_nodes);
  for (int i = 0; i < v.n_nodes; ++i) r.pareto[i].assign(pids.begin() + pptr[i], pids.begin() + pptr[i + 1]);
  r.goal_plans.assign(goal.begin(), goal.begin() + v.n_goal_plans);
  r.stats = {v.partial_plans, v.rounds, v.discarded_cp, v.removed_dominated, v.discarded_horizon,
             v.termination ? "frontier_exhausted" : "goal_below_alpha_min"};
  return r;
}

struct HookCall {
  const RoundHook* hook;
  int n_particles;
  std::exception_ptr err;
};
inline int hook_trampoline(void* user, int32_t round, const pump_explore* state, const int32_t* expanded,
                           int64_t n_expanded) {
  auto* hc = static_cast<HookCall*>(user);
  try {
    ExploreResult st = materialize(state, hc->n_particles);
    st.stats.termination.clear();  // not decided yet when the reference's hook runs
    const std::vector<int> grp(expanded, expanded + n_expanded);
    (*hc->hook)(round, st, grp);
    return 0;
  } catch (...) {
    hc->err = std::current_exception();
    return 1;
  }
}
}  // namespace detail

// explore (planner.hpp:74-267): the wavefront runs on the GPU.  With a
// RoundHook the rounds run one at a time and the hook sees the state after
// every round (planner.hpp:245), materialized on the host.
inline ExploreResult explore(const SampleGraph& g, const DeviationBank& bank, const ExploreParams& params,
                             const RoundHook& hook = nullptr) {
  detail::ensure_bank(bank);
  detail::GraphArrays ga = detail::from_graph(g);
  detail::GraphHandle gh;
  detail::check(pump_graph_upload(detail::ctx(), &ga.v, &gh.h));
  pump_explore_params p{params.alpha_min, params.alpha_max, params.lambda, params.r_n};
  pump_explore* eh = nullptr;
  if (hook) {
    detail::HookCall hc{&hook, bank.n_particles, nullptr};
    const int rc = pump_explore_run_hooked(detail::ctx(), gh.h, &p, detail::hook_trampoline, &hc, &eh);
    if (hc.err) std::rethrow_exception(hc.err);
    detail::check(rc);
  } else {
    detail::check(pump_explore_run(detail::ctx(), gh.h, &p, &eh));
  }
  std::unique_ptr<pump_explore, int (*)(pump_explore*)> guard(eh, pump_explore_free);
  return detail::materialize(eh, bank.n_particles);
}

inline std::vector<int> plan_path(const ExploreResult& res, int plan_id) {  // planner.hpp:270-276
  std::vector<int> path;
  for (int id = plan_id; id != -1; id = res.plans[id].parent) path.push_back(res.plans[id].head);
  std::reverse(path.begin(), path.end());
  return path;
}

struct Trajectory {
  std::vector<Waypoint> points;
  double duration() const { return points.empty() ? 0 : points.back().t; }
  std::vector<VectorXd> positions() const {
    std::vector<VectorXd> out;
    for (const auto& p : points) out.push_back(p.state.position);
    return out;
  }
};

inline Trajectory path_trajectory(const SampleGraph& g, const std::vector<int>& path, double dt) {  // :292-315
  Trajectory traj;
  double offset = 0;
  for (std::size_t j = 0; j + 1 < path.size(); ++j) {
    const Edge* edge = nullptr;
    for (const auto& e : g.adj[path[j]])
      if (e.to == path[j + 1]) {
        edge = &e;
        break;
      }
    if (!edge) throw std::logic_error("path_trajectory: missing edge");
    auto wps = motion_waypoints(edge->motion, dt);
    for (std::size_t k = (j == 0 ? 0 : 1); k < wps.size(); ++k) {
      Waypoint wp = wps[k];
      wp.t += offset;
      traj.points.push_back(std::move(wp));
    }
    offset += edge->motion.tau;
  }
  if (path.size() == 1) traj.points.push_back({0.0, g.nodes[path[0]], VectorXd::Zero(g.nodes[path[0]].dim())});
  return traj;
}

inline double trajectory_cost(const Trajectory& traj) {  // planner.hpp:319-330
  double c = traj.duration();
  for (std::size_t j = 0; j + 1 < traj.points.size(); ++j) {
    const auto& w0 = traj.points[j];
    const auto& w1 = traj.points[j + 1];
    const double h = w1.t - w0.t;
    VectorXd um = 0.5 * (w0.control + w1.control);
    c += h / 6.0 * (w0.control.squaredNorm() + 4.0 * um.squaredNorm() + w1.control.squaredNorm());
  }
  return c;
}

// ============================================================== pump.hpp
struct SelectionOutcome {
  bool success = false;
  int plan_id = -1;
  double mc = 0;
  std::vector<std::pair<int, double>> mc_evals;
};

template <typename McFn>
SelectionOutcome bisect_select(const std::vector<int>& sorted_ids, McFn&& mc, double alpha) {  // pump.hpp:23-51
  SelectionOutcome out;
  const int n = static_cast<int>(sorted_ids.size());
  if (n == 0) return out;
  std::vector<double> memo(n, -1.0);
  auto eval = [&](int m) {
    if (memo[m - 1] < 0) {
      memo[m - 1] = mc(sorted_ids[m - 1]);
      out.mc_evals.push_back({sorted_ids[m - 1], memo[m - 1]});
    }
    return memo[m - 1];
  };
  int l = 1, u = n;
  while (l < u) {
    const int m = (l + u + 1) / 2;
    if (eval(m) > alpha)
      u = m - 1;
    else
      l = m;
  }
  if (eval(l) > alpha) return out;
  out.success = true;
  out.plan_id = sorted_ids[l - 1];
  out.mc = memo[l - 1];
  return out;
}

struct SmoothResult {
  Trajectory traj;
  double cost = 0, mc = 0, s = 0;
};

namespace detail {
inline bool nominal_free(const Workspace& w, const Trajectory& traj, double eps_cc) {  // pump.hpp:64-75
  for (const auto& p : traj.points)
    if (!point_free(w, p.state.position)) return false;
  for (std::size_t j = 0; j + 1 < traj.points.size(); ++j) {
    const double h = traj.points[j + 1].t - traj.points[j].t;
    if (h <= 0) continue;
    if (motion_collides(w, fixed_time_connect(traj.points[j].state, traj.points[j + 1].state, h), eps_cc)) return false;
  }
  return true;
}
}  // namespace detail

// smooth (pump.hpp:84-146) on the GPU: the same device chain run_pump uses
// (blend + nominal check + MC of each bisection probe in depth-2 speculative
// batches, one synchronisation; pump_smooth)
inline SmoothResult smooth(const Trajectory& plan_traj, double plan_mc, double alpha, const ClosedLoopDynamics& cl,
                           const Workspace& w, int n_mc, std::uint64_t mc_seed, double eps_cc, int workers = 1) {
  (void)workers;
  const int n = static_cast<int>(plan_traj.points.size()), dw = cl.dw;
  std::vector<double> t(n + 1), p(static_cast<size_t>(n) * dw + 1), v(p.size()), u(p.size());
  for (int q = 0; q < n; ++q) {
    const Waypoint& wp = plan_traj.points[q];
    t[q] = wp.t;
    for (int k = 0; k < dw; ++k) {
      p[q * dw + k] = wp.state.position[k];
      v[q * dw + k] = wp.state.velocity[k];
      u[q * dw + k] = wp.control[k];
    }
  }
  detail::LoopView lv(cl);
  detail::WsView wv(w);
  std::vector<double> op(p.size()), ov(p.size()), ou(p.size());
  double out3[3] = {0, 0, 0};
  detail::check(pump_smooth(detail::ctx(), &lv.v, &wv.v, n, t.data(), p.data(), v.data(), u.data(), plan_mc, alpha,
                            n_mc, mc_seed, eps_cc, op.data(), ov.data(), ou.data(), out3));
  SmoothResult r;
  for (int q = 0; q < n; ++q)
    r.traj.points.push_back({t[q], {detail::vec(op.data() + q * dw, dw), detail::vec(ov.data() + q * dw, dw)},
                             detail::vec(ou.data() + q * dw, dw)});
  r.cost = out3[0];
  r.mc = out3[1];
  r.s = out3[2];
  return r;
}

// ========================================================== scenario.hpp
struct Seeds {
  std::uint64_t bank = 1, mc = 2, rrt = 3;
};
struct RrtConfig {
  int trials = 1000, max_iterations = 200;
  double goal_bias = 0.05;
};

struct Scenario {  // scenario.hpp:34-77
  std::string name;
  Workspace workspace;
  State x_init;
  GoalRegion goal;
  MatrixXd process_noise, measurement_noise, initial_covariance;
  LqgWeights tracking;
  double dt = 0.1;
  int samples = 1000;
  double connection_radius = 0, alpha = 0.05, eta = 0, lambda = 0.5;
  int particles = 128, mc_samples = 10000, bank_horizon = 2048;
  double max_speed = 1.0, tau_max = 0, collision_resolution = 0;
  Seeds seeds;
  RrtConfig rrt;

  int workspace_dim() const { return workspace.dim(); }
  int state_dim() const { return 2 * workspace_dim(); }
  double effective_eta() const { return eta > 0 ? eta : (alpha >= 0.01 ? 2.0 : 10.0); }
  double effective_tau_max() const {
    if (tau_max > 0) return tau_max;
    return 10.0 * (workspace.bounds.hi - workspace.bounds.lo).norm() / std::max(max_speed, 1e-9);
  }
  double effective_eps_cc() const {
    return collision_resolution > 0 ? collision_resolution : workspace.min_obstacle_edge() / 100.0;
  }
  double effective_r_n() const {
    return connection_radius > 0 ? connection_radius
                                 : suggested_connection_radius(samples, workspace_dim(), workspace, max_speed);
  }
};

namespace detail {
inline Aabb box_of(const pumpb::Box& b) {
  return {vec(b.lo.data(), b.dim()), vec(b.hi.data(), b.dim())};
}
inline Scenario from_b(const pumpb::Scenario& s) {
  Scenario o;
  o.name = s.name;
  o.workspace.bounds = box_of(s.workspace.bounds);
  for (const auto& b : s.workspace.obstacles) o.workspace.obstacles.push_back(box_of(b));
  const int dw = s.workspace_dim();
  o.x_init = {vec(s.start_pos.data(), dw), vec(s.start_vel.data(), dw)};
  o.goal = {box_of(s.goal), s.goal_max_speed};
  o.process_noise = from_la(s.process_noise);
  o.measurement_noise = from_la(s.measurement_noise);
  o.initial_covariance = from_la(s.initial_covariance);
  o.tracking = {from_la(s.tracking.Q), from_la(s.tracking.R), from_la(s.tracking.F)};
  o.dt = s.dt;
  o.samples = s.samples;
  o.connection_radius = s.connection_radius;
  o.alpha = s.alpha;
  o.eta = s.eta;
  o.lambda = s.lambda;
  o.particles = s.particles;
  o.mc_samples = s.mc_samples;
  o.bank_horizon = s.bank_horizon;
  o.max_speed = s.max_speed;
  o.tau_max = s.tau_max;
  o.collision_resolution = s.collision_resolution;
  o.seeds = {s.seeds.bank, s.seeds.mc, s.seeds.rrt};
  o.rrt = {s.rrt.trials, s.rrt.max_iterations, s.rrt.goal_bias};
  return o;
}
inline json vjson(const VectorXd& v) {
  json a = json::array();
  for (Eigen::Index i = 0; i < v.size(); ++i) a.push_back(v[i]);
  return a;
}
inline json mjson(const MatrixXd& m) {
  json a = json::array();
  for (Eigen::Index i = 0; i < m.rows(); ++i) {
    json r = json::array();
    for (Eigen::Index j = 0; j < m.cols(); ++j) r.push_back(m(i, j));
    a.push_back(r);
  }
  return a;
}
// Scenario -> JSON in the reference schema (doubles round-trip exactly)
inline json to_json(const Scenario& s) {
  json obs = json::array();
  for (const auto& o : s.workspace.obstacles) obs.push_back({{"lo", vjson(o.lo)}, {"hi", vjson(o.hi)}});
  return {{"name", s.name},
          {"workspace", {{"bounds", {{"lo", vjson(s.workspace.bounds.lo)}, {"hi", vjson(s.workspace.bounds.hi)}}},
                         {"obstacles", obs}}},
          {"start", {{"position", vjson(s.x_init.position)}, {"velocity", vjson(s.x_init.velocity)}}},
          {"goal", {{"lo", vjson(s.goal.box.lo)}, {"hi", vjson(s.goal.box.hi)}, {"max_speed", s.goal.max_speed}}},
          {"noise", {{"process", mjson(s.process_noise)}, {"measurement", mjson(s.measurement_noise)},
                     {"initial", mjson(s.initial_covariance)}}},
          {"tracking", {{"Q", mjson(s.tracking.Q)}, {"R", mjson(s.tracking.R)}, {"F", mjson(s.tracking.F)}}},
          {"dt", s.dt}, {"samples", s.samples}, {"connection_radius", s.connection_radius}, {"alpha", s.alpha},
          {"eta", s.eta}, {"lambda", s.lambda}, {"particles", s.particles}, {"mc_samples", s.mc_samples},
          {"bank_horizon", s.bank_horizon}, {"max_speed", s.max_speed}, {"tau_max", s.tau_max},
          {"collision_resolution", s.collision_resolution},
          {"seeds", {{"bank", s.seeds.bank}, {"mc", s.seeds.mc}, {"rrt", s.seeds.rrt}}},
          {"rrt", {{"trials", s.rrt.trials}, {"max_iterations", s.rrt.max_iterations},
                   {"goal_bias", s.rrt.goal_bias}}}};
}
}  // namespace detail

inline Scenario parse_scenario(const json& j) { return detail::from_b(pumpb::parse_scenario(j)); }
inline Scenario load_scenario(const std::string& path) { return detail::from_b(pumpb::load_scenario(path)); }

struct ModelBundle {
  ContinuousModel cm;
  DiscreteModel dm;
  GainSchedule gains;
  ClosedLoopDynamics cl;
};
// scenario.hpp:285-301: assembles the matrices from whatever fields the caller
// set (code-built Scenarios with empty start/goal are fine); no re-validation
inline ModelBundle build_models(const Scenario& s) {
  pumpb::LqgWeights lw{detail::to_la(s.tracking.Q), detail::to_la(s.tracking.R), detail::to_la(s.tracking.F)};
  pumpb::ModelBundle m = pumpb::build_models(static_cast<int>(s.workspace.bounds.lo.size()), s.dt,
                                             detail::to_la(s.process_noise), detail::to_la(s.measurement_noise),
                                             detail::to_la(s.initial_covariance), lw);
  ModelBundle o;
  o.cm = {detail::from_la(m.cm.A), detail::from_la(m.cm.B), detail::from_la(m.cm.C), detail::from_la(m.cm.V),
          detail::from_la(m.cm.W)};
  o.dm = detail::from_b(m.dm);
  o.gains = {detail::from_la(m.gains.L), detail::from_la(m.gains.K), detail::from_la(m.gains.sigma0)};
  o.cl = detail::from_b(m.cl);
  return o;
}

// ============================================================== pump.hpp
struct PumpResult {  // pump.hpp:148-165
  bool success = false;
  Trajectory trajectory;
  double cost = 0, certified_cp = 0, cp_hat = 0, pre_smoothing_cost = 0, smoothing_s = 0;
  std::vector<int> path;
  double build_graph_seconds = 0, explore_seconds = 0, selection_seconds = 0;
  long partial_plans = 0;
  std::string termination;
  std::vector<std::pair<double, double>> pareto;
  std::vector<std::pair<int, double>> mc_evals;
};

// run_pump (pump.hpp:170-263): the whole solve runs in the library
inline PumpResult run_pump(const Scenario& s, int workers = 1, const SampleGraph* prebuilt = nullptr) {
  (void)workers;
  const std::string text = detail::to_json(s).dump();
  pump_scenario* sh = nullptr;
  detail::check(pump_scenario_parse(text.c_str(), &sh));
  std::unique_ptr<pump_scenario, int (*)(pump_scenario*)> sg(sh, pump_scenario_free);
  detail::GraphHandle gh;
  detail::GraphArrays ga;
  if (prebuilt) {
    ga = detail::from_graph(*prebuilt);
    detail::check(pump_graph_upload(detail::ctx(), &ga.v, &gh.h));
  }
  pump_result* rh = nullptr;
  detail::check(pump_run(detail::ctx(), sh, gh.h, &rh));
  std::unique_ptr<pump_result, int (*)(pump_result*)> rg(rh, pump_result_free);
  pump_result_summary sum{};
  detail::check(pump_result_summary_get(rh, &sum));
  const int dw = sum.dw, nt = sum.n_traj_points;
  std::vector<int32_t> path(sum.path_len + 1), ids(sum.n_mc_evals + 1);
  std::vector<double> pc(sum.n_pareto + 1), pcp(sum.n_pareto + 1), mcs(sum.n_mc_evals + 1), tt(nt + 1),
      tp(static_cast<size_t>(nt) * dw + 1), tv(tp.size()), tu(tp.size());
  detail::check(pump_result_arrays(rh, path.data(), pc.data(), pcp.data(), ids.data(), mcs.data(), tt.data(),
                                   tp.data(), tv.data(), tu.data()));
  PumpResult r;
  r.success = sum.success != 0;
  r.cost = sum.cost;
  r.certified_cp = sum.certified_cp;
  r.cp_hat = sum.cp_hat;
  r.pre_smoothing_cost = sum.pre_smoothing_cost;
  r.smoothing_s = sum.smoothing_s;
  r.path.assign(path.begin(), path.begin() + sum.path_len);
  r.build_graph_seconds = sum.build_graph_seconds;
  r.explore_seconds = sum.explore_seconds;
  r.selection_seconds = sum.selection_seconds;
  r.partial_plans = static_cast<long>(sum.partial_plans);
  r.termination = sum.termination ? "frontier_exhausted" : "goal_below_alpha_min";
  for (int i = 0; i < sum.n_pareto; ++i) r.pareto.push_back({pc[i], pcp[i]});
  for (int i = 0; i < sum.n_mc_evals; ++i) r.mc_evals.push_back({ids[i], mcs[i]});
  for (int i = 0; i < nt; ++i)
    r.trajectory.points.push_back({tt[i], {detail::vec(tp.data() + i * dw, dw), detail::vec(tv.data() + i * dw, dw)},
                                   detail::vec(tu.data() + i * dw, dw)});
  return r;
}

// ============================================================== rrt.hpp
struct RrtResult {  // rrt.hpp:11-18
  bool success = false;
  Trajectory trajectory;
  double cost = 0;
  double certified_cp = 0;
  int trials_reaching_goal = 0;
  int certification_attempts = 0;
};

// repeated_rrt (rrt.hpp:50-147): the trials run on the GPU (one warp each),
// certification in cost order on the GPU; `workers` is accepted, unused
inline RrtResult repeated_rrt(const Scenario& s, int trials, double alpha, int n_mc, int workers = 1) {
  (void)workers;
  if (trials < 1) throw std::invalid_argument("repeated_rrt: trials must be at least 1");
  const std::string text = detail::to_json(s).dump();
  pump_scenario* sh = nullptr;
  detail::check(pump_scenario_parse(text.c_str(), &sh));
  std::unique_ptr<pump_scenario, int (*)(pump_scenario*)> sg(sh, pump_scenario_free);
  pump_result* rh = nullptr;
  detail::check(pump_rrt_run(detail::ctx(), sh, trials, alpha, n_mc, &rh));
  std::unique_ptr<pump_result, int (*)(pump_result*)> rg(rh, pump_result_free);
  pump_result_summary sum{};
  detail::check(pump_result_summary_get(rh, &sum));
  const int dw = sum.dw, nt = sum.n_traj_points;
  std::vector<double> tt(nt + 1), tp(static_cast<size_t>(nt) * dw + 1), tv(tp.size()), tu(tp.size());
  detail::check(pump_result_arrays(rh, nullptr, nullptr, nullptr, nullptr, nullptr, tt.data(), tp.data(), tv.data(),
                                   tu.data()));
  RrtResult r;
  r.success = sum.success != 0;
  r.cost = sum.cost;
  r.certified_cp = sum.certified_cp;
  r.trials_reaching_goal = sum.rrt_trials_reaching_goal;
  r.certification_attempts = sum.rrt_certification_attempts;
  for (int i = 0; i < nt; ++i)
    r.trajectory.points.push_back({tt[i], {detail::vec(tp.data() + i * dw, dw), detail::vec(tv.data() + i * dw, dw)},
                                   detail::vec(tu.data() + i * dw, dw)});
  return r;
}

// ============================================================ report.hpp
namespace detail {
inline void write_text(const std::string& path, const std::string& text) {
  std::ofstream out(path, std::ios::binary);
  if (!out) throw std::runtime_error("cannot open output file: " + path);
  out << text;
  if (!out) throw std::runtime_error("failed writing output file: " + path);
}
}  // namespace detail

inline json trajectory_json(const Trajectory& traj) {  // report.hpp:31-40
  json points = json::array();
  for (const auto& p : traj.points)
    points.push_back({{"t", p.t},
                      {"position", detail::vjson(p.state.position)},
                      {"velocity", detail::vjson(p.state.velocity)},
                      {"control", detail::vjson(p.control)}});
  return {{"schema_version", 1}, {"points", points}};
}

inline Trajectory parse_trajectory(const json& j) {  // report.hpp:42-62
  if (!j.contains("points") || !j["points"].is_array()) throw std::runtime_error("trajectory: missing points array");
  Trajectory traj;
  for (const auto& p : j["points"]) {
    Waypoint wp;
    wp.t = p.at("t").get<double>();
    auto pos = pumpb::sdetail::parse_vector(p.at("position"), "trajectory.position");
    const int n = static_cast<int>(pos.size());
    wp.state.position = detail::vec(pos.data(), n);
    auto vel = pumpb::sdetail::parse_vector(p.at("velocity"), "trajectory.velocity", n);
    wp.state.velocity = detail::vec(vel.data(), n);
    if (p.contains("control")) {
      auto u = pumpb::sdetail::parse_vector(p.at("control"), "trajectory.control", n);
      wp.control = detail::vec(u.data(), n);
    } else {
      wp.control = VectorXd::Zero(n);
    }
    traj.points.push_back(std::move(wp));
  }
  for (std::size_t i = 1; i < traj.points.size(); ++i)
    if (traj.points[i].t <= traj.points[i - 1].t) throw std::runtime_error("trajectory: times must be strictly increasing");
  return traj;
}

inline Trajectory load_trajectory(const std::string& path) {
  std::ifstream in(path);
  if (!in) throw std::runtime_error("cannot open trajectory file: " + path);
  json j;
  in >> j;
  return parse_trajectory(j);
}

inline json rrt_report_json(const Scenario& s, const RrtResult& r, int trials, int workers) {  // report.hpp:99-111
  return {{"schema_version", 1},
          {"scenario", s.name},
          {"algorithm", "rrt"},
          {"workers", workers},
          {"success", r.success},
          {"cost", r.cost},
          {"certified_cp", r.certified_cp},
          {"alpha", s.alpha},
          {"trials", trials},
          {"trials_reaching_goal", r.trials_reaching_goal},
          {"certification_attempts", r.certification_attempts}};
}

inline json plan_report_json(const Scenario& s, const PumpResult& r, int workers) {  // report.hpp:72-97
  json pareto = json::array();
  for (const auto& [cost, cp] : r.pareto) pareto.push_back({{"cost", cost}, {"cp_hat", cp}});
  json evals = json::array();
  for (const auto& [id, mc] : r.mc_evals) evals.push_back({{"plan", id}, {"mc", mc}});
  return {{"schema_version", 1},
          {"scenario", s.name},
          {"algorithm", "pump"},
          {"workers", workers},
          {"success", r.success},
          {"cost", r.cost},
          {"pre_smoothing_cost", r.pre_smoothing_cost},
          {"certified_cp", r.certified_cp},
          {"cp_hat", r.cp_hat},
          {"alpha", s.alpha},
          {"smoothing_s", r.smoothing_s},
          {"path", r.path},
          {"partial_plans", r.partial_plans},
          {"termination", r.termination},
          {"goal_plans", pareto},
          {"mc_evaluations", evals},
          {"timing",
           {{"build_graph_seconds", r.build_graph_seconds},
            {"explore_seconds", r.explore_seconds},
            {"selection_seconds", r.selection_seconds}}}};
}

inline std::string pareto_csv(const PumpResult& r) {  // report.hpp:113-120
  std::string out = "cost,cp_hat\n";
  for (const auto& [cost, cp] : r.pareto) {
    json row = {cost, cp};
    out += row[0].dump() + "," + row[1].dump() + "\n";
  }
  return out;
}

// ============================================================ compare.hpp
// The Fig. 4 estimator study (compare.hpp:38-96 with the estimators of
// cp.hpp:51-169).  The sampling estimators run on the GPU through the calls
// above (mc_certify, presample_bank, hsmc_extend); the analytical ones are a
// handful of 12x12 products per waypoint and stay on the host, written with
// the same (Eigen-compatible) products and summation order as the reference.
inline double gauss_tail(double x) { return 0.5 * std::erfc(x / std::sqrt(2.0)); }  // P(N(0,1) > x)

namespace detail {
// half-spaces of a region without repeats: a later (a, b) equal to an earlier
// one (b equal, a equal componentwise) is skipped (cp.hpp:56-70)
inline std::vector<const HalfSpace*> distinct_halfspaces(const ConvexRegion& region) {
  std::vector<const HalfSpace*> kept;
  for (const HalfSpace& h : region.halfspaces) {
    const bool seen = std::any_of(kept.begin(), kept.end(), [&](const HalfSpace* g) {
      return g->b == h.b && g->a.size() == h.a.size() && (g->a - h.a).cwiseAbs().maxCoeff() == 0;
    });
    if (!seen) kept.push_back(&h);
  }
  return kept;
}
}  // namespace detail

// union bound over the region's half-spaces with exact Gaussian marginals (cp.hpp:75-91)
inline double pointwise_cp(const MatrixXd& cov, const ConvexRegion& region) {
  double sum = 0;
  for (const HalfSpace* h : detail::distinct_halfspaces(region)) {
    const double var = h->a.dot(cov * h->a);
    sum += var < 1e-30 ? (h->b <= 0 ? 1.0 : 0.0) : gauss_tail(h->b / std::sqrt(var));
    if (sum >= 1.0) return 1.0;
  }
  return sum;
}

inline double additive_cp(const std::vector<double>& pointwise) {  // cp.hpp:94-98
  double sum = 0;
  for (double p : pointwise) sum += p;
  return std::min(1.0, sum);
}

inline double multiplicative_cp(const std::vector<double>& pointwise) {  // cp.hpp:101-105
  double free_all = 1;
  for (double p : pointwise) free_all *= 1.0 - p;
  return 1.0 - free_all;
}

// Gaussian filter over the joint deviation with one-sided moment-matched
// truncation per half-space (cp.hpp:113-169).
inline double conditional_multiplicative_cp(const DiscreteModel& dm, const GainSchedule& gs, const MatrixXd& sigma0,
                                            const std::vector<const ConvexRegion*>& regions) {
  const ClosedLoopDynamics cl = closed_loop(dm, gs, sigma0);
  const int d = cl.d, nz = 2 * d;
  VectorXd mean = VectorXd::Zero(nz);
  MatrixXd cov = MatrixXd::Zero(nz, nz);
  cov.topLeftCorner(d, d) = sigma0;
  const MatrixXd vq = cl.Sv * cl.Sv.transpose(), wq = cl.Sw * cl.Sw.transpose();
  double survive = 1.0;
  for (std::size_t t = 0; t < regions.size(); ++t) {
    if (regions[t]) {
      double p_step = 0;
      for (const HalfSpace* h : detail::distinct_halfspaces(*regions[t])) {
        VectorXd g = VectorXd::Zero(nz);
        g.head(d) = cl.C.transpose() * h->a;  // the half-space seen from the joint state
        const double mu = g.dot(mean), var = g.dot(cov * g);
        if (var < 1e-14) {  // no spread along g: a deterministic test
          if (mu > h->b) p_step = 1.0;
          continue;
        }
        const double sd = std::sqrt(var), beta = (h->b - mu) / sd;
        const double tail = gauss_tail(beta), keep = 1.0 - tail;
        p_step += tail;
        if (keep < 1e-12) {
          p_step = 1.0;
          continue;
        }
        const double ratio = std::exp(-0.5 * beta * beta) / std::sqrt(2.0 * 3.14159265358979323846) / keep;
        const double mu_t = mu - sd * ratio;
        const double var_t = std::max(var * (1.0 - beta * ratio - ratio * ratio), 0.0);
        const VectorXd cg = cov * g;
        mean += ((mu_t - mu) / var) * cg;
        cov += ((var_t - var) / (var * var)) * (cg * cg.transpose());
      }
      survive *= 1.0 - std::min(1.0, p_step);
      if (survive <= 0) return 1.0;
    }
    if (t + 1 < regions.size()) {
      mean = cl.F * mean;
      cov = cl.F * cov * cl.F.transpose() + cl.Gv * vq * cl.Gv.transpose() + cl.Gw * wq * cl.Gw.transpose();
    }
  }
  return 1.0 - survive;
}

// the stored trajectory as a piecewise cubic Hermite of its waypoint states (compare.hpp:13-24)
inline State trajectory_state_at(const Trajectory& traj, double t) {
  if (traj.points.empty()) throw std::invalid_argument("trajectory_state_at: empty");
  if (t <= traj.points.front().t) return traj.points.front().state;
  if (t >= traj.points.back().t) return traj.points.back().state;
  std::size_t j = 0;
  while (j + 2 < traj.points.size() && traj.points[j + 1].t <= t) ++j;
  const Waypoint& a = traj.points[j];
  const Waypoint& b = traj.points[j + 1];
  return fixed_time_connect(a.state, b.state, b.t - a.t).state_at(t - a.t);
}

struct CpComparisonRow {
  std::string method;
  int waypoints = 0;
  double estimate = 0, mc_reference = 0, seconds = 0;
};

// compare.hpp:38-96: for each waypoint count, re-discretize the trajectory,
// then every estimator against the MC reference at that resolution
inline std::vector<CpComparisonRow> cp_compare(const Scenario& s, const Trajectory& traj,
                                               const std::vector<int>& waypoint_counts, int particles, int n_mc,
                                               int workers = 1) {
  using clk = std::chrono::steady_clock;
  auto secs = [](clk::time_point a) { return std::chrono::duration<double>(clk::now() - a).count(); };
  std::vector<CpComparisonRow> rows;
  const double eps_cc = s.effective_eps_cc();
  for (int count : waypoint_counts) {
    if (count < 2) throw std::invalid_argument("cp_compare: need at least 2 waypoints");
    const int T = count - 1;
    Scenario sk = s;
    sk.dt = traj.duration() / T;
    const ModelBundle mb = build_models(sk);
    std::vector<VectorXd> y(count);
    std::vector<ConvexRegion> regions(count);
    for (int t = 0; t <= T; ++t) {
      const State st = trajectory_state_at(traj, t * sk.dt);
      y[t] = st.position;
      regions[t] = local_convex_region(s.workspace, st.position, st.velocity);
    }
    auto t0 = clk::now();
    const double mc = mc_certify(y, mb.cl, s.workspace, n_mc, s.seeds.mc, eps_cc, workers).value;
    rows.push_back({"mc", count, mc, mc, secs(t0)});

    const std::vector<MatrixXd> covs = propagate_covariances(mb.dm, mb.gains, s.initial_covariance, T);
    t0 = clk::now();
    std::vector<double> pw(count);
    for (int t = 0; t <= T; ++t) pw[t] = pointwise_cp(covs[t], regions[t]);
    const double pw_secs = secs(t0);
    rows.push_back({"additive", count, additive_cp(pw), mc, pw_secs});
    rows.push_back({"multiplicative", count, multiplicative_cp(pw), mc, pw_secs});

    t0 = clk::now();
    std::vector<const ConvexRegion*> rp(count);
    for (int t = 0; t <= T; ++t) rp[t] = &regions[t];
    const double cm = conditional_multiplicative_cp(mb.dm, mb.gains, s.initial_covariance, rp);
    rows.push_back({"conditional_multiplicative", count, cm, mc, secs(t0)});

    t0 = clk::now();
    const DeviationBank bank = presample_bank(mb.dm, mb.gains, s.initial_covariance, T, particles, s.seeds.bank, workers);
    std::vector<HsmcStep> steps(count);
    for (int t = 0; t <= T; ++t) steps[t] = {t, &regions[t]};
    const double hs = hsmc_extend(ParticleMask::full(particles), bank, steps).second;
    rows.push_back({"hsmc", count, hs, mc, secs(t0)});
  }
  return rows;
}

inline std::string cp_compare_csv(const std::vector<CpComparisonRow>& rows) {  // report.hpp:122-129
  std::string out = "method,waypoints,estimate,mc_reference,wall_time\n";
  for (const auto& r : rows)
    out += r.method + "," + std::to_string(r.waypoints) + "," + json(r.estimate).dump() + "," +
           json(r.mc_reference).dump() + "," + json(r.seconds).dump() + "\n";
  return out;
}

}  // namespace pump
