// ORACLE — TEST INFRASTRUCTURE ONLY.
//
// CPU restatement of the PUMP reference hot path (/root/reference/proj,
// header-only C++, which cannot be compiled here: it needs Eigen, absent
// from this image — SURVEY.md §0.2).  Only tests/, __graft_entry__.smoke()
// and bench.py's CPU-baseline leg may load it, and only as the checker or
// the timed CPU baseline; the product (libpump_gpu.so) never links it.
//
// Every function cites the reference file:line it restates.  Operation
// order follows the reference build (-O3, SSE2, no FMA):
// gemv rows and small-vector reductions are sequential from +0, a*b+c is
// never contracted (compile with -ffp-contract=off).
//
// Normals: mode PORTABLE evaluates log/cos with csrc/common/pmath.h (bit-
// identical to the GPU); mode GLIBC calls std::log/std::cos, i.e. the literal
// reference (whose bits vary with the host ISA).
//
// Pinning: the oracle is checked against every known-answer test the
// reference's own test-suite holds for this path (tests/test_oracle.py,
// ported from proj/tests/test_cp.cpp, test_lti.cpp, test_plan.cpp,
// test_steer.cpp, test_geom.cpp, acceptance.cpp) and against
// oracle/_ref (the reference headers compiled over oracle/eigen_shim).
#pragma once

#include <cstdint>
#include <functional>
#include <string>
#include <vector>

namespace oracle {

enum NormalMode { kPortable = 0, kGlibc = 1 };
void set_normal_mode(int mode);
int normal_mode();

// ----------------------------------------------------------------- rng.hpp
std::uint64_t mix64(std::uint64_t x);
std::uint64_t counter_hash(std::uint64_t seed, std::uint64_t a, std::uint64_t b, std::uint64_t c);
double to_unit(std::uint64_t x);
double uniform(std::uint64_t seed, std::uint64_t a, std::uint64_t b, std::uint64_t c);
double normal(std::uint64_t seed, std::uint64_t a, std::uint64_t b, std::uint64_t channel);
constexpr std::uint64_t kInitial = 0, kProcess = 1u << 20, kMeasurement = 2u << 20;

void parallel_for(std::size_t n, int workers, const std::function<void(std::size_t, std::size_t)>& chunk);

// ------------------------------------------------------------------ types
using Vec = std::vector<double>;

struct Loop {  // ClosedLoopDynamics, row-major
  int d = 0, dw = 0;
  Vec F, Gv, Gw, Sv, Sw, S0, C;
};

struct World {  // Workspace
  int dw = 0;
  Vec blo, bhi;
  int n_obs = 0;
  Vec olo, ohi;  // n_obs x dw
};

struct St {  // State
  Vec p, v;
};

struct Mot {  // Motion
  St from, to;
  double tau = 0, cost = 0;
  bool ok = false;
  Vec acc0, jerk;
};

struct Wp {  // Waypoint
  double t = 0;
  St s;
  Vec u;
};

struct Hs {  // HalfSpace
  Vec a;
  double b = 0;
  bool fallback = false;
};

struct Region {
  Vec center;
  std::vector<Hs> hs;
};

struct Edge {
  int to = -1;
  Mot m;
  int n_steps = 0;
  std::vector<Region> regions;
};

struct Graph {
  std::vector<St> nodes;
  std::vector<std::vector<Edge>> adj;
  std::vector<int> goal_nodes;
  double r_n = 0, dt = 0;
};

struct Goal {
  Vec lo, hi;
  double max_speed = 0;
};

struct Bank {
  int n = 0, horizon = 0, dw = 0;
  std::uint64_t seed = 0;
  Vec dy;
};

struct Mask {
  int n = 0;
  std::vector<std::uint64_t> w;
  static Mask full(int n);
  int popcount() const;
  double cp() const;
};

struct Plan {
  int head = 0, parent = -1;
  double cost = 0, cp = 0;
  int t_end = 0;
  Mask mask;
};

struct ExParams {
  double alpha_min = 0, alpha_max = 1, lambda = 0.5, r_n = 1;
  int workers = 1;
};

struct ExResult {
  std::vector<Plan> plans;
  std::vector<std::vector<int>> pareto;
  std::vector<int> goal_plans;
  long partial_plans = 0, discarded_cp = 0, removed_dominated = 0, discarded_horizon = 0;
  int rounds = 0;
  std::string termination;
};

using Hook = std::function<void(int, const ExResult&, const std::vector<int>&)>;

// --------------------------------------------------------------- functions
Bank presample_bank(const Loop& cl, int t_max, int n, std::uint64_t seed, int workers);

double steer_cost(const St& a, const St& b, double tau);
Mot fixed_time_connect(const St& a, const St& b, double tau);
Mot connect(const St& a, const St& b, double tau_max, double ratio);
double scan_ratio(double tau_max);
St state_at(const Mot& m, double s);
Vec control_at(const Mot& m, double s);
std::vector<Wp> waypoints(const Mot& m, double dt);

bool point_free(const World& w, const double* y);
bool segment_hits(const double* p0, const double* p1, const double* lo, const double* hi, int dw);
bool segment_collides(const World& w, const double* p0, const double* p1);
bool motion_collides(const World& w, const Mot& m, double eps_cc);
Hs project_halfspace(const Vec& d, const Vec& ydot);
Region local_convex_region(const World& w, const Vec& y, const Vec& ydot);

std::pair<Mask, double> hsmc_extend(const Mask& mask, const Bank& bank,
                                    const std::vector<std::pair<int, const Region*>>& steps);

long mc_hits(const std::vector<Vec>& y_nom, const Loop& cl, const World& w, long r0, long r1,
             std::uint64_t seed, double eps_cc, int workers, std::vector<char>* flags = nullptr);

double halton(std::uint64_t index, int base);
bool goal_contains(const Goal& g, const St& s);
std::vector<St> sample_free(int n, const World& w, double max_speed, const Goal& goal);

Graph build_graph(std::vector<St> nodes, const World& w, const Goal& goal, double r_n, double dt, double eps_cc,
                  double tau_max, int workers);

ExResult explore(const Graph& g, const Bank& bank, const ExParams& p, const Hook& hook = nullptr);

std::vector<int> plan_path(const ExResult& r, int id);
std::vector<Wp> path_trajectory(const Graph& g, const std::vector<int>& path, double dt);
double trajectory_cost(const std::vector<Wp>& traj);

struct Selection {
  bool success = false;
  int plan_id = -1;
  double mc = 0;
  std::vector<std::pair<int, double>> evals;
};
Selection bisect_select(const std::vector<int>& sorted_ids, const std::function<double(int)>& mc, double alpha);

struct Smooth {
  std::vector<Wp> traj;
  double cost = 0, mc = 0, s = 0;
};
bool nominal_free(const World& w, const std::vector<Wp>& traj, double eps_cc);
Smooth smooth(const std::vector<Wp>& plan, double plan_mc, double alpha, const Loop& cl, const World& w, int n_mc,
              std::uint64_t seed, double eps_cc, int workers);

struct PumpOut {
  bool success = false;
  std::vector<Wp> traj;
  double cost = 0, certified_cp = 0, cp_hat = 0, pre_smoothing_cost = 0, smoothing_s = 0;
  std::vector<int> path;
  double build_graph_seconds = 0, explore_seconds = 0, selection_seconds = 0;
  long partial_plans = 0;
  std::string termination;
  std::vector<std::pair<double, double>> pareto;
  std::vector<std::pair<int, double>> mc_evals;
  long n_edges = 0, n_plans = 0;
};

struct PumpIn {  // what run_pump needs from a Scenario (scenario.hpp:34-77)
  World w;
  St x_init;
  Goal goal;
  Loop cl;
  double dt = 0.1, r_n = 1, eps_cc = 0.01, tau_max = 1, alpha = 0.05, eta = 2, lambda = 0.5, max_speed = 1;
  int samples = 100, particles = 128, mc_samples = 10000, bank_horizon = 2048;
  std::uint64_t seed_bank = 1, seed_mc = 2;
};
PumpOut run_pump(const PumpIn& in, int workers, const Graph* prebuilt = nullptr);

// ------------------------------------------------------------- rrt.hpp
double motion_partial_cost(const Mot& m, double s);
Mot truncate_motion(const Mot& m, double target_cost);
struct RrtIn {
  PumpIn p;
  int trials = 1000, max_iterations = 200;
  double goal_bias = 0.05;
  std::uint64_t seed_rrt = 3;
};
struct RrtOut {
  bool success = false;
  std::vector<Wp> traj;
  double cost = 0, certified_cp = 0;
  int trials_reaching_goal = 0, certification_attempts = 0;
};
RrtOut repeated_rrt(const RrtIn& in, int trials, double alpha, int n_mc, int workers);

}  // namespace oracle
