// Fast scenario reader vs the nlohmann loader (host/scenario_fast.hpp vs
// host/scenario.hpp): for every JSON text given (one file each on the command
// line), either the fast reader defers (nullopt) or both build identical
// Scenarios, bit for bit; where the nlohmann loader throws, the fast reader
// must defer.  Prints one line per input: accepted | deferred | error-deferred.
#include <cstdio>
#include <cstring>
#include <fstream>
#include <sstream>

#include "host/scenario_fast.hpp"

using namespace pumpb;

static bool same_bits(const std::vector<double>& a, const std::vector<double>& b) {
  return a.size() == b.size() && (a.empty() || std::memcmp(a.data(), b.data(), a.size() * 8) == 0);
}
static bool same_mat(const Mat& a, const Mat& b) { return a.r == b.r && a.c == b.c && same_bits(a.a, b.a); }
static bool same_box(const Box& a, const Box& b) { return same_bits(a.lo, b.lo) && same_bits(a.hi, b.hi); }
static bool same_d(double a, double b) { return std::memcmp(&a, &b, 8) == 0; }

static bool equal(const Scenario& a, const Scenario& b) {
  bool ok = a.name == b.name && same_box(a.workspace.bounds, b.workspace.bounds) &&
            a.workspace.obstacles.size() == b.workspace.obstacles.size();
  for (size_t i = 0; ok && i < a.workspace.obstacles.size(); ++i)
    ok = same_box(a.workspace.obstacles[i], b.workspace.obstacles[i]);
  ok = ok && same_bits(a.start_pos, b.start_pos) && same_bits(a.start_vel, b.start_vel) && same_box(a.goal, b.goal) &&
       same_d(a.goal_max_speed, b.goal_max_speed) && same_mat(a.process_noise, b.process_noise) &&
       same_mat(a.measurement_noise, b.measurement_noise) && same_mat(a.initial_covariance, b.initial_covariance) &&
       same_mat(a.tracking.Q, b.tracking.Q) && same_mat(a.tracking.R, b.tracking.R) &&
       same_mat(a.tracking.F, b.tracking.F) && same_d(a.dt, b.dt) && a.samples == b.samples &&
       same_d(a.connection_radius, b.connection_radius) && same_d(a.alpha, b.alpha) && same_d(a.eta, b.eta) &&
       same_d(a.lambda, b.lambda) && a.particles == b.particles && a.mc_samples == b.mc_samples &&
       a.bank_horizon == b.bank_horizon && same_d(a.max_speed, b.max_speed) && same_d(a.tau_max, b.tau_max) &&
       same_d(a.collision_resolution, b.collision_resolution) && a.seeds.bank == b.seeds.bank &&
       a.seeds.mc == b.seeds.mc && a.seeds.rrt == b.seeds.rrt && a.rrt.trials == b.rrt.trials &&
       a.rrt.max_iterations == b.rrt.max_iterations && same_d(a.rrt.goal_bias, b.rrt.goal_bias);
  return ok;
}

int main(int argc, char** argv) {
  int bad = 0;
  for (int i = 1; i < argc; ++i) {
    std::ifstream in(argv[i]);
    std::stringstream ss;
    ss << in.rdbuf();
    const std::string text = ss.str();
    auto fast = parse_scenario_fast(text);
    bool slow_ok = true;
    Scenario slow;
    try {
      slow = parse_scenario_text(text);
    } catch (const std::exception&) {
      slow_ok = false;
    }
    const char* verdict;
    if (!slow_ok) {
      verdict = fast ? "MISMATCH (fast accepted what the loader rejects)" : "error-deferred";
    } else if (!fast) {
      verdict = "deferred";
    } else {
      verdict = equal(*fast, slow) ? "accepted" : "MISMATCH (different scenario)";
    }
    if (std::strncmp(verdict, "MISMATCH", 8) == 0) ++bad;
    std::printf("%s %s\n", verdict, argv[i]);
  }
  return bad ? 1 : 0;
}
