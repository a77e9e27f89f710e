// pump command-line front end (tools/pump_cli.cpp of the reference, same
// subcommands, flags and exit codes) over the drop-in API: `plan` runs the
// whole solve on the GPU, `certify` Monte-Carlo-certifies a trajectory on the
// GPU, `rrt` runs the repeated-RRT baseline (trials and certification on the
// GPU), `cp-compare` runs the Fig. 4 estimator study (MC, bank and HSMC on
// the GPU).  Argument parsing is hand-rolled (CLI11 is not in the image).
#include <cstdio>
#include <cstdlib>
#include <filesystem>
#include <string>
#include <vector>

#include "pump/compare.hpp"
#include "pump/report.hpp"

namespace {

constexpr int kExitSuccess = 0;
constexpr int kExitInputError = 1;
constexpr int kExitPlannerFailure = 2;

struct Opts {
  std::string scenario, out = ".", trajectory;
  std::uint64_t seed = 0;
  int workers = 1;
  std::vector<int> waypoints;  // cp-compare
  int mc_samples = 0;          // cp-compare
};

pump::Scenario load(const Opts& o) {
  pump::Scenario s = pump::load_scenario(o.scenario);
  if (o.seed != 0) {  // pump_cli.cpp:33-41
    s.seeds.bank = o.seed;
    s.seeds.mc = o.seed + 1;
    s.seeds.rrt = o.seed + 2;
  }
  return s;
}

std::string out_path(const Opts& o, const std::string& name) {
  std::filesystem::create_directories(o.out);
  return (std::filesystem::path(o.out) / name).string();
}

int run_plan(const Opts& o) {
  pump::Scenario s = load(o);
  pump::PumpResult r = pump::run_pump(s, o.workers);
  pump::detail::write_text(out_path(o, "report.json"), pump::plan_report_json(s, r, o.workers).dump(2) + "\n");
  pump::detail::write_text(out_path(o, "pareto.csv"), pump::pareto_csv(r));
  if (r.success)
    pump::detail::write_text(out_path(o, "trajectory.json"), pump::trajectory_json(r.trajectory).dump(2) + "\n");
  std::printf("%s cost=%.6f certified_cp=%.6f alpha=%g partial_plans=%ld\n", r.success ? "success" : "failure",
              r.cost, r.certified_cp, s.alpha, r.partial_plans);
  return r.success ? kExitSuccess : kExitPlannerFailure;
}

int run_cp_compare(const Opts& o) {  // pump_cli.cpp:77-90
  pump::Scenario s = load(o);
  pump::Trajectory traj = pump::load_trajectory(o.trajectory);
  std::vector<int> waypoints = o.waypoints.empty() ? std::vector<int>{25, 50, 100, 200} : o.waypoints;
  auto rows = pump::cp_compare(s, traj, waypoints, s.particles, o.mc_samples > 0 ? o.mc_samples : s.mc_samples,
                               o.workers);
  pump::detail::write_text(out_path(o, "cp_compare.csv"), pump::cp_compare_csv(rows));
  for (const auto& r : rows)
    std::printf("%-28s waypoints=%-4d estimate=%.6f mc=%.6f %.3fs\n", r.method.c_str(), r.waypoints, r.estimate,
                r.mc_reference, r.seconds);
  return kExitSuccess;
}

int run_rrt(const Opts& o) {  // pump_cli.cpp:63-76
  pump::Scenario s = load(o);
  pump::RrtResult r = pump::repeated_rrt(s, s.rrt.trials, s.alpha, s.mc_samples, o.workers);
  pump::json report = pump::rrt_report_json(s, r, s.rrt.trials, o.workers);
  pump::detail::write_text(out_path(o, "report.json"), report.dump(2) + "\n");
  if (r.success)
    pump::detail::write_text(out_path(o, "trajectory.json"), pump::trajectory_json(r.trajectory).dump(2) + "\n");
  std::printf("%s cost=%.6f certified_cp=%.6f trials_reaching_goal=%d\n", r.success ? "success" : "failure", r.cost,
              r.certified_cp, r.trials_reaching_goal);
  return r.success ? kExitSuccess : kExitPlannerFailure;
}

int run_certify(const Opts& o) {
  pump::Scenario s = load(o);
  pump::Trajectory traj = pump::load_trajectory(o.trajectory);
  pump::ModelBundle mb = pump::build_models(s);
  pump::CpEstimate est =
      pump::mc_certify(traj.positions(), mb.cl, s.workspace, s.mc_samples, s.seeds.mc, s.effective_eps_cc(), o.workers);
  pump::json report = {{"schema_version", 1}, {"scenario", s.name},       {"algorithm", "certify"},
                       {"certified_cp", est.value}, {"mc_samples", est.samples}, {"alpha", s.alpha},
                       {"within_alpha", est.value <= s.alpha}};
  pump::detail::write_text(out_path(o, "report.json"), report.dump(2) + "\n");
  std::printf("certified_cp=%.6f mc_samples=%d alpha=%g %s\n", est.value, est.samples, s.alpha,
              est.value <= s.alpha ? "within_alpha" : "exceeds_alpha");
  return est.value <= s.alpha ? kExitSuccess : kExitPlannerFailure;
}

int usage() {
  std::fprintf(stderr,
               "usage: pump {plan|certify|rrt|cp-compare} --scenario FILE [--seed N] [--workers N] [--out DIR] "
               "[--trajectory FILE] [--waypoints N...] [--mc-samples N]\n");
  return kExitInputError;
}

}  // namespace

int main(int argc, char** argv) {
  if (argc < 2) return usage();
  const std::string cmd = argv[1];
  Opts o;
  for (int i = 2; i < argc; ++i) {
    const std::string a = argv[i];
    auto next = [&]() -> std::string {
      if (i + 1 >= argc) {
        std::fprintf(stderr, "error: %s needs a value\n", a.c_str());
        std::exit(kExitInputError);
      }
      return argv[++i];
    };
    if (a == "--scenario") o.scenario = next();
    else if (a == "--out") o.out = next();
    else if (a == "--trajectory") o.trajectory = next();
    else if (a == "--seed") o.seed = std::strtoull(next().c_str(), nullptr, 10);
    else if (a == "--mc-samples") o.mc_samples = std::atoi(next().c_str());
    else if (a == "--waypoints") {  // one or more counts (CLI11 vector option)
      o.waypoints.push_back(std::atoi(next().c_str()));
      while (i + 1 < argc && std::string(argv[i + 1]).rfind("--", 0) != 0) o.waypoints.push_back(std::atoi(argv[++i]));
    }
    else if (a == "--workers") {
      o.workers = std::atoi(next().c_str());
      if (o.workers < 1) return usage();
    } else {
      std::fprintf(stderr, "error: unknown option %s\n", a.c_str());
      return kExitInputError;
    }
  }
  if (o.scenario.empty()) return usage();
  try {
    if (cmd == "plan") return run_plan(o);
    if (cmd == "certify") {
      if (o.trajectory.empty()) return usage();
      return run_certify(o);
    }
    if (cmd == "rrt") return run_rrt(o);
    if (cmd == "cp-compare") {
      if (o.trajectory.empty()) return usage();
      return run_cp_compare(o);
    }
  } catch (const std::exception& e) {
    std::fprintf(stderr, "error: %s\n", e.what());
    return kExitInputError;
  }
  return usage();
}
