// ORACLE/_REF — TEST INFRASTRUCTURE ONLY.
// The reference's OWN headers (/root/reference/proj/include/pump/*.hpp,
// compiled in place, never copied) built against the Eigen-subset shim in
// include/compat, exposed through a tiny C surface so tests can cross-check
// the oracle restatement against the literal reference code paths (glibc
// normals, reference control flow).  Built by oracle/ref/Makefile into
// oracle/_ref/libpumpref.so.
#include <chrono>
#include <cstring>
#include <string>

#include "pump/cp.hpp"
#include "pump/graph.hpp"
#include "pump/planner.hpp"
#include "pump/scenario.hpp"

// Every mc_certify call the selection phase makes (pump.hpp:223-255) is
// recorded when a trace is armed, so the bench's reference arm can replay
// the same certification work on a rollout sample (ref_bench_step).  The
// reference headers are not modified: the call sites in pump.hpp / rrt.hpp /
// compare.hpp, included after this shim, resolve `mc_certify` to it.
namespace pump {
struct McCall {
  std::vector<VectorXd> y;
  int n_mc;
  std::uint64_t seed;
  double eps_cc;
};
inline thread_local std::vector<McCall>* g_mc_trace = nullptr;
inline CpEstimate mc_certify_traced(const std::vector<VectorXd>& y_nom, const ClosedLoopDynamics& cl,
                                    const Workspace& w, int n_mc, std::uint64_t seed, double eps_cc,
                                    int workers = 1) {
  if (g_mc_trace) g_mc_trace->push_back({y_nom, n_mc, seed, eps_cc});
  return mc_certify(y_nom, cl, w, n_mc, seed, eps_cc, workers);
}
}  // namespace pump
#define mc_certify mc_certify_traced
#include "pump/pump.hpp"
#include "pump/compare.hpp"
#include "pump/report.hpp"
#include "pump/rrt.hpp"
#undef mc_certify

namespace {
thread_local std::string g_err;
pump::Scenario scn(const char* text) { return pump::parse_scenario(pump::json::parse(text)); }
}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

// presample_bank of the scenario's models: (T+1) x n x dw doubles
int ref_presample_bank(const char* text, int T, int n, unsigned long long seed, int workers, double* out) {
  try {
    pump::Scenario s = scn(text);
    pump::ModelBundle mb = pump::build_models(s);
    pump::DeviationBank b = pump::presample_bank(mb.dm, mb.gains, s.initial_covariance, T, n, seed, workers);
    std::memcpy(out, b.dy.data(), b.dy.size() * sizeof(double));
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 1;
  }
}

// closed-loop F (2d x 2d, row-major) of build_models
int ref_closed_loop_F(const char* text, double* F) {
  try {
    pump::ModelBundle mb = pump::build_models(scn(text));
    const int nz = static_cast<int>(mb.cl.F.rows());
    for (int i = 0; i < nz; ++i)
      for (int j = 0; j < nz; ++j) F[i * nz + j] = mb.cl.F(i, j);
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 1;
  }
}

// run_pump: scalars[0..7] = success, cost, certified_cp, cp_hat, partial_plans,
// smoothing_s, pre_smoothing_cost, n_path; path -> path (cap 4096);
// mc evals -> (eval_ids, eval_vals, *n_evals); pareto (cost, cp) -> *n_pareto;
// trajectory positions (n_traj x dw) -> traj_pos, *n_traj
int ref_run_pump(const char* text, int workers, double* scalars, int* path, int* eval_ids, double* eval_vals,
                 int* n_evals, double* pareto_cost, double* pareto_cp, int* n_pareto, double* traj_t,
                 double* traj_pos, int* n_traj) {
  try {
    pump::Scenario s = scn(text);
    pump::PumpResult r = pump::run_pump(s, workers);
    scalars[0] = r.success ? 1 : 0;
    scalars[1] = r.cost;
    scalars[2] = r.certified_cp;
    scalars[3] = r.cp_hat;
    scalars[4] = static_cast<double>(r.partial_plans);
    scalars[5] = r.smoothing_s;
    scalars[6] = r.pre_smoothing_cost;
    scalars[7] = static_cast<double>(r.path.size());
    for (size_t i = 0; i < r.path.size() && i < 4096; ++i) path[i] = r.path[i];
    *n_evals = static_cast<int>(r.mc_evals.size());
    for (size_t i = 0; i < r.mc_evals.size() && i < 4096; ++i) {
      eval_ids[i] = r.mc_evals[i].first;
      eval_vals[i] = r.mc_evals[i].second;
    }
    *n_pareto = static_cast<int>(r.pareto.size());
    for (size_t i = 0; i < r.pareto.size() && i < 4096; ++i) {
      pareto_cost[i] = r.pareto[i].first;
      pareto_cp[i] = r.pareto[i].second;
    }
    const int dw = s.workspace_dim();
    *n_traj = static_cast<int>(r.trajectory.points.size());
    for (size_t i = 0; i < r.trajectory.points.size() && i < 100000; ++i) {
      traj_t[i] = r.trajectory.points[i].t;
      for (int k = 0; k < dw; ++k) traj_pos[i * dw + k] = r.trajectory.points[i].state.position[k];
    }
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 1;
  }
}

// repeated_rrt (rrt.hpp:50-147): out4 = success, cost, certified_cp,
// n_points; out2 = trials_reaching_goal, certification_attempts; trajectory
// times / positions (cap points, positions n x dw)
int ref_repeated_rrt(const char* text, int trials, double alpha, int n_mc, int workers, double* out4, int* out2,
                     int cap, double* traj_t, double* traj_pos) {
  try {
    pump::Scenario s = scn(text);
    pump::RrtResult r = pump::repeated_rrt(s, trials, alpha, n_mc, workers);
    out4[0] = r.success ? 1.0 : 0.0;
    out4[1] = r.cost;
    out4[2] = r.certified_cp;
    out4[3] = static_cast<double>(r.trajectory.points.size());
    out2[0] = r.trials_reaching_goal;
    out2[1] = r.certification_attempts;
    const int dw = s.workspace_dim();
    for (std::size_t i = 0; i < r.trajectory.points.size() && static_cast<int>(i) < cap; ++i) {
      traj_t[i] = r.trajectory.points[i].t;
      for (int k = 0; k < dw; ++k) traj_pos[i * dw + k] = r.trajectory.points[i].state.position[k];
    }
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 1;
  }
}

// cp_compare (compare.hpp:38-96) on a trajectory given as report.hpp JSON
// text: est[5 i + m] for count i, methods in the reference's row order (mc,
// additive, multiplicative, conditional_multiplicative, hsmc)
int ref_cp_compare(const char* text, const char* traj_text, const int* counts, int n_counts, int particles, int n_mc,
                   int workers, double* est) {
  try {
    pump::Scenario s = scn(text);
    pump::Trajectory traj = pump::parse_trajectory(pump::json::parse(traj_text));
    auto rows = pump::cp_compare(s, traj, std::vector<int>(counts, counts + n_counts), particles, n_mc, workers);
    for (std::size_t r = 0; r < rows.size(); ++r) est[r] = rows[r].estimate;
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 1;
  }
}

// The reference's own writers (report.hpp:31-129, pump_cli.cpp:48-109) on
// result values read back from another writer's files: kind 0 = plan
// (report.json, pareto.csv, trajectory.json), 1 = rrt (report.json,
// trajectory.json), 2 = certify (report.json).  The texts are returned
// concatenated with a '\x1f' separator in the CLI's exact bytes.
int ref_render(int kind, const char* scenario_text, const char* report_text, const char* traj_text, int workers,
               char* out, long cap, long* len) {
  try {
    pump::Scenario s = scn(scenario_text);
    const pump::json rep = pump::json::parse(report_text);
    std::string text;
    if (kind == 0) {
      pump::PumpResult r;
      r.success = rep.at("success").get<bool>();
      r.cost = rep.at("cost").get<double>();
      r.pre_smoothing_cost = rep.at("pre_smoothing_cost").get<double>();
      r.certified_cp = rep.at("certified_cp").get<double>();
      r.cp_hat = rep.at("cp_hat").get<double>();
      r.smoothing_s = rep.at("smoothing_s").get<double>();
      r.path = rep.at("path").get<std::vector<int>>();
      r.partial_plans = rep.at("partial_plans").get<long>();
      r.termination = rep.at("termination").get<std::string>();
      for (const auto& g : rep.at("goal_plans")) r.pareto.push_back({g.at("cost").get<double>(), g.at("cp_hat").get<double>()});
      for (const auto& e : rep.at("mc_evaluations")) r.mc_evals.push_back({e.at("plan").get<int>(), e.at("mc").get<double>()});
      r.build_graph_seconds = rep.at("timing").at("build_graph_seconds").get<double>();
      r.explore_seconds = rep.at("timing").at("explore_seconds").get<double>();
      r.selection_seconds = rep.at("timing").at("selection_seconds").get<double>();
      text = pump::plan_report_json(s, r, workers).dump(2) + "\n" + "\x1f" + pump::pareto_csv(r);
      if (traj_text && *traj_text)
        text += "\x1f" + pump::trajectory_json(pump::parse_trajectory(pump::json::parse(traj_text))).dump(2) + "\n";
    } else if (kind == 1) {
      pump::RrtResult r;
      r.success = rep.at("success").get<bool>();
      r.cost = rep.at("cost").get<double>();
      r.certified_cp = rep.at("certified_cp").get<double>();
      r.trials_reaching_goal = rep.at("trials_reaching_goal").get<int>();
      r.certification_attempts = rep.at("certification_attempts").get<int>();
      text = pump::rrt_report_json(s, r, rep.at("trials").get<int>(), workers).dump(2) + "\n";
      if (traj_text && *traj_text)
        text += "\x1f" + pump::trajectory_json(pump::parse_trajectory(pump::json::parse(traj_text))).dump(2) + "\n";
    } else {
      const double v = rep.at("certified_cp").get<double>();
      const pump::json report = {{"schema_version", 1},
                                 {"scenario", s.name},
                                 {"algorithm", "certify"},
                                 {"certified_cp", v},
                                 {"mc_samples", rep.at("mc_samples").get<int>()},
                                 {"alpha", s.alpha},
                                 {"within_alpha", v <= s.alpha}};
      text = report.dump(2) + "\n";
    }
    *len = static_cast<long>(text.size());
    if (out && cap >= *len) std::memcpy(out, text.data(), text.size());
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 1;
  }
}

// ------------------------------------------------ bench.py reference arm
// A bounded sample of one reference solve (run_pump, pump.hpp:170-263), for
// workloads whose full solve takes tens of seconds on the host: setup builds
// the graph and runs one full solve (timed, and recording its MC calls);
// each step then re-times, through the reference's own functions,
//   - sample_free + the build_graph row loop (graph.hpp:63-95, the body
//     restated over the reference's connect / motion_collides /
//     motion_waypoints / point_free / local_convex_region) for the rows
//     v = offset (mod stride), scaled by stride;
//   - presample_bank + explore on the full graph (unsampled);
//   - every recorded mc_certify call over its first n_mc / mc_stride
//     rollouts (rollouts are independent), scaled by mc_stride.
struct RefBench {
  pump::Scenario s;
  pump::ModelBundle mb;
  pump::SampleGraph g;
  std::vector<pump::McCall> trace;
};

int ref_bench_setup(const char* text, int workers, double* out, void** handle) {
  try {
    using clk = std::chrono::steady_clock;
    auto* b = new RefBench;
    b->s = scn(text);
    pump::Scenario& s = b->s;
    b->mb = pump::build_models(s);
    auto t0 = clk::now();
    std::vector<pump::State> nodes;
    nodes.push_back(s.x_init);
    for (auto& st : pump::sample_free(s.samples, s.workspace, s.max_speed, s.goal)) nodes.push_back(std::move(st));
    b->g = pump::build_graph(std::move(nodes), s.workspace, s.goal, s.effective_r_n(), s.dt, s.effective_eps_cc(),
                             s.effective_tau_max(), workers);
    auto t1 = clk::now();
    pump::g_mc_trace = &b->trace;
    pump::PumpResult r = pump::run_pump(s, workers, &b->g);
    pump::g_mc_trace = nullptr;
    auto t2 = clk::now();
    out[0] = std::chrono::duration<double>(t1 - t0).count();
    out[1] = std::chrono::duration<double>(t2 - t1).count();
    out[2] = r.explore_seconds;
    out[3] = r.selection_seconds;
    out[4] = static_cast<double>(r.partial_plans);
    out[5] = static_cast<double>(b->trace.size());
    out[6] = r.success ? 1.0 : 0.0;
    out[7] = r.cost;
    out[8] = static_cast<double>(b->g.nodes.size());
    *handle = b;
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 1;
  }
}

int ref_bench_step(void* handle, int workers, int row_stride, int row_offset, int mc_stride, double* out) {
  try {
    using clk = std::chrono::steady_clock;
    auto secs = [](clk::time_point a, clk::time_point c) { return std::chrono::duration<double>(c - a).count(); };
    RefBench& b = *static_cast<RefBench*>(handle);
    const pump::Scenario& s = b.s;
    const double r_n = s.effective_r_n(), eps_cc = s.effective_eps_cc(), tau_max = s.effective_tau_max();
    // sampling + graph rows
    auto t0 = clk::now();
    std::vector<pump::State> nodes;
    nodes.push_back(s.x_init);
    for (auto& st : pump::sample_free(s.samples, s.workspace, s.max_speed, s.goal)) nodes.push_back(std::move(st));
    const int n = static_cast<int>(nodes.size());
    auto t_s = clk::now();
    std::vector<int> rows;
    for (int v = row_offset; v < n; v += row_stride) rows.push_back(v);
    std::vector<long> kept(rows.size(), 0);
    pump::parallel_for(rows.size(), workers, [&](std::size_t lo, std::size_t hi) {
      for (std::size_t q = lo; q < hi; ++q) {
        const pump::State& a = nodes[rows[q]];
        for (int u = 0; u < n; ++u) {
          if (u == rows[q]) continue;
          const pump::State& bb = nodes[u];
          if (2.0 * (bb.velocity - a.velocity).norm() >= r_n) continue;
          pump::Motion m = pump::connect(a, bb, tau_max);
          if (!m.ok || m.cost >= r_n || m.tau <= 0) continue;
          if (pump::motion_collides(s.workspace, m, eps_cc)) continue;
          auto wps = pump::motion_waypoints(m, s.dt);
          std::vector<pump::ConvexRegion> regions;
          regions.reserve(wps.size());
          bool valid = true;
          for (std::size_t j = 1; j < wps.size(); ++j) {
            if (!pump::point_free(s.workspace, wps[j].state.position)) {
              valid = false;
              break;
            }
            regions.push_back(pump::local_convex_region(s.workspace, wps[j].state.position, wps[j].state.velocity));
          }
          if (valid) kept[q]++;
        }
      }
    });
    auto t1 = clk::now();
    // bank + explore on the full graph (pump.hpp:194-208)
    pump::DeviationBank bank = pump::presample_bank(b.mb.dm, b.mb.gains, s.initial_covariance, s.bank_horizon,
                                                    s.particles, s.seeds.bank, workers);
    pump::ExploreParams ep;
    const double eta = s.effective_eta();
    ep.alpha_min = s.alpha / eta;
    ep.alpha_max = std::min(1.0, eta * s.alpha);
    ep.lambda = s.lambda;
    ep.r_n = r_n;
    ep.workers = workers;
    pump::ExploreResult ex = pump::explore(b.g, bank, ep);
    auto t2 = clk::now();
    // the selection phase's certifications on a rollout sample
    long hits = 0;
    for (const auto& c : b.trace) {
      const int n_s = std::max(1, c.n_mc / mc_stride);
      hits += static_cast<long>(pump::mc_certify(c.y, b.mb.cl, s.workspace, n_s, c.seed, c.eps_cc, workers).value *
                                n_s);
    }
    auto t3 = clk::now();
    long edges = 0;
    for (long k : kept) edges += k;
    out[0] = secs(t0, t_s);  // sample_free (full)
    out[1] = secs(t_s, t1);  // sampled rows
    out[2] = secs(t1, t2);   // bank + explore (full)
    out[3] = secs(t2, t3);   // sampled certifications
    out[4] = static_cast<double>(rows.size());
    out[5] = static_cast<double>(edges);
    out[6] = static_cast<double>(ex.stats.partial_plans);
    out[7] = static_cast<double>(hits);
    // estimate of the full solve (seconds)
    out[8] = out[0] + out[1] * (static_cast<double>(n) / std::max<size_t>(1, rows.size())) + out[2] +
             out[3] * mc_stride;
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 1;
  }
}

void ref_bench_free(void* handle) { delete static_cast<RefBench*>(handle); }

}  // extern "C"
