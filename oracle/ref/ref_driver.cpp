// ORACLE/_REF — TEST INFRASTRUCTURE ONLY.
// The reference's OWN headers (/root/reference/proj/include/pump/*.hpp,
// compiled in place, never copied) built against the Eigen-subset shim in
// include/compat, exposed through a tiny C surface so tests can cross-check
// the oracle restatement against the literal reference code paths (glibc
// normals, reference control flow).  Built by oracle/ref/Makefile into
// oracle/_ref/libpumpref.so.
#include <cstring>
#include <string>

#include "pump/pump.hpp"
#include "pump/compare.hpp"
#include "pump/report.hpp"
#include "pump/rrt.hpp"
#include "pump/scenario.hpp"

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

}  // extern "C"
