// ORACLE — TEST INFRASTRUCTURE ONLY.  extern "C" surface of the CPU
// restatement so tests/ (ctypes) and bench.py's cpu_baseline leg can drive it
// with exactly the same flat layouts as libpump_gpu.so (include/pump_gpu.h).
#include <cstring>
#include <memory>
#include <stdexcept>
#include <string>

#include "../include/pump_gpu.h"
#include "../paper_1607_06886_b200/csrc/host/scenario.hpp"
#include "pump_oracle.hpp"

using namespace oracle;

namespace {
thread_local std::string g_err;

template <class F>
int guard(F&& f) {
  try {
    g_err.clear();
    f();
    return PUMP_OK;
  } catch (const pumpb::ScenarioError& e) {
    g_err = e.what();
    return PUMP_E_SCENARIO;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return PUMP_E_INVALID_ARGUMENT;
  } catch (const std::out_of_range& e) {
    g_err = e.what();
    return PUMP_E_OUT_OF_RANGE;
  } catch (const std::logic_error& e) {
    g_err = e.what();
    return PUMP_E_LOGIC;
  } catch (const std::exception& e) {
    g_err = e.what();
    return PUMP_E_RUNTIME;
  }
}

Loop loop_from(const pump_closed_loop* c) {
  Loop l;
  l.d = c->d;
  l.dw = c->dw;
  const int d = c->d, dw = c->dw;
  l.F.assign(c->F, c->F + 4 * d * d);
  l.Gv.assign(c->Gv, c->Gv + 2 * d * d);
  l.Gw.assign(c->Gw, c->Gw + 2 * d * dw);
  l.Sv.assign(c->Sv, c->Sv + d * d);
  l.Sw.assign(c->Sw, c->Sw + dw * dw);
  l.S0.assign(c->S0, c->S0 + d * d);
  l.C.assign(c->C, c->C + dw * d);
  return l;
}

World world_from(const pump_workspace* w) {
  World o;
  o.dw = w->dw;
  o.n_obs = w->n_obs;
  o.blo.assign(w->bounds_lo, w->bounds_lo + w->dw);
  o.bhi.assign(w->bounds_hi, w->bounds_hi + w->dw);
  if (w->n_obs > 0) {
    o.olo.assign(w->obs_lo, w->obs_lo + w->n_obs * w->dw);
    o.ohi.assign(w->obs_hi, w->obs_hi + w->n_obs * w->dw);
  }
  return o;
}

Loop loop_from_mb(const pumpb::ClosedLoop& c) {
  Loop l;
  l.d = c.d;
  l.dw = c.dw;
  l.F = c.F.a;
  l.Gv = c.Gv.a;
  l.Gw = c.Gw.a;
  l.Sv = c.Sv.a;
  l.Sw = c.Sw.a;
  l.S0 = c.S0.a;
  l.C = c.C.a;
  return l;
}

World world_from_scn(const pumpb::World& w) {
  World o;
  o.dw = w.dim();
  o.blo = w.bounds.lo;
  o.bhi = w.bounds.hi;
  o.n_obs = static_cast<int>(w.obstacles.size());
  for (const auto& b : w.obstacles) {
    o.olo.insert(o.olo.end(), b.lo.begin(), b.lo.end());
    o.ohi.insert(o.ohi.end(), b.hi.begin(), b.hi.end());
  }
  return o;
}

Bank bank_from(int n, int horizon, int dw, const double* dy) {
  Bank b;
  b.n = n;
  b.horizon = horizon;
  b.dw = dw;
  b.dy.assign(dy, dy + static_cast<std::size_t>(horizon + 1) * n * dw);
  return b;
}

struct OGraph {
  Graph g;
};
struct OExplore {
  ExResult r;
};
struct ORun {
  PumpOut r;
  int dw = 0;
};

}  // namespace

extern "C" {

const char* oracle_last_error(void) { return g_err.c_str(); }
void oracle_set_normal_mode(int mode) { set_normal_mode(mode); }

double oracle_normal(uint64_t seed, uint64_t a, uint64_t b, uint64_t ch) { return normal(seed, a, b, ch); }
double oracle_uniform(uint64_t seed, uint64_t a, uint64_t b, uint64_t c) { return uniform(seed, a, b, c); }
uint64_t oracle_counter_hash(uint64_t seed, uint64_t a, uint64_t b, uint64_t c) { return counter_hash(seed, a, b, c); }

// n normals for keys (seed, a[i], b[i], ch[i])
void oracle_normals(uint64_t seed, int64_t n, const uint64_t* a, const uint64_t* b, const uint64_t* ch, double* out) {
  for (int64_t i = 0; i < n; ++i) out[i] = normal(seed, a[i], b[i], ch[i]);
}

int oracle_presample_bank(const pump_closed_loop* cl, int t_max, int n, uint64_t seed, int workers, double* dy_out) {
  return guard([&] {
    Bank b = presample_bank(loop_from(cl), t_max, n, seed, workers);
    std::memcpy(dy_out, b.dy.data(), b.dy.size() * sizeof(double));
  });
}

int oracle_hsmc_extend_batch(int n, int horizon, int dw, const double* dy, int64_t n_tasks, int n_words,
                             const uint64_t* masks_in, const int64_t* step_off, const int32_t* step_t,
                             const int64_t* step_hs_off, const double* hs_a, const double* hs_b, uint64_t* masks_out,
                             int32_t* pop_out, int workers) {
  return guard([&] {
    Bank bank = bank_from(n, horizon, dw, dy);
    std::exception_ptr first;
    parallel_for(static_cast<std::size_t>(n_tasks), workers, [&](std::size_t lo, std::size_t hi) {
      std::vector<Region> regions;
      std::vector<std::pair<int, const Region*>> steps;
      for (std::size_t t = lo; t < hi; ++t) {
        regions.clear();
        steps.clear();
        for (int64_t s = step_off[t]; s < step_off[t + 1]; ++s) {
          Region r;
          for (int64_t h = step_hs_off[s]; h < step_hs_off[s + 1]; ++h) {
            Hs x;
            x.a.assign(hs_a + h * dw, hs_a + (h + 1) * dw);
            x.b = hs_b[h];
            r.hs.push_back(x);
          }
          regions.push_back(std::move(r));
        }
        int k = 0;
        for (int64_t s = step_off[t]; s < step_off[t + 1]; ++s, ++k) steps.push_back({step_t[s], &regions[k]});
        Mask m;
        m.n = n;
        m.w.assign(masks_in + t * n_words, masks_in + (t + 1) * n_words);
        auto [out, cp] = hsmc_extend(m, bank, steps);
        (void)cp;
        std::memcpy(masks_out + t * n_words, out.w.data(), n_words * sizeof(uint64_t));
        pop_out[t] = out.popcount();
      }
    });
  });
}

int oracle_mc_hits(const pump_closed_loop* cl, const pump_workspace* ws, int n_points, const double* y_nom,
                   int64_t r0, int64_t r1, uint64_t seed, double eps_cc, int workers, int64_t* hits,
                   uint8_t* flags) {
  return guard([&] {
    std::vector<Vec> y(n_points);
    for (int t = 0; t < n_points; ++t) y[t].assign(y_nom + t * cl->dw, y_nom + (t + 1) * cl->dw);
    std::vector<char> f;
    *hits = mc_hits(y, loop_from(cl), world_from(ws), r0, r1, seed, eps_cc, workers, flags ? &f : nullptr);
    if (flags)
      for (std::size_t i = 0; i < f.size(); ++i) flags[i] = static_cast<uint8_t>(f[i]);
  });
}

// smooth (pump.hpp:84-146) of a plan trajectory: out3 = {cost, mc, s}
int oracle_smooth(const pump_closed_loop* cl, const pump_workspace* ws, int n_points, const double* t,
                  const double* pos, const double* vel, const double* ctrl, double plan_mc, double alpha, int n_mc,
                  uint64_t seed, double eps_cc, int workers, double* out_pos, double* out_vel, double* out_ctrl,
                  double* out3) {
  return guard([&] {
    const int dw = cl->dw;
    std::vector<Wp> plan(n_points);
    for (int q = 0; q < n_points; ++q) {
      plan[q].t = t[q];
      plan[q].s.p.assign(pos + q * dw, pos + (q + 1) * dw);
      plan[q].s.v.assign(vel + q * dw, vel + (q + 1) * dw);
      plan[q].u.assign(ctrl + q * dw, ctrl + (q + 1) * dw);
    }
    Smooth r = smooth(plan, plan_mc, alpha, loop_from(cl), world_from(ws), n_mc, seed, eps_cc, workers);
    for (int q = 0; q < n_points; ++q)
      for (int k = 0; k < dw; ++k) {
        out_pos[q * dw + k] = r.traj[q].s.p[k];
        out_vel[q * dw + k] = r.traj[q].s.v[k];
        out_ctrl[q * dw + k] = r.traj[q].u[k];
      }
    out3[0] = r.cost;
    out3[1] = r.mc;
    out3[2] = r.s;
  });
}

int oracle_mc_certify(const pump_closed_loop* cl, const pump_workspace* ws, int n_points, const double* y_nom,
                      int n_mc, uint64_t seed, double eps_cc, int workers, double* value) {
  if (n_mc < 1) {
    g_err = "mc_certify: need at least one rollout";
    return PUMP_E_INVALID_ARGUMENT;
  }
  int64_t hits = 0;
  int rc = oracle_mc_hits(cl, ws, n_points, y_nom, 0, n_mc, seed, eps_cc, workers, &hits, nullptr);
  if (rc == PUMP_OK) *value = static_cast<double>(hits) / n_mc;
  return rc;
}

// connect (steer.hpp:111-182): out = {ok, tau, cost}, acc0/jerk[dw]
int oracle_connect(int dw, const double* ap, const double* av, const double* bp, const double* bv, double tau_max,
                   double* out3, double* acc0, double* jerk) {
  return guard([&] {
    St a{Vec(ap, ap + dw), Vec(av, av + dw)}, b{Vec(bp, bp + dw), Vec(bv, bv + dw)};
    Mot m = connect(a, b, tau_max, scan_ratio(tau_max));
    out3[0] = m.ok ? 1.0 : 0.0;
    out3[1] = m.tau;
    out3[2] = m.cost;
    for (int k = 0; k < dw && m.ok; ++k) {
      acc0[k] = m.acc0[k];
      jerk[k] = m.jerk[k];
    }
  });
}

double oracle_steer_cost(int dw, const double* ap, const double* av, const double* bp, const double* bv, double tau) {
  St a{Vec(ap, ap + dw), Vec(av, av + dw)}, b{Vec(bp, bp + dw), Vec(bv, bv + dw)};
  return steer_cost(a, b, tau);
}

// motion given by (from, to, tau, acc0, jerk)
int oracle_motion_collides(const pump_workspace* ws, const double* fp, const double* fv, const double* tp,
                           const double* tv, double tau, const double* acc0, const double* jerk, double eps_cc,
                           int* out) {
  return guard([&] {
    const int dw = ws->dw;
    Mot m;
    m.from = {Vec(fp, fp + dw), Vec(fv, fv + dw)};
    m.to = {Vec(tp, tp + dw), Vec(tv, tv + dw)};
    m.tau = tau;
    m.ok = true;
    m.acc0.assign(acc0, acc0 + dw);
    m.jerk.assign(jerk, jerk + dw);
    *out = motion_collides(world_from(ws), m, eps_cc) ? 1 : 0;
  });
}

int oracle_point_free(const pump_workspace* ws, const double* y) { return point_free(world_from(ws), y) ? 1 : 0; }
int oracle_segment_collides(const pump_workspace* ws, const double* p0, const double* p1) {
  return segment_collides(world_from(ws), p0, p1) ? 1 : 0;
}

// local_convex_region: writes up to cap half-spaces (a: cap x dw, b, fallback); *n_out = count
int oracle_local_convex_region(const pump_workspace* ws, const double* y, const double* ydot, int cap, double* a,
                               double* b, uint8_t* fb, int* n_out) {
  return guard([&] {
    const int dw = ws->dw;
    Region r = local_convex_region(world_from(ws), Vec(y, y + dw), Vec(ydot, ydot + dw));
    *n_out = static_cast<int>(r.hs.size());
    if (static_cast<int>(r.hs.size()) > cap) throw std::runtime_error("capacity");
    for (std::size_t i = 0; i < r.hs.size(); ++i) {
      for (int k = 0; k < dw; ++k) a[i * dw + k] = r.hs[i].a[k];
      b[i] = r.hs[i].b;
      fb[i] = r.hs[i].fallback ? 1 : 0;
    }
  });
}

double oracle_halton(uint64_t index, int base) { return halton(index, base); }

// ------------------------------------------------------------------ graph
int oracle_build_graph(int n_nodes, int dw, const double* pos, const double* vel, const pump_workspace* ws,
                       const pump_goal* goal, double r_n, double dt, double eps_cc, double tau_max, int workers,
                       void** out) {
  return guard([&] {
    std::vector<St> nodes(n_nodes);
    for (int i = 0; i < n_nodes; ++i) nodes[i] = {Vec(pos + i * dw, pos + (i + 1) * dw), Vec(vel + i * dw, vel + (i + 1) * dw)};
    Goal g{Vec(goal->lo, goal->lo + dw), Vec(goal->hi, goal->hi + dw), goal->max_speed};
    auto* og = new OGraph;
    try {
      og->g = build_graph(std::move(nodes), world_from(ws), g, r_n, dt, eps_cc, tau_max, workers);
    } catch (...) {
      delete og;
      throw;
    }
    *out = og;
  });
}

int oracle_graph_counts(void* h, pump_graph_view* v) {
  const Graph& g = static_cast<OGraph*>(h)->g;
  v->n_nodes = static_cast<int32_t>(g.nodes.size());
  v->dw = g.nodes.empty() ? 0 : static_cast<int32_t>(g.nodes[0].p.size());
  v->n_edges = v->n_waypoints = v->n_halfspaces = 0;
  for (const auto& row : g.adj)
    for (const auto& e : row) {
      v->n_edges++;
      v->n_waypoints += e.n_steps;
      for (const auto& r : e.regions) v->n_halfspaces += static_cast<int64_t>(r.hs.size());
    }
  v->n_goal = static_cast<int32_t>(g.goal_nodes.size());
  v->r_n = g.r_n;
  v->dt = g.dt;
  return PUMP_OK;
}

int oracle_graph_export(void* h, pump_graph_view* v) {
  const Graph& g = static_cast<OGraph*>(h)->g;
  const int dw = g.nodes.empty() ? 0 : static_cast<int>(g.nodes[0].p.size());
  int64_t e = 0, wp = 0, hs = 0;
  for (std::size_t i = 0; i < g.nodes.size(); ++i) {
    for (int k = 0; k < dw; ++k) {
      if (v->node_pos) v->node_pos[i * dw + k] = g.nodes[i].p[k];
      if (v->node_vel) v->node_vel[i * dw + k] = g.nodes[i].v[k];
    }
  }
  if (v->row_ptr) v->row_ptr[0] = 0;
  if (v->edge_wp_off) v->edge_wp_off[0] = 0;
  if (v->wp_hs_off) v->wp_hs_off[0] = 0;
  for (std::size_t i = 0; i < g.adj.size(); ++i) {
    for (const auto& ed : g.adj[i]) {
      if (v->edge_to) v->edge_to[e] = ed.to;
      if (v->edge_cost) v->edge_cost[e] = ed.m.cost;
      if (v->edge_tau) v->edge_tau[e] = ed.m.tau;
      for (int k = 0; k < dw; ++k) {
        if (v->edge_acc0) v->edge_acc0[e * dw + k] = ed.m.acc0[k];
        if (v->edge_jerk) v->edge_jerk[e * dw + k] = ed.m.jerk[k];
      }
      if (v->edge_nsteps) v->edge_nsteps[e] = ed.n_steps;
      for (const auto& r : ed.regions) {
        for (const auto& x : r.hs) {
          for (int k = 0; k < dw; ++k)
            if (v->hs_a) v->hs_a[hs * dw + k] = x.a[k];
          if (v->hs_b) v->hs_b[hs] = x.b;
          if (v->hs_fallback) v->hs_fallback[hs] = x.fallback ? 1 : 0;
          ++hs;
        }
        ++wp;
        if (v->wp_hs_off) v->wp_hs_off[wp] = hs;
      }
      ++e;
      if (v->edge_wp_off) v->edge_wp_off[e] = wp;
    }
    if (v->row_ptr) v->row_ptr[i + 1] = e;
  }
  if (v->goal_nodes)
    for (std::size_t i = 0; i < g.goal_nodes.size(); ++i) v->goal_nodes[i] = g.goal_nodes[i];
  return PUMP_OK;
}

// Rebuild an oracle graph from a flat view (e.g. the GPU's graph), so the
// oracle explore can run on exactly the same edges.
int oracle_graph_from_view(const pump_graph_view* v, void** out) {
  return guard([&] {
    auto* og = new OGraph;
    Graph& g = og->g;
    const int dw = v->dw;
    g.r_n = v->r_n;
    g.dt = v->dt;
    g.nodes.resize(v->n_nodes);
    for (int i = 0; i < v->n_nodes; ++i)
      g.nodes[i] = {Vec(v->node_pos + i * dw, v->node_pos + (i + 1) * dw),
                    Vec(v->node_vel + i * dw, v->node_vel + (i + 1) * dw)};
    g.adj.resize(v->n_nodes);
    for (int i = 0; i < v->n_nodes; ++i) {
      for (int64_t e = v->row_ptr[i]; e < v->row_ptr[i + 1]; ++e) {
        Edge ed;
        ed.to = v->edge_to[e];
        ed.m.from = g.nodes[i];
        ed.m.to = g.nodes[ed.to];
        ed.m.tau = v->edge_tau[e];
        ed.m.cost = v->edge_cost[e];
        ed.m.ok = true;
        ed.m.acc0.assign(v->edge_acc0 + e * dw, v->edge_acc0 + (e + 1) * dw);
        ed.m.jerk.assign(v->edge_jerk + e * dw, v->edge_jerk + (e + 1) * dw);
        ed.n_steps = v->edge_nsteps[e];
        for (int64_t w = v->edge_wp_off[e]; w < v->edge_wp_off[e + 1]; ++w) {
          Region r;
          for (int64_t h = v->wp_hs_off[w]; h < v->wp_hs_off[w + 1]; ++h) {
            Hs x;
            x.a.assign(v->hs_a + h * dw, v->hs_a + (h + 1) * dw);
            x.b = v->hs_b[h];
            x.fallback = v->hs_fallback ? v->hs_fallback[h] != 0 : false;
            r.hs.push_back(std::move(x));
          }
          ed.regions.push_back(std::move(r));
        }
        g.adj[i].push_back(std::move(ed));
      }
    }
    g.goal_nodes.assign(v->goal_nodes, v->goal_nodes + v->n_goal);
    *out = og;
  });
}

void oracle_graph_free(void* h) { delete static_cast<OGraph*>(h); }

// ---------------------------------------------------------------- explore
int oracle_explore(void* gh, int n, int horizon, int dw, const double* dy, const pump_explore_params* p, int workers,
                   void** out) {
  return guard([&] {
    Bank bank = bank_from(n, horizon, dw, dy);
    ExParams ep;
    ep.alpha_min = p->alpha_min;
    ep.alpha_max = p->alpha_max;
    ep.lambda = p->lambda;
    ep.r_n = p->r_n;
    ep.workers = workers;
    auto* oe = new OExplore;
    oe->r = explore(static_cast<OGraph*>(gh)->g, bank, ep);
    *out = oe;
  });
}

// Pareto invariants of acceptance.cpp:475-571 checked through the round
// hook: counts[0] dominance violations, [1] double expansions, [2] cp
// violations, [3] rounds.
int oracle_explore_invariants(void* gh, int n, int horizon, int dw, const double* dy, const pump_explore_params* p,
                              int64_t* counts) {
  return guard([&] {
    Bank bank = bank_from(n, horizon, dw, dy);
    ExParams ep;
    ep.alpha_min = p->alpha_min;
    ep.alpha_max = p->alpha_max;
    ep.lambda = p->lambda;
    ep.r_n = p->r_n;
    std::vector<char> seen;
    int64_t dom = 0, dup = 0, cpv = 0, rounds = 0;
    Hook hook = [&](int, const ExResult& st, const std::vector<int>& expanded) {
      rounds++;
      for (int id : expanded) {
        if (id >= static_cast<int>(seen.size())) seen.resize(id + 1, 0);
        if (seen[id]) dup++;
        seen[id] = 1;
      }
      for (const auto& set : st.pareto)
        for (std::size_t i = 0; i < set.size(); ++i) {
          const Plan& pi = st.plans[set[i]];
          if (pi.cp >= ep.alpha_max && set[i] != 0) cpv++;
          for (std::size_t j = 0; j < set.size(); ++j) {
            if (i == j) continue;
            const Plan& pj = st.plans[set[j]];
            if (pi.cost > pj.cost && pi.cp >= pj.cp) dom++;
          }
        }
    };
    explore(static_cast<OGraph*>(gh)->g, bank, ep, hook);
    counts[0] = dom;
    counts[1] = dup;
    counts[2] = cpv;
    counts[3] = rounds;
  });
}

// The reference's RoundHook view of every round (planner.hpp:245), flattened
// for the GPU hook parity test: per round [round, n_expanded, expanded...,
// n_plans, partial_plans, discarded_cp, removed_dominated, discarded_horizon,
// n_nodes, |pareto[v]|..., pareto ids...].  *len = items written (or needed).
int oracle_explore_trace(void* gh, int n, int horizon, int dw, const double* dy, const pump_explore_params* p,
                         int64_t* out, int64_t cap, int64_t* len) {
  return guard([&] {
    Bank bank = bank_from(n, horizon, dw, dy);
    ExParams ep;
    ep.alpha_min = p->alpha_min;
    ep.alpha_max = p->alpha_max;
    ep.lambda = p->lambda;
    ep.r_n = p->r_n;
    int64_t k = 0;
    auto put = [&](int64_t x) {
      if (k < cap) out[k] = x;
      ++k;
    };
    Hook hook = [&](int round, const ExResult& st, const std::vector<int>& expanded) {
      put(round);
      put(static_cast<int64_t>(expanded.size()));
      for (int id : expanded) put(id);
      put(static_cast<int64_t>(st.plans.size()));
      put(st.partial_plans);
      put(st.discarded_cp);
      put(st.removed_dominated);
      put(st.discarded_horizon);
      put(static_cast<int64_t>(st.pareto.size()));
      for (const auto& set : st.pareto) put(static_cast<int64_t>(set.size()));
      for (const auto& set : st.pareto)
        for (int id : set) put(id);
    };
    explore(static_cast<OGraph*>(gh)->g, bank, ep, hook);
    *len = k;
  });
}

int oracle_explore_counts(void* h, pump_explore_view* v) {
  const ExResult& r = static_cast<OExplore*>(h)->r;
  v->n_plans = static_cast<int64_t>(r.plans.size());
  v->n_words = r.plans.empty() ? 0 : static_cast<int32_t>(r.plans[0].mask.w.size());
  v->n_nodes = static_cast<int32_t>(r.pareto.size());
  v->n_pareto = 0;
  for (const auto& s : r.pareto) v->n_pareto += static_cast<int64_t>(s.size());
  v->n_goal_plans = static_cast<int64_t>(r.goal_plans.size());
  v->partial_plans = r.partial_plans;
  v->discarded_cp = r.discarded_cp;
  v->removed_dominated = r.removed_dominated;
  v->discarded_horizon = r.discarded_horizon;
  v->rounds = r.rounds;
  v->termination = r.termination == "frontier_exhausted" ? 1 : 0;
  return PUMP_OK;
}

int oracle_explore_export(void* h, pump_explore_view* v) {
  const ExResult& r = static_cast<OExplore*>(h)->r;
  const int W = r.plans.empty() ? 0 : static_cast<int>(r.plans[0].mask.w.size());
  for (std::size_t i = 0; i < r.plans.size(); ++i) {
    const Plan& p = r.plans[i];
    if (v->head) v->head[i] = p.head;
    if (v->parent) v->parent[i] = p.parent;
    if (v->cost) v->cost[i] = p.cost;
    if (v->cp_hat) v->cp_hat[i] = p.cp;
    if (v->t_end) v->t_end[i] = p.t_end;
    if (v->masks)
      for (int k = 0; k < W; ++k) v->masks[i * W + k] = p.mask.w[k];
  }
  int64_t o = 0;
  if (v->pareto_ptr) v->pareto_ptr[0] = 0;
  for (std::size_t i = 0; i < r.pareto.size(); ++i) {
    for (int id : r.pareto[i]) {
      if (v->pareto_ids) v->pareto_ids[o] = id;
      ++o;
    }
    if (v->pareto_ptr) v->pareto_ptr[i + 1] = o;
  }
  if (v->goal_plans)
    for (std::size_t i = 0; i < r.goal_plans.size(); ++i) v->goal_plans[i] = r.goal_plans[i];
  return PUMP_OK;
}

void oracle_explore_free(void* h) { delete static_cast<OExplore*>(h); }

// ---------------------------------------------------------------- run_pump
static PumpIn pump_in_from(const pumpb::Scenario& s) {
  PumpIn in;
  in.w = world_from_scn(s.workspace);
  in.x_init = {s.start_pos, s.start_vel};
  in.goal = {s.goal.lo, s.goal.hi, s.goal_max_speed};
  in.cl = loop_from_mb(s.models().cl);
  in.dt = s.dt;
  in.r_n = s.effective_r_n();
  in.eps_cc = s.effective_eps_cc();
  in.tau_max = s.effective_tau_max();
  in.alpha = s.alpha;
  in.eta = s.effective_eta();
  in.lambda = s.lambda;
  in.max_speed = s.max_speed;
  in.samples = s.samples;
  in.particles = s.particles;
  in.mc_samples = s.mc_samples;
  in.bank_horizon = s.bank_horizon;
  in.seed_bank = s.seeds.bank;
  in.seed_mc = s.seeds.mc;
  return in;
}

// json_text: scenario; prebuilt: oracle graph handle or NULL
int oracle_run_pump(const char* json_text, int workers, void* prebuilt, void** out) {
  return guard([&] {
    pumpb::Scenario s = pumpb::parse_scenario_text(json_text);
    PumpIn in = pump_in_from(s);
    auto* r = new ORun;
    r->dw = s.workspace_dim();
    try {
      r->r = run_pump(in, workers, prebuilt ? &static_cast<OGraph*>(prebuilt)->g : nullptr);
    } catch (...) {
      delete r;
      throw;
    }
    *out = r;
  });
}

// Nodes of the solve (x_init + sample_free), so tests can feed the very
// same nodes to the GPU graph builder.
int oracle_scenario_nodes(const char* json_text, int cap, double* pos, double* vel, int* n_out) {
  return guard([&] {
    pumpb::Scenario s = pumpb::parse_scenario_text(json_text);
    PumpIn in = pump_in_from(s);
    auto nodes = sample_free(in.samples, in.w, in.max_speed, in.goal);
    nodes.insert(nodes.begin(), in.x_init);
    *n_out = static_cast<int>(nodes.size());
    if (static_cast<int>(nodes.size()) > cap) return;
    const int dw = in.w.dw;
    for (std::size_t i = 0; i < nodes.size(); ++i)
      for (int k = 0; k < dw; ++k) {
        pos[i * dw + k] = nodes[i].p[k];
        vel[i * dw + k] = nodes[i].v[k];
      }
  });
}

int oracle_result_summary(void* h, pump_result_summary* o) {
  const ORun* rr = static_cast<ORun*>(h);
  const PumpOut& r = rr->r;
  std::memset(o, 0, sizeof(*o));
  o->success = r.success ? 1 : 0;
  o->termination = r.termination == "frontier_exhausted" ? 1 : 0;
  o->path_len = static_cast<int32_t>(r.path.size());
  o->n_pareto = static_cast<int32_t>(r.pareto.size());
  o->n_mc_evals = static_cast<int32_t>(r.mc_evals.size());
  o->n_traj_points = static_cast<int32_t>(r.traj.size());
  o->dw = rr->dw;
  o->partial_plans = r.partial_plans;
  o->cost = r.cost;
  o->certified_cp = r.certified_cp;
  o->cp_hat = r.cp_hat;
  o->pre_smoothing_cost = r.pre_smoothing_cost;
  o->smoothing_s = r.smoothing_s;
  o->build_graph_seconds = r.build_graph_seconds;
  o->explore_seconds = r.explore_seconds;
  o->selection_seconds = r.selection_seconds;
  o->n_edges = r.n_edges;
  o->n_plans = r.n_plans;
  return PUMP_OK;
}

int oracle_result_arrays(void* h, int32_t* path, double* pc, double* pcp, int32_t* ids, double* mcs, double* tt,
                         double* tp, double* tv, double* tu) {
  const ORun* rr = static_cast<ORun*>(h);
  const PumpOut& r = rr->r;
  const int dw = rr->dw;
  for (std::size_t i = 0; i < r.path.size(); ++i)
    if (path) path[i] = r.path[i];
  for (std::size_t i = 0; i < r.pareto.size(); ++i) {
    if (pc) pc[i] = r.pareto[i].first;
    if (pcp) pcp[i] = r.pareto[i].second;
  }
  for (std::size_t i = 0; i < r.mc_evals.size(); ++i) {
    if (ids) ids[i] = r.mc_evals[i].first;
    if (mcs) mcs[i] = r.mc_evals[i].second;
  }
  for (std::size_t i = 0; i < r.traj.size(); ++i) {
    if (tt) tt[i] = r.traj[i].t;
    for (int k = 0; k < dw; ++k) {
      if (tp) tp[i * dw + k] = r.traj[i].s.p[k];
      if (tv) tv[i * dw + k] = r.traj[i].s.v[k];
      if (tu) tu[i * dw + k] = r.traj[i].u[k];
    }
  }
  return PUMP_OK;
}

void oracle_result_free(void* h) { delete static_cast<ORun*>(h); }

}  // extern "C"

extern "C" {
// build_models(s).cl of a JSON scenario (shared host synthesis, models.hpp);
// scalars: [eps_cc, r_n, tau_max, alpha, eta, lambda, dt, max_speed]
int oracle_scenario_closed_loop(const char* json_text, int32_t* d, int32_t* dw, double* F, double* Gv, double* Gw,
                                double* Sv, double* Sw, double* S0, double* Cm, double* scalars) {
  return guard([&] {
    pumpb::Scenario s = pumpb::parse_scenario_text(json_text);
    *dw = s.workspace_dim();
    *d = 2 * *dw;
    if (scalars) {
      scalars[0] = s.effective_eps_cc();
      scalars[1] = s.effective_r_n();
      scalars[2] = s.effective_tau_max();
      scalars[3] = s.alpha;
      scalars[4] = s.effective_eta();
      scalars[5] = s.lambda;
      scalars[6] = s.dt;
      scalars[7] = s.max_speed;
    }
    if (!F) return;
    pumpb::ClosedLoop cl = s.models().cl;
    std::memcpy(F, cl.F.a.data(), cl.F.a.size() * 8);
    std::memcpy(Gv, cl.Gv.a.data(), cl.Gv.a.size() * 8);
    std::memcpy(Gw, cl.Gw.a.data(), cl.Gw.a.size() * 8);
    std::memcpy(Sv, cl.Sv.a.data(), cl.Sv.a.size() * 8);
    std::memcpy(Sw, cl.Sw.a.data(), cl.Sw.a.size() * 8);
    std::memcpy(S0, cl.S0.a.data(), cl.S0.a.size() * 8);
    std::memcpy(Cm, cl.C.a.data(), cl.C.a.size() * 8);
  });
}

// bisect_select (pump.hpp:23-51) over ids 0..n-1 with given MC values:
// returns success; *plan, *mc; evals (ids in probe order) -> eval_ids[*n_evals]
int oracle_bisect_select(int n, const double* values, double alpha, int* plan, double* mc, int* eval_ids,
                         int* n_evals) {
  std::vector<int> ids(n);
  for (int i = 0; i < n; ++i) ids[i] = i;
  Selection s = bisect_select(ids, [&](int id) { return values[id]; }, alpha);
  *plan = s.plan_id;
  *mc = s.mc;
  *n_evals = static_cast<int>(s.evals.size());
  for (size_t i = 0; i < s.evals.size(); ++i) eval_ids[i] = s.evals[i].first;
  return s.success ? 1 : 0;
}

// fixed_time_connect (steer.hpp:97-107): out = {cost}, acc0/jerk[dw]
void oracle_fixed_time_connect(int dw, const double* ap, const double* av, const double* bp, const double* bv,
                               double tau, double* cost, double* acc0, double* jerk) {
  St a{Vec(ap, ap + dw), Vec(av, av + dw)}, b{Vec(bp, bp + dw), Vec(bv, bv + dw)};
  Mot m = fixed_time_connect(a, b, tau);
  *cost = m.cost;
  for (int k = 0; k < dw; ++k) {
    acc0[k] = m.acc0[k];
    jerk[k] = m.jerk[k];
  }
}

// motion_waypoints (steer.hpp:192-212) of a motion; returns the count (<= cap written)
int oracle_waypoints(int dw, const double* fp, const double* fv, const double* tp, const double* tv, double tau,
                     const double* acc0, const double* jerk, double dt, int cap, double* t_out, double* p_out,
                     double* v_out, double* u_out) {
  Mot m;
  m.from = {Vec(fp, fp + dw), Vec(fv, fv + dw)};
  m.to = {Vec(tp, tp + dw), Vec(tv, tv + dw)};
  m.tau = tau;
  m.ok = true;
  m.acc0.assign(acc0, acc0 + dw);
  m.jerk.assign(jerk, jerk + dw);
  auto w = waypoints(m, dt);
  for (int i = 0; i < static_cast<int>(w.size()) && i < cap; ++i) {
    t_out[i] = w[i].t;
    for (int k = 0; k < dw; ++k) {
      p_out[i * dw + k] = w[i].s.p[k];
      v_out[i * dw + k] = w[i].s.v[k];
      u_out[i * dw + k] = w[i].u[k];
    }
  }
  return static_cast<int>(w.size());
}
}

// ------------------------------------------------------------ repeated_rrt
// rrt.hpp:50-147 for a scenario; trials <= 0 / alpha < 0 / n_mc <= 0 take the
// scenario's rrt.trials / alpha / mc_samples.  out3 = {success, cost,
// certified_cp}, out2 = {trials_reaching_goal, certification_attempts};
// the trajectory (when successful) into t / pos / vel / u (cap points).
extern "C" int oracle_repeated_rrt(const char* json_text, int trials, double alpha, int n_mc, int workers, double* out3,
                                   int32_t* out2, int32_t cap, double* t, double* pos, double* vel, double* u,
                                   int32_t* n_pts) {
  return guard([&] {
    pumpb::Scenario s = pumpb::parse_scenario_text(json_text);
    RrtIn in;
    in.p = pump_in_from(s);
    in.trials = s.rrt.trials;
    in.max_iterations = s.rrt.max_iterations;
    in.goal_bias = s.rrt.goal_bias;
    in.seed_rrt = s.seeds.rrt;
    const RrtOut r = repeated_rrt(in, trials > 0 ? trials : s.rrt.trials, alpha >= 0 ? alpha : s.alpha,
                                  n_mc > 0 ? n_mc : s.mc_samples, workers);
    out3[0] = r.success ? 1.0 : 0.0;
    out3[1] = r.cost;
    out3[2] = r.certified_cp;
    out2[0] = r.trials_reaching_goal;
    out2[1] = r.certification_attempts;
    *n_pts = static_cast<int32_t>(r.traj.size());
    const int dw = s.workspace_dim();
    if (static_cast<int>(r.traj.size()) > cap) return;
    for (std::size_t i = 0; i < r.traj.size(); ++i) {
      if (t) t[i] = r.traj[i].t;
      for (int k = 0; k < dw; ++k) {
        if (pos) pos[i * dw + k] = r.traj[i].s.p[k];
        if (vel) vel[i * dw + k] = r.traj[i].s.v[k];
        if (u) u[i * dw + k] = r.traj[i].u[k];
      }
    }
  });
}
