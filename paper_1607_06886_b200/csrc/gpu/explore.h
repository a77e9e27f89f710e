// Device-resident explore (planner.hpp:74-267) state and driver.
#pragma once

#include <functional>
#include <vector>

#include "graph.h"

namespace pumpg {

struct ExploreStatus {  // read back once per round (pinned)
  long long G, T, K, n_plans, open_count, i, max_bucket, min_bucket, pool_n;
  long long best_goal_bits, min_group_bits;
  long long disc_cp, disc_hor, removed, n_surv, evicted_open, err, touched, hs_tests;
  long long max_goal_tend;  // largest t_end of any plan committed at a goal node
  long long hs_read;        // half-spaces of every expanded edge (SURVEY §8d HBM-byte model)
  // pipelined rounds (k_round_gate): halt 0 run, 1 the loop-top termination
  // holds, 2 a buffer is too small / the round needs the per-kernel path
  long long halt, n_keys, rounds, partial_plans, commit_bytes;
};

struct DevExplore {
  int n = 0, W = 0, N = 0;
  int64_t cap = 0;  // arena capacity (plans)
  DBuf head, parent, cost, cp, t_end, mask, bucket, flags;
  DBuf mem_off, mem_cnt, mem_a, mem_b;  // per-node Pareto members (segmented, ascending ids)
  bool mem_flip = false;
  DBuf pool_a, pool_b;  // open plans not yet collected (ascending ids)
  bool pool_flip = false;
  DBuf group, task_off, task_grp, task_e;  // per task t: its plan (task_grp) and edge (task_e)
  DBuf is_goal, new_cnt, touched, drop, surv, fpos;
  DBuf cand_keep, cand_head, cand_src, cand_tend, cand_cost, cand_cp, cand_mask, cand_rank, new_slot;
  DBuf status_d;
  ExploreStatus* status_h = nullptr;  // pinned: [0] read back synchronously, [1..2] the window's in-flight rounds
  cudaEvent_t status_ev[2] = {nullptr, nullptr};
  // results
  int64_t n_plans = 0, partial_plans = 0, disc_cp = 0, disc_hor = 0, removed = 0, hs_tests = 0, hs_read = 0;
  int rounds = 0;
  unsigned coop_epoch = 0;  // tags the cooperative round's scan status words
  int termination = 0;  // 0 goal_below_alpha_min, 1 frontier_exhausted
  double kernel_ms = 0;
  ~DevExplore();
};

struct ExploreArgs {
  double alpha_min, alpha_max, lambda, r_n;
  // called after every round's status readback (run_pump extends the MC
  // table on the side stream up to the goal plans' largest t_end)
  std::function<void(const ExploreStatus&)> on_round = nullptr;
  // the hook only needs the latest status, not every round's: pipelined
  // batches stay on and it runs once per status read
  bool on_round_batched = false;
  // RoundHook (planner.hpp:51-52, 245): rounds run one at a time and, after
  // each, the observer gets the round number and the group it expanded; the
  // arena, member sets and statistics in the DevExplore are current then
  std::function<void(int round, const std::vector<int32_t>& expanded)> on_round_state = nullptr;
};

void run_explore_device(DevExplore& X, Ctx& c, const DevGraph& G, const ExploreArgs& a);
// microseconds per grid barrier of the round kernel's grid and per dependent L2 load
void probe_round_latency(Ctx& c, double* us_barrier, double* us_load);

}  // namespace pumpg

struct pump_explore {
  pumpg::DevExplore x;
  pump_ctx* owner = nullptr;
  std::vector<int32_t> goal_nodes;
};
