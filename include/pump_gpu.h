/*
 * pump_gpu.h — C ABI of libpump_gpu.so, the B200 (sm_100a) data-parallel core
 * of PUMP (arXiv 1607.06886).
 *
 * The reference library is header-only C++ (namespace pump) with no FFI of
 * its own; its hot-path entry points are the C++ functions cited next to each
 * declaration below.  This header is the thin C layer those C++ entry points
 * sit on in this build: POD structs, caller-owned buffers, int status codes
 * mapped 1:1 onto the reference's exception types (see pump_last_error()).
 * include/pump/ headers re-expose the reference's C++ signatures on top of it;
 * INTEGRATION.md shows the ctypes / C++ bindings.
 *
 * Conventions
 *  - Matrices are dense, row-major, binary64.
 *  - Every call is synchronous from the caller's view (stream-ordered inside).
 *  - One pump_ctx per host thread; a ctx owns one CUDA device + stream and the
 *    device-resident particle bank / graph buffers.
 *  - No CPU fallback: if the CUDA runtime or an sm_100a device is missing the
 *    call fails with PUMP_E_CUDA.
 */
#ifndef PUMP_GPU_H
#define PUMP_GPU_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Status codes <-> reference exception types. */
enum {
  PUMP_OK = 0,
  PUMP_E_INVALID_ARGUMENT = 1, /* std::invalid_argument   (lti.hpp:51, cp.hpp:217, graph.hpp:53, geom.hpp:191) */
  PUMP_E_OUT_OF_RANGE = 2,     /* std::out_of_range       (cp.hpp:186-187) */
  PUMP_E_RUNTIME = 3,          /* std::runtime_error      (geom.hpp:220, lti.hpp:130-171, sample.hpp:84) */
  PUMP_E_SCENARIO = 4,         /* pump::ScenarioError     (scenario.hpp:18-20) */
  PUMP_E_CUDA = 5,             /* device / driver failure (no reference analogue) */
  PUMP_E_CAPACITY = 6,         /* caller buffer or device arena too small */
  PUMP_E_LOGIC = 7,            /* std::logic_error        (planner.hpp:303) */
  PUMP_E_HOOK = 8              /* a round hook asked to stop (pump_explore_run_hooked) */
};

/* Message of the last failing call on this thread ("" if none). */
const char* pump_last_error(void);
int pump_abi_version(void);

/* ------------------------------------------------------------------ types */

/* ClosedLoopDynamics (lti.hpp:181-190): z_{t+1} = F z + Gv (Sv nv) + Gw (Sw nw). */
typedef struct pump_closed_loop {
  int32_t d, dw;     /* state dim d = 2 dw for the double integrator */
  const double* F;   /* 2d x 2d */
  const double* Gv;  /* 2d x d  */
  const double* Gw;  /* 2d x dw */
  const double* Sv;  /* d x d   */
  const double* Sw;  /* dw x dw */
  const double* S0;  /* d x d   */
  const double* C;   /* dw x d  */
} pump_closed_loop;

/* Workspace (geom.hpp:41-52): bounds minus a union of closed AABBs. */
typedef struct pump_workspace {
  int32_t dw, n_obs;
  const double* bounds_lo; /* dw */
  const double* bounds_hi; /* dw */
  const double* obs_lo;    /* n_obs x dw */
  const double* obs_hi;    /* n_obs x dw */
} pump_workspace;

/* GoalRegion (sample.hpp:22-29). */
typedef struct pump_goal {
  const double* lo; /* dw */
  const double* hi; /* dw */
  double max_speed;
} pump_goal;

/* Flat SampleGraph (graph.hpp:18-37): CSR rows in ascending neighbour order,
 * per-edge Motion (tau, cost, acc0, jerk), per-waypoint ConvexRegion
 * (waypoints 1..n_steps of each edge, graph.hpp:80-87) as half-space lists. */
typedef struct pump_graph_view {
  int32_t n_nodes, dw;
  int64_t n_edges, n_waypoints, n_halfspaces;
  int32_t n_goal;
  double r_n, dt;
  double* node_pos;      /* n_nodes x dw */
  double* node_vel;      /* n_nodes x dw */
  int64_t* row_ptr;      /* n_nodes + 1 */
  int32_t* edge_to;      /* n_edges */
  double* edge_cost;     /* n_edges */
  double* edge_tau;      /* n_edges */
  double* edge_acc0;     /* n_edges x dw */
  double* edge_jerk;     /* n_edges x dw */
  int32_t* edge_nsteps;  /* n_edges */
  int64_t* edge_wp_off;  /* n_edges + 1  (edge e owns waypoints [off[e], off[e+1])) */
  int64_t* wp_hs_off;    /* n_waypoints + 1 */
  double* hs_a;          /* n_halfspaces x dw */
  double* hs_b;          /* n_halfspaces */
  uint8_t* hs_fallback;  /* n_halfspaces */
  int32_t* goal_nodes;   /* n_goal, ascending */
} pump_graph_view;

/* ExploreParams (planner.hpp:26-32). */
typedef struct pump_explore_params {
  double alpha_min, alpha_max, lambda, r_n;
} pump_explore_params;

/* ExploreResult (planner.hpp:17-48) flattened. termination: 0 =
 * "goal_below_alpha_min", 1 = "frontier_exhausted". */
typedef struct pump_explore_view {
  int64_t n_plans;
  int32_t n_words, n_nodes;
  int64_t n_pareto, n_goal_plans;
  int64_t partial_plans, discarded_cp, removed_dominated, discarded_horizon;
  int32_t rounds, termination;
  int32_t* head;        /* n_plans */
  int32_t* parent;      /* n_plans */
  double* cost;         /* n_plans */
  double* cp_hat;       /* n_plans */
  int32_t* t_end;       /* n_plans */
  uint64_t* masks;      /* n_plans x n_words (may be NULL on export) */
  int64_t* pareto_ptr;  /* n_nodes + 1 */
  int32_t* pareto_ids;  /* n_pareto (ascending ids per node) */
  int32_t* goal_plans;  /* n_goal_plans */
} pump_explore_view;

/* PumpResult (pump.hpp:148-165) scalar part. */
typedef struct pump_result_summary {
  int32_t success, termination;
  int32_t path_len, n_pareto, n_mc_evals, n_traj_points, dw;
  int64_t partial_plans;
  double cost, certified_cp, cp_hat, pre_smoothing_cost, smoothing_s;
  double build_graph_seconds, explore_seconds, selection_seconds;
  /* device-side breakdown (CUDA events), not in the reference report */
  double bank_ms, explore_kernel_ms, mc_ms;
  int64_t n_edges, n_plans, mc_rollouts;
  /* repeated_rrt results (pump_rrt_run; 0 for pump_run) */
  int32_t rrt_trials_reaching_goal, rrt_certification_attempts;
  /* explore: half-spaces of every expanded edge (the HBM-byte model's region reads) */
  int64_t explore_hs_read;
} pump_result_summary;

typedef struct pump_ctx pump_ctx;
typedef struct pump_graph pump_graph;
typedef struct pump_explore pump_explore;
typedef struct pump_result pump_result;
typedef struct pump_scenario pump_scenario;

/* ---------------------------------------------------------------- context */
int pump_ctx_create(int device, pump_ctx** out);
int pump_ctx_destroy(pump_ctx* ctx);
/* CUDA-event time of the last kernel family launched by the ctx, ms. */
double pump_ctx_last_kernel_ms(pump_ctx* ctx);
/* Number of kernel launches issued by this ctx since creation. */
int64_t pump_ctx_launch_count(pump_ctx* ctx);
/* The context's CUDA stream (cudaStream_t) every call of this ctx is ordered
 * on: callers time or order their own work against it. */
int pump_ctx_stream(pump_ctx* ctx, void** stream_out);
/* Measurement hooks (bench.py): per-kernel-family CUDA-event timing on the
 * launching stream; read returns total ms, launch counts and algorithmic work
 * units per family (PUMP_FAM_* order, PUMP_FAM_COUNT entries) and resets them. */
enum {
  PUMP_FAM_BANK_NOISE, PUMP_FAM_BANK_REC, PUMP_FAM_HSMC, PUMP_FAM_MC, PUMP_FAM_CONNECT, PUMP_FAM_COLLIDE,
  PUMP_FAM_EMIT, PUMP_FAM_REGIONS, PUMP_FAM_EXPAND, PUMP_FAM_COMMIT, PUMP_FAM_DOM, PUMP_FAM_SCAN,
  PUMP_FAM_SPLIT, PUMP_FAM_MISC, PUMP_FAM_PAIR, PUMP_FAM_MC_TABLE, PUMP_FAM_COUNT
};
int pump_ctx_profile(pump_ctx* ctx, int enable);
int pump_ctx_profile_read(pump_ctx* ctx, double* ms, int64_t* counts, int64_t* work);
/* out[0] host->device bytes, out[1] device->host bytes, out[2] MC rollout-steps,
 * out[3] device allocations made so far (process-wide), out[4] collectives
 * issued (NCCL or host).  `out` holds 5 values. */
int pump_ctx_io_bytes(pump_ctx* ctx, int64_t* out);
/* Overwrite a 256 MiB buffer (> 126 MB L2) on the ctx stream and synchronize. */
int pump_ctx_flush_l2(pump_ctx* ctx);
/* FP64 DMUL+DADD issue-rate microbenchmark, Gop/s (roofline denominator). */
int pump_peak_fp64(pump_ctx* ctx, double* gops);
/* Latency floor of the explore round: microseconds per grid barrier of the
 * cooperative round kernel's grid, and per dependent L2-resident load. */
int pump_probe_round_latency(pump_ctx* ctx, double* us_barrier, double* us_l2_load);

/* ------------------------------------------------- host geometry queries */
/* Single-call queries for the drop-in C++ headers; they run the same
 * __host__ __device__ code as the kernels (bit-identical results). */
/* connect (steer.hpp:111-182): out3 = {ok, tau, cost}; acc0/jerk[dw] when ok */
int pump_connect(int32_t dw, const double* ap, const double* av, const double* bp, const double* bv, double tau_max,
                 double* out3, double* acc0, double* jerk);
double pump_steer_cost(int32_t dw, const double* ap, const double* av, const double* bp, const double* bv,
                       double tau);                                                   /* steer.hpp:84-94 */
int pump_fixed_time_connect(int32_t dw, const double* ap, const double* av, const double* bp, const double* bv,
                            double tau, double* cost, double* acc0, double* jerk);    /* steer.hpp:97-107 */
int pump_point_free(const pump_workspace* ws, const double* y);                       /* geom.hpp:56-61 */
int pump_segment_hits_aabb(int32_t dw, const double* p0, const double* p1, const double* lo,
                           const double* hi);                                         /* geom.hpp:64-80 */
int pump_motion_collides(const pump_workspace* ws, const double* fp, const double* fv, const double* tp,
                         const double* tv, double tau, const double* acc0, const double* jerk, double eps_cc,
                         int32_t* out);                                               /* geom.hpp:96-123 */
int pump_local_convex_region(const pump_workspace* ws, const double* y, const double* ydot, int32_t cap,
                             double* a, double* b, uint8_t* fallback, int32_t* n_out); /* geom.hpp:189-225 */
int pump_sample_free(int32_t n, const pump_workspace* ws, double max_speed, const pump_goal* goal, int32_t cap,
                     double* pos, double* vel, int32_t* n_out);                       /* sample.hpp:56-89 */
/* motion_waypoints (steer.hpp:192-212): returns the count (writes <= cap). */
int32_t pump_waypoints(int32_t dw, const double* fp, const double* fv, const double* tp, const double* tv,
                       double tau, const double* acc0, const double* jerk, double dt, int32_t cap, double* t_out,
                       double* p_out, double* v_out, double* u_out);

/* ------------------------------------------------------------ multi-GPU */
/* Sharded MC certification: rank r simulates rollouts
 * [n r / W, n (r+1) / W) of every certification in pump_run and the int64
 * hit counts are summed with ncclAllReduce on the ctx stream.  The 128-byte
 * ncclUniqueId comes from rank 0's pump_nccl_unique_id, broadcast by the
 * caller (e.g. torch.distributed). */
int pump_nccl_unique_id(uint8_t* out128);
int pump_ctx_set_comm(pump_ctx* ctx, int rank, int world, const uint8_t* id128);
/* The same sharding over caller-supplied host collectives instead of NCCL
 * (e.g. a torch.distributed gloo group: several ranks may then share one
 * GPU, since no kernel waits on another rank).  allreduce: in-place int64 sum
 * of `count` values over all ranks.  gather: every rank contributes its
 * len[rank] bytes `send`; on return `recv` holds rank r's bytes at offset
 * off[r] for every r (off/len have `world` entries).  Both return 0 on
 * success.  Device data is staged through host memory around each call.
 * world <= 1 (or NULL functions) removes them. */
typedef int (*pump_allreduce_i64_fn)(void* user, int64_t* values, int64_t count);
typedef int (*pump_gather_fn)(void* user, const void* send, void* recv, const int64_t* off, const int64_t* len,
                              int32_t world);
int pump_ctx_set_collectives(pump_ctx* ctx, int rank, int world, pump_allreduce_i64_fn allreduce,
                             pump_gather_fn gather, void* user);
int pump_shard_range(int64_t n, int rank, int world, int64_t* lo, int64_t* hi);

/* ------------------------------------------------------------- scenario */
/* load_scenario / parse_scenario / build_models (scenario.hpp:144-301). */
int pump_scenario_parse(const char* json_text, pump_scenario** out);
int pump_scenario_load(const char* path, pump_scenario** out);
int pump_scenario_free(pump_scenario* s);
/* Closed-loop matrices of build_models(s).cl; buffers sized by d, dw
 * (pass NULL buffers to query d, dw only). */
int pump_scenario_closed_loop(const pump_scenario* s, int32_t* d, int32_t* dw, double* F, double* Gv, double* Gw,
                              double* Sv, double* Sw, double* S0, double* C);
/* JSON-scenario scalars: eps_cc, r_n, tau_max, alpha, eta, lambda, dt. */
int pump_scenario_params(const pump_scenario* s, double out[8], int64_t iout[8]);
/* repeated_rrt (rrt.hpp:50-147), the goal-biased kinodynamic RRT baseline of
 * the paper's Table 1, on the GPU (one warp per trial) with the reference's
 * certification order.  trials <= 0 / alpha < 0 / n_mc <= 0 take the
 * scenario's rrt.trials / alpha / mc_samples.  The result carries success,
 * cost, certified_cp, the trajectory (pump_result_arrays) and
 * rrt_trials_reaching_goal / rrt_certification_attempts. */
int pump_rrt_run(pump_ctx* ctx, const pump_scenario* scenario, int32_t trials, double alpha, int32_t n_mc,
                 pump_result** out);
/* The node set run_pump plans over (pump.hpp:184-189): x_init, then the
 * accepted Halton states (sample.hpp:56-89), then the appended goal sample if
 * any.  Writes n_out; fills pos/vel (n x dw, row-major) when both are given
 * (PUMP_E_OUT_OF_RANGE if n > cap).  Host only. */
int pump_scenario_nodes(const pump_scenario* s, int32_t cap, double* pos, double* vel, int32_t* n_out);

/* ---------------------------------------------------- particle bank (K_bank) */
/* presample_bank (lti.hpp:257-292).  The bank stays resident in the ctx;
 * dy_out (nullable) receives (t_max+1) x n x dw doubles. */
int pump_presample_bank(pump_ctx* ctx, const pump_closed_loop* cl, int32_t t_max, int32_t n, uint64_t seed,
                        double* dy_out);
/* Replace the ctx bank by a caller-provided one (hand-built banks). */
int pump_bank_upload(pump_ctx* ctx, int32_t n, int32_t horizon, int32_t dw, const double* dy);

/* ------------------------------------------------------ HSMC (K_hsmc) */
/* Batched hsmc_extend (cp.hpp:180-208) against the ctx bank.  Task i extends
 * masks_in[i*n_words..] along steps [step_off[i], step_off[i+1]); step s
 * checks bank row step_t[s] against half-spaces [step_hs_off[s],
 * step_hs_off[s+1]) of (hs_a, hs_b).  A step with an empty list is the
 * reference's null/empty region.  Out: masks_out, popcounts; cp = 1 -
 * popcount/n.  Returns PUMP_E_OUT_OF_RANGE if any step_t is outside
 * [0, horizon] (checked before the empty-region skip, as cp.hpp:186-188). */
int pump_hsmc_extend_batch(pump_ctx* ctx, int64_t n_tasks, int32_t n_words, const uint64_t* masks_in,
                           const int64_t* step_off, const int32_t* step_t, const int64_t* step_hs_off,
                           const double* hs_a, const double* hs_b, uint64_t* masks_out, int32_t* popcount_out);

/* ----------------------------------------------- MC certification (K_mc) */
/* Batched mc_certify (cp.hpp:214-268): trajectory j = y_nom rows
 * [traj_off[j], traj_off[j+1]) (dw doubles each).  Rollouts
 * [rollout_lo, rollout_hi) of n_mc are simulated for every trajectory (the
 * multi-GPU shard); hits_out[j] = number of colliding rollouts in the range.
 * value = hits / n_mc once summed over shards (bit-identical for any split). */
int pump_mc_certify_batch(pump_ctx* ctx, const pump_closed_loop* cl, const pump_workspace* ws, int32_t n_traj,
                          const int64_t* traj_off, const double* y_nom, int64_t rollout_lo, int64_t rollout_hi,
                          uint64_t seed, double eps_cc, int64_t* hits_out);
/* Single-trajectory convenience with the reference's signature semantics;
 * value_out = n_hit / n_mc. */
/* smooth (pump.hpp:84-146): blend the plan trajectory (n_points waypoints:
 * times t, positions / velocities / controls n_points x dw) toward the
 * fixed-time optimal motion between its end states; the blend fraction is
 * bisected (s = 1, then 10 midpoints), each probe a nominal collision check
 * and an MC certification with (n_mc, seed, eps_cc), in depth-2 speculative
 * device batches exactly as run_pump does.  plan_mc is the plan's own MC CP
 * (kept when no blend certifies).  Out: the accepted trajectory (same times),
 * out3 = {cost, certified CP, s}. */
int pump_smooth(pump_ctx* ctx, const pump_closed_loop* cl, const pump_workspace* ws, int32_t n_points,
                const double* t, const double* pos, const double* vel, const double* ctrl, double plan_mc,
                double alpha, int32_t n_mc, uint64_t seed, double eps_cc, double* out_pos, double* out_vel,
                double* out_ctrl, double* out3);
int pump_mc_certify(pump_ctx* ctx, const pump_closed_loop* cl, const pump_workspace* ws, int32_t n_points,
                    const double* y_nom, int32_t n_mc, uint64_t seed, double eps_cc, double* value_out);

/* ------------------------------------------------ graph build (K_graph) */
/* build_graph (graph.hpp:50-95) for nodes (pos, vel: n x dw). tau_ratio is
 * pow(tau_max / (tau_max*1e-7), 1/63), pass <= 0 to let the library compute
 * it with the host libm exactly as steer.hpp:133 does. */
int pump_build_graph(pump_ctx* ctx, int32_t n_nodes, int32_t dw, const double* pos, const double* vel,
                     const pump_workspace* ws, const pump_goal* goal, double r_n, double dt, double eps_cc,
                     double tau_max, pump_graph** out);
/* The edges of source rows [row_lo, row_hi) only (a multi-GPU rank's slice,
 * SURVEY §8e): row_ptr is 0 before the slice and the slice's edge count after
 * it; regions are built for the slice's edges.  The slices of a partition of
 * [0, n) concatenate (edges, waypoints, half-spaces) and sum (row_ptr) to the
 * full graph.  With a communicator set, pump_build_graph does exactly this per
 * rank and gathers the slices over NCCL. */
int pump_build_graph_rows(pump_ctx* ctx, int32_t n_nodes, int32_t dw, const double* pos, const double* vel,
                          const pump_workspace* ws, const pump_goal* goal, double r_n, double dt, double eps_cc,
                          double tau_max, int32_t row_lo, int32_t row_hi, pump_graph** out);
/* Upload a prebuilt graph (pump.hpp:170 "prebuilt"). Reads every field. */
int pump_graph_upload(pump_ctx* ctx, const pump_graph_view* view, pump_graph** out);
/* Sizes into view (pointers untouched); then export into caller buffers
 * (any NULL pointer is skipped). */
int pump_graph_counts(const pump_graph* g, pump_graph_view* view);
int pump_graph_export(const pump_graph* g, pump_graph_view* view);
int pump_graph_free(pump_graph* g);

/* ----------------------------------------------------- explore (K_hsmc..) */
/* explore (planner.hpp:74-267) on the ctx bank; wavefront on one GPU. */
int pump_explore_run(pump_ctx* ctx, const pump_graph* g, const pump_explore_params* p, pump_explore** out);
/* RoundHook (planner.hpp:51-52, 245): explore with an observer called after
 * every round (rounds then run one at a time, unpipelined).  `state` is the
 * exploration so far: pump_explore_counts / pump_explore_export on it return
 * the arena, the per-node Pareto sets and the statistics as the reference's
 * hook sees them (goal_plans empty until the run ends); `expanded` lists the
 * group the round expanded.  A nonzero return stops the run with
 * PUMP_E_HOOK (the C++ drop-in rethrows the hook's own exception). */
typedef int (*pump_round_hook)(void* user, int32_t round, const pump_explore* state, const int32_t* expanded,
                               int64_t n_expanded);
int pump_explore_run_hooked(pump_ctx* ctx, const pump_graph* g, const pump_explore_params* p, pump_round_hook hook,
                            void* user, pump_explore** out);
int pump_explore_counts(const pump_explore* e, pump_explore_view* view);
int pump_explore_export(const pump_explore* e, pump_explore_view* view);
int pump_explore_free(pump_explore* e);

/* ------------------------------------------------------ full pipeline */
/* run_pump (pump.hpp:170-263). prebuilt may be NULL. */
int pump_run(pump_ctx* ctx, const pump_scenario* s, const pump_graph* prebuilt, pump_result** out);
int pump_result_summary_get(const pump_result* r, pump_result_summary* out);
/* Caller buffers sized from the summary counts (NULL to skip). */
int pump_result_arrays(const pump_result* r, int32_t* path, double* pareto_cost, double* pareto_cp,
                       int32_t* mc_eval_ids, double* mc_eval_values, double* traj_t, double* traj_pos,
                       double* traj_vel, double* traj_ctrl);
int pump_result_free(pump_result* r);

#ifdef __cplusplus
}
#endif

#endif /* PUMP_GPU_H */
