// Device-resident SampleGraph (graph.hpp:25-37) in CSR form.
#pragma once

#include "../ctx.h"

namespace pumpg {

struct DevGraph {
  int n = 0, dw = 0;
  double r_n = 0, dt = 0;
  // H: half-spaces over all waypoints (the reference's count); H_pk: records
  // stored in hs_pk (the edges' end waypoints share their end node's records)
  int64_t E = 0, NW = 0, H = 0, H_pk = 0, n_cand = 0, n_connect = 0;
  DBuf pos, vel;                                          // n x dw
  DBuf row_ptr;                                           // n + 1 (int64)
  DBuf e_from, e_to, e_cost, e_tau, e_acc0, e_jerk, e_nsteps;
  DBuf wp_off;                                            // E + 1 (int64)
  DBuf hs_off;                                            // NW (+ n): first half-space of each waypoint (then node)
  int64_t hs_cap = 0;                                     // half-space slots in hs_pk/hs_fb
  DBuf hs_cnt;                                            // NW: half-spaces of each waypoint
  // half-spaces packed 32 B each {a_0 .. a_{dw-1}, (pad), b at [3]}: one
  // pair of 16-byte loads per half-space in the explore expand kernel
  DBuf hs_pk, hs_fb;                                      // H x 4 doubles, H
  std::vector<int32_t> goal_nodes;                        // host, ascending
  std::vector<double> h_pos, h_vel;                       // host copies of the nodes
};

// Edges of source rows [row_lo, row_hi) (default: all).  With gather, the
// row slices of all ranks of c's communicator are concatenated over NCCL into
// the full graph on every rank (rows are contiguous per rank and edges are
// row-major, so the global arrays are the rank-ordered concatenation and
// row_ptr is the sum of the ranks' local row_ptr).  Regions are then built
// for every edge present.
void build_graph_device(DevGraph& G, Ctx& c, int n, int dw, const double* h_pos, const double* h_vel,
                        const DevWorld& w, double r_n, double dt, double eps_cc, double tau_max, double ratio,
                        int row_lo = 0, int row_hi = -1, bool gather = false);

}  // namespace pumpg

struct pump_graph {
  pumpg::DevGraph g;
  pump_ctx* owner = nullptr;
};
