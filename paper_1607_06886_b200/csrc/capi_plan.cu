// C ABI: build_graph / explore / run_pump (include/pump_gpu.h) and the host
// orchestration of the full solve (pump.hpp:170-263).  Host glue that the
// reference runs on the CPU after exploration (path walk, waypoint
// concatenation, front reduction, Alg. 4 bisection replay, smoothing
// bisection) runs here in C++ with the same __host__ __device__ geometry the
// kernels use; every Monte-Carlo certification runs on the GPU (K_mc).
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstring>
#include <limits>
#include <cstdlib>
#include <map>
#include <numeric>

#include "ctx.h"
#include "gpu/dispatch.cuh"
#include "gpu/explore.h"
#include "gpu/graph.h"
#include "gpu/scan.cuh"
#include "guard.h"

using namespace pumpg;

namespace pumpg {

// ---------------------------------------------------------------- host glue
struct HWp {  // Waypoint (steer.hpp:184-188)
  double t;
  double p[6], v[6], u[6];
};

struct HMotion {
  double p0[6], v0[6], p1[6], v1[6], a[6], j[6];
  double tau;
};

template <int DW>
static MotionD<DW> as_motion(const HMotion& h) {
  MotionD<DW> m;
  for (int k = 0; k < DW; ++k) {
    m.p0[k] = h.p0[k];
    m.v0[k] = h.v0[k];
    m.p1[k] = h.p1[k];
    m.v1[k] = h.v1[k];
    m.a[k] = h.a[k];
    m.j[k] = h.j[k];
  }
  m.tau = h.tau;
  return m;
}

// fixed_time_coeffs (steer.hpp:63-79) + cost
static double fixed_time(HMotion& m, int dw) {
  const double tau = m.tau;
  double effort = 0;
  for (int k = 0; k < dw; ++k) {
    double dp = m.p1[k] - m.p0[k] - m.v0[k] * tau;
    double dv = m.v1[k] - m.v0[k];
    m.a[k] = 6 * dp / (tau * tau) - 2 * dv / tau;
    m.j[k] = -12 * dp / (tau * tau * tau) + 6 * dv / (tau * tau);
    effort += 12 * dp * dp / (tau * tau * tau) - 12 * dp * dv / (tau * tau) + 4 * dv * dv / tau;
  }
  return tau + effort;
}

static void state_at(const HMotion& m, int dw, double s, double* p, double* v) {
  dispatch_dw(dw, [&]<int DW>() { motion_state<DW>(as_motion<DW>(m), s, p, v); });
}

static void control_at(const HMotion& m, int dw, double s, double* u) {  // steer.hpp:53-57
  if (m.tau <= 0) {
    for (int k = 0; k < dw; ++k) u[k] = 0;
    return;
  }
  s = std::clamp(s, 0.0, m.tau);
  for (int k = 0; k < dw; ++k) u[k] = m.a[k] + m.j[k] * s;
}

static std::vector<HWp> motion_waypoints(const HMotion& m, int dw, double dt) {  // steer.hpp:192-212
  std::vector<HWp> out;
  HWp w{};
  if (m.tau <= 0) {
    w.t = 0;
    std::memcpy(w.p, m.p0, sizeof(w.p));
    std::memcpy(w.v, m.v0, sizeof(w.v));
    out.push_back(w);
    return out;
  }
  const int k = static_cast<int>(std::floor(m.tau / dt + 1e-9));
  const double rem = m.tau - k * dt;
  for (int i = 0; i <= k; ++i) {
    const double t = i * dt;
    w.t = t;
    state_at(m, dw, t, w.p, w.v);
    control_at(m, dw, t, w.u);
    out.push_back(w);
  }
  if (rem > 1e-9) {
    w.t = m.tau;
    std::memcpy(w.p, m.p1, sizeof(w.p));
    std::memcpy(w.v, m.v1, sizeof(w.v));
    control_at(m, dw, m.tau, w.u);
    out.push_back(w);
  } else {
    out.back().t = m.tau;
    std::memcpy(out.back().p, m.p1, sizeof(w.p));
    std::memcpy(out.back().v, m.v1, sizeof(w.v));
  }
  return out;
}

static double seq_sqn(const double* x, int n) {
  double s = 0.0;
  for (int k = 0; k < n; ++k) s = s + x[k] * x[k];
  return s;
}

static double trajectory_cost(const std::vector<HWp>& t, int dw) {  // planner.hpp:319-330
  double c = t.empty() ? 0 : t.back().t;
  for (size_t j = 0; j + 1 < t.size(); ++j) {
    const double h = t[j + 1].t - t[j].t;
    double um[6];
    for (int k = 0; k < dw; ++k) um[k] = 0.5 * (t[j].u[k] + t[j + 1].u[k]);
    c += h / 6.0 * (seq_sqn(t[j].u, dw) + 4.0 * seq_sqn(um, dw) + seq_sqn(t[j + 1].u, dw));
  }
  return c;
}

struct HostWorld {
  int dw = 0;
  std::vector<double> lo, hi;
  double blo[6] = {0}, bhi[6] = {0};
  WorldD view() const {
    WorldD w;
    w.n_obs = static_cast<int>(lo.size()) / (dw ? dw : 1);
    w.lo = lo.data();
    w.hi = hi.data();
    for (int k = 0; k < 6; ++k) {
      w.blo[k] = blo[k];
      w.bhi[k] = bhi[k];
    }
    return w;
  }
};

static bool point_free_h(const HostWorld& w, const double* y) {
  bool r = false;
  dispatch_dw(w.dw, [&]<int DW>() { r = point_free<DW>(w.view(), y); });
  return r;
}

// ------------------------------------------------------------ smoothing kernels
// Smoothing probes on the device (pump.hpp:84-146): for each probed blend
// fraction s the blended trajectory (1 - s) plan + s opt (positions and
// velocities, the host blend's expressions), then nominal_free of it
// (pump.hpp:64-75: every waypoint point_free, every positive-length segment's
// cubic Hermite motion_collides).  The positions feed the MC batch directly.
//
// The reference's bisection (pump.hpp:118-141) is chained on the stream in
// depth-2 speculative batches: batch 0 probes s = 1 and the first two
// bisection levels {0.5, 0.75, 0.25}; batch b >= 1 first replays the two steps
// of the previous batch (certified = free and hits / n_mc <= alpha, the host's
// expressions) and then probes m = 0.5 (lo + hi) with both of its children
// 0.5 (m + hi) and 0.5 (lo + m).  Five batches cover the 10 steps.  Once s = 1
// certifies every later probe is marked done (no check, no MC).  The host
// reads the history once and replays the bisection from it.
constexpr int kSmoothSlots = 16;  // 4 + 4 batches x 3
constexpr int kSmoothBatches = 5;
struct SmoothChain {
  // bisection state entering batch b (b = 0: the initial [0, 1]): batch b
  // reads entry b and writes entry b + 1, so the blocks of one launch never
  // read what its first block writes
  double lo[kSmoothBatches + 1], hi[kSmoothBatches + 1];
  int32_t done_b[kSmoothBatches + 1];
  int32_t done, pad;
  double s[kSmoothSlots];
  unsigned long long hits[kSmoothSlots];
  int32_t live[kSmoothSlots];  // 1 until the nominal check fails (0: no MC; also when done)
  unsigned long long steps;
};
__global__ void k_smooth_init(SmoothChain* c) {
  const int q = threadIdx.x;
  if (q < kSmoothSlots) {
    c->live[q] = 1;
    c->hits[q] = 0;
  }
  if (q == 0) {
    c->lo[0] = 0;
    c->hi[0] = 1;
    c->done_b[0] = 0;
    c->done = 0;
    c->steps = 0;
  }
}
__device__ __forceinline__ bool smooth_cert(const SmoothChain* c, int q, int64_t n_mc, double alpha) {
  return c->live[q] != 0 && static_cast<double>(c->hits[q]) / n_mc <= alpha;
}
// one bisection step on probe slots (m, m_hi child, m_lo child)
__device__ __forceinline__ void smooth_two_steps(const SmoothChain* c, int q, int64_t n_mc, double alpha, double& lo,
                                                 double& hi) {
  const bool cm = smooth_cert(c, q, n_mc, alpha);
  if (cm)
    lo = c->s[q];
  else
    hi = c->s[q];
  const int qc = cm ? q + 1 : q + 2;  // the child the bisection visits next
  if (smooth_cert(c, qc, n_mc, alpha))
    lo = c->s[qc];
  else
    hi = c->s[qc];
}
// batch b's decision (the previous batches' verdicts are final): its probes
// s[0..np) and whether the bisection is done
__device__ __forceinline__ void smooth_decide(const SmoothChain* c, int batch, int64_t n_mc, double alpha,
                                              double* sv, double& lo, double& hi, int& done) {
  lo = c->lo[batch];
  hi = c->hi[batch];
  done = c->done_b[batch];
  if (batch == 0) {
    sv[0] = 1.0;
    const double m = 0.5 * (lo + hi);
    sv[1] = m;
    sv[2] = 0.5 * (m + hi);
    sv[3] = 0.5 * (lo + m);
    return;
  }
  const int q0 = 4 + 3 * (batch - 1);
  if (!done) {
    if (batch == 1) {
      if (smooth_cert(c, 0, n_mc, alpha))
        done = 1;  // s = 1 certifies: no bisection
      else
        smooth_two_steps(c, 1, n_mc, alpha, lo, hi);
    } else {
      smooth_two_steps(c, q0 - 3, n_mc, alpha, lo, hi);
    }
  }
  const double m = 0.5 * (lo + hi);
  sv[0] = m;
  sv[1] = 0.5 * (m + hi);
  sv[2] = 0.5 * (lo + m);
}

// One batch in one launch: every block takes the batch's decision itself
// (block 0 records it), then a warp per (probe, waypoint) blends the
// waypoint and its successor, stores the waypoint for the MC batch, and runs
// the nominal check: point_free with the lanes over the boxes, the segment's
// obstacle cull (motion_cull: the boxes not separated from the motion's
// widened bounding box) likewise, then every lane runs motion_collides on the
// warp's candidates (identical data, no divergence).  Same tests, same
// verdicts.  LIST = 0: worlds of at most 64 kCullWords boxes (bitmask);
// LIST = kCullList: larger worlds, the candidates listed in ascending order by
// ballot, all boxes tested past LIST of them (motion_cull's list mode).
template <int DW, int LIST>
__global__ void __launch_bounds__(128) k_smooth_probe(SmoothChain* chn, int batch, int64_t n_mc, double alpha, WorldD w,
                                                      int n_wp, const double* __restrict__ pt,
                                                      const double* __restrict__ pp, const double* __restrict__ pv,
                                                      MotionD<DW> opt, double eps_cc, double* __restrict__ y,
                                                      double* __restrict__ yv,
                                                      const unsigned long long* __restrict__ maxdev,
                                                      uint16_t* __restrict__ g_list, int32_t* __restrict__ g_nl,
                                                      uint8_t* __restrict__ g_skip) {
  extern __shared__ double smem[];
  __shared__ double s_sv[4];
  __shared__ int s_done;
  const int q0 = batch == 0 ? 0 : 4 + 3 * (batch - 1), n_probe = batch == 0 ? 4 : 3;
  if (threadIdx.x == 0) {
    double sv[4], lo, hi;
    int done;
    smooth_decide(chn, batch, n_mc, alpha, sv, lo, hi, done);
    for (int k = 0; k < n_probe; ++k) s_sv[k] = sv[k];
    s_done = done;
    if (blockIdx.x == 0) {
      chn->lo[batch + 1] = lo;
      chn->hi[batch + 1] = hi;
      chn->done_b[batch + 1] = done;
      chn->done = done;
      for (int k = 0; k < n_probe; ++k) {
        chn->s[q0 + k] = sv[k];
        if (done) chn->live[q0 + k] = 0;
      }
    }
  }
  const WorldD ws = stage_world<DW>(w, smem);  // (its __syncthreads publishes s_sv / s_done)
  if (s_done) return;
  const int64_t x = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (x >= static_cast<int64_t>(n_probe) * n_wp) return;
  const int64_t pr = x / n_wp;
  const int j = static_cast<int>(x % n_wp);
  const double sp = s_sv[pr];
  // the blend of waypoints j and j + 1 (k_smooth_blend's expressions)
  double y_j[DW], yv_j[DW], y_n[DW], yv_n[DW];
  {
    double op[DW], ov[DW];
    motion_state<DW>(opt, pt[j], op, ov);
#pragma unroll
    for (int k = 0; k < DW; ++k) {
      y_j[k] = (1 - sp) * pp[j * DW + k] + sp * op[k];
      yv_j[k] = (1 - sp) * pv[j * DW + k] + sp * ov[k];
    }
    if (lane == 0) {
#pragma unroll
      for (int k = 0; k < DW; ++k) {
        y[x * DW + k] = y_j[k];
        yv[x * DW + k] = yv_j[k];
      }
    }
    if (j + 1 < n_wp) {
      motion_state<DW>(opt, pt[j + 1], op, ov);
#pragma unroll
      for (int k = 0; k < DW; ++k) {
        y_n[k] = (1 - sp) * pp[(j + 1) * DW + k] + sp * op[k];
        yv_n[k] = (1 - sp) * pv[(j + 1) * DW + k] + sp * ov[k];
      }
    }
  }
  if (chn->live[q0 + pr] == 0) return;  // another waypoint of this probe already failed
  // the MC batch's candidate lists (k_mc_steps' rows): step 0 and step j + 1
  // (the segment j -> j + 1) of this probe
  if (maxdev) {
    if (j == 0) mc_step_row<DW, kStepCap>(ws, y_j, nullptr, maxdev, 0, pr * n_wp, lane, g_list, g_nl, g_skip);
    if (j + 1 < n_wp)
      mc_step_row<DW, kStepCap>(ws, y_n, y_j, maxdev, j + 1, pr * n_wp + j + 1, lane, g_list, g_nl, g_skip);
  }
  const double* yp = y_j;
  // point_free (geom.hpp:56-61): bounds, then every box, lanes over the boxes
  bool hit = false;
  for (int o = lane; o < ws.n_obs && !hit; o += 32) hit = box_contains<DW>(ws.lo + o * DW, ws.hi + o * DW, yp);
  bool ok = box_contains<DW>(ws.blo, ws.bhi, yp) && !__any_sync(0xffffffffu, hit);
  if (ok && j + 1 < n_wp) {
    const double h = pt[j + 1] - pt[j];
    if (h > 0) {
      MotionD<DW> m;
#pragma unroll
      for (int k = 0; k < DW; ++k) {
        m.p0[k] = yp[k];
        m.v0[k] = yv_j[k];
        m.p1[k] = y_n[k];
        m.v1[k] = yv_n[k];
      }
      m.tau = h;
      coeffs_dev<DW>(m.p0, m.v0, m.p1, m.v1, m.tau, m.a, m.j);
      // motion_cull with the lanes over the boxes (the same separation test)
      MotionCullT<LIST> c;
      double bl[DW], bh[DW];
      motion_bbox<DW>(m, bl, bh);
      c.inside = true;
#pragma unroll
      for (int k = 0; k < DW; ++k) c.inside = c.inside && bl[k] > ws.blo[k] && bh[k] < ws.bhi[k];
      c.masked = true;
      if constexpr (LIST > 0) {
        for (int q = 0; q < kCullWords; ++q) c.cand[q] = 0;
        c.nlist = 0;
        c.any = false;
        for (int o0 = 0; o0 < ws.n_obs && c.masked; o0 += 32) {
          const int o = o0 + lane;
          bool cand = false;
          if (o < ws.n_obs) {
            bool sep = false;
#pragma unroll
            for (int k = 0; k < DW; ++k) sep = sep || (bh[k] < ws.lo[o * DW + k]) || (bl[k] > ws.hi[o * DW + k]);
            cand = !sep;
          }
          unsigned bal = __ballot_sync(0xffffffffu, cand);
          if (bal) c.any = true;
          for (; bal; bal &= bal - 1) {
            if (c.nlist == LIST) {
              c.masked = false;  // too many candidates: every box is tested
              break;
            }
            c.list[c.nlist++] = static_cast<uint16_t>(o0 + __ffs(bal) - 1);
          }
        }
        ok = !motion_collides<DW, LIST>(m, ws, eps_cc, &c);
      } else {
      c.nlist = -1;
      for (int q = 0; q < kCullWords; ++q) {
        uint64_t word = 0;
        for (int half = 0; half < 2; ++half) {
          const int o = q * 64 + half * 32 + lane;
          bool cand = false;
          if (o < ws.n_obs) {
            bool sep = false;
#pragma unroll
            for (int k = 0; k < DW; ++k) sep = sep || (bh[k] < ws.lo[o * DW + k]) || (bl[k] > ws.hi[o * DW + k]);
            cand = !sep;
          }
          word |= static_cast<uint64_t>(__ballot_sync(0xffffffffu, cand)) << (32 * half);
        }
        c.cand[q] = word;
      }
      c.any = (c.cand[0] | c.cand[1] | c.cand[2] | c.cand[3]) != 0;
      ok = !motion_collides<DW>(m, ws, eps_cc, &c);
      }
    }
  }
  if (!ok && lane == 0) chn->live[q0 + pr] = 0;
}


// ------------------------------------------------------------ path kernels
// Walk parent pointers of selected plans and resolve each hop to its edge
// (first edge v->u in the ascending row, as planner.hpp:297-302).
__global__ void k_paths(int n_sel, const int32_t* sel, const int32_t* head, const int32_t* parent,
                        const int64_t* row_ptr, const int32_t* e_to, int max_len, int32_t* nodes, int64_t* edges,
                        int32_t* lens) {
  const int s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= n_sel) return;
  int len = 0;
  for (int id = sel[s]; id != -1 && len < max_len; id = parent[id]) nodes[static_cast<int64_t>(s) * max_len + len++] = head[id];
  int32_t* nd = nodes + static_cast<int64_t>(s) * max_len;
  for (int a = 0, b = len - 1; a < b; ++a, --b) {
    const int t = nd[a];
    nd[a] = nd[b];
    nd[b] = t;
  }
  for (int h = 0; h + 1 < len; ++h) {
    const int v = nd[h], u = nd[h + 1];
    int64_t lo = row_ptr[v], hi = row_ptr[v + 1];  // first index with e_to >= u
    while (lo < hi) {
      const int64_t mid = (lo + hi) >> 1;
      if (e_to[mid] < u)
        lo = mid + 1;
      else
        hi = mid;
    }
    edges[static_cast<int64_t>(s) * max_len + h] = (lo < row_ptr[v + 1] && e_to[lo] == u) ? lo : -1;
  }
  lens[s] = len;
}

__global__ void k_gather_members(int n_goal, const int32_t* goal_nodes, const int64_t* mem_off,
                                 const int64_t* out_off, const int32_t* ids, const double* cost, const double* cp,
                                 const int32_t* t_end, int32_t* out_ids, double* out_cost, double* out_cp,
                                 int32_t* out_tend) {
  const int g = blockIdx.x;
  if (g >= n_goal) return;
  const int v = goal_nodes[g];
  const int64_t a = mem_off[v], o = out_off[g], m = out_off[g + 1] - out_off[g];
  for (int64_t k = threadIdx.x; k < m; k += blockDim.x) {
    const int id = ids[a + k];
    out_ids[o + k] = id;
    out_cost[o + k] = cost[id];
    out_cp[o + k] = cp[id];
    out_tend[o + k] = t_end[id];
  }
}

// path_trajectory (planner.hpp:292-315) of every front plan on the device: a
// warp per plan walks its edges in order (the time offset is the running sum
// of the edge durations, as the reference adds them) and the lanes write each
// edge's waypoints (motion_waypoints, steer.hpp:192-212: i dt for i <= k, the
// end state at tau; a later edge drops its first waypoint).  A plan's
// waypoint count is t_end + 1, so the host knows every offset up front.
template <int DW>
__global__ void k_traj_build(int ns, int max_len, const int32_t* __restrict__ nodes, const int64_t* __restrict__ edges,
                             const int32_t* __restrict__ lens, const int64_t* __restrict__ off,
                             const double* __restrict__ pos, const double* __restrict__ vel,
                             const double* __restrict__ e_tau, const double* __restrict__ e_acc0,
                             const double* __restrict__ e_jerk, double dt, double* __restrict__ wt,
                             double* __restrict__ wp, double* __restrict__ wv, double* __restrict__ wu) {
  const int s = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (s >= ns) return;
  const int len = lens[s];
  const int32_t* nd = nodes + static_cast<int64_t>(s) * max_len;
  const int64_t* ed = edges + static_cast<int64_t>(s) * max_len;
  int64_t w = off[s];
  if (len == 1 && lane == 0) {
    wt[w] = 0;
#pragma unroll
    for (int k = 0; k < DW; ++k) {
      wp[w * DW + k] = pos[nd[0] * DW + k];
      wv[w * DW + k] = vel[nd[0] * DW + k];
      wu[w * DW + k] = 0;
    }
  }
  double offset = 0;
  for (int j = 0; j + 1 < len; ++j) {
    const int64_t e = ed[j];
    MotionD<DW> m;
    m.tau = e_tau[e];
    const int v = nd[j], u = nd[j + 1];
#pragma unroll
    for (int k = 0; k < DW; ++k) {
      m.p0[k] = pos[v * DW + k];
      m.v0[k] = vel[v * DW + k];
      m.p1[k] = pos[u * DW + k];
      m.v1[k] = vel[u * DW + k];
      m.a[k] = e_acc0[e * DW + k];
      m.j[k] = e_jerk[e * DW + k];
    }
    int kk = 0, cnt = 1;
    bool extra = false;
    if (m.tau > 0) {
      kk = static_cast<int>(floor(m.tau / dt + 1e-9));
      const double rem = m.tau - kk * dt;
      extra = rem > 1e-9;
      cnt = kk + 1 + (extra ? 1 : 0);
    }
    const int i0 = j == 0 ? 0 : 1;
    for (int i = i0 + lane; i < cnt; i += 32) {
      double t = 0, p[DW], vv[DW], uu[DW];
      if (m.tau <= 0) {
#pragma unroll
        for (int k = 0; k < DW; ++k) {
          p[k] = m.p0[k];
          vv[k] = m.v0[k];
          uu[k] = 0;
        }
      } else if (extra && i == kk + 1) {
        t = m.tau;
#pragma unroll
        for (int k = 0; k < DW; ++k) {
          p[k] = m.p1[k];
          vv[k] = m.v1[k];
          uu[k] = m.a[k] + m.j[k] * m.tau;
        }
      } else {
        t = i * dt;
        motion_state<DW>(m, t, p, vv);
        const double sc = t < 0 ? 0.0 : (m.tau < t ? m.tau : t);  // std::clamp(t, 0, tau)
#pragma unroll
        for (int k = 0; k < DW; ++k) uu[k] = m.a[k] + m.j[k] * sc;
        if (!extra && i == kk) {  // the last waypoint is the end state at tau
          t = m.tau;
#pragma unroll
          for (int k = 0; k < DW; ++k) {
            p[k] = m.p1[k];
            vv[k] = m.v1[k];
          }
        }
      }
      const int64_t x = w + (i - i0);
      wt[x] = t + offset;
#pragma unroll
      for (int k = 0; k < DW; ++k) {
        wp[x * DW + k] = p[k];
        wv[x * DW + k] = vv[k];
        wu[x * DW + k] = uu[k];
      }
    }
    w += cnt - i0;
    offset += m.tau;
  }
}

// Batched MC over trajectories (rollouts [0, n_mc)); values = hits / n_mc
// MC values of nt trajectories already on the device (positions d_y, point
// offsets d_off); this rank's rollouts, hit counts summed over the ranks
static std::vector<double> mc_values_dev(Ctx& c, const HostLoop& L, const DevWorld& w, int nt, const int64_t* d_off,
                                         const double* d_y, int max_pts, int n_mc, uint64_t seed, double eps_cc,
                                         double* mc_ms, int64_t* rollouts) {
  DBuf& d_h = c.buf("r_mc_hits", (nt + 1) * 8 + 256);
  PUMP_CUDA(cudaMemsetAsync(d_h.p, 0, (nt + 1) * 8, c.stream));
  // this rank's rollouts (all of them on one GPU), then the hit counts of all
  // ranks are summed over NVLink (bit-identical for any world size)
  int64_t r0 = 0, r1 = n_mc;
  shard_range(n_mc, c.rank, c.world, &r0, &r1);
  if (c.mc_join_pending) {
    static const bool dbg_join = std::getenv("PUMP_DEBUG_TIMING") != nullptr;
    if (dbg_join) {  // how long the MC table on the side stream keeps the certification waiting
      c.sync();
      const auto a = std::chrono::steady_clock::now();
      PUMP_CUDA(cudaEventSynchronize(c.join));
      std::fprintf(stderr, "[pump t] mc table wait          %8.3f ms\n",
                   1e3 * std::chrono::duration<double>(std::chrono::steady_clock::now() - a).count());
    }
    PUMP_CUDA(cudaStreamWaitEvent(c.stream, c.join, 0));
    c.mc_join_pending = false;
  }
  c.tic();
  launch_mc(L, w, nt, d_off, d_y, max_pts, r0, r1, seed, eps_cc, d_h.as<unsigned long long>(), c.stream, &c.launches,
            d_h.as<unsigned long long>() + nt, &c.mc_table);
  allreduce_sum_i64(c, d_h.as<int64_t>(), nt);
  *mc_ms += c.toc();
  *rollouts += (r1 - r0) * nt;
  std::vector<int64_t> hits(nt + 1);
  c.d2h(hits.data(), d_h.p, (nt + 1) * 8);
  c.sync();
  kprof_work(F_MC, hits[nt]);
  c.mc_rollout_steps += hits[nt];
  std::vector<double> v(nt);
  for (int j = 0; j < nt; ++j) v[j] = static_cast<double>(hits[j]) / n_mc;
  return v;
}

static std::vector<double> mc_values(Ctx& c, const HostLoop& L, const DevWorld& w,
                                     const std::vector<std::vector<HWp>>& trajs, int n_mc, uint64_t seed,
                                     double eps_cc, double* mc_ms, int64_t* rollouts) {
  const int dw = L.dw;
  std::vector<int64_t> off(trajs.size() + 1, 0);
  for (size_t j = 0; j < trajs.size(); ++j) off[j + 1] = off[j] + static_cast<int64_t>(trajs[j].size());
  std::vector<double> y(static_cast<size_t>(off.back()) * dw);
  int max_pts = 0;
  for (size_t j = 0; j < trajs.size(); ++j) {
    if (trajs[j].empty()) throw std::invalid_argument("mc_certify: empty trajectory");
    max_pts = std::max<int>(max_pts, static_cast<int>(trajs[j].size()));
    for (size_t t = 0; t < trajs[j].size(); ++t)
      for (int k = 0; k < dw; ++k) y[(off[j] + t) * dw + k] = trajs[j][t].p[k];
  }
  const int nt = static_cast<int>(trajs.size());
  DBuf& d_off = c.buf("r_mc_off", (nt + 1) * 8 + 256);
  DBuf& d_y = c.buf("r_mc_y", y.size() * 8 + 256);
  c.h2d(d_off.p, off.data(), (nt + 1) * 8);
  c.h2d(d_y.p, y.data(), y.size() * 8);
  return mc_values_dev(c, L, w, nt, d_off.as<int64_t>(), d_y.as<double>(), max_pts, n_mc, seed, eps_cc, mc_ms,
                       rollouts);
}

}  // namespace pumpg

struct pump_result {
  pump_result_summary s{};
  std::vector<int32_t> path;
  std::vector<double> pareto_cost, pareto_cp;
  std::vector<int32_t> mc_ids;
  std::vector<double> mc_vals;
  std::vector<pumpg::HWp> traj;
  int dw = 0;
};

namespace pumpg {

static void graph_goal_nodes(DevGraph& G, const double* pos, const double* vel, const pump_goal* goal) {
  const int dw = G.dw;
  G.goal_nodes.clear();
  for (int i = 0; i < G.n; ++i) {
    bool in = true;
    for (int k = 0; k < dw; ++k)
      if (pos[i * dw + k] < goal->lo[k] || pos[i * dw + k] > goal->hi[k]) in = false;
    if (in && std::sqrt(seq_sqn(vel + i * dw, dw)) <= goal->max_speed) G.goal_nodes.push_back(i);
  }
}

static double scan_ratio(double tau_max) {  // steer.hpp:130-133 (host libm, as the reference)
  const double tau_lo = tau_max * 1e-7;
  return std::pow(tau_max / tau_lo, 1.0 / (64 - 1));
}

// sample_free (sample.hpp:56-89)
static double halton(uint64_t index, int base) {
  double f = 1.0, r = 0.0;
  while (index > 0) {
    f /= base;
    r += f * (index % base);
    index /= base;
  }
  return r;
}

static void halton_state(uint64_t index, const double* lo, const double* hi, int dw, double ms, double* p, double* v) {
  static const int kPrimes[] = {2, 3, 5, 7, 11, 13, 17, 19, 23, 29, 31, 37};
  for (int k = 0; k < dw; ++k) {
    double u = halton(index, kPrimes[k]);
    p[k] = lo[k] + u * (hi[k] - lo[k]);
    double q = halton(index, kPrimes[dw + k]);
    v[k] = -ms + q * 2 * ms;
  }
}

static void sample_nodes(const pumpb::Scenario& s, const HostWorld& w, std::vector<double>& pos,
                         std::vector<double>& vel) {
  const int dw = s.workspace_dim();
  pos.assign(s.start_pos.begin(), s.start_pos.end());
  vel.assign(s.start_vel.begin(), s.start_vel.end());
  auto goal_contains = [&](const double* p, const double* v) {
    for (int k = 0; k < dw; ++k)
      if (p[k] < s.goal.lo[k] || p[k] > s.goal.hi[k]) return false;
    return std::sqrt(seq_sqn(v, dw)) <= s.goal_max_speed;
  };
  bool have_goal = false;
  uint64_t index = 1;
  int got = 0;
  double p[6], v[6];
  while (got < s.samples) {
    halton_state(index++, s.workspace.bounds.lo.data(), s.workspace.bounds.hi.data(), dw, s.max_speed, p, v);
    if (!point_free_h(w, p)) continue;
    have_goal = have_goal || goal_contains(p, v);
    pos.insert(pos.end(), p, p + dw);
    vel.insert(vel.end(), v, v + dw);
    ++got;
  }
  if (!have_goal) {
    for (int k = 0; k < dw; ++k) {
      p[k] = 0.5 * (s.goal.lo[k] + s.goal.hi[k]);
      v[k] = 0.0;
    }
    if (point_free_h(w, p)) {
      pos.insert(pos.end(), p, p + dw);
      vel.insert(vel.end(), v, v + dw);
    } else {
      bool placed = false;
      for (uint64_t gi = 1; gi <= 100000 && !placed; ++gi) {
        halton_state(gi, s.goal.lo.data(), s.goal.hi.data(), dw, s.goal_max_speed, p, v);
        if (std::sqrt(seq_sqn(v, dw)) > s.goal_max_speed) continue;
        if (!point_free_h(w, p)) continue;
        pos.insert(pos.end(), p, p + dw);
        vel.insert(vel.end(), v, v + dw);
        placed = true;
      }
      if (!placed) throw std::runtime_error("sample_free: goal region appears entirely in collision");
    }
  }
}

// ---- node sampling on the device (sample.hpp:56-89, pump.hpp:184-189):
// the Halton candidates of a whole index window are drawn and tested in
// parallel, then the first `samples` free ones are taken in index order (a
// scan of the free flags), which is exactly the reference's sequential
// accept loop.  Same arithmetic as halton_state / point_free above.
static inline size_t al(size_t x) { return (x + 255) & ~size_t(255); }

struct SampleBox {
  double lo[6], hi[6], ms;     // workspace bounds, max speed
  double glo[6], ghi[6], gms;  // goal region
};

__device__ double halton_dev(uint64_t index, int base) {
  double f = 1.0, r = 0.0;
  while (index > 0) {
    f /= base;
    r += f * (index % base);
    index /= base;
  }
  return r;
}

template <int DW>
__global__ void k_halton_cand(SampleBox B, WorldD w, uint64_t idx0, int64_t M, double* __restrict__ cp,
                              double* __restrict__ cv, uint8_t* __restrict__ fr, uint8_t* __restrict__ ing) {
  const int64_t x = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (x >= M) return;
  constexpr int kPrimes[12] = {2, 3, 5, 7, 11, 13, 17, 19, 23, 29, 31, 37};
  const uint64_t index = idx0 + static_cast<uint64_t>(x);
  double p[DW], v[DW];
#pragma unroll
  for (int k = 0; k < DW; ++k) {
    const double u = halton_dev(index, kPrimes[k]);
    p[k] = B.lo[k] + u * (B.hi[k] - B.lo[k]);
    const double q = halton_dev(index, kPrimes[DW + k]);
    v[k] = -B.ms + q * 2 * B.ms;
  }
  const bool free = point_free<DW>(w, p);
  bool in = free;
#pragma unroll
  for (int k = 0; k < DW; ++k) in = in && !(p[k] < B.glo[k] || p[k] > B.ghi[k]);
  in = in && sqrt(sqnorm<DW>(v)) <= B.gms;
#pragma unroll
  for (int k = 0; k < DW; ++k) {
    cp[x * DW + k] = p[k];
    cv[x * DW + k] = v[k];
  }
  fr[x] = free ? 1 : 0;
  ing[x] = in ? 1 : 0;
}

// take the free candidates ranked below `need` into rows row0 + rank
__global__ void k_halton_take(int dw, int64_t M, int64_t need, int64_t row0, const int64_t* __restrict__ rank,
                              const uint8_t* __restrict__ fr, const uint8_t* __restrict__ ing,
                              const double* __restrict__ cp, const double* __restrict__ cv, double* __restrict__ pos,
                              double* __restrict__ vel, int* __restrict__ goal_flag) {
  const int64_t x = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (x >= M || !fr[x]) return;
  const int64_t r = rank[x];
  if (r >= need) return;
  for (int k = 0; k < dw; ++k) {
    pos[(row0 + r) * dw + k] = cp[x * dw + k];
    vel[(row0 + r) * dw + k] = cv[x * dw + k];
  }
  if (ing[x]) atomicOr(goal_flag, 1);
}

// the goal fallback of sample_free (sample.hpp:63-88): the first goal Halton
// index in [1, kGoalTries] whose state is within the goal speed and free
constexpr int kGoalTries = 100000;
template <int DW>
__global__ void k_goal_halton(SampleBox B, WorldD w, int* __restrict__ first) {
  const int gi = 1 + blockIdx.x * blockDim.x + threadIdx.x;
  if (gi > kGoalTries) return;
  constexpr int kPrimes[12] = {2, 3, 5, 7, 11, 13, 17, 19, 23, 29, 31, 37};
  double p[DW], v[DW];
#pragma unroll
  for (int k = 0; k < DW; ++k) {
    const double u = halton_dev(static_cast<uint64_t>(gi), kPrimes[k]);
    p[k] = B.glo[k] + u * (B.ghi[k] - B.glo[k]);
    const double q = halton_dev(static_cast<uint64_t>(gi), kPrimes[DW + k]);
    v[k] = -B.gms + q * 2 * B.gms;
  }
  if (sqrt(sqnorm<DW>(v)) > B.gms) return;
  if (!point_free<DW>(w, p)) return;
  atomicMin(first, gi);
}

// goal nodes (graph_goal_nodes) on the device: flag, scan, ascending scatter
__global__ void k_goal_flags(int n, int dw, const double* __restrict__ pos, const double* __restrict__ vel, SampleBox B,
                             uint8_t* __restrict__ flag) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  bool in = true;
  double sq = 0.0;
  for (int k = 0; k < dw; ++k) {
    const double p = pos[i * dw + k], v = vel[i * dw + k];
    in = in && !(p < B.glo[k] || p > B.ghi[k]);
    sq = sq + v * v;  // seq_sqn
  }
  flag[i] = (in && sqrt(sq) <= B.gms) ? 1 : 0;
}
__global__ void k_goal_scatter(int n, const uint8_t* __restrict__ flag, const int64_t* __restrict__ off,
                               int32_t* __restrict__ out) {  // out[0] = count, out[1 + j] = goal node j
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i == n) out[0] = static_cast<int32_t>(off[n]);
  if (i >= n || !flag[i]) return;
  out[1 + off[i]] = i;
}

// sample_free on the device; `overlap` (host work) runs while the first
// batch's kernels do.  Returns the node count (the nodes stay in G.pos / G.vel).
template <class Overlap>
static int sample_nodes_device(Ctx& c, const pumpb::Scenario& s, const HostWorld& hw, const DevWorld& dwld,
                               DevGraph& G, Overlap&& overlap) {
  const int dw = s.workspace_dim();
  const int64_t need_total = s.samples;
  const int64_t rows_cap = 1 + need_total + 1;
  G.pos.ensure(al(rows_cap * dw * 8));
  G.vel.ensure(al(rows_cap * dw * 8));
  c.h2d(G.pos.p, s.start_pos.data(), dw * 8);
  c.h2d(G.vel.p, s.start_vel.data(), dw * 8);
  SampleBox B{};
  for (int k = 0; k < dw; ++k) {
    B.lo[k] = s.workspace.bounds.lo[k];
    B.hi[k] = s.workspace.bounds.hi[k];
    B.glo[k] = s.goal.lo[k];
    B.ghi[k] = s.goal.hi[k];
  }
  B.ms = s.max_speed;
  B.gms = s.goal_max_speed;
  WorldD wd;
  wd.n_obs = dwld.n_obs;
  wd.lo = dwld.d_lo;
  wd.hi = dwld.d_hi;
  for (int k = 0; k < 6; ++k) {
    wd.blo[k] = dwld.blo[k];
    wd.bhi[k] = dwld.bhi[k];
  }
  int64_t got = 0;
  int have_goal = 0;
  uint64_t idx0 = 1;
  int64_t M = need_total + need_total / 2 + 256;
  DBuf& gflag = c.buf("s_goal_flag", 256);
  PUMP_CUDA(cudaMemsetAsync(gflag.p, 0, 4, c.stream));
  while (got < need_total) {
    DBuf& cp = c.buf("s_cp", al(M * dw * 8));
    DBuf& cv = c.buf("s_cv", al(M * dw * 8));
    DBuf& fr = c.buf("s_fr", al(M + 8));
    DBuf& ing = c.buf("s_ing", al(M + 8));
    DBuf& rank = c.buf("s_rank", al((M + 2) * 8));
    DBuf& stmp = c.buf("s_scantmp", scan_temp_bytes(M + 16));
    dispatch_dw(dw, [&]<int DW>() {
      k_halton_cand<DW><<<grid_for(M, 128), 128, 0, c.stream>>>(B, wd, idx0, M, cp.as<double>(), cv.as<double>(),
                                                                fr.as<uint8_t>(), ing.as<uint8_t>());
    });
    ++c.launches;
    exclusive_scan<uint8_t>(fr.as<uint8_t>(), rank.as<int64_t>(), M, stmp.p, c.stream, &c.launches);
    k_halton_take<<<grid_for(M, 256), 256, 0, c.stream>>>(dw, M, need_total - got, 1 + got, rank.as<int64_t>(),
                                                          fr.as<uint8_t>(), ing.as<uint8_t>(), cp.as<double>(),
                                                          cv.as<double>(), G.pos.as<double>(), G.vel.as<double>(),
                                                          gflag.as<int>());
    ++c.launches;
    PUMP_CUDA(cudaGetLastError());
    if (idx0 == 1) overlap();
    int64_t acc = 0;
    c.d2h(&acc, rank.as<int64_t>() + M, 8);
    c.d2h(&have_goal, gflag.p, 4);
    c.sync();
    got += std::min(acc, need_total - got);
    idx0 += static_cast<uint64_t>(M);
    M = 2 * (need_total - got) + 256;
  }
  if (idx0 == 1) overlap();  // (no sample needed)
  const int64_t n = 1 + need_total;
  if (!have_goal) {  // goal centre, else a goal Halton sample (sample.hpp:63-88), on the host
    double p[6], v[6];
    for (int k = 0; k < dw; ++k) {
      p[k] = 0.5 * (s.goal.lo[k] + s.goal.hi[k]);
      v[k] = 0.0;
    }
    bool placed = point_free_h(hw, p);
    if (!placed) {  // the goal Halton sequence, searched on the device
      DBuf& fb = c.buf("s_goal_first", 256);
      const int none = kGoalTries + 1;
      c.h2d(fb.p, &none, 4);
      dispatch_dw(dw, [&]<int DW>() {
        k_goal_halton<DW><<<grid_for(kGoalTries, 256), 256, 0, c.stream>>>(B, wd, fb.as<int>());
      });
      ++c.launches;
      int first = none;
      c.d2h(&first, fb.p, 4);
      c.sync();
      if (first <= kGoalTries) {
        halton_state(static_cast<uint64_t>(first), s.goal.lo.data(), s.goal.hi.data(), dw, s.goal_max_speed, p, v);
        placed = true;
      }
    }
    if (!placed) throw std::runtime_error("sample_free: goal region appears entirely in collision");
    c.h2d(G.pos.as<double>() + n * dw, p, dw * 8);
    c.h2d(G.vel.as<double>() + n * dw, v, dw * 8);
    return static_cast<int>(n + 1);
  }
  return static_cast<int>(n);
}

static HostWorld host_world(const pumpb::World& sw) {
  HostWorld w;
  w.dw = sw.dim();
  for (int k = 0; k < w.dw; ++k) {
    w.blo[k] = sw.bounds.lo[k];
    w.bhi[k] = sw.bounds.hi[k];
  }
  for (const auto& b : sw.obstacles) {
    w.lo.insert(w.lo.end(), b.lo.begin(), b.lo.end());
    w.hi.insert(w.hi.end(), b.hi.begin(), b.hi.end());
  }
  return w;
}

static HostLoop loop_of(const pumpb::ClosedLoop& cl) {
  HostLoop L;
  L.d = cl.d;
  L.dw = cl.dw;
  L.F = cl.F.a;
  L.Gv = cl.Gv.a;
  L.Gw = cl.Gw.a;
  L.Sv = cl.Sv.a;
  L.Sw = cl.Sw.a;
  L.S0 = cl.S0.a;
  L.C = cl.C.a;
  return L;
}

// run_pump (pump.hpp:170-263)
// smooth (pump.hpp:84-146) on the device: the plan trajectory blended toward
// the fixed-time optimal motion between its end states, the blend fraction
// bisected (s = 1, then 10 midpoints), each probe a nominal collision check
// + one MC certification.  Used by run_pump and by pump_smooth.
struct SmoothOut {
  std::vector<HWp> traj;
  double cost = 0, mc = 0, s = 0;
};
static SmoothOut smooth_device(Ctx& c, const std::vector<HWp>& plan, double plan_mc, double alpha,
                               const HostLoop& L, const DevWorld& dwld, int64_t n_mc, uint64_t seed, double eps_cc,
                               int dw, double* mc_ms, int64_t* mc_rollouts) {
  // smoothing (pump.hpp:84-146).  The reference bisects the blend fraction
  // s sequentially (s = 1, then 10 midpoints), each probe a nominal
  // collision check + one MC certification.  The probes form a dyadic tree,
  // so whole subtrees are evaluated speculatively in one batched MC launch
  // (candidates whose blended nominal collides get no MC, as in the
  // reference) and the bisection is then replayed from the memo: the accepted
  // s, trajectory and certified CP are exactly the reference's.
  std::vector<HWp> best = plan;
  double best_cost = trajectory_cost(plan, dw), best_mc = plan_mc, best_s = 0;
  if (plan.size() >= 2) {
    HMotion opt{};
    std::memcpy(opt.p0, plan.front().p, sizeof(opt.p0));
    std::memcpy(opt.v0, plan.front().v, sizeof(opt.v0));
    std::memcpy(opt.p1, plan.back().p, sizeof(opt.p1));
    std::memcpy(opt.v1, plan.back().v, sizeof(opt.v1));
    opt.tau = plan.back().t;
    fixed_time(opt, dw);
    auto blend = [&](double sv) {
      std::vector<HWp> t(plan.size());
      for (size_t q = 0; q < plan.size(); ++q) {
        const HWp& wp = plan[q];
        HWp& b = t[q];
        b = HWp{};
        b.t = wp.t;
        double op[6], ov[6], ou[6];
        state_at(opt, dw, wp.t, op, ov);
        control_at(opt, dw, wp.t, ou);
        for (int k = 0; k < dw; ++k) {
          b.p[k] = (1 - sv) * wp.p[k] + sv * op[k];
          b.v[k] = (1 - sv) * wp.v[k] + sv * ov[k];
          b.u[k] = (1 - sv) * wp.u[k] + sv * ou[k];
        }
      }
      return t;
    };
    struct Probe {
      std::vector<HWp> traj;
      bool free = false;
      double mc = 1.0;
    };
    std::map<double, Probe> probes;
    // the device chain: five depth-2 speculative batches, each blending its
    // probes, checking their nominal and certifying them in one pass
    const int n_wp = static_cast<int>(plan.size());
    {
      // the plan's times, positions and velocities in one upload
      std::vector<double> pl(static_cast<size_t>(n_wp) * (1 + 2 * dw));
      for (int q = 0; q < n_wp; ++q) {
        pl[q] = plan[q].t;
        for (int k = 0; k < dw; ++k) {
          pl[n_wp + q * dw + k] = plan[q].p[k];
          pl[n_wp * (1 + dw) + q * dw + k] = plan[q].v[k];
        }
      }
      c.h2d(c.buf("sm_plan", pl.size() * 8 + 256).p, pl.data(), pl.size() * 8);
    }
    auto certified = [&](double sv) {
      const Probe& p = probes.at(sv);
      return p.free && p.mc <= alpha;
    };
    auto accept = [&](double sv) {
      Probe& p = probes.at(sv);
      if (p.traj.empty()) p.traj = blend(sv);  // device probes keep only the verdicts
      best = p.traj;
      best_cost = trajectory_cost(p.traj, dw);
      best_mc = p.mc;
      best_s = sv;
    };
    // five batches enqueued at once, each deciding on the device from the
    // previous batch's verdicts; one synchronisation for the whole bisection
    const int64_t items = static_cast<int64_t>(4) * n_wp;
    DBuf& d_y = c.buf("sm_y", items * dw * 8 + 256);
    DBuf& d_yv = c.buf("sm_yv", items * dw * 8 + 256);
    DBuf& d_ch = c.buf("sm_chain", sizeof(SmoothChain) + 256);
    DBuf& d_off = c.buf("sm_choff", 256);
    const int64_t offs[5] = {0, n_wp, 2 * static_cast<int64_t>(n_wp), 3 * static_cast<int64_t>(n_wp),
                             4 * static_cast<int64_t>(n_wp)};
    c.h2d(d_off.p, offs, sizeof(offs));
    SmoothChain* ch = d_ch.as<SmoothChain>();
    WorldD wd;
    wd.n_obs = dwld.n_obs;
    wd.lo = dwld.d_lo;
    wd.hi = dwld.d_hi;
    for (int k = 0; k < 6; ++k) {
      wd.blo[k] = dwld.blo[k];
      wd.bhi[k] = dwld.bhi[k];
    }
    int64_t r0 = 0, r1 = n_mc;
    shard_range(n_mc, c.rank, c.world, &r0, &r1);
    if (c.mc_join_pending) {
      PUMP_CUDA(cudaStreamWaitEvent(c.stream, c.join, 0));
      c.mc_join_pending = false;
    }
    // the probes' MC step lists are written by the probe kernel when the
    // table holds every probe step (else launch_mc lists them itself)
    mc_table_prepare(c.mc_table, L, r0, r1, seed, n_wp - 1, c.stream, &c.launches);
    const bool lists = mc_table_covers(c.mc_table, L, r0, r1, seed, n_wp - 1) && r1 - r0 <= kTabRollouts;
    if (lists) mc_step_buffers(c.mc_table, 4, n_wp);
    c.tic();
    k_smooth_init<<<1, 32, 0, c.stream>>>(ch);
    ++c.launches;
    for (int b = 0; b < kSmoothBatches; ++b) {
      const int q0 = b == 0 ? 0 : 4 + 3 * (b - 1), np = b == 0 ? 4 : 3;
      const int64_t it = static_cast<int64_t>(np) * n_wp;
      dispatch_dw(dw, [&]<int DW>() {
        HMotion o = opt;
        auto kern = wd.n_obs <= 64 * kCullWords ? k_smooth_probe<DW, 0> : k_smooth_probe<DW, kCullList>;
        const size_t sm = static_cast<size_t>(2 * wd.n_obs * DW) * 8 + 16;
        if (sm > 48 * 1024)
          PUMP_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(sm)));
        const double* plan_d = c.scratch["sm_plan"].as<double>();
        kern<<<grid_for(it * 32, 128), 128, sm, c.stream>>>(ch, b, n_mc, alpha, wd, n_wp, plan_d, plan_d + n_wp,
                                                            plan_d + n_wp * (1 + dw), as_motion<DW>(o), eps_cc,
                                                            d_y.as<double>(), d_yv.as<double>(),
                                                            lists ? c.mc_table.maxdev.as<unsigned long long>() : nullptr,
                                                            c.mc_table.step_list.as<uint16_t>(),
                                                            c.mc_table.step_nl.as<int32_t>(),
                                                            c.mc_table.step_skip.as<uint8_t>());
      });
      c.launches += 1;
      launch_mc(L, dwld, np, d_off.as<int64_t>(), d_y.as<double>(), n_wp, r0, r1, seed, eps_cc,
                &ch->hits[q0], c.stream, &c.launches, &ch->steps, &c.mc_table, &ch->live[q0], lists);
      allreduce_sum_i64(c, reinterpret_cast<int64_t*>(&ch->hits[q0]), np);
      PUMP_CUDA(cudaGetLastError());
    }
    SmoothChain hc{};
    c.d2h(&hc, ch, sizeof(SmoothChain));
    *mc_ms += c.toc();
    c.sync();
    kprof_work(F_MC, static_cast<int64_t>(hc.steps));
    c.mc_rollout_steps += static_cast<int64_t>(hc.steps);
    for (int q = 0; q < kSmoothSlots; ++q) {  // every probe the batches evaluated
      if (probes.count(hc.s[q]) || (q > 0 && hc.done)) continue;
      Probe p;
      p.free = hc.live[q] != 0;
      if (p.free) {
        p.mc = static_cast<double>(hc.hits[q]) / n_mc;
        *mc_rollouts += r1 - r0;
      }
      probes.emplace(hc.s[q], std::move(p));
    }
    // replay (pump.hpp:118-141) from the history (probes.at throws if a
    // probe the bisection visits was not evaluated on the device)
    if (certified(1.0)) {
      accept(1.0);
    } else {
      double lo = 0, hi = 1;
      for (int k = 1; k <= 10; ++k) {
        const double mid = 0.5 * (lo + hi);
        if (!probes.count(mid)) throw std::runtime_error("smoothing: device bisection diverged from the host replay");
        if (certified(mid)) {
          accept(mid);
          lo = mid;
        } else {
          hi = mid;
        }
      }
    }
  }
  SmoothOut o;
  o.traj = std::move(best);
  o.cost = best_cost;
  o.mc = best_mc;
  o.s = best_s;
  return o;
}

static void run_pump_device(Ctx& c, const pumpb::Scenario& s, const DevGraph* prebuilt, pump_result& R) {
  c.mc_table.invalidate();  // the MC table is built inside every solve (no state across solves)
  using clk = std::chrono::steady_clock;
  auto secs = [](clk::time_point a, clk::time_point b) { return std::chrono::duration<double>(b - a).count(); };
  const int dw = s.workspace_dim();
  R.dw = dw;
  const double eps_cc = s.effective_eps_cc();
  const double r_n = s.effective_r_n();
  HostWorld hw = host_world(s.workspace);
  // upload the workspace once
  pump_workspace pw{dw, static_cast<int32_t>(s.workspace.obstacles.size()), s.workspace.bounds.lo.data(),
                    s.workspace.bounds.hi.data(), hw.lo.data(), hw.hi.data()};
  DevWorld dwld = upload_world(c, &pw, "run_ws_");

  auto t0 = clk::now();
  // The models (host: discretisation, Riccati, closed loop) and the particle
  // bank (presample_bank, lti.hpp:257-292) depend only on the model and seed:
  // the models are synthesised while the sampler's first batch runs, and the
  // bank runs on the side stream while the graph is built (a few
  // latency-bound warps next to the FP64-bound graph kernels); explore waits
  // for it through the join event.
  HostLoop L;
  auto models_and_bank = [&]() {
    const auto tm0 = clk::now();
    pumpb::ModelBundle mb = s.models();
    L = loop_of(mb.cl);
    if (std::getenv("PUMP_DEBUG_TIMING"))
      std::fprintf(stderr, "[pump g] %-24s %8.3f ms\n", "models", 1e3 * secs(tm0, clk::now()));
    const size_t bytes = static_cast<size_t>(s.bank_horizon + 1) * s.particles * dw * sizeof(double);
    c.bank.ensure(bytes);
    DBuf& scr = c.buf("bank_scratch", bank_scratch_bytes(L, s.particles, s.bank_horizon));
    PUMP_CUDA(cudaEventRecord(c.fork, c.stream));
    PUMP_CUDA(cudaStreamWaitEvent(c.side, c.fork, 0));
    launch_bank(L, s.particles, s.bank_horizon, s.seeds.bank, c.bank.as<double>(), scr.p, c.side, &c.launches);
    PUMP_CUDA(cudaEventRecord(c.join, c.side));
    c.bank_n = s.particles;
    c.bank_horizon = s.bank_horizon;
    c.bank_dw = dw;
  };
  if (!c.run_graph) c.run_graph = std::make_shared<DevGraph>();
  if (!c.run_explore) c.run_explore = std::make_shared<DevExplore>();
  DevGraph& local = *c.run_graph;
  const DevGraph* graph = prebuilt;
  if (!graph) {
    const int n = sample_nodes_device(c, s, hw, dwld, local, models_and_bank);
    if (std::getenv("PUMP_DEBUG_TIMING"))
      std::fprintf(stderr, "[pump g] %-24s %8.3f ms (from solve start)\n", "sample_nodes",
                   1e3 * secs(t0, clk::now()));
    // goal nodes (graph_goal_nodes) on the device, read back after the graph
    // build's own synchronisations: no host copy of the sampled nodes
    DBuf& gfl = c.buf("r_goal_flag", al(n + 8));
    DBuf& gof = c.buf("r_goal_off", al((n + 2) * 8));
    DBuf& gls = c.buf("r_goal_list", al((n + 2) * 4));
    DBuf& gtmp = c.buf("r_goal_tmp", scan_temp_bytes(n + 16));
    {
      SampleBox GB{};
      for (int k = 0; k < dw; ++k) {
        GB.glo[k] = s.goal.lo[k];
        GB.ghi[k] = s.goal.hi[k];
      }
      GB.gms = s.goal_max_speed;
      k_goal_flags<<<grid_for(n, 256), 256, 0, c.stream>>>(n, dw, local.pos.as<double>(), local.vel.as<double>(), GB,
                                                          gfl.as<uint8_t>());
      exclusive_scan<uint8_t>(gfl.as<uint8_t>(), gof.as<int64_t>(), n, gtmp.p, c.stream, &c.launches);
      k_goal_scatter<<<grid_for(n + 1, 256), 256, 0, c.stream>>>(n, gfl.as<uint8_t>(), gof.as<int64_t>(),
                                                                gls.as<int32_t>());
      c.launches += 2;
    }
    // multi-GPU: each rank builds the rows of its slice; the slices are
    // gathered over NVLink into the full graph on every rank
    int64_t rlo = 0, rhi = n;
    if (c.world > 1) shard_range(n, c.rank, c.world, &rlo, &rhi);
    build_graph_device(local, c, n, dw, nullptr, nullptr,  // the sampler left the nodes in local.pos / vel
                       dwld, r_n, s.dt, eps_cc, s.effective_tau_max(), scan_ratio(s.effective_tau_max()),
                       static_cast<int>(rlo), static_cast<int>(rhi), c.world > 1);
    int32_t ng = 0;
    c.d2h(&ng, gls.p, 4);
    c.sync();
    local.goal_nodes.resize(ng);
    if (ng > 0) {
      c.d2h(local.goal_nodes.data(), gls.as<int32_t>() + 1, static_cast<size_t>(ng) * 4);
      c.sync();
    }
    local.h_pos.clear();  // (run_pump keeps its nodes on the device)
    local.h_vel.clear();
    graph = &local;
  } else {
    models_and_bank();
  }
  auto t1 = clk::now();
  R.s.build_graph_seconds = secs(t0, t1);
  R.s.n_edges = graph->E;

  // explore consumes the bank built on the side stream
  PUMP_CUDA(cudaStreamWaitEvent(c.stream, c.join, 0));
  R.s.bank_ms = 0.0;  // overlapped with the graph build (bank kernels are in the profiler's bank families)
  DevExplore& X = *c.run_explore;
  const double eta = s.effective_eta();
  ExploreArgs ea{s.alpha / eta, std::min(1.0, eta * s.alpha), s.lambda, r_n};
  // The certified trajectories are paths of goal-node plans, so the largest
  // t_end of any plan committed at a goal node bounds their length: grow the
  // MC table (mc.cu) to it on the low-priority side stream while the
  // latency-bound wavefront runs.
  int64_t mr0 = 0, mr1 = s.mc_samples;
  shard_range(s.mc_samples, c.rank, c.world, &mr0, &mr1);
  bool side_forked = false;
  static const bool dbg_r = std::getenv("PUMP_DEBUG_TIMING") != nullptr;
  ea.on_round = [&](const ExploreStatus& h) {
    if (dbg_r)
      std::fprintf(stderr, "[pump r] %8.3f ms plans %lld open %lld max_goal_tend %lld\n", 1e3 * secs(t1, clk::now()),
                   h.n_plans, h.open_count, h.max_goal_tend);
    // before any goal plan: track the wavefront.  A plan's cost is at least
    // its duration (c(tau) >= tau per edge), so open plans of bucket i end
    // near step i width / dt; growing the table behind that estimate spreads
    // its kernels over the rounds instead of starting them at the last one
    int64_t w64 = h.max_goal_tend;
    if (w64 <= 0) {
      w64 = static_cast<int64_t>(std::floor(static_cast<double>(h.i) * s.lambda * r_n / s.dt)) - 16;
      if (w64 < 16) return;
      const int have = static_cast<int>(std::min<int64_t>(s.bank_horizon, w64 - 16));
      if (mc_table_covers(c.mc_table, L, mr0, mr1, s.seeds.mc, have)) return;  // grow in slices of >= 16 steps
    }
    const int want = static_cast<int>(std::min<int64_t>(s.bank_horizon, w64));
    if (want < 0) return;
    if (mc_table_covers(c.mc_table, L, mr0, mr1, s.seeds.mc, want)) return;
    if (!side_forked) {
      PUMP_CUDA(cudaEventRecord(c.fork, c.stream));
      PUMP_CUDA(cudaStreamWaitEvent(c.side, c.fork, 0));
      side_forked = true;
    }
    mc_table_prepare(c.mc_table, L, mr0, mr1, s.seeds.mc, want, c.side, &c.launches);
    PUMP_CUDA(cudaEventRecord(c.join, c.side));
    c.mc_join_pending = true;
  };
  // per-round hook (not batched): the table must start growing as soon as the
  // first goal plans appear, so the certification does not wait for it later
  // (batched, the front MC waited ~0.35 ms longer on quad3d_indoor).  Growing
  // it eagerly from the kept candidates' largest t_end instead measured slower
  // (the over-built table's kernels crowd the explore rounds' SMs).
  ea.on_round_batched = false;  // (pipelined batches re-measured in round 2: forest equal, indoor +0.4 ms)
  run_explore_device(X, c, *graph, ea);
  auto t2 = clk::now();
  static const bool dbg_t = std::getenv("PUMP_DEBUG_TIMING") != nullptr;
  auto mark = [&](const char* what) {
    if (dbg_t) std::fprintf(stderr, "[pump t] %-24s %8.3f ms\n", what, 1e3 * secs(t2, clk::now()));
  };
  R.s.explore_seconds = secs(t1, t2);
  R.s.explore_kernel_ms = X.kernel_ms;
  R.s.partial_plans = X.partial_plans;
  R.s.termination = X.termination;
  R.s.n_plans = X.n_plans;
  R.s.explore_hs_read = X.hs_read;

  // goal plans = concat over goal nodes (ascending) of pareto[v] (planner.hpp:264-265)
  std::vector<int32_t> gids, gtend;
  std::vector<double> gcost, gcp;
  {
    const int ng = static_cast<int>(graph->goal_nodes.size());
    std::vector<int32_t> cnt(graph->n);
    c.d2h(cnt.data(), X.mem_cnt.p, graph->n * 4);
    c.sync();
    std::vector<int64_t> goff(ng + 1, 0);
    for (int g = 0; g < ng; ++g) goff[g + 1] = goff[g] + cnt[graph->goal_nodes[g]];
    const int64_t total = goff[ng];
    if (total > 0) {
      DBuf& d_gn = c.buf("r_gn", ng * 4 + 256);
      DBuf& d_go = c.buf("r_go", (ng + 1) * 8 + 256);
      DBuf& d_id = c.buf("r_gid", total * 4 + 256);
      DBuf& d_c = c.buf("r_gc", total * 8 + 256);
      DBuf& d_p = c.buf("r_gp", total * 8 + 256);
      DBuf& d_t = c.buf("r_gt", total * 4 + 256);
      c.h2d(d_gn.p, graph->goal_nodes.data(), ng * 4);
      c.h2d(d_go.p, goff.data(), (ng + 1) * 8);
      const DBuf& ids = X.mem_flip ? X.mem_b : X.mem_a;
      k_gather_members<<<ng, 128, 0, c.stream>>>(ng, d_gn.as<int32_t>(), X.mem_off.as<int64_t>(),
                                                 d_go.as<int64_t>(), ids.as<int32_t>(), X.cost.as<double>(),
                                                 X.cp.as<double>(), X.t_end.as<int32_t>(), d_id.as<int32_t>(),
                                                 d_c.as<double>(), d_p.as<double>(), d_t.as<int32_t>());
      ++c.launches;
      gids.resize(total);
      gcost.resize(total);
      gcp.resize(total);
      gtend.resize(total);
      c.d2h(gtend.data(), d_t.p, total * 4);
      c.d2h(gids.data(), d_id.p, total * 4);
      c.d2h(gcost.data(), d_c.p, total * 8);
      c.d2h(gcp.data(), d_p.p, total * 8);
      c.sync();
    }
  }
  // global front (pump.hpp:212-235)
  std::vector<int> order(gids.size());
  std::iota(order.begin(), order.end(), 0);
  std::stable_sort(order.begin(), order.end(), [&](int a, int b) {
    if (gcost[a] != gcost[b]) return gcost[a] < gcost[b];
    if (gcp[a] != gcp[b]) return gcp[a] < gcp[b];
    return gids[a] < gids[b];
  });
  std::vector<int> front;  // indices into gids
  double min_cp = std::numeric_limits<double>::infinity();
  for (int k : order)
    if (gcp[k] < min_cp) {
      front.push_back(k);
      min_cp = gcp[k];
    }
  for (int k : front) {
    R.pareto_cost.push_back(gcost[k]);
    R.pareto_cp.push_back(gcp[k]);
  }
  std::vector<int> sorted_ids;  // ascending cp_hat
  std::vector<int> sorted_tend;
  for (auto it = front.rbegin(); it != front.rend(); ++it) {
    sorted_ids.push_back(gids[*it]);
    sorted_tend.push_back(gtend[*it]);
  }

  // Alg. 4 bisection (pump.hpp:23-51): every front plan is certified in one
  // batched MC launch (speculatively), then the bisection is replayed from
  // the memo so mc_evaluations lists exactly the probes the reference makes.
  // The certifications below all read the common-random-number MC table up
  // to the longest front trajectory (t_end + 1 waypoints; smoothing keeps the
  // length): build it on the side stream now, under the host work of
  // resolving the paths and their waypoints.
  if (!front.empty()) {
    int t_max = 0;
    for (int k : front) t_max = std::max(t_max, static_cast<int>(gtend[k]));
    int64_t r0 = 0, r1 = s.mc_samples;
    shard_range(s.mc_samples, c.rank, c.world, &r0, &r1);
    PUMP_CUDA(cudaEventRecord(c.fork, c.stream));
    PUMP_CUDA(cudaStreamWaitEvent(c.side, c.fork, 0));
    mc_table_prepare(c.mc_table, L, r0, r1, s.seeds.mc, t_max, c.side, &c.launches);
    PUMP_CUDA(cudaEventRecord(c.join, c.side));
    c.mc_join_pending = true;  // the first certification waits for it (mc_values)
  }
  mark("front");
  // The front plans' node paths and trajectories on the device (k_paths,
  // k_traj_build): plan q has t_end + 1 waypoints, so the offsets are known
  // here; their positions feed the MC batch directly and only the selected
  // plan is copied back.
  const int nf = static_cast<int>(sorted_ids.size());
  constexpr int kMaxLen = 4096;
  std::vector<int64_t> woff(nf + 1, 0);
  std::vector<double> memo;
  if (nf > 0) {
    int max_pts = 0;
    for (int q = 0; q < nf; ++q) {
      woff[q + 1] = woff[q] + sorted_tend[q] + 1;
      max_pts = std::max(max_pts, sorted_tend[q] + 1);
    }
    const int64_t total = woff[nf];
    std::vector<int64_t> in(nf + 1 + (nf + 1) / 2 + 1, 0);  // offsets, then the plan ids (int32 pairs)
    std::memcpy(in.data(), woff.data(), (nf + 1) * 8);
    std::memcpy(in.data() + nf + 1, sorted_ids.data(), nf * 4);
    DBuf& d_in = c.buf("p_in", in.size() * 8 + 256);
    c.h2d(d_in.p, in.data(), in.size() * 8);
    const int64_t* d_woff = d_in.as<int64_t>();
    const int32_t* d_sel = reinterpret_cast<const int32_t*>(d_in.as<int64_t>() + nf + 1);
    DBuf& d_nodes = c.buf("p_nodes", static_cast<size_t>(nf) * kMaxLen * 4 + 256);
    DBuf& d_edges = c.buf("p_edges", static_cast<size_t>(nf) * kMaxLen * 8 + 256);
    DBuf& d_lens = c.buf("p_lens", nf * 4 + 256);
    DBuf& d_wt = c.buf("p_wt", total * 8 + 256);
    DBuf& d_wp = c.buf("p_wp", total * dw * 8 + 256);
    DBuf& d_wv = c.buf("p_wv", total * dw * 8 + 256);
    DBuf& d_wu = c.buf("p_wu", total * dw * 8 + 256);
    const DevGraph& G = *graph;
    k_paths<<<(nf + 127) / 128, 128, 0, c.stream>>>(nf, d_sel, X.head.as<int32_t>(), X.parent.as<int32_t>(),
                                                    G.row_ptr.as<int64_t>(), G.e_to.as<int32_t>(), kMaxLen,
                                                    d_nodes.as<int32_t>(), d_edges.as<int64_t>(), d_lens.as<int32_t>());
    dispatch_dw(dw, [&]<int DW>() {
      k_traj_build<DW><<<(nf * 32 + 127) / 128, 128, 0, c.stream>>>(
          nf, kMaxLen, d_nodes.as<int32_t>(), d_edges.as<int64_t>(), d_lens.as<int32_t>(), d_woff,
          G.pos.as<double>(), G.vel.as<double>(), G.e_tau.as<double>(), G.e_acc0.as<double>(), G.e_jerk.as<double>(),
          G.dt, d_wt.as<double>(), d_wp.as<double>(), d_wv.as<double>(), d_wu.as<double>());
    });
    c.launches += 2;
    PUMP_CUDA(cudaGetLastError());
    memo = mc_values_dev(c, L, dwld, nf, d_woff, d_wp.as<double>(), max_pts, s.mc_samples, s.seeds.mc, eps_cc,
                         &R.s.mc_ms, &R.s.mc_rollouts);
  }
  mark("paths + trajectories");
  std::vector<char> seen(nf, 0);
  auto eval = [&](int m) {
    if (!seen[m - 1]) {
      seen[m - 1] = 1;
      R.mc_ids.push_back(sorted_ids[m - 1]);
      R.mc_vals.push_back(memo[m - 1]);
    }
    return memo[m - 1];
  };
  bool success = false;
  int sel = -1;
  if (nf > 0) {
    int l = 1, u = nf;
    while (l < u) {
      const int m = (l + u + 1) / 2;
      if (eval(m) > s.alpha)
        u = m - 1;
      else
        l = m;
    }
    if (!(eval(l) > s.alpha)) {
      success = true;
      sel = l - 1;
    }
  }
  if (!success) {
    R.s.selection_seconds = secs(t2, clk::now());
    R.s.success = 0;
    return;
  }
  mark("front mc");
  const int sel_id = sorted_ids[sel];
  std::vector<HWp> plan_sel;
  double cph = 0.0, cst = 0.0;
  {
    // the selected plan's node path and waypoints, its cp_hat and cost (one readback)
    const int64_t n_wp = woff[sel + 1] - woff[sel];
    int32_t len = 0;
    c.d2h(&len, c.scratch["p_lens"].as<int32_t>() + sel, 4);
    std::vector<int32_t> nodes(kMaxLen);
    c.d2h(nodes.data(), c.scratch["p_nodes"].as<int32_t>() + static_cast<int64_t>(sel) * kMaxLen, kMaxLen * 4);
    std::vector<double> wt(n_wp), wpv(n_wp * dw), wvv(n_wp * dw), wuv(n_wp * dw);
    c.d2h(wt.data(), c.scratch["p_wt"].as<double>() + woff[sel], n_wp * 8);
    c.d2h(wpv.data(), c.scratch["p_wp"].as<double>() + woff[sel] * dw, n_wp * dw * 8);
    c.d2h(wvv.data(), c.scratch["p_wv"].as<double>() + woff[sel] * dw, n_wp * dw * 8);
    c.d2h(wuv.data(), c.scratch["p_wu"].as<double>() + woff[sel] * dw, n_wp * dw * 8);
    c.d2h(&cph, X.cp.as<double>() + sel_id, 8);
    c.d2h(&cst, X.cost.as<double>() + sel_id, 8);
    c.sync();
    R.path.assign(nodes.begin(), nodes.begin() + len);
    plan_sel.resize(n_wp);
    for (int64_t q = 0; q < n_wp; ++q) {
      HWp& h = plan_sel[q];
      h = HWp{};
      h.t = wt[q];
      for (int k = 0; k < dw; ++k) {
        h.p[k] = wpv[q * dw + k];
        h.v[k] = wvv[q * dw + k];
        h.u[k] = wuv[q * dw + k];
      }
    }
  }
  R.s.cp_hat = cph;
  R.s.pre_smoothing_cost = cst;
  {
    SmoothOut sm = smooth_device(c, plan_sel, memo[sel], s.alpha, L, dwld, s.mc_samples, s.seeds.mc, eps_cc, dw,
                                 &R.s.mc_ms, &R.s.mc_rollouts);
    R.traj = std::move(sm.traj);
    R.s.cost = sm.cost;
    R.s.certified_cp = sm.mc;
    R.s.smoothing_s = sm.s;
  }
  mark("smoothing");
  R.s.success = 1;
  R.s.selection_seconds = secs(t2, clk::now());
}

// ==================================================================== RRT
// repeated_rrt (rrt.hpp:50-147), the Table 1 baseline: one warp per trial.
// Each iteration draws the target (counter-hash uniforms, rrt.hpp:27-44),
// finds the nearest tree node (lanes over the nodes, warp argmin with the
// first index on ties, as the reference's strict `<` scan), then lane 0
// steers (connect, the graph build's code), truncates the motion at cost r_n
// (steer.hpp:214-243) and checks it (motion_collides); the tree lives in
// global memory.  The host assembles the reached trials' trajectories,
// orders them by cost and certifies them in that order on the MC table.
struct RrtArgs {
  int trials, max_it, n_max;
  uint64_t seed;
  double goal_bias, max_speed, goal_ms, tau_max, ratio, r_n, eps_cc;
  double blo[6], bhi[6], glo[6], ghi[6], x0p[6], x0v[6];
  double* np;    // [trial][n_max][dw] node positions
  double* nv;    // node velocities
  int32_t* par;  // [trial][n_max]
  double* itau;  // incoming motion: tau, acc0[dw], jerk[dw]
  double* ia;
  double* ij;
  int32_t* reached;  // goal node index or -1
};

__device__ __forceinline__ double uniform_dev(uint64_t seed, uint64_t a, uint64_t b, uint64_t c) {
  return to_unit(mix64(mix64(hash_seed_a(seed, a) + b) + c));
}

// motion_partial_cost (steer.hpp:214-225), the reference's operation order
template <int DW>
__host__ __device__ __forceinline__ double partial_cost(const double* a, const double* j, double tau, double s) {
  if (s <= 0) return 0;
  s = s < tau ? s : tau;
  double c = s;
#pragma unroll
  for (int k = 0; k < DW; ++k) c += a[k] * a[k] * s + a[k] * j[k] * s * s + j[k] * j[k] * s * s * s / 3;
  return c;
}

template <int DW>
__global__ void __launch_bounds__(128) k_rrt(RrtArgs A, WorldD w) {
  extern __shared__ double smem[];
  const WorldD ws = stage_world<DW>(w, smem);
  const int lane = threadIdx.x & 31;
  const int trial = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (trial >= A.trials) return;
  double* np = A.np + static_cast<int64_t>(trial) * A.n_max * DW;
  double* nv = A.nv + static_cast<int64_t>(trial) * A.n_max * DW;
  int32_t* par = A.par + static_cast<int64_t>(trial) * A.n_max;
  double* itau = A.itau + static_cast<int64_t>(trial) * A.n_max;
  double* ia = A.ia + static_cast<int64_t>(trial) * A.n_max * DW;
  double* ij = A.ij + static_cast<int64_t>(trial) * A.n_max * DW;
  if (lane == 0) {
    for (int k = 0; k < DW; ++k) {
      np[k] = A.x0p[k];
      nv[k] = A.x0v[k];
    }
    par[0] = -1;
    itau[0] = 0;
  }
  __syncwarp();
  int n_nodes = 1, reached = -1;
  for (int iter = 0; iter < A.max_it; ++iter) {
    double tp[DW], tv[DW];
    {
      const double bias = uniform_dev(A.seed, trial, iter, 0);
      const bool g = bias < A.goal_bias;
      const double vmax = g ? A.goal_ms : A.max_speed;
#pragma unroll
      for (int k = 0; k < DW; ++k) {
        const double lo = g ? A.glo[k] : A.blo[k], hi = g ? A.ghi[k] : A.bhi[k];
        const double u = uniform_dev(A.seed, trial, iter, 1 + k);
        tp[k] = lo + u * (hi - lo);
        const double v = uniform_dev(A.seed, trial, iter, 1 + DW + k);
        tv[k] = -vmax + v * 2 * vmax;
      }
    }
    if (!point_free<DW>(ws, tp)) continue;
    // nearest node: squaredNorm(p - tp) + squaredNorm(v - tv), first strict minimum
    double bd = __builtin_inf();
    int bi = 0x7fffffff;
    for (int ni = lane; ni < n_nodes; ni += 32) {
      double dp[DW], dv[DW];
#pragma unroll
      for (int k = 0; k < DW; ++k) {
        dp[k] = np[ni * DW + k] - tp[k];
        dv[k] = nv[ni * DW + k] - tv[k];
      }
      const double dist = sqnorm<DW>(dp) + sqnorm<DW>(dv);
      if (dist < bd) {
        bd = dist;
        bi = ni;
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const double od = __shfl_xor_sync(0xffffffffu, bd, o);
      const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
      if (od < bd || (od == bd && oi < bi)) {
        bd = od;
        bi = oi;
      }
    }
    const int nearest = bi;
    int added = 0;
    if (lane == 0) {
      double ap[DW], av[DW];
#pragma unroll
      for (int k = 0; k < DW; ++k) {
        ap[k] = np[nearest * DW + k];
        av[k] = nv[nearest * DW + k];
      }
      double tau = 0, cost = 0;
      const bool ok = connect_dev<DW>(ap, av, tp, tv, A.tau_max, A.ratio, tau, cost);
      if (ok && tau > 0) {
        MotionD<DW> m;
        m.tau = tau;
#pragma unroll
        for (int k = 0; k < DW; ++k) {
          m.p0[k] = ap[k];
          m.v0[k] = av[k];
          m.p1[k] = tp[k];
          m.v1[k] = tv[k];
        }
        coeffs_dev<DW>(ap, av, tp, tv, tau, m.a, m.j);
        if (cost > A.r_n) {  // truncate_motion (steer.hpp:228-243)
          double lo = 0, hi = tau;
          for (int it = 0; it < 60; ++it) {
            const double mid = 0.5 * (lo + hi);
            if (partial_cost<DW>(m.a, m.j, tau, mid) < A.r_n)
              lo = mid;
            else
              hi = mid;
          }
          const double tt = 0.5 * (lo + hi);
          motion_state<DW>(m, tt, m.p1, m.v1);
          m.tau = tt;
        }
        if (m.tau > 0 && !motion_collides<DW>(m, ws, A.eps_cc)) {
          const int id = n_nodes;
#pragma unroll
          for (int k = 0; k < DW; ++k) {
            np[id * DW + k] = m.p1[k];
            nv[id * DW + k] = m.v1[k];
            ia[id * DW + k] = m.a[k];
            ij[id * DW + k] = m.j[k];
          }
          par[id] = nearest;
          itau[id] = m.tau;
          added = 1;
          bool in = true;  // GoalRegion::contains (sample.hpp:26-28)
#pragma unroll
          for (int k = 0; k < DW; ++k) in = in && !(m.p1[k] < A.glo[k] || m.p1[k] > A.ghi[k]);
          if (in && sqrt(sqnorm<DW>(m.v1)) <= A.goal_ms) added = 2;
        }
      }
    }
    added = __shfl_sync(0xffffffffu, added, 0);
    __syncwarp();
    if (added) {
      ++n_nodes;
      if (added == 2) {
        reached = n_nodes - 1;
        break;
      }
    }
  }
  if (lane == 0) A.reached[trial] = reached;
}

struct RrtOutcome {
  bool success = false;
  std::vector<HWp> traj;
  double cost = 0, certified_cp = 0;
  int reached = 0, attempts = 0;
};

static RrtOutcome run_rrt_device(Ctx& c, const pumpb::Scenario& s, int trials, double alpha, int n_mc) {
  if (trials < 1) throw std::invalid_argument("repeated_rrt: trials must be at least 1");
  c.mc_table.invalidate();
  const int dw = s.workspace_dim();
  pumpb::ModelBundle mb = s.models();
  HostLoop L = loop_of(mb.cl);
  HostWorld hw = host_world(s.workspace);
  pump_workspace pw{dw, static_cast<int32_t>(s.workspace.obstacles.size()), s.workspace.bounds.lo.data(),
                    s.workspace.bounds.hi.data(), hw.lo.data(), hw.hi.data()};
  DevWorld dwld = upload_world(c, &pw, "rrt_ws_");
  const int n_max = s.rrt.max_iterations + 1;
  RrtArgs A{};
  A.trials = trials;
  A.max_it = s.rrt.max_iterations;
  A.n_max = n_max;
  A.seed = s.seeds.rrt;
  A.goal_bias = s.rrt.goal_bias;
  A.max_speed = s.max_speed;
  A.goal_ms = s.goal_max_speed;
  A.tau_max = s.effective_tau_max();
  A.ratio = scan_ratio(A.tau_max);
  A.r_n = s.effective_r_n();
  A.eps_cc = s.effective_eps_cc();
  for (int k = 0; k < dw; ++k) {
    A.blo[k] = s.workspace.bounds.lo[k];
    A.bhi[k] = s.workspace.bounds.hi[k];
    A.glo[k] = s.goal.lo[k];
    A.ghi[k] = s.goal.hi[k];
    A.x0p[k] = s.start_pos[k];
    A.x0v[k] = s.start_vel[k];
  }
  const size_t tn = static_cast<size_t>(trials) * n_max;
  DBuf& bp = c.buf("rrt_np", al(tn * dw * 8));
  DBuf& bv = c.buf("rrt_nv", al(tn * dw * 8));
  DBuf& bpar = c.buf("rrt_par", al(tn * 4));
  DBuf& btau = c.buf("rrt_tau", al(tn * 8));
  DBuf& ba = c.buf("rrt_a", al(tn * dw * 8));
  DBuf& bj = c.buf("rrt_j", al(tn * dw * 8));
  DBuf& brc = c.buf("rrt_reached", al(static_cast<size_t>(trials) * 4));
  A.np = bp.as<double>();
  A.nv = bv.as<double>();
  A.par = bpar.as<int32_t>();
  A.itau = btau.as<double>();
  A.ia = ba.as<double>();
  A.ij = bj.as<double>();
  A.reached = brc.as<int32_t>();
  WorldD wd;
  wd.n_obs = dwld.n_obs;
  wd.lo = dwld.d_lo;
  wd.hi = dwld.d_hi;
  for (int k = 0; k < 6; ++k) {
    wd.blo[k] = dwld.blo[k];
    wd.bhi[k] = dwld.bhi[k];
  }
  const size_t wsmem = 2 * static_cast<size_t>(dwld.n_obs) * dw * sizeof(double);
  dispatch_dw(dw, [&]<int DW>() {
    if (wsmem > 48 * 1024)
      PUMP_CUDA(cudaFuncSetAttribute(k_rrt<DW>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)wsmem));
    k_rrt<DW><<<grid_for(static_cast<int64_t>(trials) * 32, 128), 128, wsmem, c.stream>>>(A, wd);
  });
  ++c.launches;
  PUMP_CUDA(cudaGetLastError());
  std::vector<int32_t> reached(trials);
  c.d2h(reached.data(), brc.p, trials * 4);
  c.sync();
  // reached trials: walk the chain on the host and assemble the trajectory
  // (rrt.hpp:95-113) from the nodes and incoming motions
  struct Tr {
    int trial;
    std::vector<HWp> traj;
    double cost;
  };
  std::vector<Tr> got;
  std::vector<double> hp, hv, ht, ha, hj;
  std::vector<int32_t> hpar;
  for (int t = 0; t < trials; ++t) {
    if (reached[t] < 0) continue;
    const size_t base = static_cast<size_t>(t) * n_max;
    const int nn = reached[t] + 1;
    hp.resize(static_cast<size_t>(nn) * dw);
    hv.resize(static_cast<size_t>(nn) * dw);
    ha.resize(static_cast<size_t>(nn) * dw);
    hj.resize(static_cast<size_t>(nn) * dw);
    ht.resize(nn);
    hpar.resize(nn);
    c.d2h(hp.data(), bp.as<double>() + base * dw, nn * dw * 8);
    c.d2h(hv.data(), bv.as<double>() + base * dw, nn * dw * 8);
    c.d2h(ha.data(), ba.as<double>() + base * dw, nn * dw * 8);
    c.d2h(hj.data(), bj.as<double>() + base * dw, nn * dw * 8);
    c.d2h(ht.data(), btau.as<double>() + base, nn * 8);
    c.d2h(hpar.data(), bpar.as<int32_t>() + base, nn * 4);
    c.sync();
    std::vector<int> chain;
    for (int id = reached[t]; id != -1; id = hpar[id]) chain.push_back(id);
    std::reverse(chain.begin(), chain.end());
    Tr tr;
    tr.trial = t;
    double offset = 0;
    for (size_t q = 0; q < chain.size(); ++q) {
      const int id = chain[q];
      if (q == 0) {
        HWp w0{};
        w0.t = 0.0;
        for (int k = 0; k < dw; ++k) {
          w0.p[k] = hp[id * dw + k];
          w0.v[k] = hv[id * dw + k];
        }
        tr.traj.push_back(w0);
        continue;
      }
      const int pid = hpar[id];
      HMotion m{};
      for (int k = 0; k < dw; ++k) {
        m.p0[k] = hp[pid * dw + k];
        m.v0[k] = hv[pid * dw + k];
        m.p1[k] = hp[id * dw + k];
        m.v1[k] = hv[id * dw + k];
        m.a[k] = ha[id * dw + k];
        m.j[k] = hj[id * dw + k];
      }
      m.tau = ht[id];
      auto wps = motion_waypoints(m, dw, s.dt);
      for (size_t k = 1; k < wps.size(); ++k) {
        HWp wp = wps[k];
        wp.t += offset;
        tr.traj.push_back(wp);
      }
      offset += m.tau;
    }
    tr.cost = trajectory_cost(tr.traj, dw);
    got.push_back(std::move(tr));
  }
  RrtOutcome out;
  out.reached = static_cast<int>(got.size());
  std::stable_sort(got.begin(), got.end(), [](const Tr& a, const Tr& b) { return a.cost < b.cost; });
  // certify in cost order until one passes; batches of 8 certified together
  // (the reference stops at the first pass: attempts = its position + 1)
  constexpr size_t kBatch = 8;
  for (size_t b0 = 0; b0 < got.size() && !out.success; b0 += kBatch) {
    std::vector<std::vector<HWp>> batch;
    for (size_t q = b0; q < std::min(got.size(), b0 + kBatch); ++q) batch.push_back(got[q].traj);
    double mc_ms = 0;
    int64_t rollouts = 0;
    auto v = mc_values(c, L, dwld, batch, n_mc, s.seeds.mc, A.eps_cc, &mc_ms, &rollouts);
    for (size_t q = 0; q < batch.size(); ++q) {
      out.attempts++;
      if (v[q] <= alpha) {
        out.success = true;
        out.traj = got[b0 + q].traj;
        out.cost = got[b0 + q].cost;
        out.certified_cp = v[q];
        break;
      }
    }
  }
  return out;
}

}  // namespace pumpg

extern "C" {

// ------------------------------------------------------------------ graph
static int build_graph_rows(pump_ctx* ctx, int32_t n_nodes, int32_t dw, const double* pos, const double* vel,
                            const pump_workspace* ws, const pump_goal* goal, double r_n, double dt, double eps_cc,
                            double tau_max, int32_t row_lo, int32_t row_hi, bool gather, pump_graph** out) {
  return guard([&] {
    Ctx& c = ctx->c;
    if (!ws || ws->dw != dw) throw std::invalid_argument("build_graph: workspace dimension mismatch");
    if (r_n <= 0) throw std::invalid_argument("build_graph: r_n must be positive");
    DevWorld w = upload_world(c, ws, "g_ws_");
    auto* g = new pump_graph;
    try {
      g->owner = ctx;
      build_graph_device(g->g, c, n_nodes, dw, pos, vel, w, r_n, dt, eps_cc, tau_max, scan_ratio(tau_max), row_lo,
                         row_hi, gather);
      g->g.h_pos.assign(pos, pos + static_cast<size_t>(n_nodes) * dw);
      g->g.h_vel.assign(vel, vel + static_cast<size_t>(n_nodes) * dw);
      graph_goal_nodes(g->g, pos, vel, goal);
    } catch (...) {
      delete g;
      throw;
    }
    *out = g;
  });
}

int pump_build_graph(pump_ctx* ctx, int32_t n_nodes, int32_t dw, const double* pos, const double* vel,
                     const pump_workspace* ws, const pump_goal* goal, double r_n, double dt, double eps_cc,
                     double tau_max, pump_graph** out) {
  if (!ctx) return PUMP_E_INVALID_ARGUMENT;
  int64_t lo = 0, hi = n_nodes;
  const bool shard = ctx->c.has_comm();
  if (shard) shard_range(n_nodes, ctx->c.rank, ctx->c.world, &lo, &hi);
  return build_graph_rows(ctx, n_nodes, dw, pos, vel, ws, goal, r_n, dt, eps_cc, tau_max, static_cast<int32_t>(lo),
                          static_cast<int32_t>(hi), shard, out);
}

int pump_build_graph_rows(pump_ctx* ctx, int32_t n_nodes, int32_t dw, const double* pos, const double* vel,
                          const pump_workspace* ws, const pump_goal* goal, double r_n, double dt, double eps_cc,
                          double tau_max, int32_t row_lo, int32_t row_hi, pump_graph** out) {
  return build_graph_rows(ctx, n_nodes, dw, pos, vel, ws, goal, r_n, dt, eps_cc, tau_max, row_lo, row_hi, false,
                          out);
}

int pump_rrt_run(pump_ctx* ctx, const pump_scenario* scn, int32_t trials, double alpha, int32_t n_mc,
                 pump_result** out) {
  return guard([&] {
    if (!ctx || !scn || !out) throw std::invalid_argument("repeated_rrt: null argument");
    const auto& s = scn->s;
    auto* r = new pump_result;
    try {
      const RrtOutcome o = run_rrt_device(ctx->c, s, trials > 0 ? trials : s.rrt.trials, alpha >= 0 ? alpha : s.alpha,
                                          n_mc > 0 ? n_mc : s.mc_samples);
      r->dw = s.workspace_dim();
      r->s.dw = r->dw;
      r->s.success = o.success ? 1 : 0;
      r->s.cost = o.cost;
      r->s.certified_cp = o.certified_cp;
      r->s.rrt_trials_reaching_goal = o.reached;
      r->s.rrt_certification_attempts = o.attempts;
      r->traj = o.traj;
      r->s.n_traj_points = static_cast<int32_t>(o.traj.size());
    } catch (...) {
      delete r;
      throw;
    }
    *out = r;
  });
}

int pump_smooth(pump_ctx* ctx, const pump_closed_loop* cl, const pump_workspace* ws, int32_t n_points,
                const double* t, const double* pos, const double* vel, const double* ctrl, double plan_mc,
                double alpha, int32_t n_mc, uint64_t seed, double eps_cc, double* out_pos, double* out_vel,
                double* out_ctrl, double* out3) {
  return guard([&] {
    Ctx& c = ctx->c;
    if (n_mc < 1) throw std::invalid_argument("mc_certify: need at least one rollout");
    if (n_points < 1) throw std::invalid_argument("smooth: empty trajectory");
    const HostLoop L = host_loop(cl);
    const int dw = L.dw;
    if (ws->dw != dw) throw std::invalid_argument("smooth: workspace / closed-loop dimension mismatch");
    const DevWorld dwld = upload_world(c, ws, "sm_ws_");
    std::vector<HWp> plan(n_points);
    for (int q = 0; q < n_points; ++q) {
      HWp& h = plan[q];
      h = HWp{};
      h.t = t[q];
      for (int k = 0; k < dw; ++k) {
        h.p[k] = pos[q * dw + k];
        h.v[k] = vel[q * dw + k];
        h.u[k] = ctrl[q * dw + k];
      }
    }
    // the certifications read a common-random-number table built for this call
    c.mc_table.invalidate();
    double mc_ms = 0;
    int64_t rollouts = 0;
    SmoothOut o = smooth_device(c, plan, plan_mc, alpha, L, dwld, n_mc, seed, eps_cc, dw, &mc_ms, &rollouts);
    for (int q = 0; q < n_points; ++q)
      for (int k = 0; k < dw; ++k) {
        out_pos[q * dw + k] = o.traj[q].p[k];
        out_vel[q * dw + k] = o.traj[q].v[k];
        out_ctrl[q * dw + k] = o.traj[q].u[k];
      }
    out3[0] = o.cost;
    out3[1] = o.mc;
    out3[2] = o.s;
  });
}

int pump_scenario_nodes(const pump_scenario* s, int32_t cap, double* pos, double* vel, int32_t* n_out) {
  return guard([&] {
    if (!s || !n_out) throw std::invalid_argument("scenario_nodes: null argument");
    HostWorld hw = host_world(s->s.workspace);
    std::vector<double> p, v;
    sample_nodes(s->s, hw, p, v);
    const int dw = s->s.workspace_dim();
    const int n = static_cast<int>(p.size()) / dw;
    *n_out = n;
    if (pos && vel) {
      if (n > cap) throw std::out_of_range("scenario_nodes: capacity " + std::to_string(cap) + " < " + std::to_string(n));
      std::copy(p.begin(), p.end(), pos);
      std::copy(v.begin(), v.end(), vel);
    }
  });
}

int pump_graph_upload(pump_ctx* ctx, const pump_graph_view* v, pump_graph** out) {
  return guard([&] {
    Ctx& c = ctx->c;
    auto* gp = new pump_graph;
    DevGraph& G = gp->g;
    try {
      gp->owner = ctx;
      const int n = v->n_nodes, dw = v->dw;
      const int64_t E = v->n_edges, NW = v->n_waypoints, H = v->n_halfspaces;
      G.n = n;
      G.dw = dw;
      G.r_n = v->r_n;
      G.dt = v->dt;
      G.E = E;
      G.NW = NW;
      G.H = H;
      G.H_pk = H;
      auto up = [&](DBuf& b, const void* src, size_t bytes) {
        b.ensure(bytes + 256);
        c.h2d(b.p, src, bytes);
      };
      up(G.pos, v->node_pos, n * dw * 8);
      up(G.vel, v->node_vel, n * dw * 8);
      up(G.row_ptr, v->row_ptr, (n + 1) * 8);
      up(G.e_to, v->edge_to, E * 4);
      up(G.e_cost, v->edge_cost, E * 8);
      up(G.e_tau, v->edge_tau, E * 8);
      up(G.e_acc0, v->edge_acc0, E * dw * 8);
      up(G.e_jerk, v->edge_jerk, E * dw * 8);
      up(G.e_nsteps, v->edge_nsteps, E * 4);
      up(G.wp_off, v->edge_wp_off, (E + 1) * 8);
      up(G.hs_off, v->wp_hs_off, (NW + 1) * 8);
      std::vector<int32_t> cnt(NW + 1, 0);
      for (int64_t w = 0; w < NW; ++w) cnt[w] = static_cast<int32_t>(v->wp_hs_off[w + 1] - v->wp_hs_off[w]);
      up(G.hs_cnt, cnt.data(), (NW + 1) * 4);
      std::vector<double> pk(static_cast<size_t>(H) * 4 + 4, 0.0);
      for (int64_t h = 0; h < H; ++h) {
        for (int k = 0; k < dw; ++k) pk[h * 4 + k] = v->hs_a[h * dw + k];
        pk[h * 4 + 3] = v->hs_b[h];
      }
      up(G.hs_pk, pk.data(), H * 32);
      G.hs_fb.ensure(H + 256);
      if (v->hs_fallback) c.h2d(G.hs_fb.p, v->hs_fallback, H);
      std::vector<int32_t> from(E);
      for (int i = 0; i < n; ++i)
        for (int64_t e = v->row_ptr[i]; e < v->row_ptr[i + 1]; ++e) from[e] = i;
      up(G.e_from, from.data(), E * 4);
      G.goal_nodes.assign(v->goal_nodes, v->goal_nodes + v->n_goal);
      G.h_pos.assign(v->node_pos, v->node_pos + static_cast<size_t>(n) * dw);
      G.h_vel.assign(v->node_vel, v->node_vel + static_cast<size_t>(n) * dw);
      c.sync();
    } catch (...) {
      delete gp;
      throw;
    }
    *out = gp;
  });
}

int pump_graph_counts(const pump_graph* g, pump_graph_view* v) {
  return guard([&] {
    const DevGraph& G = g->g;
    v->n_nodes = G.n;
    v->dw = G.dw;
    v->n_edges = G.E;
    v->n_waypoints = G.NW;
    v->n_halfspaces = G.H;
    v->n_goal = static_cast<int32_t>(G.goal_nodes.size());
    v->r_n = G.r_n;
    v->dt = G.dt;
  });
}

int pump_graph_export(const pump_graph* g, pump_graph_view* v) {
  return guard([&] {
    Ctx& c = g->owner->c;
    const DevGraph& G = g->g;
    const int n = G.n, dw = G.dw;
    auto dn = [&](void* dst, const DBuf& b, size_t bytes) {
      if (dst && bytes) c.d2h(dst, b.p, bytes);
    };
    if (v->node_pos) std::memcpy(v->node_pos, G.h_pos.data(), n * dw * 8);
    if (v->node_vel) std::memcpy(v->node_vel, G.h_vel.data(), n * dw * 8);
    dn(v->row_ptr, G.row_ptr, (n + 1) * 8);
    dn(v->edge_to, G.e_to, G.E * 4);
    dn(v->edge_cost, G.e_cost, G.E * 8);
    dn(v->edge_tau, G.e_tau, G.E * 8);
    dn(v->edge_acc0, G.e_acc0, G.E * dw * 8);
    dn(v->edge_jerk, G.e_jerk, G.E * dw * 8);
    dn(v->edge_nsteps, G.e_nsteps, G.E * 4);
    dn(v->edge_wp_off, G.wp_off, (G.E + 1) * 8);
    // half-spaces: waypoint w owns [hs_off[w], hs_off[w] + hs_cnt[w]) on the
    // device; the exported view is the reference's waypoint-ordered CSR
    if (v->wp_hs_off || v->hs_a || v->hs_b || v->hs_fallback) {
      const int64_t NW = G.NW, H = G.H_pk;  // (stored records; waypoints may share them)
      std::vector<int64_t> start(NW + 1);
      std::vector<int32_t> cnt(NW + 1);
      std::vector<double> pk(static_cast<size_t>(H) * 4 + 4);
      std::vector<uint8_t> fb(H + 1);
      c.d2h(start.data(), G.hs_off.p, NW * 8);
      c.d2h(cnt.data(), G.hs_cnt.p, NW * 4);
      c.d2h(pk.data(), G.hs_pk.p, H * 32);
      c.d2h(fb.data(), G.hs_fb.p, H);
      c.sync();
      int64_t o = 0;
      if (v->wp_hs_off) v->wp_hs_off[0] = 0;
      for (int64_t w = 0; w < NW; ++w) {
        for (int32_t h = 0; h < cnt[w]; ++h, ++o) {
          const int64_t src = start[w] + h;
          for (int k = 0; k < dw; ++k)
            if (v->hs_a) v->hs_a[o * dw + k] = pk[src * 4 + k];
          if (v->hs_b) v->hs_b[o] = pk[src * 4 + 3];
          if (v->hs_fallback) v->hs_fallback[o] = fb[src];
        }
        if (v->wp_hs_off) v->wp_hs_off[w + 1] = o;
      }
    }
    if (v->goal_nodes) std::memcpy(v->goal_nodes, G.goal_nodes.data(), G.goal_nodes.size() * 4);
    c.sync();
  });
}

int pump_graph_free(pump_graph* g) {
  delete g;
  return PUMP_OK;
}

// ---------------------------------------------------------------- explore
int pump_explore_run(pump_ctx* ctx, const pump_graph* g, const pump_explore_params* p, pump_explore** out) {
  return guard([&] {
    auto* e = new pump_explore;
    try {
      ExploreArgs a{p->alpha_min, p->alpha_max, p->lambda, p->r_n};
      run_explore_device(e->x, ctx->c, g->g, a);
      e->owner = ctx;
      e->goal_nodes = g->g.goal_nodes;
    } catch (...) {
      delete e;
      throw;
    }
    *out = e;
  });
}

namespace {
struct HookStop {};
}  // namespace

int pump_explore_run_hooked(pump_ctx* ctx, const pump_graph* g, const pump_explore_params* p, pump_round_hook hook,
                            void* user, pump_explore** out) {
  int rc = PUMP_OK;
  const int st = guard([&] {
    auto* e = new pump_explore;
    try {
      e->owner = ctx;  // goal_nodes stay empty during the rounds (goal_plans are collected at the end)
      ExploreArgs a{p->alpha_min, p->alpha_max, p->lambda, p->r_n};
      if (hook)
        a.on_round_state = [&](int round, const std::vector<int32_t>& grp) {
          if (hook(user, round, e, grp.data(), static_cast<int64_t>(grp.size())) != 0) throw HookStop{};
        };
      try {
        run_explore_device(e->x, ctx->c, g->g, a);
      } catch (const HookStop&) {
        rc = PUMP_E_HOOK;
        delete e;
        return;
      }
      e->goal_nodes = g->g.goal_nodes;
    } catch (...) {
      delete e;
      throw;
    }
    *out = e;
  });
  return st != PUMP_OK ? st : rc;
}

int pump_explore_counts(const pump_explore* e, pump_explore_view* v) {
  return guard([&] {
    const DevExplore& X = e->x;
    Ctx& c = e->owner->c;
    v->n_plans = X.n_plans;
    v->n_words = X.W;
    v->n_nodes = X.n;
    std::vector<int32_t> cnt(X.n);
    c.d2h(cnt.data(), X.mem_cnt.p, X.n * 4);
    c.sync();
    int64_t tot = 0;
    for (int x : cnt) tot += x;
    v->n_pareto = tot;
    v->n_goal_plans = 0;
    for (int gnode : e->goal_nodes) v->n_goal_plans += cnt[gnode];
    v->partial_plans = X.partial_plans;
    v->discarded_cp = X.disc_cp;
    v->removed_dominated = X.removed;
    v->discarded_horizon = X.disc_hor;
    v->rounds = X.rounds;
    v->termination = X.termination;
  });
}

int pump_explore_export(const pump_explore* e, pump_explore_view* v) {
  return guard([&] {
    const DevExplore& X = e->x;
    Ctx& c = e->owner->c;
    const int64_t P = X.n_plans;
    auto dn = [&](void* dst, const DBuf& b, size_t bytes) {
      if (dst && bytes) c.d2h(dst, b.p, bytes);
    };
    dn(v->head, X.head, P * 4);
    dn(v->parent, X.parent, P * 4);
    dn(v->cost, X.cost, P * 8);
    dn(v->cp_hat, X.cp, P * 8);
    dn(v->t_end, X.t_end, P * 4);
    dn(v->masks, X.mask, P * X.W * 8);
    std::vector<int32_t> cnt(X.n);
    std::vector<int64_t> off(X.n + 1);
    c.d2h(cnt.data(), X.mem_cnt.p, X.n * 4);
    c.d2h(off.data(), X.mem_off.p, (X.n + 1) * 8);
    c.sync();
    const DBuf& ids = X.mem_flip ? X.mem_b : X.mem_a;
    const int64_t span = off[X.n];
    std::vector<int32_t> all(span + 1);
    if (span > 0) c.d2h(all.data(), ids.p, span * 4);
    c.sync();
    int64_t o = 0;
    if (v->pareto_ptr) v->pareto_ptr[0] = 0;
    for (int i = 0; i < X.n; ++i) {
      for (int k = 0; k < cnt[i]; ++k) {
        if (v->pareto_ids) v->pareto_ids[o] = all[off[i] + k];
        ++o;
      }
      if (v->pareto_ptr) v->pareto_ptr[i + 1] = o;
    }
    int64_t q = 0;
    for (int gnode : e->goal_nodes)
      for (int k = 0; k < cnt[gnode]; ++k) {
        if (v->goal_plans) v->goal_plans[q] = all[off[gnode] + k];
        ++q;
      }
  });
}

int pump_explore_free(pump_explore* e) {
  delete e;
  return PUMP_OK;
}

// ------------------------------------------------------------- pipeline
int pump_run(pump_ctx* ctx, const pump_scenario* s, const pump_graph* prebuilt, pump_result** out) {
  return guard([&] {
    auto* r = new pump_result;
    try {
      run_pump_device(ctx->c, s->s, prebuilt ? &prebuilt->g : nullptr, *r);
      r->s.path_len = static_cast<int32_t>(r->path.size());
      r->s.n_pareto = static_cast<int32_t>(r->pareto_cost.size());
      r->s.n_mc_evals = static_cast<int32_t>(r->mc_ids.size());
      r->s.n_traj_points = static_cast<int32_t>(r->traj.size());
      r->s.dw = r->dw;
    } catch (...) {
      delete r;
      throw;
    }
    *out = r;
  });
}

int pump_result_summary_get(const pump_result* r, pump_result_summary* out) {
  *out = r->s;
  return PUMP_OK;
}

int pump_result_arrays(const pump_result* r, int32_t* path, double* pc, double* pcp, int32_t* ids, double* mcs,
                       double* tt, double* tp, double* tv, double* tu) {
  const int dw = r->dw;
  if (path) std::copy(r->path.begin(), r->path.end(), path);
  if (pc) std::copy(r->pareto_cost.begin(), r->pareto_cost.end(), pc);
  if (pcp) std::copy(r->pareto_cp.begin(), r->pareto_cp.end(), pcp);
  if (ids) std::copy(r->mc_ids.begin(), r->mc_ids.end(), ids);
  if (mcs) std::copy(r->mc_vals.begin(), r->mc_vals.end(), mcs);
  for (size_t i = 0; i < r->traj.size(); ++i) {
    if (tt) tt[i] = r->traj[i].t;
    for (int k = 0; k < dw; ++k) {
      if (tp) tp[i * dw + k] = r->traj[i].p[k];
      if (tv) tv[i * dw + k] = r->traj[i].v[k];
      if (tu) tu[i * dw + k] = r->traj[i].u[k];
    }
  }
  return PUMP_OK;
}

int pump_result_free(pump_result* r) {
  delete r;
  return PUMP_OK;
}

int pump_probe_round_latency(pump_ctx* ctx, double* us_barrier, double* us_l2_load) {
  return guard([&] { pumpg::probe_round_latency(ctx->c, us_barrier, us_l2_load); });
}

}  // extern "C"
