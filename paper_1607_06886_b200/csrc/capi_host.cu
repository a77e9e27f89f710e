// Host-side helpers of the C ABI: single-call steering, collision, convex
// region, sampling and waypoint queries for the drop-in C++ headers
// (include/pump/).  They run the very __host__ __device__ code the kernels
// run (gpu/dev.cuh), so a host query and a kernel agree bit for bit.
#include <cmath>
#include <cstring>
#include <vector>

#include "ctx.h"
#include "gpu/dispatch.cuh"
#include "guard.h"

using namespace pumpg;

namespace {

struct HostWs {
  std::vector<double> lo, hi;
  WorldD w{};
  explicit HostWs(const pump_workspace* ws) {
    if (!ws || ws->dw < 1 || ws->dw > 6) throw std::invalid_argument("workspace: bad dimensions");
    const size_t m = static_cast<size_t>(ws->n_obs) * ws->dw;
    if (m) {
      lo.assign(ws->obs_lo, ws->obs_lo + m);
      hi.assign(ws->obs_hi, ws->obs_hi + m);
    }
    w.n_obs = ws->n_obs;
    w.lo = lo.data();
    w.hi = hi.data();
    for (int k = 0; k < ws->dw; ++k) {
      w.blo[k] = ws->bounds_lo[k];
      w.bhi[k] = ws->bounds_hi[k];
    }
  }
};

template <int DW>
MotionD<DW> motion_of(const double* fp, const double* fv, const double* tp, const double* tv, double tau,
                      const double* acc0, const double* jerk) {
  MotionD<DW> m;
  for (int k = 0; k < DW; ++k) {
    m.p0[k] = fp[k];
    m.v0[k] = fv[k];
    m.p1[k] = tp[k];
    m.v1[k] = tv[k];
    m.a[k] = acc0[k];
    m.j[k] = jerk[k];
  }
  m.tau = tau;
  return m;
}

double halton(uint64_t index, int base) {  // sample.hpp:12-20
  double f = 1.0, r = 0.0;
  while (index > 0) {
    f /= base;
    r += f * (index % base);
    index /= base;
  }
  return r;
}

}  // namespace

extern "C" {

// connect (steer.hpp:111-182): out3 = {ok, tau, cost}; acc0/jerk when ok
int pump_connect(int32_t dw, const double* ap, const double* av, const double* bp, const double* bv, double tau_max,
                 double* out3, double* acc0, double* jerk) {
  return guard([&] {
    const double ratio = std::pow(tau_max / (tau_max * 1e-7), 1.0 / (64 - 1));  // steer.hpp:133
    dispatch_dw(dw, [&]<int DW>() {
      double tau = 0, cost = 0;
      const bool ok = connect_dev<DW>(ap, av, bp, bv, tau_max, ratio, tau, cost);
      out3[0] = ok ? 1.0 : 0.0;
      out3[1] = tau;
      out3[2] = cost;
      if (ok && tau > 0) {
        coeffs_dev<DW>(ap, av, bp, bv, tau, acc0, jerk);
      } else if (ok) {
        for (int k = 0; k < DW; ++k) acc0[k] = jerk[k] = 0.0;
      }
    });
  });
}

double pump_steer_cost(int32_t dw, const double* ap, const double* av, const double* bp, const double* bv,
                       double tau) {
  double c = 0;
  dispatch_dw(dw, [&]<int DW>() { c = steer_cost<DW>(ap, av, bp, bv, tau); });
  return c;
}

// fixed_time_connect (steer.hpp:97-107): cost, acc0, jerk
int pump_fixed_time_connect(int32_t dw, const double* ap, const double* av, const double* bp, const double* bv,
                            double tau, double* cost, double* acc0, double* jerk) {
  return guard([&] {
    double effort = 0;
    for (int k = 0; k < dw; ++k) {
      const double dp = bp[k] - ap[k] - av[k] * tau;
      const double dv = bv[k] - av[k];
      acc0[k] = 6 * dp / (tau * tau) - 2 * dv / tau;
      jerk[k] = -12 * dp / (tau * tau * tau) + 6 * dv / (tau * tau);
      effort += 12 * dp * dp / (tau * tau * tau) - 12 * dp * dv / (tau * tau) + 4 * dv * dv / tau;
    }
    *cost = tau + effort;
  });
}

int pump_point_free(const pump_workspace* ws, const double* y) {
  HostWs h(ws);
  bool r = false;
  dispatch_dw(ws->dw, [&]<int DW>() { r = point_free<DW>(h.w, y); });
  return r ? 1 : 0;
}

int pump_segment_hits_aabb(int32_t dw, const double* p0, const double* p1, const double* lo, const double* hi) {
  bool r = false;
  dispatch_dw(dw, [&]<int DW>() { r = segment_hits<DW>(p0, p1, lo, hi); });
  return r ? 1 : 0;
}

// motion_collides (geom.hpp:96-123) of the motion (from, to, tau, acc0, jerk)
int pump_motion_collides(const pump_workspace* ws, const double* fp, const double* fv, const double* tp,
                         const double* tv, double tau, const double* acc0, const double* jerk, double eps_cc,
                         int32_t* out) {
  return guard([&] {
    HostWs h(ws);
    dispatch_dw(ws->dw, [&]<int DW>() {
      *out = motion_collides<DW>(motion_of<DW>(fp, fv, tp, tv, tau, acc0, jerk), h.w, eps_cc) ? 1 : 0;
    });
  });
}

// local_convex_region (geom.hpp:189-225): up to cap half-spaces
int pump_local_convex_region(const pump_workspace* ws, const double* y, const double* ydot, int32_t cap, double* a,
                             double* b, uint8_t* fb, int32_t* n_out) {
  return guard([&] {
    HostWs h(ws);
    if (ws->n_obs > 4096) throw std::invalid_argument("local_convex_region: more than 4096 obstacles");
    dispatch_dw(ws->dw, [&]<int DW>() {
      if (!point_free<DW>(h.w, y)) throw std::invalid_argument("local_convex_region: waypoint is in collision");
      std::vector<double> ta(static_cast<size_t>(ws->n_obs + 1) * DW), tb(ws->n_obs + 1);
      std::vector<uint8_t> tf(ws->n_obs + 1);
      const int n = convex_region<DW>(h.w, y, ydot, ta.data(), tb.data(), tf.data());
      if (n < 0) throw std::runtime_error("local_convex_region: pruning loop failed to make progress");
      *n_out = n;
      if (n > cap) throw CapacityError("local_convex_region: output capacity too small");
      std::memcpy(a, ta.data(), static_cast<size_t>(n) * DW * 8);
      std::memcpy(b, tb.data(), static_cast<size_t>(n) * 8);
      std::memcpy(fb, tf.data(), static_cast<size_t>(n));
    });
  });
}

// sample_free (sample.hpp:56-89): writes up to cap states, *n_out = count
int pump_sample_free(int32_t n, const pump_workspace* ws, double max_speed, const pump_goal* goal, int32_t cap,
                     double* pos, double* vel, int32_t* n_out) {
  return guard([&] {
    if (n < 1) throw std::invalid_argument("sample_free: n must be at least 1");
    HostWs h(ws);
    const int dw = ws->dw;
    static const int kPrimes[] = {2, 3, 5, 7, 11, 13, 17, 19, 23, 29, 31, 37};
    if (2 * dw > 12) throw std::invalid_argument("sample_free: workspace dimension above 6");
    std::vector<double> P, V;
    auto state = [&](uint64_t index, const double* lo, const double* hi, double ms, double* p, double* v) {
      for (int k = 0; k < dw; ++k) {
        const double u = halton(index, kPrimes[k]);
        p[k] = lo[k] + u * (hi[k] - lo[k]);
        const double q = halton(index, kPrimes[dw + k]);
        v[k] = -ms + q * 2 * ms;
      }
    };
    auto pf = [&](const double* p) {
      bool r = false;
      dispatch_dw(dw, [&]<int DW>() { r = point_free<DW>(h.w, p); });
      return r;
    };
    auto nrm = [&](const double* v) {
      double s = 0.0;
      for (int k = 0; k < dw; ++k) s = s + v[k] * v[k];
      return std::sqrt(s);
    };
    auto in_goal = [&](const double* p, const double* v) {
      for (int k = 0; k < dw; ++k)
        if (p[k] < goal->lo[k] || p[k] > goal->hi[k]) return false;
      return nrm(v) <= goal->max_speed;
    };
    bool have_goal = false;
    uint64_t index = 1;
    double p[6], v[6];
    int got = 0;
    while (got < n) {
      state(index++, ws->bounds_lo, ws->bounds_hi, max_speed, p, v);
      if (!pf(p)) continue;
      have_goal = have_goal || in_goal(p, v);
      P.insert(P.end(), p, p + dw);
      V.insert(V.end(), v, v + dw);
      ++got;
    }
    if (!have_goal) {
      for (int k = 0; k < dw; ++k) {
        p[k] = 0.5 * (goal->lo[k] + goal->hi[k]);
        v[k] = 0.0;
      }
      if (pf(p)) {
        P.insert(P.end(), p, p + dw);
        V.insert(V.end(), v, v + dw);
      } else {
        bool placed = false;
        for (uint64_t gi = 1; gi <= 100000 && !placed; ++gi) {
          state(gi, goal->lo, goal->hi, goal->max_speed, p, v);
          if (nrm(v) > goal->max_speed) continue;
          if (!pf(p)) continue;
          P.insert(P.end(), p, p + dw);
          V.insert(V.end(), v, v + dw);
          placed = true;
        }
        if (!placed) throw std::runtime_error("sample_free: goal region appears entirely in collision");
      }
    }
    *n_out = static_cast<int32_t>(P.size() / dw);
    if (*n_out > cap) throw CapacityError("sample_free: output capacity too small");
    std::memcpy(pos, P.data(), P.size() * 8);
    std::memcpy(vel, V.data(), V.size() * 8);
  });
}

// motion_waypoints (steer.hpp:192-212): returns the count, writes <= cap
int32_t pump_waypoints(int32_t dw, const double* fp, const double* fv, const double* tp, const double* tv, double tau,
                       const double* acc0, const double* jerk, double dt, int32_t cap, double* t_out, double* p_out,
                       double* v_out, double* u_out) {
  if (dt <= 0) return -PUMP_E_INVALID_ARGUMENT;
  int count = 0;
  auto put = [&](double t, const double* p, const double* v, const double* u) {
    if (count < cap) {
      t_out[count] = t;
      for (int k = 0; k < dw; ++k) {
        p_out[count * dw + k] = p[k];
        v_out[count * dw + k] = v[k];
        u_out[count * dw + k] = u[k];
      }
    }
    ++count;
  };
  double zero[6] = {0, 0, 0, 0, 0, 0};
  if (tau <= 0) {
    put(0.0, fp, fv, zero);
    return count;
  }
  auto control = [&](double s, double* u) {
    s = s < 0 ? 0 : (s > tau ? tau : s);
    for (int k = 0; k < dw; ++k) u[k] = acc0[k] + jerk[k] * s;
  };
  const int k = static_cast<int>(std::floor(tau / dt + 1e-9));
  const double rem = tau - k * dt;
  for (int i = 0; i <= k; ++i) {
    const double t = i * dt;
    double p[6], v[6], u[6];
    dispatch_dw(dw, [&]<int DW>() {
      const MotionD<DW> m = motion_of<DW>(fp, fv, tp, tv, tau, acc0, jerk);
      motion_state<DW>(m, t, p, v);
    });
    control(t, u);
    if (i == k && !(rem > 1e-9)) {
      put(tau, tp, tv, u);  // last waypoint replaced by the target state
    } else {
      put(t, p, v, u);
    }
  }
  if (rem > 1e-9) {
    double u[6];
    control(tau, u);
    put(tau, tp, tv, u);
  }
  return count;
}

}  // extern "C"
