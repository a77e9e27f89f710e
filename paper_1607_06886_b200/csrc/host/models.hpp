// Host-side model synthesis: ZOH discretization, steady-state LQG gains and
// the joint closed-loop deviation recursion.  Restates lti.hpp:75-241 and
// scenario.hpp:285-301 with the small dense helpers of linalg.hpp.  Runs
// once per solve on <= 12x12 matrices; the GPU never sees anything but the
// resulting ClosedLoop matrices.
#pragma once

#include <stdexcept>
#include <vector>

#include "linalg.hpp"

namespace pumpb {

using la::Mat;

struct ContinuousModel {
  Mat A, B, C, V, W;
};

struct DiscreteModel {
  Mat A, B, C, V, W;
  double dt = 0;
  int state_dim() const { return A.r; }
  int output_dim() const { return C.r; }
};

struct LqgWeights {
  Mat Q, R, F;
};

struct GainSchedule {
  Mat L, K, sigma0;
};

// lti.hpp:181-190 — the joint (dx, dx_hat) recursion
//   z_{t+1} = F z_t + Gv (Sv nv) + Gw (Sw nw)
struct ClosedLoop {
  int d = 0, dw = 0;
  Mat F, Gv, Gw, Sv, Sw, S0, C;
};

inline void require(bool ok, const char* msg) {
  if (!ok) throw std::invalid_argument(msg);
}

// lti.hpp:75-109
inline DiscreteModel discretize(const ContinuousModel& cm, double dt) {
  const int d = cm.A.r, l = cm.B.c, dw = cm.C.r;
  require(dt > 0, "discretize: dt must be positive");
  require(cm.B.r == d, "discretize: B row dimension mismatch");
  require(cm.C.c == d, "discretize: C column dimension mismatch");
  require(cm.V.r == d && cm.V.c == d, "discretize: V dimension mismatch");
  require(cm.W.r == dw && cm.W.c == dw, "discretize: W dimension mismatch");
  require(la::is_psd(cm.V), "discretize: V_c must be symmetric PSD");
  require(la::is_psd(cm.W), "discretize: W_c must be symmetric PSD");
  DiscreteModel dm;
  dm.dt = dt;
  dm.C = cm.C;
  dm.W = cm.W;
  for (size_t i = 0; i < dm.W.a.size(); ++i) dm.W.a[i] = cm.W.a[i] / dt;
  Mat m1 = Mat::zero(d + l, d + l);
  la::set_block(m1, 0, 0, dt * cm.A);
  la::set_block(m1, 0, d, dt * cm.B);
  Mat e1 = la::expm(m1);
  dm.A = la::block(e1, 0, 0, d, d);
  dm.B = la::block(e1, 0, d, d, l);
  Mat m2 = Mat::zero(2 * d, 2 * d);
  la::set_block(m2, 0, 0, (-dt) * cm.A);
  la::set_block(m2, 0, d, dt * cm.V);
  la::set_block(m2, d, d, dt * la::transpose(cm.A));
  Mat e2 = la::expm(m2);
  Mat v = la::transpose(la::block(e2, d, d, d, d)) * la::block(e2, 0, d, d, d);
  dm.V = la::symmetrize(v);
  return dm;
}

// lti.hpp:113-175
inline GainSchedule lqg_synthesize(const DiscreteModel& dm, const LqgWeights& w, const Mat& sigma0) {
  const int d = dm.state_dim();
  const double tol = 1e-10;
  const int max_iter = 10000;
  Mat At = la::transpose(dm.A), Bt = la::transpose(dm.B);
  Mat p = w.F;
  bool converged = false;
  for (int it = 0; it < max_iter; ++it) {
    Mat bpb = w.R + Bt * p * dm.B;
    Mat bpa = Bt * p * dm.A;
    Mat next = w.Q + At * p * dm.A - la::transpose(bpa) * la::solve(bpb, bpa);
    next = la::symmetrize(next);
    double diff = la::max_abs(next - p);
    p = next;
    if (!la::all_finite(p)) throw std::runtime_error("lqg_synthesize: control Riccati diverged");
    if (diff < tol) {
      converged = true;
      break;
    }
  }
  if (!converged) throw std::runtime_error("lqg_synthesize: control Riccati did not converge");
  GainSchedule gs;
  gs.sigma0 = sigma0;
  Mat bpb = w.R + Bt * p * dm.B;
  gs.L = (-1.0) * la::solve(bpb, Bt * p * dm.A);

  Mat Ct = la::transpose(dm.C);
  auto kalman_gain = [&](const Mat& cov) -> Mat {
    Mat innov = dm.C * cov * Ct + dm.W;
    if (la::max_abs(innov) < 1e-300) return Mat::zero(d, dm.output_dim());
    return cov * Ct * la::solve(innov, Mat::eye(innov.r));
  };
  Mat s = sigma0;
  converged = false;
  for (int it = 0; it < max_iter; ++it) {
    Mat gain = kalman_gain(s);
    Mat upd = s - gain * dm.C * s;
    Mat next = dm.A * upd * At + dm.V;
    next = la::symmetrize(next);
    double diff = la::max_abs(next - s);
    s = next;
    if (!la::all_finite(s)) throw std::runtime_error("lqg_synthesize: filter Riccati diverged");
    if (diff < tol) {
      converged = true;
      break;
    }
  }
  if (!converged) throw std::runtime_error("lqg_synthesize: filter Riccati did not converge");
  gs.K = kalman_gain(s);
  return gs;
}

// lti.hpp:192-217
inline ClosedLoop closed_loop(const DiscreteModel& dm, const GainSchedule& gs, const Mat& sigma0) {
  const int d = dm.state_dim(), dw = dm.output_dim();
  ClosedLoop cl;
  cl.d = d;
  cl.dw = dw;
  cl.C = dm.C;
  Mat bl = dm.B * gs.L;
  Mat kc = gs.K * dm.C;
  Mat I = Mat::eye(d);
  cl.F = Mat::zero(2 * d, 2 * d);
  la::set_block(cl.F, 0, 0, dm.A);
  la::set_block(cl.F, 0, d, bl);
  la::set_block(cl.F, d, 0, kc * dm.A);
  la::set_block(cl.F, d, d, (I - kc) * (dm.A + bl) + kc * bl);
  cl.Gv = Mat::zero(2 * d, d);
  la::set_block(cl.Gv, 0, 0, I);
  la::set_block(cl.Gv, d, 0, kc);
  cl.Gw = Mat::zero(2 * d, dw);
  la::set_block(cl.Gw, d, 0, gs.K);
  cl.Sv = la::psd_sqrt(dm.V);
  cl.Sw = la::psd_sqrt(dm.W);
  cl.S0 = la::psd_sqrt(sigma0);
  return cl;
}

// lti.hpp:221-240: workspace marginal covariances C Cov(dx_t) C'.
inline std::vector<Mat> propagate_covariances(const ClosedLoop& cl, const Mat& sigma0, int T) {
  require(T >= 0, "propagate_covariances: T must be nonnegative");
  const int d = cl.d;
  Mat sz = Mat::zero(2 * d, 2 * d);
  la::set_block(sz, 0, 0, sigma0);
  Mat vq = cl.Sv * la::transpose(cl.Sv), wq = cl.Sw * la::transpose(cl.Sw);
  Mat Ft = la::transpose(cl.F), Gvt = la::transpose(cl.Gv), Gwt = la::transpose(cl.Gw),
      Ct = la::transpose(cl.C);
  std::vector<Mat> out;
  for (int t = 0;; ++t) {
    out.push_back(cl.C * la::block(sz, 0, 0, d, d) * Ct);
    if (t == T) break;
    sz = cl.F * sz * Ft + cl.Gv * vq * Gvt + cl.Gw * wq * Gwt;
  }
  return out;
}

struct ModelBundle {
  ContinuousModel cm;
  DiscreteModel dm;
  GainSchedule gains;
  ClosedLoop cl;
};

// scenario.hpp:285-301: per-axis double integrator in dw dimensions.
inline ModelBundle build_models(int dw, double dt, const Mat& process_noise, const Mat& measurement_noise,
                                const Mat& initial_covariance, const LqgWeights& tracking) {
  const int d = 2 * dw;
  ModelBundle mb;
  mb.cm.A = Mat::zero(d, d);
  la::set_block(mb.cm.A, 0, dw, Mat::eye(dw));
  mb.cm.B = Mat::zero(d, dw);
  la::set_block(mb.cm.B, dw, 0, Mat::eye(dw));
  mb.cm.C = Mat::zero(dw, d);
  la::set_block(mb.cm.C, 0, 0, Mat::eye(dw));
  mb.cm.V = process_noise;
  mb.cm.W = measurement_noise;
  mb.dm = discretize(mb.cm, dt);
  mb.gains = lqg_synthesize(mb.dm, tracking, initial_covariance);
  mb.cl = closed_loop(mb.dm, mb.gains, initial_covariance);
  return mb;
}

}  // namespace pumpb
