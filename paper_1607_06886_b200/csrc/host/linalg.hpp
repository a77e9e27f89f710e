// Small dense linear algebra for the host-side model synthesis (<= 12x12,
// once per solve).  This replaces the Eigen subset the reference uses for
// discretize / lqg_synthesize / closed_loop (lti.hpp:55-217).  It is NOT on
// the accelerated path: the GPU kernels consume the resulting closed-loop
// matrices as inputs, and the CPU oracle consumes the very same matrices, so
// GPU-vs-oracle parity does not depend on how these are computed.
//
// Row-major storage throughout.
#pragma once

#include <algorithm>
#include <cmath>
#include <stdexcept>
#include <vector>

namespace pumpb::la {

struct Mat {
  int r = 0, c = 0;
  std::vector<double> a;
  Mat() = default;
  Mat(int rows, int cols, double v = 0.0) : r(rows), c(cols), a(static_cast<size_t>(rows) * cols, v) {}
  double& operator()(int i, int j) { return a[static_cast<size_t>(i) * c + j]; }
  double operator()(int i, int j) const { return a[static_cast<size_t>(i) * c + j]; }
  static Mat zero(int rows, int cols) { return Mat(rows, cols, 0.0); }
  static Mat eye(int n) {
    Mat m(n, n);
    for (int i = 0; i < n; ++i) m(i, i) = 1.0;
    return m;
  }
};

inline Mat operator+(const Mat& x, const Mat& y) {
  Mat o(x.r, x.c);
  for (size_t i = 0; i < o.a.size(); ++i) o.a[i] = x.a[i] + y.a[i];
  return o;
}
inline Mat operator-(const Mat& x, const Mat& y) {
  Mat o(x.r, x.c);
  for (size_t i = 0; i < o.a.size(); ++i) o.a[i] = x.a[i] - y.a[i];
  return o;
}
inline Mat operator*(double s, const Mat& x) {
  Mat o(x.r, x.c);
  for (size_t i = 0; i < o.a.size(); ++i) o.a[i] = s * x.a[i];
  return o;
}
inline Mat operator*(const Mat& x, const Mat& y) {
  if (x.c != y.r) throw std::invalid_argument("la: product dimension mismatch");
  Mat o(x.r, y.c);
  for (int i = 0; i < x.r; ++i)
    for (int j = 0; j < y.c; ++j) {
      double s = 0;
      for (int k = 0; k < x.c; ++k) s += x(i, k) * y(k, j);
      o(i, j) = s;
    }
  return o;
}
inline Mat transpose(const Mat& x) {
  Mat o(x.c, x.r);
  for (int i = 0; i < x.r; ++i)
    for (int j = 0; j < x.c; ++j) o(j, i) = x(i, j);
  return o;
}
inline double max_abs(const Mat& x) {
  double m = 0;
  for (double v : x.a) m = std::max(m, std::fabs(v));
  return m;
}
inline bool all_finite(const Mat& x) {
  for (double v : x.a)
    if (!std::isfinite(v)) return false;
  return true;
}
inline Mat block(const Mat& x, int r0, int c0, int rows, int cols) {
  Mat o(rows, cols);
  for (int i = 0; i < rows; ++i)
    for (int j = 0; j < cols; ++j) o(i, j) = x(r0 + i, c0 + j);
  return o;
}
inline void set_block(Mat& x, int r0, int c0, const Mat& b) {
  for (int i = 0; i < b.r; ++i)
    for (int j = 0; j < b.c; ++j) x(r0 + i, c0 + j) = b(i, j);
}
inline Mat symmetrize(const Mat& x) { return 0.5 * (x + transpose(x)); }

// Solve A X = B by Gaussian elimination with partial pivoting (A square).
inline Mat solve(Mat A, Mat B) {
  const int n = A.r;
  if (A.c != n || B.r != n) throw std::invalid_argument("la: solve dimension mismatch");
  for (int col = 0; col < n; ++col) {
    int piv = col;
    for (int i = col + 1; i < n; ++i)
      if (std::fabs(A(i, col)) > std::fabs(A(piv, col))) piv = i;
    if (A(piv, col) == 0.0) throw std::runtime_error("la: singular system");
    if (piv != col) {
      for (int j = 0; j < n; ++j) std::swap(A(col, j), A(piv, j));
      for (int j = 0; j < B.c; ++j) std::swap(B(col, j), B(piv, j));
    }
    for (int i = col + 1; i < n; ++i) {
      double f = A(i, col) / A(col, col);
      if (f == 0.0) continue;
      for (int j = col; j < n; ++j) A(i, j) -= f * A(col, j);
      for (int j = 0; j < B.c; ++j) B(i, j) -= f * B(col, j);
    }
  }
  Mat X(n, B.c);
  for (int j = 0; j < B.c; ++j)
    for (int i = n - 1; i >= 0; --i) {
      double s = B(i, j);
      for (int k = i + 1; k < n; ++k) s -= A(i, k) * X(k, j);
      X(i, j) = s / A(i, i);
    }
  return X;
}

// Matrix exponential: scaling and squaring with a degree-18 Taylor core.
inline Mat expm(const Mat& A) {
  const int n = A.r;
  double nrm = 0;
  for (int i = 0; i < n; ++i) {
    double s = 0;
    for (int j = 0; j < n; ++j) s += std::fabs(A(i, j));
    nrm = std::max(nrm, s);
  }
  int sq = 0;
  if (nrm > 0.25) sq = static_cast<int>(std::ceil(std::log2(nrm / 0.25)));
  Mat X = std::ldexp(1.0, -sq) * A;
  Mat E = Mat::eye(n), term = Mat::eye(n);
  for (int k = 1; k <= 18; ++k) {
    term = (1.0 / k) * (term * X);
    E = E + term;
  }
  for (int i = 0; i < sq; ++i) E = E * E;
  return E;
}

// Cyclic Jacobi eigen-decomposition of a symmetric matrix.
inline void sym_eig(const Mat& S, std::vector<double>& evals, Mat& V) {
  const int n = S.r;
  Mat A = S;
  V = Mat::eye(n);
  for (int sweep = 0; sweep < 100; ++sweep) {
    double off = 0;
    for (int i = 0; i < n; ++i)
      for (int j = i + 1; j < n; ++j) off += A(i, j) * A(i, j);
    if (off < 1e-300) break;
    for (int p = 0; p < n; ++p)
      for (int q = p + 1; q < n; ++q) {
        if (A(p, q) == 0.0) continue;
        double theta = (A(q, q) - A(p, p)) / (2 * A(p, q));
        double t = (theta >= 0 ? 1.0 : -1.0) / (std::fabs(theta) + std::sqrt(theta * theta + 1));
        double c = 1 / std::sqrt(t * t + 1), s = t * c;
        for (int k = 0; k < n; ++k) {
          double akp = A(k, p), akq = A(k, q);
          A(k, p) = c * akp - s * akq;
          A(k, q) = s * akp + c * akq;
        }
        for (int k = 0; k < n; ++k) {
          double apk = A(p, k), aqk = A(q, k);
          A(p, k) = c * apk - s * aqk;
          A(q, k) = s * apk + c * aqk;
        }
        for (int k = 0; k < n; ++k) {
          double vkp = V(k, p), vkq = V(k, q);
          V(k, p) = c * vkp - s * vkq;
          V(k, q) = s * vkp + c * vkq;
        }
      }
  }
  evals.resize(n);
  for (int i = 0; i < n; ++i) evals[i] = A(i, i);
}

// lti.hpp:58-64
inline bool is_psd(const Mat& m, double tol = 1e-9) {
  if (m.r != m.c) return false;
  if (max_abs(m - transpose(m)) > tol * (1.0 + max_abs(m))) return false;
  std::vector<double> ev;
  Mat V;
  sym_eig(m, ev, V);
  double mn = ev.empty() ? 0 : *std::min_element(ev.begin(), ev.end());
  return mn >= -tol * (1.0 + max_abs(m));
}

// lti.hpp:66-71: symmetric PSD square root, negative eigenvalues clamped.
inline Mat psd_sqrt(const Mat& m) {
  const int n = m.r;
  if (max_abs(m) == 0.0) return Mat::zero(n, n);
  std::vector<double> ev;
  Mat V;
  sym_eig(m, ev, V);
  Mat D = Mat::zero(n, n);
  for (int i = 0; i < n; ++i) D(i, i) = std::sqrt(std::max(ev[i], 0.0));
  Mat out = V * D * transpose(V);
  // exact zeros stay exact zeros (diagonal inputs give diagonal roots)
  bool diag = true;
  for (int i = 0; i < n && diag; ++i)
    for (int j = 0; j < n; ++j)
      if (i != j && m(i, j) != 0.0) {
        diag = false;
        break;
      }
  if (diag) {
    out = Mat::zero(n, n);
    for (int i = 0; i < n; ++i) out(i, i) = std::sqrt(std::max(m(i, i), 0.0));
  }
  return out;
}

}  // namespace pumpb::la
