// K_mc: Monte-Carlo CP certification rollouts (cp.hpp:214-268) on sm_100a.
//
// One thread per (trajectory, rollout).  Each rollout simulates the closed
// loop around the nominal trajectory with the reference's counter-hash
// normals, checks every realized point and every eps_cc-subdivided segment
// against the workspace, and stops at the first hit.
//
// Per step the state-independent noise of the transition t -> t+1
// (9 normals in 3-D, u = Gv(Sv nv), w = Gw(Sw nw)) is produced first, in
// straight-line code, so its long hash/log/cos latency overlaps the
// state-dependent collision checks of y_t; then z <- ((F z) + u) + w, which
// is exactly the reference's rounding (lti.hpp:287).  The per-(rollout, t)
// hash prefix is shared by all channels of a step and the t+1 prefix of the
// measurement noise is carried into the next step.  Nominal trajectory and
// obstacles are staged in shared memory; hits are reduced with a warp
// ballot + popc, one atomicAdd per warp; rollout-steps are counted the same
// way for the roofline.
#include <cooperative_groups.h>
#include <cmath>
#include <cstdlib>

#include "dispatch.cuh"

namespace pumpg {

constexpr int kMcBlock = 128;
constexpr int kMcTabBlock = 256;  // k_mc_tab: the staged span (nominal rows, boxes, step lists) shared by 8 warps

template <int D, int DW>
__global__ void __launch_bounds__(kMcBlock) k_mc(const LoopP<D, DW> L, WorldD w, const int64_t* __restrict__ traj_off,
                                                 const double* __restrict__ ynom_all, int64_t r0, int64_t r1,
                                                 uint64_t seed, double eps_cc, unsigned long long* __restrict__ hits,
                                                 unsigned long long* __restrict__ steps_out) {
  extern __shared__ double smem[];
  const int j = blockIdx.y;
  const int64_t p_begin = traj_off[j];
  const int n_pts = static_cast<int>(traj_off[j + 1] - p_begin);
  const int T = n_pts - 1;
  double* s_y = smem;               // n_pts * DW
  double* s_lo = s_y + n_pts * DW;  // n_obs * DW
  double* s_hi = s_lo + w.n_obs * DW;
  for (int x = threadIdx.x; x < n_pts * DW; x += blockDim.x) s_y[x] = ynom_all[p_begin * DW + x];
  for (int x = threadIdx.x; x < w.n_obs * DW; x += blockDim.x) {
    s_lo[x] = w.lo[x];
    s_hi[x] = w.hi[x];
  }
  __syncthreads();
  WorldD ws = w;
  ws.lo = s_lo;
  ws.hi = s_hi;
  const double e = eps_cc > 1e-12 ? eps_cc : 1e-12;  // std::max(eps_cc, 1e-12)

  const int64_t i = r0 + static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  bool collided = false;
  int steps = 0;
  if (i < r1) {
    const uint64_t sa = hash_seed_a(seed, static_cast<uint64_t>(i));
    uint64_t pt = mix64(sa + 0ull);
    double z[2 * D];
    {
      double nv[D];
#pragma unroll
      for (int k = 0; k < D; ++k) nv[k] = normal_from_prefix(pt, static_cast<uint64_t>(k));  // kInitial
#pragma unroll
      for (int r = 0; r < D; ++r) z[r] = row_dot<D>(L.S0 + r * D, nv);
#pragma unroll
      for (int r = D; r < 2 * D; ++r) z[r] = 0.0;
    }
    double prev[DW];
    for (int t = 0; t <= T; ++t) {
      ++steps;
      // (A) noise of the transition t -> t+1, independent of the state
      double u[2 * D], wv[2 * D];
      uint64_t pt1 = 0;
      if (t < T) {
        pt1 = mix64(sa + static_cast<uint64_t>(t + 1));
        double nv[D], nw[DW], t1[D], t2[DW];
#pragma unroll
        for (int k = 0; k < D; ++k) nv[k] = normal_from_prefix(pt, kProcess + k);
#pragma unroll
        for (int k = 0; k < DW; ++k) nw[k] = normal_from_prefix(pt1, kMeasurement + k);
#pragma unroll
        for (int r = 0; r < D; ++r) t1[r] = row_dot<D>(L.Sv + r * D, nv);
#pragma unroll
        for (int r = 0; r < DW; ++r) t2[r] = row_dot<DW>(L.Sw + r * DW, nw);
#pragma unroll
        for (int r = 0; r < 2 * D; ++r) {
          u[r] = row_dot<D>(L.Gv + r * D, t1);
          wv[r] = row_dot<DW>(L.Gw + r * DW, t2);
        }
      }
      // (B) realized point and segment checks (cp.hpp:232-248)
      double y[DW];
#pragma unroll
      for (int k = 0; k < DW; ++k) y[k] = s_y[t * DW + k] + row_dot<D>(L.C + k * D, z);
      if (!point_free<DW>(ws, y)) {
        collided = true;
        break;
      }
      if (t > 0) {
        double diff[DW];
#pragma unroll
        for (int k = 0; k < DW; ++k) diff[k] = y[k] - prev[k];
        const double len = sqrt(sqnorm<DW>(diff));
        int segs = static_cast<int>(ceil(len / e));
        if (segs < 1) segs = 1;
        double p0[DW];
#pragma unroll
        for (int k = 0; k < DW; ++k) p0[k] = prev[k];
        for (int s2 = 1; s2 <= segs && !collided; ++s2) {
          const double f = static_cast<double>(s2) / segs;
          double p1[DW];
#pragma unroll
          for (int k = 0; k < DW; ++k) p1[k] = prev[k] + (y[k] - prev[k]) * f;
          if (!point_free<DW>(ws, p1) || segment_collides<DW>(ws, p0, p1)) collided = true;
#pragma unroll
          for (int k = 0; k < DW; ++k) p0[k] = p1[k];
        }
        if (collided) break;
      }
#pragma unroll
      for (int k = 0; k < DW; ++k) prev[k] = y[k];
      // (C) z <- ((F z) + u) + w
      if (t < T) {
        double zn[2 * D];
#pragma unroll
        for (int r = 0; r < 2 * D; ++r) zn[r] = (row_dot<2 * D>(L.F + r * 2 * D, z) + u[r]) + wv[r];
#pragma unroll
        for (int r = 0; r < 2 * D; ++r) z[r] = zn[r];
        pt = pt1;
      }
    }
  }
  const unsigned bal = __ballot_sync(0xffffffffu, collided);
  const unsigned tot = __reduce_add_sync(0xffffffffu, static_cast<unsigned>(steps));
  if ((threadIdx.x & 31) == 0) {
    if (bal) atomicAdd(hits + j, static_cast<unsigned long long>(__popc(bal)));
    if (steps_out) atomicAdd(steps_out, static_cast<unsigned long long>(tot));
  }
}

// ------------------------------------------------------------------------
// Axis-separable closed loop (the per-axis double integrator with diagonal
// noise and tracking weights): every matrix only couples the four z entries
// {k, dw+k, d+k, d+dw+k} of one workspace axis k.  Dropping the structural
// zeros from a sequential sum c = 0 + sum_j M_rj x_j leaves every partial
// sum unchanged for finite operands (0*x adds +-0, and c + (+-0) == c for
// c != 0, while +0 + (-0) == +0), so the per-axis form below is bit-exact
// to the dense recursion.  One lane per axis (LPR lanes per rollout): the
// dynamics need no communication; y and the collision verdict are combined
// with shuffles; obstacle culling and segment checks are split across the
// rollout's lanes.

bool separable(const HostLoop& L) {
  const int d = L.d, dw = L.dw, nz = 2 * d;
  if (d != 2 * dw) return false;
  auto ax = [&](int i) { return (i % d) % dw; };
  for (int r = 0; r < nz; ++r) {
    for (int c = 0; c < nz; ++c)
      if (ax(r) != ax(c) && L.F[r * nz + c] != 0.0) return false;
    for (int c = 0; c < d; ++c)
      if (ax(r) != c % dw && L.Gv[r * d + c] != 0.0) return false;
    for (int c = 0; c < dw; ++c)
      if (ax(r) != c && L.Gw[r * dw + c] != 0.0) return false;
  }
  for (int a = 0; a < d; ++a)
    for (int b = 0; b < d; ++b)
      if (a % dw != b % dw && (L.Sv[a * d + b] != 0.0 || L.S0[a * d + b] != 0.0)) return false;
  for (int a = 0; a < dw; ++a)
    for (int b = 0; b < dw; ++b)
      if (a != b && L.Sw[a * dw + b] != 0.0) return false;
  for (int k = 0; k < dw; ++k)
    for (int j = 0; j < d; ++j)
      if (j % dw != k && L.C[k * d + j] != 0.0) return false;
  for (double x : L.F)
    if (!std::isfinite(x)) return false;
  return true;
}

SepBlocks sep_blocks(const HostLoop& L) {
  SepBlocks B{};
  const int d = L.d, dw = L.dw, nz = 2 * d;
  for (int k = 0; k < dw; ++k) {
    const int g[4] = {k, dw + k, d + k, d + dw + k};
    const int h[2] = {k, dw + k};
    for (int r = 0; r < 4; ++r) {
      for (int c = 0; c < 4; ++c) B.F[k][r * 4 + c] = L.F[g[r] * nz + g[c]];
      for (int a = 0; a < 2; ++a) B.Gv[k][r * 2 + a] = L.Gv[g[r] * d + h[a]];
      B.Gw[k][r] = L.Gw[g[r] * dw + k];
    }
    for (int a = 0; a < 2; ++a)
      for (int b = 0; b < 2; ++b) {
        B.Sv[k][a * 2 + b] = L.Sv[h[a] * d + h[b]];
        B.S0[k][a * 2 + b] = L.S0[h[a] * d + h[b]];
      }
    B.Sw[k] = L.Sw[k * dw + k];
    for (int a = 0; a < 2; ++a) B.C[k][a] = L.C[k * d + h[a]];
  }
  return B;
}

// One lane per axis: a rollout is a group of DW consecutive lanes; a warp
// holds 32 / DW groups (DW = 3: 10 groups, lanes 30-31 idle).
template <int DW>
constexpr int lanes_per_rollout() {
  return DW;
}
template <int DW>
constexpr int groups_per_warp() {
  return 32 / DW;
}

template <int DW, int MINB>
__global__ void __launch_bounds__(kMcBlock, MINB) k_mc_sep(const SepBlocks B, WorldD w, const int64_t* __restrict__ traj_off,
                                                     const double* __restrict__ ynom_all, int64_t r0, int64_t r1,
                                                     uint64_t seed, double eps_cc, unsigned long long* __restrict__ hits,
                                                     unsigned long long* __restrict__ steps_out) {
  constexpr int LPR = lanes_per_rollout<DW>();
  extern __shared__ double smem[];
  const int j = blockIdx.y;
  const int64_t p_begin = traj_off[j];
  const int n_pts = static_cast<int>(traj_off[j + 1] - p_begin);
  const int T = n_pts - 1;
  double* s_y = smem;               // n_pts * DW
  double* s_lo = s_y + n_pts * DW;  // n_obs * DW, inflated for culling: lo - M
  double* s_hi = s_lo + w.n_obs * DW;
  double* s_clo = s_hi + w.n_obs * DW;  // exact boxes for the reference tests
  double* s_chi = s_clo + w.n_obs * DW;
  for (int x = threadIdx.x; x < n_pts * DW; x += blockDim.x) s_y[x] = ynom_all[p_begin * DW + x];
  for (int x = threadIdx.x; x < w.n_obs * DW; x += blockDim.x) {
    const int k = x % DW;
    const double bl = w.blo[k] < 0 ? -w.blo[k] : w.blo[k], bh = w.bhi[k] < 0 ? -w.bhi[k] : w.bhi[k];
    const double lo = w.lo[x], hi = w.hi[x];
    // margin >= box_separated's for any point inside the bounds (dev.cuh)
    const double M = 1e-9 * (1.0 + (lo < 0 ? -lo : lo) + (hi < 0 ? -hi : hi) + 2.0 * (bl > bh ? bl : bh));
    s_lo[x] = lo - M;
    s_hi[x] = hi + M;
    s_clo[x] = lo;
    s_chi[x] = hi;
  }
  __syncthreads();
  const double e = eps_cc > 1e-12 ? eps_cc : 1e-12;  // std::max(eps_cc, 1e-12)
  constexpr int GPW = groups_per_warp<DW>();
  const int lane = threadIdx.x & 31;
  const int q = lane % LPR;                 // axis of this lane
  const int g = lane / LPR;                 // rollout group in the warp (g == GPW: idle lanes)
  const int gbase = lane - q;               // first lane of the rollout group
  const int k = q;
  const int64_t i = r0 + (static_cast<int64_t>(blockIdx.x) * (kMcBlock / 32) + (threadIdx.x >> 5)) * GPW + g;
  const bool active = g < GPW && i < r1;
  const unsigned gmask = gbase + LPR <= 32 ? ((1u << LPR) - 1u) << gbase : 0xffffffffu << gbase;
  bool collided = false;
  int steps = 0;
  // per-axis blocks in shared memory (39 doubles per axis; the 3 axes of a
  // warp access land in distinct banks)
  __shared__ double s_blk[3][40];
  for (int x = threadIdx.x; x < 3 * 40; x += blockDim.x) {
    const int ax = x / 40, o = x % 40;
    double v = 0.0;
    if (ax < DW) {
      if (o < 16) v = B.F[ax][o];
      else if (o < 24) v = B.Gv[ax][o - 16];
      else if (o < 28) v = B.Gw[ax][o - 24];
      else if (o < 32) v = B.Sv[ax][o - 28];
      else if (o < 36) v = B.S0[ax][o - 32];
      else if (o < 38) v = B.C[ax][o - 36];
      else if (o == 38) v = B.Sw[ax];
    }
    s_blk[ax][o] = v;
  }
  __syncthreads();
  const double* F = &s_blk[k][0];
  const double* Gv = &s_blk[k][16];
  const double* Gw = &s_blk[k][24];
  const double* Sv = &s_blk[k][28];
  const double* S0 = &s_blk[k][32];
  const double* C = &s_blk[k][36];
  const double Sw = s_blk[k][38];
  const uint64_t ch0 = static_cast<uint64_t>(k), ch1 = static_cast<uint64_t>(DW + k);

  double z[4];
  uint64_t sa = 0, pt = 0;
  if (active) {
    sa = hash_seed_a(seed, static_cast<uint64_t>(i));
    pt = mix64(sa + 0ull);
    const double n0 = normal_from_prefix(pt, ch0), n1 = normal_from_prefix(pt, ch1);  // kInitial channels
    z[0] = (0.0 + S0[0] * n0) + S0[1] * n1;
    z[1] = (0.0 + S0[2] * n0) + S0[3] * n1;
    z[2] = 0.0;
    z[3] = 0.0;
  }
  double prev[DW];
  for (int t = 0; t <= T; ++t) {
    // group-uniform loop: all lanes of a rollout stay in lock step
    const bool live = active && !collided;
    if (!__any_sync(0xffffffffu, live)) break;
    double u[4] = {0, 0, 0, 0}, wv[4] = {0, 0, 0, 0};
    uint64_t pt1 = 0;
    double y_own = 0;
    if (live) {
      ++steps;
      if (t < T) {  // (A) noise of t -> t+1 for this axis
        pt1 = mix64(sa + static_cast<uint64_t>(t + 1));
        const double nv0 = normal_from_prefix(pt, kProcess + ch0);
        const double nv1 = normal_from_prefix(pt, kProcess + ch1);
        const double nw = normal_from_prefix(pt1, kMeasurement + static_cast<uint64_t>(k));
        const double t10 = (0.0 + Sv[0] * nv0) + Sv[1] * nv1;
        const double t11 = (0.0 + Sv[2] * nv0) + Sv[3] * nv1;
        const double t2 = 0.0 + Sw * nw;
#pragma unroll
        for (int r = 0; r < 4; ++r) {
          u[r] = (0.0 + Gv[2 * r] * t10) + Gv[2 * r + 1] * t11;
          wv[r] = 0.0 + Gw[r] * t2;
        }
      }
      y_own = s_y[t * DW + k] + ((0.0 + C[0] * z[0]) + C[1] * z[1]);
    }
    // (B) gather the realized point of the rollout into every lane of the group
    double y[DW];
#pragma unroll
    for (int a = 0; a < DW; ++a) y[a] = __shfl_sync(0xffffffffu, y_own, gbase + a);
    if (t == 0) {
#pragma unroll
      for (int a = 0; a < DW; ++a) prev[a] = y[a];
    }
    bool hit = false;
    if (live) {
      // bounds (every lane), then obstacles culled against bbox(prev, y)
      bool inb = true;
#pragma unroll
      for (int a = 0; a < DW; ++a) inb = inb && !(y[a] < w.blo[a] || y[a] > w.bhi[a]);
      if (!inb) {
        hit = true;
      } else {
        double bl[DW], bh[DW];
#pragma unroll
        for (int a = 0; a < DW; ++a) {
          bl[a] = prev[a] < y[a] ? prev[a] : y[a];
          bh[a] = prev[a] < y[a] ? y[a] : prev[a];
        }
        uint64_t cand = 0;  // this lane's share of the obstacles (o = q mod LPR)
        for (int o = q; o < w.n_obs && o < 64; o += LPR) {
          bool sep = false;
#pragma unroll
          for (int a = 0; a < DW; ++a) sep = sep || (bh[a] < s_lo[o * DW + a]) || (bl[a] > s_hi[o * DW + a]);
          if (!sep) cand |= 1ull << o;
        }
        // obstacles beyond the first 64 are never culled (checked below)
        uint64_t all = 0;  // union of the group's shares
#pragma unroll
        for (int x = 0; x < LPR; ++x) all |= __shfl_sync(gmask, cand, gbase + x);  // group-uniform branch
        // the point y itself (t = 0 included): lane 0 of the group
        if (q == 0) {
          for (uint64_t m = all; m; m &= m - 1) {
            const int o = __ffsll(static_cast<long long>(m)) - 1;
            if (box_contains<DW>(s_clo + o * DW, s_chi + o * DW, y)) hit = true;
          }
        }
        if (w.n_obs > 64 && q == 0) {
          for (int o = 64; o < w.n_obs; ++o)
            if (box_contains<DW>(s_clo + o * DW, s_chi + o * DW, y)) hit = true;
        }
        if (t > 0) {  // segments prev -> y, subdivided to eps_cc (cp.hpp:237-248), split across lanes
          double diff[DW];
#pragma unroll
          for (int a = 0; a < DW; ++a) diff[a] = y[a] - prev[a];
          const double len = sqrt(sqnorm<DW>(diff));
          int segs = static_cast<int>(ceil(len / e));
          if (segs < 1) segs = 1;
          for (int s2 = 1 + q; s2 <= segs; s2 += LPR) {
            double p0[DW], p1[DW];
            const double f1 = static_cast<double>(s2) / segs;
#pragma unroll
            for (int a = 0; a < DW; ++a) p1[a] = prev[a] + (y[a] - prev[a]) * f1;
            if (s2 == 1) {
#pragma unroll
              for (int a = 0; a < DW; ++a) p0[a] = prev[a];
            } else {
              const double f0 = static_cast<double>(s2 - 1) / segs;
#pragma unroll
              for (int a = 0; a < DW; ++a) p0[a] = prev[a] + (y[a] - prev[a]) * f0;
            }
            bool in1 = true;
#pragma unroll
            for (int a = 0; a < DW; ++a) in1 = in1 && !(p1[a] < w.blo[a] || p1[a] > w.bhi[a]);
            if (!in1) {
              hit = true;
              break;
            }
            for (uint64_t m = all; m; m &= m - 1) {
              const int o = __ffsll(static_cast<long long>(m)) - 1;
              if (box_contains<DW>(s_clo + o * DW, s_chi + o * DW, p1) ||
                  segment_hits<DW>(p0, p1, s_clo + o * DW, s_chi + o * DW)) {
                hit = true;
                break;
              }
            }
            for (int o = 64; o < w.n_obs && !hit; ++o)
              if (box_contains<DW>(s_clo + o * DW, s_chi + o * DW, p1) ||
                  segment_hits<DW>(p0, p1, s_clo + o * DW, s_chi + o * DW))
                hit = true;
            if (hit) break;
          }
        }
      }
    }
    // rollout verdict = OR over its lanes
    const unsigned hb = __ballot_sync(0xffffffffu, hit);
    const bool ghit = (hb & gmask) != 0u;
    if (live) {
      if (ghit) {
        collided = true;
      } else {
#pragma unroll
        for (int a = 0; a < DW; ++a) prev[a] = y[a];
        if (t < T) {  // (C) z <- ((F z) + u) + w  for this axis block
          double zn[4];
#pragma unroll
          for (int r = 0; r < 4; ++r) {
            double c = 0.0;
#pragma unroll
            for (int x = 0; x < 4; ++x) c = c + F[r * 4 + x] * z[x];
            zn[r] = (c + u[r]) + wv[r];
          }
#pragma unroll
          for (int r = 0; r < 4; ++r) z[r] = zn[r];
          pt = pt1;
        }
      }
    }
  }
  const bool leader = (q == 0) && active;
  const unsigned bal = __ballot_sync(0xffffffffu, leader && collided);
  const unsigned tot = __reduce_add_sync(0xffffffffu, leader ? static_cast<unsigned>(steps) : 0u);
  if (lane == 0) {
    if (bal) atomicAdd(hits + j, static_cast<unsigned long long>(__popc(bal)));
    if (steps_out) atomicAdd(steps_out, static_cast<unsigned long long>(tot));
  }
}

// ------------------------------------------------------------------------
// Common-random-number table (kernels.h, McTable).
//

// Build in two phases for the axis-separable loop (the default path): the
// noise of every (transition t-1 -> t, rollout, axis) is a pure function of
// the key, so k_mcnoise_sep draws all of it in parallel (3 normals and the
// Sv / Sw products per item, the operations k_mc_sep performs), and
// k_mcrec_sep then runs only the short per-axis recurrence, reading the noise
// kMcPf steps at a time.  Same operations in the same order as k_mctab_sep.
template <int DW>
__global__ void __launch_bounds__(256) k_mcnoise_sep(const SepBlocks B, int64_t r0, int64_t n, uint64_t seed, int tn0,
                                                     int steps, double* __restrict__ nz) {
  const int64_t x = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (x >= static_cast<int64_t>(steps) * n * DW) return;
  const int64_t tt = x / (n * DW);
  const int64_t rem = x - tt * n * DW;
  const int64_t li = rem / DW;
  const int k = static_cast<int>(rem - li * DW);
  const int t = tn0 + static_cast<int>(tt);
  const uint64_t sa = hash_seed_a(seed, static_cast<uint64_t>(r0 + li));
  const uint64_t pt = mix64(sa + static_cast<uint64_t>(t - 1));
  const uint64_t pt1 = mix64(sa + static_cast<uint64_t>(t));
  const uint64_t ch0 = static_cast<uint64_t>(k), ch1 = static_cast<uint64_t>(DW + k);
  const double nv0 = normal_from_prefix(pt, kProcess + ch0);
  const double nv1 = normal_from_prefix(pt, kProcess + ch1);
  const double nw = normal_from_prefix(pt1, kMeasurement + static_cast<uint64_t>(k));
  const double* Sv = B.Sv[k];
  double* o = nz + x * 3;
  o[0] = (0.0 + Sv[0] * nv0) + Sv[1] * nv1;
  o[1] = (0.0 + Sv[2] * nv0) + Sv[3] * nv1;
  o[2] = 0.0 + B.Sw[k] * nw;
}

constexpr int kMcPf = 8;
template <int DW>
__global__ void __launch_bounds__(128) k_mcrec_sep(const SepBlocks B, int64_t r0, int64_t n, uint64_t seed,
                                                   int t_from, int t_to, int tn0, const double* __restrict__ nz,
                                                   double* __restrict__ dy, double* __restrict__ zst) {
  const int64_t x = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (x >= n * DW) return;
  const int64_t li = x / DW;
  const int k = static_cast<int>(x - li * DW);
  const double* F = B.F[k];
  const double* Gv = B.Gv[k];
  const double* Gw = B.Gw[k];
  const double* C = B.C[k];
  double z[4];
  double* zs = zst + x * 4;
  if (t_from == 0) {
    const uint64_t pt = mix64(hash_seed_a(seed, static_cast<uint64_t>(r0 + li)) + 0ull);
    const double n0 = normal_from_prefix(pt, static_cast<uint64_t>(k));
    const double n1 = normal_from_prefix(pt, static_cast<uint64_t>(DW + k));  // kInitial channels
    z[0] = (0.0 + B.S0[k][0] * n0) + B.S0[k][1] * n1;
    z[1] = (0.0 + B.S0[k][2] * n0) + B.S0[k][3] * n1;
    z[2] = 0.0;
    z[3] = 0.0;
    dy[x] = (0.0 + C[0] * z[0]) + C[1] * z[1];  // t = 0
  } else {
#pragma unroll
    for (int r = 0; r < 4; ++r) z[r] = zs[r];
  }
  const int64_t stride = n * DW * 3;
  for (int tb = tn0; tb <= t_to; tb += kMcPf) {
    double q[kMcPf][3];
#pragma unroll
    for (int u = 0; u < kMcPf; ++u)
      if (tb + u <= t_to) {
        const double* src = nz + static_cast<int64_t>(tb + u - tn0) * stride + x * 3;
        q[u][0] = src[0];
        q[u][1] = src[1];
        q[u][2] = src[2];
      }
#pragma unroll
    for (int u = 0; u < kMcPf; ++u) {
      const int t = tb + u;
      if (t > t_to) break;
      double zn[4];
#pragma unroll
      for (int r = 0; r < 4; ++r) {
        const double uu = (0.0 + Gv[2 * r] * q[u][0]) + Gv[2 * r + 1] * q[u][1];
        const double wv = 0.0 + Gw[r] * q[u][2];
        double c = 0.0;
#pragma unroll
        for (int y = 0; y < 4; ++y) c = c + F[r * 4 + y] * z[y];
        zn[r] = (c + uu) + wv;
      }
#pragma unroll
      for (int r = 0; r < 4; ++r) z[r] = zn[r];
      dy[static_cast<int64_t>(t) * n * DW + x] = (0.0 + C[0] * z[0]) + C[1] * z[1];
    }
  }
#pragma unroll
  for (int r = 0; r < 4; ++r) zs[r] = z[r];
}

// Build, general loop: one thread per rollout, the k_mc recursion.
template <int D, int DW>
__global__ void __launch_bounds__(kMcBlock) k_mctab_dense(const LoopP<D, DW> L, int64_t r0, int64_t n, uint64_t seed,
                                                          int t_from, int t_to, double* __restrict__ dy,
                                                          double* __restrict__ zst) {
  const int64_t li = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (li >= n) return;
  const int64_t i = r0 + li;
  const uint64_t sa = hash_seed_a(seed, static_cast<uint64_t>(i));
  double z[2 * D];
  double* zs = zst + li * 2 * D;
  if (t_from == 0) {
    const uint64_t pt = mix64(sa + 0ull);
    double nv[D];
#pragma unroll
    for (int k = 0; k < D; ++k) nv[k] = normal_from_prefix(pt, static_cast<uint64_t>(k));  // kInitial
#pragma unroll
    for (int r = 0; r < D; ++r) z[r] = row_dot<D>(L.S0 + r * D, nv);
#pragma unroll
    for (int r = D; r < 2 * D; ++r) z[r] = 0.0;
  } else {
#pragma unroll
    for (int r = 0; r < 2 * D; ++r) z[r] = zs[r];
  }
  for (int t = t_from; t <= t_to; ++t) {
    if (t > 0) {
      const uint64_t pt = mix64(sa + static_cast<uint64_t>(t - 1));
      const uint64_t pt1 = mix64(sa + static_cast<uint64_t>(t));
      double nv[D], nw[DW], t1[D], t2[DW], u[2 * D], wv[2 * D];
#pragma unroll
      for (int k = 0; k < D; ++k) nv[k] = normal_from_prefix(pt, kProcess + k);
#pragma unroll
      for (int k = 0; k < DW; ++k) nw[k] = normal_from_prefix(pt1, kMeasurement + k);
#pragma unroll
      for (int r = 0; r < D; ++r) t1[r] = row_dot<D>(L.Sv + r * D, nv);
#pragma unroll
      for (int r = 0; r < DW; ++r) t2[r] = row_dot<DW>(L.Sw + r * DW, nw);
#pragma unroll
      for (int r = 0; r < 2 * D; ++r) {
        u[r] = row_dot<D>(L.Gv + r * D, t1);
        wv[r] = row_dot<DW>(L.Gw + r * DW, t2);
      }
      double zn[2 * D];
#pragma unroll
      for (int r = 0; r < 2 * D; ++r) zn[r] = (row_dot<2 * D>(L.F + r * 2 * D, z) + u[r]) + wv[r];
#pragma unroll
      for (int r = 0; r < 2 * D; ++r) z[r] = zn[r];
    }
#pragma unroll
    for (int k = 0; k < DW; ++k) dy[(static_cast<int64_t>(t) * n + li) * DW + k] = row_dot<D>(L.C + k * D, z);
  }
#pragma unroll
  for (int r = 0; r < 2 * D; ++r) zs[r] = z[r];
}

// Certify against the table.  A rollout's verdict is the OR of independent
// per-step tests (point y_t, segment y_{t-1} -> y_t; the reference stops at
// the first hit, which changes the work, not the verdict), so the steps are
// spread over the grid: thread = (trajectory, rollout, span of kMcSpan
// steps), y_t = ynom_t + dy_t (the addition k_mc performs), the collision
// tests of k_mc_sep (bounds, bbox-culled obstacles, eps_cc-subdivided
// segment).  A hit claims flag[j][i] (the rollout's first hit over the
// span blocks counts it into hits[j]).
constexpr int kMcChunk = 8;   // steps whose table rows a thread loads up front
// Per (trajectory, step) the candidate obstacles every rollout of the table
// can meet (see k_mc_tab), listed once per certification instead of once per
// block: the box ynom -/+ the largest |dy| over the table's rollouts at t and
// t - 1 (fl is monotone, so fl(ynom +- maxdev) bounds fl(ynom + dy)), widened
// by the sub-segment rounding margin; the inflated obstacles meeting it, a
// warp per step (ballot compaction).  A step with an empty list whose box is
// inside the workspace holds no failing test for any rollout: skip = 1.
template <int DW>
__global__ void __launch_bounds__(128) k_mc_steps(WorldD w, const int64_t* __restrict__ traj_off,
                                                  const double* __restrict__ ynom_all,
                                                  const unsigned long long* __restrict__ maxdev, int t_stride,
                                                  uint16_t* __restrict__ g_list, int32_t* __restrict__ g_nl,
                                                  uint8_t* __restrict__ g_skip, const int32_t* __restrict__ live) {
  const int j = blockIdx.y;
  if (live && !live[j]) return;
  const int lane = threadIdx.x & 31;
  const int t = blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5);
  const int64_t p_begin = traj_off[j];
  const int T = static_cast<int>(traj_off[j + 1] - p_begin) - 1;
  if (t > T) return;
  const double* y1 = ynom_all + (p_begin + t) * DW;
  mc_step_row<DW, kStepCap>(w, y1, t > 0 ? y1 - DW : nullptr, maxdev, t, static_cast<int64_t>(j) * t_stride + t, lane, g_list,
                  g_nl, g_skip);
}

template <int DW, int kMcSub>  // kMcSub sub-chunks per block: a block spans kMcSpan steps
__global__ void __launch_bounds__(kMcTabBlock) k_mc_tab(WorldD w, const int64_t* __restrict__ traj_off,
                                                     const double* __restrict__ ynom_all, int64_t r0, int64_t r1,
                                                     int64_t tab_r0, int64_t tab_n, const double* __restrict__ dy,
                                                     const unsigned long long* __restrict__ maxdev, double eps_cc,
                                                     uint32_t* __restrict__ flags, const int32_t* __restrict__ live,
                                                     int t_stride, const uint16_t* __restrict__ g_list,
                                                     const int32_t* __restrict__ g_nl,
                                                     const uint8_t* __restrict__ g_skip,
                                                     unsigned long long* __restrict__ hits,
                                                     unsigned long long* __restrict__ steps_out) {
  extern __shared__ double smem[];
  constexpr int kMcSpan = kMcChunk * kMcSub;
  __shared__ uint16_t s_list[kMcSpan + 1][kStepCap];
  __shared__ int s_nlist[kMcSpan + 1];  // -1: more than kStepCap candidates
  __shared__ int s_skip[kMcSpan + 1];
  const int j = blockIdx.y;
  if (live && !live[j]) return;  // trajectory not certified (its nominal collides): flags stay 0
  if (steps_out && blockIdx.x == 0 && blockIdx.z == 0 && threadIdx.x == 0)  // rollouts x (T_j + 1)
    atomicAdd(steps_out, static_cast<unsigned long long>(r1 - r0) *
                             static_cast<unsigned long long>(traj_off[j + 1] - traj_off[j]));
  const int64_t p_begin = traj_off[j];
  const int n_pts = static_cast<int>(traj_off[j + 1] - p_begin);
  const int T = n_pts - 1;
  const int t_lo = blockIdx.z * kMcSpan;
  if (t_lo > T) return;
  const int t_hi = min(T, t_lo + kMcSpan - 1);
  const int s_lo_t = t_lo > 0 ? t_lo - 1 : 0;  // rows staged: [s_lo_t, t_hi]
  const int rows = t_hi - s_lo_t + 1;
  // the span's step flags and lists (k_mc_steps); a span where every step
  // skips exits before staging anything
  const int64_t row0 = static_cast<int64_t>(j) * t_stride + s_lo_t;
  bool act = false;
  if (threadIdx.x <= kMcSpan) {
    const int r = threadIdx.x, t = s_lo_t + r;
    const bool in = t >= t_lo && t <= t_hi;
    const int skip = in ? g_skip[row0 + r] : 1;
    s_skip[r] = skip;
    s_nlist[r] = in ? g_nl[row0 + r] : 0;
    act = !skip;
  }
  if (!__syncthreads_or(act)) return;
  double* s_y = smem;
  double* s_lo = s_y + rows * DW;
  double* s_hi = s_lo + w.n_obs * DW;
  double* s_clo = s_hi + w.n_obs * DW;
  double* s_chi = s_clo + w.n_obs * DW;
  for (int x = threadIdx.x; x < rows * DW; x += blockDim.x) s_y[x] = ynom_all[(p_begin + s_lo_t) * DW + x];
  for (int x = threadIdx.x; x < w.n_obs * DW; x += blockDim.x) {
    const int k = x % DW;
    const double bl = w.blo[k] < 0 ? -w.blo[k] : w.blo[k], bh = w.bhi[k] < 0 ? -w.bhi[k] : w.bhi[k];
    const double lo = w.lo[x], hi = w.hi[x];
    const double M = 1e-9 * (1.0 + (lo < 0 ? -lo : lo) + (hi < 0 ? -hi : hi) + 2.0 * (bl > bh ? bl : bh));
    s_lo[x] = lo - M;
    s_hi[x] = hi + M;
    s_clo[x] = lo;
    s_chi[x] = hi;
  }
  for (int x = threadIdx.x; x < (kMcSpan + 1) * kStepCap; x += blockDim.x) {
    const int r = x / kStepCap, q = x % kStepCap;
    if (q < s_nlist[r]) s_list[r][q] = g_list[(row0 + r) * kStepCap + q];
  }
  __syncthreads();
  const double e = eps_cc > 1e-12 ? eps_cc : 1e-12;  // std::max(eps_cc, 1e-12)
  const int64_t i = r0 + static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= r1) return;
  const double* d = dy + (i - tab_r0) * DW;
  const int64_t stride = tab_n * DW;
  bool hit = false;
  // the block's span in sub-chunks of kMcChunk steps; row rb of a sub-chunk
  // seeds prev (it was the previous sub-chunk's last step)
  for (int rb = 0; rb < kMcSpan && s_lo_t + rb <= t_hi && !hit; rb += kMcChunk) {
  double dv[kMcChunk + 1][DW];  // issue every needed load of the sub-chunk up front
#pragma unroll
  for (int r = 0; r <= kMcChunk; ++r) {
    const int rr = rb + r;
    const bool need = s_lo_t + rr <= t_hi && (!s_skip[rr] || (r < kMcChunk && !s_skip[rr + 1]));
    if (need) {
#pragma unroll
      for (int k = 0; k < DW; ++k) dv[r][k] = d[static_cast<int64_t>(s_lo_t + rr) * stride + k];
    }
  }
#pragma unroll
  for (int r = 0; r <= kMcChunk; ++r) {
    const int rr = rb + r;
    const int t = s_lo_t + rr;
    if (t < t_lo || t > t_hi || hit || s_skip[rr] || (r == 0 && rb > 0)) continue;  // row 0 only seeds prev
    double prev[DW];
    const int rp = t > 0 ? r - 1 : r;  // t = 0: the step's box is the point itself
#pragma unroll
    for (int k = 0; k < DW; ++k) prev[k] = s_y[(rb + rp) * DW + k] + dv[rp][k];
    double y[DW];
#pragma unroll
    for (int k = 0; k < DW; ++k) y[k] = s_y[rr * DW + k] + dv[r][k];
    bool inb = true;
#pragma unroll
    for (int a = 0; a < DW; ++a) inb = inb && !(y[a] < w.blo[a] || y[a] > w.bhi[a]);
    if (!inb) {
      hit = true;
      continue;
    }
    double bl[DW], bh[DW];
#pragma unroll
    for (int a = 0; a < DW; ++a) {
      bl[a] = prev[a] < y[a] ? prev[a] : y[a];
      bh[a] = prev[a] < y[a] ? y[a] : prev[a];
    }
    const int nl = s_nlist[rr];
    // this rollout's culling within the step's list (bit q <-> s_list[rr][q])
    uint64_t cand = 0;
    for (int q = 0; q < nl; ++q) {
      const int o = s_list[rr][q];
      bool sep = false;
#pragma unroll
      for (int a = 0; a < DW; ++a) sep = sep || (bh[a] < s_lo[o * DW + a]) || (bl[a] > s_hi[o * DW + a]);
      if (!sep) cand |= 1ull << q;
    }
    if (nl >= 0) {
      for (uint64_t m = cand; m && !hit; m &= m - 1) {
        const int o = s_list[rr][__ffsll(static_cast<long long>(m)) - 1];
        if (box_contains<DW>(s_clo + o * DW, s_chi + o * DW, y)) hit = true;
      }
    } else {
      for (int o = 0; o < w.n_obs && !hit; ++o)
        if (box_contains<DW>(s_clo + o * DW, s_chi + o * DW, y)) hit = true;
    }
    // every subdivision point lies in bbox(prev, y) up to rounding: with no
    // candidate obstacle and the box strictly inside the bounds, no
    // sub-segment test can fail
    bool clear = nl >= 0 && cand == 0;
#pragma unroll
    for (int a2 = 0; a2 < DW; ++a2) {
      const double m = 1e-12 * (1.0 + (bl[a2] < 0 ? -bl[a2] : bl[a2]) + (bh[a2] < 0 ? -bh[a2] : bh[a2]));
      clear = clear && bl[a2] - m > w.blo[a2] && bh[a2] + m < w.bhi[a2];
    }
    if (t > 0 && !hit && !clear) {  // segments prev -> y, subdivided to eps_cc (cp.hpp:237-248)
      double diff[DW];
#pragma unroll
      for (int a = 0; a < DW; ++a) diff[a] = y[a] - prev[a];
      const double len = sqrt(sqnorm<DW>(diff));
      int segs = static_cast<int>(ceil(len / e));
      if (segs < 1) segs = 1;
      double p0[DW];
#pragma unroll
      for (int a = 0; a < DW; ++a) p0[a] = prev[a];
      for (int s2 = 1; s2 <= segs && !hit; ++s2) {
        double p1[DW];
        const double f1 = static_cast<double>(s2) / segs;
#pragma unroll
        for (int a = 0; a < DW; ++a) p1[a] = prev[a] + (y[a] - prev[a]) * f1;
        bool in1 = true;
#pragma unroll
        for (int a = 0; a < DW; ++a) in1 = in1 && !(p1[a] < w.blo[a] || p1[a] > w.bhi[a]);
        if (!in1) {
          hit = true;
          break;
        }
        if (nl >= 0) {
          for (uint64_t m = cand; m; m &= m - 1) {
            const int o = s_list[rr][__ffsll(static_cast<long long>(m)) - 1];
            if (box_contains<DW>(s_clo + o * DW, s_chi + o * DW, p1) ||
                segment_hits<DW>(p0, p1, s_clo + o * DW, s_chi + o * DW)) {
              hit = true;
              break;
            }
          }
        } else {
          for (int o = 0; o < w.n_obs && !hit; ++o)
            if (box_contains<DW>(s_clo + o * DW, s_chi + o * DW, p1) ||
                segment_hits<DW>(p0, p1, s_clo + o * DW, s_chi + o * DW))
              hit = true;
        }
#pragma unroll
        for (int a = 0; a < DW; ++a) p0[a] = p1[a];
      }
    }
  }
  }
  // a rollout can hit in several spans: the first claim counts it
  const bool first = hit && atomicExch(flags + static_cast<int64_t>(j) * (r1 - r0) + (i - r0), 1u) == 0u;
  const cooperative_groups::coalesced_group cg = cooperative_groups::coalesced_threads();
  const unsigned b = cg.ballot(first);
  if (b && cg.thread_rank() == 0) atomicAdd(hits + j, static_cast<unsigned long long>(__popc(b)));
}

// maxdev[t][k] = max_i |dy[t][i][k]| over the table's rollouts, as the bit
// pattern of a non-negative double (ordered like the value) for atomicMax
__global__ void __launch_bounds__(256) k_mctab_maxdev(const double* __restrict__ dy, int64_t n, int dw, int t_from,
                                                      unsigned long long* __restrict__ maxdev) {
  const int t = t_from + blockIdx.y;
  __shared__ unsigned long long s_m[3];
  if (threadIdx.x < 3) s_m[threadIdx.x] = 0ull;
  __syncthreads();
  unsigned long long m[3] = {0ull, 0ull, 0ull};
  const double* row = dy + static_cast<int64_t>(t) * n * dw;
  for (int64_t x = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; x < n * dw;
       x += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const double v = row[x];
    const unsigned long long b = static_cast<unsigned long long>(__double_as_longlong(v < 0 ? -v : v));
    const int k = static_cast<int>(x % dw);
    m[k] = b > m[k] ? b : m[k];
  }
  for (int k = 0; k < dw; ++k) {
    unsigned long long v = m[k];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const unsigned long long y = __shfl_xor_sync(0xffffffffu, v, o);
      v = y > v ? y : v;
    }
    if ((threadIdx.x & 31) == 0) atomicMax(&s_m[k], v);
  }
  __syncthreads();
  if (threadIdx.x < dw) atomicMax(&maxdev[t * dw + threadIdx.x], s_m[threadIdx.x]);
}

static bool same_loop(const HostLoop& a, const HostLoop& b) {
  return a.d == b.d && a.dw == b.dw && a.F == b.F && a.Gv == b.Gv && a.Gw == b.Gw && a.Sv == b.Sv && a.Sw == b.Sw &&
         a.S0 == b.S0 && a.C == b.C;
}

// Make the table cover rollouts [r0, r1) and steps t <= T.  Returns false
// when it would not fit the memory budget (the caller then runs the direct
// kernels).
static bool ensure_table(McTable& tab, const HostLoop& HL, int64_t r0, int64_t r1, uint64_t seed, int T,
                         cudaStream_t st, int64_t* launches) {
  const int64_t n = r1 - r0;
  const int dw = HL.dw, d = HL.d;
  const size_t row = static_cast<size_t>(n) * dw * 8;
  constexpr size_t kBudget = size_t(24) << 30;  // 24 GiB of HBM at most
  if (row * static_cast<size_t>(T + 1) > kBudget) return false;
  if (!tab.valid || tab.seed != seed || tab.r0 != r0 || tab.r1 != r1 || !same_loop(tab.L, HL)) {
    tab.valid = true;
    tab.seed = seed;
    tab.r0 = r0;
    tab.r1 = r1;
    tab.L = HL;
    tab.t_done = -1;
    tab.sep = HL.dw >= 2 && HL.dw <= 3 && separable(HL);
    tab.z.ensure(static_cast<size_t>(n) * std::max(4 * dw, 2 * d) * 8 + 256);
  }
  if (T <= tab.t_done) return true;
  const int t_from = tab.t_done + 1;
  if (static_cast<size_t>(T + 1) * row > tab.dy.cap) {
    // grow with headroom (the dy prefix is t-major: keep the rows built so far)
    const int want = T + 1 + (T + 1) / 2;
    const size_t bytes = std::min(static_cast<size_t>(want) * row, std::max(kBudget, static_cast<size_t>(T + 1) * row));
    tab.dy.grow(bytes, static_cast<size_t>(t_from) * row, st);
  }
  KScope ks(st, F_MC_TABLE);
  if (tab.sep) {
    // time slices of kTabSlice steps bound the noise scratch (n x slice x 3 x dw doubles)
    constexpr int kTabSlice = 64;
    const SepBlocks B = sep_blocks(HL);
    tab.nz.ensure(static_cast<size_t>(kTabSlice) * n * dw * 3 * 8 + 256);
    for (int tc0 = t_from; tc0 <= T; tc0 += kTabSlice) {
      const int tc1 = std::min(T, tc0 + kTabSlice - 1);
      const int tn0 = std::max(1, tc0);
      const int steps = tc1 - tn0 + 1;
      dispatch_dw(dw, [&]<int DW>() {
        if (steps > 0) {
          const int64_t items = static_cast<int64_t>(steps) * n * DW;
          // 60 KB of (unused) dynamic shared memory caps the kernel at 3 blocks
          // per SM, so the cooperative round kernel (24k registers, 24 KB) or an
          // expand block always fits next to it during explore
          constexpr int kNoiseSmem = 60 * 1024;
          static bool attr[64] = {};  // per device (the attribute is set in each device's context)
          int dev = 0;
          PUMP_CUDA(cudaGetDevice(&dev));
          if (dev < 0 || dev >= 64 || !attr[dev]) {
            PUMP_CUDA(cudaFuncSetAttribute(k_mcnoise_sep<DW>, cudaFuncAttributeMaxDynamicSharedMemorySize, kNoiseSmem));
            if (dev >= 0 && dev < 64) attr[dev] = true;
          }
          k_mcnoise_sep<DW><<<grid_for(items, 256), 256, kNoiseSmem, st>>>(B, r0, n, seed, tn0, steps,
                                                                           tab.nz.as<double>());
          ++*launches;
        }
        k_mcrec_sep<DW><<<grid_for(n * DW, 128), 128, 0, st>>>(B, r0, n, seed, tc0, tc1, tn0, tab.nz.as<double>(),
                                                              tab.dy.as<double>(), tab.z.as<double>());
      });
      if (tc0 + kTabSlice > T) break;
    }
  } else {
    dispatch_dims(d, dw, [&]<int D, int DW>() {
      const LoopP<D, DW> L = make_loop<D, DW>(HL);
      k_mctab_dense<D, DW><<<grid_for(n, kMcBlock), kMcBlock, 0, st>>>(L, r0, n, seed, t_from, T,
                                                                         tab.dy.as<double>(), tab.z.as<double>());
    });
  }
  kprof_work(F_MC_TABLE, n * static_cast<int64_t>(T + 1 - t_from));  // rollout-steps drawn
  // per-step max deviation of the new rows (the certification's skip test)
  const size_t md_bytes = static_cast<size_t>(T + 1) * dw * 8;
  if (md_bytes > tab.maxdev.cap) tab.maxdev.grow(md_bytes * 2, static_cast<size_t>(t_from) * dw * 8, st);
  PUMP_CUDA(cudaMemsetAsync(tab.maxdev.as<char>() + static_cast<size_t>(t_from) * dw * 8, 0,
                            static_cast<size_t>(T + 1 - t_from) * dw * 8, st));
  k_mctab_maxdev<<<dim3(static_cast<unsigned>(std::min<int64_t>((n * dw + 255) / 256, 16)), T + 1 - t_from), 256, 0,
                   st>>>(tab.dy.as<double>(), n, dw, t_from, tab.maxdev.as<unsigned long long>());
  *launches += 2;
  PUMP_CUDA(cudaGetLastError());
  tab.t_done = T;
  return true;
}

void mc_step_buffers(McTable& tab, int n_traj, int max_points) {
  const size_t rows_all = static_cast<size_t>(n_traj) * max_points;
  tab.step_list.ensure(rows_all * kStepCap * 2 + 256);
  tab.step_nl.ensure(rows_all * 4 + 256);
  tab.step_skip.ensure(rows_all + 256);
}

bool mc_table_covers(const McTable& tab, const HostLoop& HL, int64_t r0, int64_t r1, uint64_t seed, int T) {
  return tab.valid && tab.seed == seed && tab.r0 == r0 && tab.r1 == r1 && T <= tab.t_done && same_loop(tab.L, HL);
}

void mc_table_prepare(McTable& tab, const HostLoop& HL, int64_t r0, int64_t r1, uint64_t seed, int T,
                      cudaStream_t st, int64_t* launches) {
  if (r1 <= r0 || T < 0) return;
  static const bool direct = std::getenv("PUMP_MC_DIRECT") != nullptr;
  if (direct) return;
  ensure_table(tab, HL, r0, r1, seed, T, st, launches);
}

void launch_mc(const HostLoop& HL, const DevWorld& w, int n_traj, const int64_t* d_traj_off, const double* d_ynom,
               int max_points, int64_t r0, int64_t r1, uint64_t seed, double eps_cc, unsigned long long* d_hits,
               cudaStream_t st, int64_t* launches, unsigned long long* d_steps, McTable* table,
               const int32_t* d_live, bool lists_ready) {
  if (r1 <= r0 || n_traj <= 0) return;
  if (HL.dw != w.dw) throw std::invalid_argument("mc_certify: workspace / model dimension mismatch");
  static const bool direct = std::getenv("PUMP_MC_DIRECT") != nullptr;
  // Large certifications (SURVEY config 4: up to 1e7 rollouts) go through the
  // table in rollout chunks; each chunk's hits accumulate into d_hits.
  if (table && !direct && r1 - r0 > kTabRollouts) {
    for (int64_t c0 = r0; c0 < r1; c0 += kTabRollouts)
      launch_mc(HL, w, n_traj, d_traj_off, d_ynom, max_points, c0, std::min(r1, c0 + kTabRollouts), seed, eps_cc,
                d_hits, st, launches, d_steps, table, d_live);  // (lists per chunk: each chunk's table)
    return;
  }
  if (table && !direct && ensure_table(*table, HL, r0, r1, seed, max_points - 1, st, launches)) {
    WorldD wd;
    wd.n_obs = w.n_obs;
    wd.lo = w.d_lo;
    wd.hi = w.d_hi;
    for (int k = 0; k < 6; ++k) {
      wd.blo[k] = w.blo[k];
      wd.bhi[k] = w.bhi[k];
    }
    const int64_t n = r1 - r0;
    table->flags.ensure(static_cast<size_t>(n) * n_traj * 4 + 256);
    PUMP_CUDA(cudaMemsetAsync(table->flags.p, 0, static_cast<size_t>(n) * n_traj * 4, st));
    dispatch_dw(HL.dw, [&]<int DW>() {
      // per-(trajectory, step) candidate lists, once per certification
      mc_step_buffers(*table, n_traj, max_points);
      if (!lists_ready) {
        k_mc_steps<DW><<<dim3((max_points + 3) / 4, n_traj), 128, 0, st>>>(
            wd, d_traj_off, d_ynom, table->maxdev.as<unsigned long long>(), max_points,
            table->step_list.as<uint16_t>(), table->step_nl.as<int32_t>(), table->step_skip.as<uint8_t>(), d_live);
        ++*launches;
      }
      auto go = [&]<int SUB>() {
        constexpr int span = kMcChunk * SUB;
        const size_t smem = (static_cast<size_t>(span + 1) * DW + 4 * static_cast<size_t>(w.n_obs) * DW) * sizeof(double);
        if (smem > 48 * 1024)
          PUMP_CUDA(cudaFuncSetAttribute(k_mc_tab<DW, SUB>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(smem)));
        dim3 grid(grid_for(n, kMcTabBlock), n_traj, (max_points + span - 1) / span);
        k_mc_tab<DW, SUB><<<grid, kMcTabBlock, smem, st>>>(wd, d_traj_off, d_ynom, r0, r1, table->r0,
                                                        table->r1 - table->r0, table->dy.as<double>(),
                                                        table->maxdev.as<unsigned long long>(), eps_cc,
                                                        table->flags.as<uint32_t>(), d_live, max_points,
                                                        table->step_list.as<uint16_t>(), table->step_nl.as<int32_t>(),
                                                        table->step_skip.as<uint8_t>(), d_hits, d_steps);
      };
      KScope ks(st, F_MC);
      go.template operator()<2>();  // 2 x kMcChunk steps per thread (1 and 4 measured slower)
    });
    *launches += 1;
    PUMP_CUDA(cudaGetLastError());
    return;
  }
  if (HL.dw >= 2 && HL.dw <= 3 && separable(HL)) {
    const SepBlocks B = sep_blocks(HL);
    WorldD wd;
    wd.n_obs = w.n_obs;
    wd.lo = w.d_lo;
    wd.hi = w.d_hi;
    for (int k = 0; k < 6; ++k) {
      wd.blo[k] = w.blo[k];
      wd.bhi[k] = w.bhi[k];
    }
    dispatch_dw(HL.dw, [&]<int DW>() {
      const size_t smem = (static_cast<size_t>(max_points) * DW + 4 * static_cast<size_t>(w.n_obs) * DW) * sizeof(double);
      constexpr int per_block = (kMcBlock / 32) * groups_per_warp<DW>();
      dim3 grid(static_cast<unsigned>((r1 - r0 + per_block - 1) / per_block), n_traj);
      auto go = [&]<int MINB>() {
        if (smem > 48 * 1024)
          PUMP_CUDA(cudaFuncSetAttribute(k_mc_sep<DW, MINB>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(smem)));
        KScope ks(st, F_MC);
        k_mc_sep<DW, MINB><<<grid, kMcBlock, smem, st>>>(B, wd, d_traj_off, d_ynom, r0, r1, seed, eps_cc, d_hits,
                                                          d_steps);
      };
      go.template operator()<5>();  // 5 blocks per SM (4, 6, 8 measured slower)
      ++*launches;
      PUMP_CUDA(cudaGetLastError());
    });
    return;
  }
  dispatch_dims(HL.d, HL.dw, [&]<int D, int DW>() {
    const LoopP<D, DW> L = make_loop<D, DW>(HL);
    WorldD wd;
    wd.n_obs = w.n_obs;
    wd.lo = w.d_lo;
    wd.hi = w.d_hi;
    for (int k = 0; k < 6; ++k) {
      wd.blo[k] = w.blo[k];
      wd.bhi[k] = w.bhi[k];
    }
    const size_t smem = (static_cast<size_t>(max_points) * DW + 2 * static_cast<size_t>(w.n_obs) * DW) * sizeof(double);
    if (smem > 48 * 1024)
      PUMP_CUDA(cudaFuncSetAttribute(k_mc<D, DW>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
    dim3 grid(grid_for(r1 - r0, kMcBlock), n_traj);
    KScope ks(st, F_MC);
    k_mc<D, DW><<<grid, kMcBlock, smem, st>>>(L, wd, d_traj_off, d_ynom, r0, r1, seed, eps_cc, d_hits, d_steps);
    ++*launches;
    PUMP_CUDA(cudaGetLastError());
  });
}

}  // namespace pumpg
