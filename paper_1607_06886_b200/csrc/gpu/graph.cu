// K_graph: build_graph (graph.hpp:50-95) on sm_100a.
//
//  k_connect_rows   one CTA per source row v, one thread per target u:
//                   velocity prefilter, connect() (64-point geometric scan +
//                   golden section, steer.hpp:111-182), cost < r_n filter;
//                   survivors compacted in ascending-u order (warp ballots +
//                   CTA prefix) into a per-row candidate slab.
//  k_collide        one thread per candidate: motion_collides (adaptive
//                   bisection, geom.hpp:96-123, iterative DFS over (t0,t1)
//                   spans) + waypoint point_free checks (graph.hpp:80-84).
//  k_emit_edges     order-preserving compaction into the CSR edge arrays.
//  k_regions        one thread per edge waypoint: local_convex_region
//                   (geom.hpp:189-225); run twice (count, then write).
// Obstacles are staged in shared memory.  All floating point follows the
// reference's operation order (no FMA: --fmad=false).
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>

#include "dispatch.cuh"
#include "graph.h"
#include "scan.cuh"

namespace pumpg {

constexpr int kRowBlock = 256;
constexpr int kGridBlock = 128;  // k_pair_filter_grid: a block per row

struct GraphArgs {
  int n;
  const double* pos;  // n x dw
  const double* vel;
  double r_n, dt, eps_cc, tau_max, ratio;
};

// Exact-preserving pair filter (bound in dev.cuh, pair_lb / interval_clears).
// It is also bounded below by tau itself beyond thr.  If a cover of (0, thr]
// by intervals whose bounds exceed thr = r_n (1 + 1e-6) exists, the pair's
// true minimum cost exceeds r_n by a margin far above the rounding of the
// reference's cost evaluation (<= ~1e-13 relative), so connect() would return
// cost >= r_n (or ok = false) and the reference would reject the pair at
// graph.hpp:72: skipping it changes nothing.
constexpr int kLbK = 256;  // 4^4 leaves: a 4-ary interval tree, coarse to fine
struct LbGrid {
  double thr;
  double t[kLbK + 1];   // decreasing: t[0] = thr, t[K] = thr * 1e-4
  double c3[kLbK + 1];  // 12 / t^3 of each interval's upper end (c3[K]: head interval)
  double c1[kLbK];      // 1 / t of each interval's upper end
};

// The interval [t[i + SPAN], t[i]] clears if its own bound does or all four
// quarters clear (the tree only decides how much work the cover takes).
template <int SPAN>
__device__ __forceinline__ bool lb_tree(const PairLb& p, const LbGrid& L, int i) {
  if (interval_clears(p, L.t[i + SPAN], L.t[i], L.c3[i], L.c1[i], L.thr)) return true;
  if constexpr (SPAN == 1) {
    return false;
  } else {
#pragma unroll 1
    for (int q = 0; q < 4; ++q)
      if (!lb_tree<SPAN / 4>(p, L, i + q * (SPAN / 4))) return false;
    return true;
  }
}

__device__ __forceinline__ bool lb_head_clears(const PairLb& p, const LbGrid& L) {
  // head interval (0, t_K]: c >= 12 min q / t_K^3
  const double tk = L.t[kLbK];
  const double q0 = p.A, qk = p.A - 2.0 * p.B * tk + p.C * tk * tk;
  double qm = q0 < qk ? q0 : qk;
  if (p.ts > 0 && p.ts < tk) qm = p.A - p.B * p.ts;
  const double ab = p.B < 0 ? -p.B : p.B;
  qm -= 1e-12 * (p.A + 2.0 * ab * tk + p.C * tk * tk);
  if (qm < 0) qm = 0;
  return L.c3[kLbK] * qm * (1.0 - 1e-12) >= L.thr;
}

// Global bound, tried when the root interval does not clear.  On (0, thr]
// q(tau) >= q* = min over [0, thr] of the quadratic (less the rounding margin
// of interval_clears), so c(tau) >= g(tau) = tau + 12 q* / tau^3 + D / tau.
// g is convex on tau > 0 with its minimum at tau*^2 = (D + sqrt(D^2 + 144 q*)) / 2
// (g' = 1 - 36 q* / tau^4 - D / tau^2); g at the computed tau* exceeds min g by
// O(eps^2) and is evaluated to a few ulps, so g(tau*) (1 - 1e-12) is a lower
// bound of c on (0, thr]: at or above thr the pair is rejected (as by a cover).
__device__ __forceinline__ bool lb_global_clears(const PairLb& p, double thr) {
  const double q0 = p.A, q1 = p.A - 2.0 * p.B * thr + p.C * thr * thr;
  double qm = q0 < q1 ? q0 : q1;
  if (p.ts > 0 && p.ts < thr) qm = p.A - p.B * p.ts;
  const double ab = p.B < 0 ? -p.B : p.B;
  qm -= 1e-12 * (p.A + 2.0 * ab * thr + p.C * thr * thr);
  if (!(qm > 0)) return false;
  const double a = 12.0 * qm;
  const double t2 = 0.5 * (p.D + sqrt(p.D * p.D + 12.0 * a));
  const double t = sqrt(t2);
  const double g = t + a / (t2 * t) + p.D / t;
  return g * (1.0 - 1e-12) >= thr;
}

__device__ __forceinline__ bool lb_rejects(const PairLb& p, const LbGrid& L) {
  // head interval (0, t_K]: c >= 12 min q / t_K^3
  const double tk = L.t[kLbK];
  const double q0 = p.A, qk = p.A - 2.0 * p.B * tk + p.C * tk * tk;
  double qm = q0 < qk ? q0 : qk;
  if (p.ts > 0 && p.ts < tk) qm = p.A - p.B * p.ts;
  const double ab = p.B < 0 ? -p.B : p.B;
  qm -= 1e-12 * (p.A + 2.0 * ab * tk + p.C * tk * tk);
  if (qm < 0) qm = 0;
  if (!(L.c3[kLbK] * qm * (1.0 - 1e-12) >= L.thr)) return false;
  return lb_tree<kLbK>(p, L, 0);
}

LbGrid make_lb_grid(double r_n) {
  LbGrid L;
  L.thr = r_n * (1.0 + 1e-6);
  const double rho = std::pow(1e4, 1.0 / kLbK);
  for (int i = 0; i <= kLbK; ++i) {
    L.t[i] = L.thr / std::pow(rho, i);
    L.c3[i] = 12.0 / (L.t[i] * L.t[i] * L.t[i]);
    if (i < kLbK) L.c1[i] = 1.0 / L.t[i];
  }
  // round the multipliers down so the bound stays a lower bound after rounding
  for (int i = 0; i <= kLbK; ++i) L.c3[i] *= (1.0 - 1e-14);
  for (int i = 0; i < kLbK; ++i) L.c1[i] *= (1.0 - 1e-14);
  return L;
}


// Pass 1, lane-refill form.  The tree cover of lb_tree costs 1 interval test
// for most pairs and hundreds for near-threshold ones; one pair per lane left
// ~1/3 of the lanes active.  Here every lane runs the same loop body -- one
// interval test of an explicit depth-first walk over the 4-ary tree -- and a
// lane whose pair is decided takes the next u of the row (warp ballot + one
// shared atomic per warp).  Survivors land in a bitmask over a chunk of u and
// are compacted in ascending-u order after it, so the slab is identical to
// k_pair_filter's (the decision per pair is the same pure function).
constexpr int kPfChunk = 32 * kRowBlock;
template <int DW>
__global__ void __launch_bounds__(kRowBlock) k_pair_filter_q(GraphArgs g, const LbGrid lb, int cap, int row0, int refill,
                                                             int32_t* __restrict__ row_cnt,
                                                             int32_t* __restrict__ su) {
  __shared__ LbGrid sl;
  __shared__ uint32_t bits[kPfChunk / 32];
  __shared__ int wtot[kRowBlock / 32];
  __shared__ int s_next, base_s;
  {
    const double* src = reinterpret_cast<const double*>(&lb);
    double* dst = reinterpret_cast<double*>(&sl);
    for (int x = threadIdx.x; x < static_cast<int>(sizeof(LbGrid) / 8); x += blockDim.x) dst[x] = src[x];
  }
  const int v = row0 + blockIdx.x;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const unsigned lt = (1u << lane) - 1u;
  double ap[DW], av[DW];
#pragma unroll
  for (int k = 0; k < DW; ++k) {
    ap[k] = g.pos[v * DW + k];
    av[k] = g.vel[v * DW + k];
  }
  if (threadIdx.x == 0) base_s = 0;
  for (int c0 = 0; c0 < g.n; c0 += kPfChunk) {
    const int c1 = min(g.n, c0 + kPfChunk);
    bits[threadIdx.x] = 0u;  // kPfChunk / 32 == kRowBlock
    if (threadIdx.x == 0) s_next = c0;
    __syncthreads();
    bool active = false, exhausted = false;
    PairLb p{};
    int i = 0, s = 0, u = 0;
    for (;;) {
      while (!exhausted) {  // warp-uniform
        const unsigned need = __ballot_sync(0xffffffffu, !active);
        // refill in bulk: the refill body (loads, pair_lb, head test) is
        // several interval tests long, so it waits for half the warp
        if (need == 0 || (need != 0xffffffffu && __popc(need) < refill)) break;
        int base = 0;
        if (lane == 0) base = atomicAdd(&s_next, __popc(need));
        base = __shfl_sync(0xffffffffu, base, 0);
        if (base >= c1) {
          exhausted = true;
          break;
        }
        if (!active) {
          u = base + __popc(need & lt);
          if (u < c1 && u != v) {
            double bp[DW], bv[DW];
#pragma unroll
            for (int k = 0; k < DW; ++k) {
              bp[k] = g.pos[u * DW + k];
              bv[k] = g.vel[u * DW + k];
            }
            p = pair_lb<DW>(ap, av, bp, bv);
            if (!(2.0 * sqrt(p.D) >= g.r_n)) {
              if (!lb_head_clears(p, sl)) {
                atomicOr(&bits[(u - c0) >> 5], 1u << ((u - c0) & 31));
              } else {
                active = true;
                i = 0;
                s = 4;  // span 4^s: the root
              }
            }
          }
        }
      }
      if (!__any_sync(0xffffffffu, active)) break;
      if (active) {
        const int span = 1 << (2 * s);
        if (interval_clears(p, sl.t[i + span], sl.t[i], sl.c3[i], sl.c1[i], sl.thr)) {
          i += span;  // a multiple of 4^s: climb past every finished parent
          const int z = (__ffs(i) - 1) >> 1;
          s = z < 4 ? (z > s ? z : s) : 4;
          if (i == kLbK) active = false;  // covered: rejected
        } else if (s == 0) {
          atomicOr(&bits[(u - c0) >> 5], 1u << ((u - c0) & 31));  // a leaf fails: survivor
          active = false;
        } else {
          --s;
        }
      }
    }
    __syncthreads();
    // ascending-u compaction of the chunk's bitmask, one word per thread
    const uint32_t wb = bits[threadIdx.x];
    const int cnt = __popc(wb);
    int inc = cnt;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, inc, o);
      if (lane >= o) inc += y;
    }
    if (lane == 31) wtot[warp] = inc;
    __syncthreads();
    int off = base_s + inc - cnt;
    for (int w = 0; w < warp; ++w) off += wtot[w];
    uint32_t m = wb;
    while (m) {
      const int b = __ffs(m) - 1;
      m &= m - 1;
      if (off < cap) su[static_cast<int64_t>(v) * cap + off] = c0 + threadIdx.x * 32 + b;
      ++off;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      int t = 0;
      for (int w = 0; w < kRowBlock / 32; ++w) t += wtot[w];
      base_s += t;
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) row_cnt[v] = base_s;
}

// ---------------------------------------------------------------- cell grid
// Exact-preserving spatial cull in front of the pair filter.  For tau in
// (0, thr] and |vbar| <= V (V = the nodes' largest speed), the cost
// c(tau) >= 12 |dp0 - vbar tau|^2 / tau^3 >= 12 (d - V thr)^2 / thr^3 once the
// distance d = |dp0| exceeds V thr, and that exceeds thr once
// d > R = V thr + thr^2 / sqrt(12); beyond thr, c >= tau > thr.  So a node
// farther than R from v has true cost above thr = r_n (1 + 1e-6) for every
// tau (the host tightens R interval by interval, below) -- the premise the interval-tree filter itself rests on (connect would
// return cost >= r_n or ok = false; graph.hpp:72 drops the pair).  Nodes are
// bucketed into cells of edge >= R / 2 with exact per-cell bounding boxes; a
// row visits only the cells whose box lies within R (squared distance against
// R^2 (1 + 1e-9), far above the distance's rounding).  Survivors land in a
// bitmask over all n and are compacted in ascending u, so the per-row slab
// holds exactly the pairs k_pair_filter_q keeps among the cells visited.
constexpr int kCellMaxList = 2048;  // cells a row may examine (the host sizes the grid for it)
// Velocity-aware reach of a row (the cell cull of k_pair_filter_grid): a pair
// of cost <= thr has some tau <= thr with 12 |dp - vbar tau|^2 / tau^3 <=
// thr - tau, vbar = (av + bv) / 2, so for tau in an interval [tl, th]
//   |dp - av tau / 2| <= V th / 2 + sqrt((thr - tl) th^3 / 12) = rho
// (|bv| <= V): dp lies within rho of the box swept by av tau / 2.  A cell
// whose exact node box is farther than rho from every interval's swept box
// holds no pair of cost <= thr.  kSaus intervals: (0, thr/64], [thr/64,
// thr/32], then steps of thr/32 (the outer reach is set by the last ones).
constexpr int kSaus = 33;
constexpr int kSausGroups = 8;  // groups of 4 intervals (the first also holds the head)
__host__ __device__ constexpr int saus_g0(int q) { return q == 0 ? 0 : 1 + 4 * q; }
struct SausTab {
  double tl[kSaus], th[kSaus], rho2[kSaus];  // rho2 = (rho (1 + 1e-9) + 1e-12)^2
  double grho2[kSausGroups];                 // largest rho2 of a group's intervals
  double ext;                                // largest reach of any interval (rho + V th / 2)
};
struct CellGrid {
  double lo[3];
  double inv_h;
  int dims[3];
};

__device__ __forceinline__ unsigned long long ord_of(double x) {
  const unsigned long long b = static_cast<unsigned long long>(__double_as_longlong(x));
  return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}
__host__ __device__ __forceinline__ double dbl_of(unsigned long long o) {
  const unsigned long long b = (o >> 63) ? (o & 0x7fffffffffffffffull) : ~o;
  double x;
  memcpy(&x, &b, 8);
  return x;
}

// stats[0..DW) = ord(min pos), stats[3..3+DW) = ord(max pos), stats[6] = ord(max |v|^2)
template <int DW>
__global__ void k_node_stats(int n, const double* __restrict__ pos, const double* __restrict__ vel,
                             unsigned long long* __restrict__ stats) {
  double lo[DW], hi[DW], v2 = 0.0;
#pragma unroll
  for (int k = 0; k < DW; ++k) {
    lo[k] = INFINITY;
    hi[k] = -INFINITY;
  }
  for (int u = blockIdx.x * blockDim.x + threadIdx.x; u < n; u += gridDim.x * blockDim.x) {
    double s = 0.0;
#pragma unroll
    for (int k = 0; k < DW; ++k) {
      const double p = pos[u * DW + k], w = vel[u * DW + k];
      lo[k] = fmin(lo[k], p);
      hi[k] = fmax(hi[k], p);
      s += w * w;
    }
    v2 = fmax(v2, s);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
#pragma unroll
    for (int k = 0; k < DW; ++k) {
      lo[k] = fmin(lo[k], __shfl_xor_sync(0xffffffffu, lo[k], o));
      hi[k] = fmax(hi[k], __shfl_xor_sync(0xffffffffu, hi[k], o));
    }
    v2 = fmax(v2, __shfl_xor_sync(0xffffffffu, v2, o));
  }
  if ((threadIdx.x & 31) == 0) {
#pragma unroll
    for (int k = 0; k < DW; ++k) {
      atomicMin(&stats[k], ord_of(lo[k]));
      atomicMax(&stats[3 + k], ord_of(hi[k]));
    }
    atomicMax(&stats[6], ord_of(v2));
  }
}

__global__ void k_cell_box_init(int n_cells, unsigned long long* __restrict__ cbox) {
  const int x = blockIdx.x * blockDim.x + threadIdx.x;
  if (x >= n_cells * 6) return;
  cbox[x] = (x % 6) < 3 ? ~0ull : 0ull;  // min words start at the top of the order, max words at the bottom
}

template <int DW>
__device__ __forceinline__ int cell_coord(const CellGrid& G, const double* p, int k) {
  const double x = floor((p[k] - G.lo[k]) * G.inv_h);
  return x < 0 ? 0 : (x >= G.dims[k] ? G.dims[k] - 1 : static_cast<int>(x));
}

// per node: its cell, rank within the cell, and the cell's exact bounding box
template <int DW>
__global__ void k_cell_count(int n, const double* __restrict__ pos, const CellGrid G, int32_t* __restrict__ cnt,
                             unsigned long long* __restrict__ cbox, int32_t* __restrict__ ncell,
                             int32_t* __restrict__ nrank) {
  const int u = blockIdx.x * blockDim.x + threadIdx.x;
  if (u >= n) return;
  double p[DW];
#pragma unroll
  for (int k = 0; k < DW; ++k) p[k] = pos[u * DW + k];
  int id = 0;
#pragma unroll
  for (int k = DW - 1; k >= 0; --k) id = id * G.dims[k] + cell_coord<DW>(G, p, k);
  ncell[u] = id;
  nrank[u] = atomicAdd(&cnt[id], 1);
#pragma unroll
  for (int k = 0; k < DW; ++k) {
    atomicMin(&cbox[static_cast<int64_t>(id) * 6 + k], ord_of(p[k]));
    atomicMax(&cbox[static_cast<int64_t>(id) * 6 + 3 + k], ord_of(p[k]));
  }
}

template <int DW>
__global__ void k_cell_scatter(int n, const double* __restrict__ pos, const double* __restrict__ vel,
                               const int32_t* __restrict__ ncell, const int32_t* __restrict__ nrank,
                               const int64_t* __restrict__ cstart, int32_t* __restrict__ sidx,
                               double* __restrict__ spos, double* __restrict__ svel) {
  const int u = blockIdx.x * blockDim.x + threadIdx.x;
  if (u >= n) return;
  const int64_t j = cstart[ncell[u]] + nrank[u];
  sidx[j] = u;
#pragma unroll
  for (int k = 0; k < DW; ++k) {
    spos[j * DW + k] = pos[u * DW + k];
    svel[j * DW + k] = vel[u * DW + k];
  }
}

// Pass 1 over the cells within R of the row's node; the per-pair decision and
// the lane-refill walk are k_pair_filter_q's.
template <int DW>
__global__ void __launch_bounds__(kGridBlock) k_pair_filter_grid(
    GraphArgs g, const LbGrid* __restrict__ lbp, const CellGrid G, const SausTab SZ, int cap, int row0, int refill,
    const int32_t* __restrict__ ccnt, const int64_t* __restrict__ cstart,
    const unsigned long long* __restrict__ cbox, const int32_t* __restrict__ sidx, const double* __restrict__ spos,
    const double* __restrict__ svel, int32_t* __restrict__ row_cnt, int32_t* __restrict__ su, int use_global) {
  // the interval table from global memory (L1-resident; staging its 6 KB
  // into shared memory per row cost more than the walks' reads of it)
  const LbGrid& sl = *lbp;
  __shared__ int cl_start[kCellMaxList];
  __shared__ int cl_pref[kCellMaxList + 1];
  __shared__ int wtot[kGridBlock / 32];
  __shared__ int s_next, s_ncl, s_nsurv;
  __shared__ int s_surv[32];  // the first 32 survivors (a row has ~8): sorted by one warp
  extern __shared__ uint32_t bits[];  // ceil(n / 32) words
  const int v = row0 + blockIdx.x;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const unsigned lt = (1u << lane) - 1u;
  const int nw = (g.n + 31) >> 5;
  double ap[DW], av[DW];
#pragma unroll
  for (int k = 0; k < DW; ++k) {
    ap[k] = g.pos[v * DW + k];
    av[k] = g.vel[v * DW + k];
  }
  for (int x = threadIdx.x; x < nw; x += blockDim.x) bits[x] = 0u;
  if (threadIdx.x == 0) {
    s_ncl = 0;
    s_next = 0;
    s_nsurv = 0;
  }
  __syncthreads();
  // candidate cells: the boxes swept by av tau / 2 over the reach intervals
  // (SausTab), their union's extent bounding the cell range; a non-empty cell
  // is kept when its exact node box is within rho of some interval's box
  __shared__ double s_sw[kSaus][2 * DW];
  __shared__ double s_gw[kSausGroups][2 * DW];  // per group of intervals: the union of their boxes
  __shared__ int s_c0[DW], s_c1[DW];
  for (int i = threadIdx.x; i < kSaus; i += blockDim.x) {
#pragma unroll
    for (int k = 0; k < DW; ++k) {
      const double a0 = av[k] * SZ.tl[i] * 0.5, a1 = av[k] * SZ.th[i] * 0.5;
      s_sw[i][k] = a0 < a1 ? a0 : a1;
      s_sw[i][DW + k] = a0 < a1 ? a1 : a0;
    }
  }
  if (threadIdx.x < kSausGroups) {  // group q: intervals [saus_g0(q), saus_g0(q + 1)) (av tau / 2 is monotone in tau)
    const int q = threadIdx.x;
#pragma unroll
    for (int k = 0; k < DW; ++k) {
      const double a0 = av[k] * SZ.tl[saus_g0(q)] * 0.5, a1 = av[k] * SZ.th[saus_g0(q + 1) - 1] * 0.5;
      s_gw[q][k] = a0 < a1 ? a0 : a1;
      s_gw[q][DW + k] = a0 < a1 ? a1 : a0;
    }
  }
  if (threadIdx.x < DW) {  // the cell range: every interval's box widened by its rho (ext bounds both)
    const int k = threadIdx.x;
    const double c = av[k] * SZ.th[kSaus - 1] * 0.5;
    double e0 = ap[k] + (c < 0 ? c : 0.0) - SZ.ext, e1 = ap[k] + (c > 0 ? c : 0.0) + SZ.ext;
    const double x0 = floor((e0 - G.lo[k]) * G.inv_h), x1 = floor((e1 - G.lo[k]) * G.inv_h);
    s_c0[k] = x0 < 0 ? 0 : (x0 >= G.dims[k] ? G.dims[k] - 1 : static_cast<int>(x0));
    s_c1[k] = x1 < 0 ? 0 : (x1 >= G.dims[k] ? G.dims[k] - 1 : static_cast<int>(x1));
  }
  __syncthreads();
  {
    int ext[DW], tot = 1;
#pragma unroll
    for (int k = 0; k < DW; ++k) {
      ext[k] = s_c1[k] - s_c0[k] + 1;
      tot *= ext[k];
    }
    for (int o = threadIdx.x; o < tot; o += blockDim.x) {
      int r = o, id = 0, mul = 1;
#pragma unroll
      for (int k = 0; k < DW; ++k) {
        const int cxy = s_c0[k] + r % ext[k];
        r /= ext[k];
        id += cxy * mul;
        mul *= G.dims[k];
      }
      const int cnt = ccnt[id];
      if (cnt == 0) continue;
      double bl[DW], bh[DW];
#pragma unroll
      for (int k = 0; k < DW; ++k) {
        bl[k] = dbl_of(cbox[static_cast<int64_t>(id) * 6 + k]) - ap[k];
        bh[k] = dbl_of(cbox[static_cast<int64_t>(id) * 6 + 3 + k]) - ap[k];
      }
      auto near = [&](const double* sw, double rho2) {
        double d2 = 0.0;
#pragma unroll
        for (int k = 0; k < DW; ++k) {
          const double g1 = bl[k] - sw[DW + k], g2 = sw[k] - bh[k];
          const double gap = g1 > 0 ? g1 : (g2 > 0 ? g2 : 0.0);
          d2 += gap * gap;
        }
        return d2 <= rho2;
      };
      // the groups with the widest reach first; a group's intervals only when
      // the cell is within the group's largest rho of the union of their boxes
      bool keep = false;
      for (int q = kSausGroups - 1; q >= 0 && !keep; --q) {
        if (!near(s_gw[q], SZ.grho2[q])) continue;
        for (int i = saus_g0(q + 1) - 1; i >= saus_g0(q) && !keep; --i) keep = near(s_sw[i], SZ.rho2[i]);
      }
      if (!keep) continue;
      const int slot = atomicAdd(&s_ncl, 1);
      cl_start[slot] = static_cast<int>(cstart[id]);
      cl_pref[slot + 1] = cnt;
    }
  }
  __syncthreads();
  const int ncl = s_ncl;
  if (warp == 0) {  // inclusive prefix of the list's counts: 16 entries per lane + a warp scan
    constexpr int kPer = kCellMaxList / 32;
    int run = 0;
    for (int q = 0; q < kPer; ++q) {
      const int e = lane * kPer + q;
      if (e < ncl) run += cl_pref[e + 1];
    }
    int inc = run;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, inc, o);
      if (lane >= o) inc += y;
    }
    int acc = inc - run;
    for (int q = 0; q < kPer; ++q) {
      const int e = lane * kPer + q;
      if (e < ncl) {
        acc += cl_pref[e + 1];
        cl_pref[e + 1] = acc;
      }
    }
    if (lane == 0) cl_pref[0] = 0;
  }
  __syncthreads();
  const int total = cl_pref[ncl];
  auto keep_surv = [&](int uu) {
    atomicOr(&bits[uu >> 5], 1u << (uu & 31));
    const int k = atomicAdd(&s_nsurv, 1);
    if (k < 32) s_surv[k] = uu;
  };
  bool active = false, exhausted = false;
  PairLb p{};
  int i = 0, s = 0, u = 0;
  for (;;) {
    while (!exhausted) {  // warp-uniform
      const unsigned need = __ballot_sync(0xffffffffu, !active);
      if (need == 0 || (need != 0xffffffffu && __popc(need) < refill)) break;
      int base = 0;
      if (lane == 0) base = atomicAdd(&s_next, __popc(need));
      base = __shfl_sync(0xffffffffu, base, 0);
      if (base >= total) {
        exhausted = true;
        break;
      }
      if (!active) {
        const int j = base + __popc(need & lt);
        if (j < total) {
          int lo = 0, hi = ncl;  // largest c with cl_pref[c] <= j
          while (hi - lo > 1) {
            const int mid = (lo + hi) >> 1;
            if (cl_pref[mid] <= j)
              lo = mid;
            else
              hi = mid;
          }
          const int js = cl_start[lo] + (j - cl_pref[lo]);
          u = sidx[js];
          if (u != v) {
            double bp[DW], bv[DW];
#pragma unroll
            for (int k = 0; k < DW; ++k) {
              bp[k] = spos[static_cast<int64_t>(js) * DW + k];
              bv[k] = svel[static_cast<int64_t>(js) * DW + k];
            }
            p = pair_lb<DW>(ap, av, bp, bv);
            if (!(2.0 * sqrt(p.D) >= g.r_n)) {
              if (!lb_head_clears(p, sl)) {
                keep_surv(u);
              } else {
                active = true;
                i = 0;
                s = 4;
              }
            }
          }
        }
      }
    }
    if (!__any_sync(0xffffffffu, active)) break;
    if (active) {
      const int span = 1 << (2 * s);
      if (interval_clears(p, sl.t[i + span], sl.t[i], sl.c3[i], sl.c1[i], sl.thr)) {
        i += span;
        const int z = (__ffs(i) - 1) >> 1;
        s = z < 4 ? (z > s ? z : s) : 4;
        if (i == kLbK) active = false;
      } else if (s == 0) {
        keep_surv(u);
        active = false;
      } else if (s == 4 && use_global && lb_global_clears(p, sl.thr)) {
        active = false;  // the root did not clear, the global bound does: rejected
      } else {
        --s;
      }
    }
  }
  __syncthreads();
  const int nsurv = s_nsurv;
  if (nsurv <= 32) {  // the short list in ascending order: a lane's rank among the listed nodes
    if (warp == 0) {
      const int x = lane < nsurv ? s_surv[lane] : 0x7fffffff;
      int rank = 0;
      for (int q = 0; q < nsurv; ++q) rank += __shfl_sync(0xffffffffu, x, q) < x ? 1 : 0;
      if (lane < nsurv && rank < cap) su[static_cast<int64_t>(v) * cap + rank] = x;
      if (lane == 0) row_cnt[v] = nsurv;
    }
    return;
  }
  // ascending-u compaction of the bitmask, kGridBlock words per pass
  int base_run = 0;
  for (int w0 = 0; w0 < nw; w0 += kGridBlock) {
    const int x = w0 + threadIdx.x;
    const uint32_t wb = x < nw ? bits[x] : 0u;
    const int cnt = __popc(wb);
    int inc = cnt;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, inc, o);
      if (lane >= o) inc += y;
    }
    if (lane == 31) wtot[warp] = inc;
    __syncthreads();
    int off = base_run + inc - cnt, blk = 0;
    for (int w = 0; w < kGridBlock / 32; ++w) {
      if (w < warp) off += wtot[w];
      blk += wtot[w];
    }
    uint32_t m = wb;
    while (m) {
      const int b = __ffs(m) - 1;
      m &= m - 1;
      if (off < cap) su[static_cast<int64_t>(v) * cap + off] = x * 32 + b;
      ++off;
    }
    base_run += blk;
    __syncthreads();
  }
  if (threadIdx.x == 0) row_cnt[v] = base_run;
}

// largest per-row survivor count (the slab refit check) without a host copy of the counts
__global__ void k_max_count(int n, const int32_t* __restrict__ cnt, int* __restrict__ out) {
  int m = 0;
  for (int v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gridDim.x * blockDim.x) m = max(m, cnt[v]);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) m = max(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0) atomicMax(out, m);
}

// candidate count, edge count and waypoint count into one fixed place (one copy back)
__global__ void k_graph_totals(const int64_t* __restrict__ d_ncand, const int64_t* __restrict__ d_E,
                               const int64_t* __restrict__ wp_off, int64_t* __restrict__ out) {
  out[0] = *d_ncand;
  out[1] = *d_E;
  out[2] = wp_off[*d_E];
}

__device__ __forceinline__ int find_row(const int64_t* __restrict__ off, int n, int64_t c) {
  int lo = 0, hi = n;  // largest r with off[r] <= c
  while (hi - lo > 1) {
    const int mid = (lo + hi) >> 1;
    if (off[mid] <= c)
      lo = mid;
    else
      hi = mid;
  }
  return lo;
}

// Pass 2: connect() (steer.hpp:111-182) on the compacted survivors, one
// thread each: every lane of every warp does useful DDIV-heavy work.
template <int DW>
__global__ void __launch_bounds__(128) k_connect(GraphArgs g, int cap, int64_t n_surv,
                                                 const int64_t* __restrict__ soff, const int32_t* __restrict__ su,
                                                 uint8_t* __restrict__ keep, int32_t* __restrict__ s_v,
                                                 int32_t* __restrict__ s_u, double* __restrict__ s_tau,
                                                 double* __restrict__ s_cost) {
  const int64_t s = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (s >= n_surv) return;
  const int v = find_row(soff, g.n, s);
  const int u = su[static_cast<int64_t>(v) * cap + (s - soff[v])];
  double ap[DW], av[DW], bp[DW], bv[DW];
#pragma unroll
  for (int k = 0; k < DW; ++k) {
    ap[k] = g.pos[v * DW + k];
    av[k] = g.vel[v * DW + k];
    bp[k] = g.pos[u * DW + k];
    bv[k] = g.vel[u * DW + k];
  }
  double tau = 0, cost = 0;
  const bool ok = connect_dev<DW, true>(ap, av, bp, bv, g.tau_max, g.ratio, tau, cost, g.r_n * (1.0 + 1e-6));
  keep[s] = (ok && !(cost >= g.r_n) && !(tau <= 0)) ? 1 : 0;  // graph.hpp:72
  s_v[s] = v;
  s_u[s] = u;
  s_tau[s] = tau;
  s_cost[s] = cost;
}

// order-preserving compaction of kept survivors into the candidate arrays
__global__ void k_cand_compact(int n, int64_t n_surv, const uint8_t* __restrict__ keep,
                               const int64_t* __restrict__ cpos, const int64_t* __restrict__ soff,
                               const int32_t* __restrict__ s_v, const int32_t* __restrict__ s_u,
                               const double* __restrict__ s_tau, const double* __restrict__ s_cost,
                               int32_t* __restrict__ c_v, int32_t* __restrict__ c_u, double* __restrict__ c_tau,
                               double* __restrict__ c_cost, int64_t* __restrict__ cand_off) {
  const int64_t s = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (s <= n) cand_off[s] = cpos[soff[s]];
  if (s >= n_surv || !keep[s]) return;
  const int64_t c = cpos[s];
  c_v[c] = s_v[s];
  c_u[c] = s_u[s];
  c_tau[c] = s_tau[s];
  c_cost[c] = s_cost[s];
}


template <int DW, int LIST>
__global__ void __launch_bounds__(128, 6) k_collide(GraphArgs g, WorldD w, const int64_t* __restrict__ d_ncand,
                                                 const int32_t* __restrict__ c_v, const int32_t* __restrict__ c_u,
                                                 const double* __restrict__ c_tau, uint8_t* __restrict__ valid,
                                                 int32_t* __restrict__ nsteps) {
  extern __shared__ double smem[];
  const WorldD ws = stage_world<DW>(w, smem);
  const int64_t c = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (c >= *d_ncand) return;
  const int v = c_v[c], u = c_u[c];
  MotionD<DW> m;
  m.tau = c_tau[c];
#pragma unroll
  for (int k = 0; k < DW; ++k) {
    m.p0[k] = g.pos[v * DW + k];
    m.v0[k] = g.vel[v * DW + k];
    m.p1[k] = g.pos[u * DW + k];
    m.v1[k] = g.vel[u * DW + k];
  }
  coeffs_dev<DW>(m.p0, m.v0, m.p1, m.v1, m.tau, m.a, m.j);
  const MotionCullT<LIST> cull = motion_cull<DW, LIST>(m, ws);
  bool ok = !motion_collides<DW, LIST>(m, ws, g.eps_cc, &cull);
  int L = 0;
  if (ok) {
    // motion_waypoints (steer.hpp:192-212): k = floor(tau/dt + 1e-9)
    const int k = static_cast<int>(floor(m.tau / g.dt + 1e-9));
    const double rem = m.tau - k * g.dt;
    L = rem > 1e-9 ? k + 1 : k;
    // the waypoints lie on the motion, inside the box the cull was made for:
    // with the box inside the bounds and clear of every obstacle all are free
    const bool all_free = cull.inside && !cull.any;
    for (int j = 1; j <= L && ok && !all_free; ++j) {
      double p[DW], vv[DW];
      if (j == L) {
#pragma unroll
        for (int q = 0; q < DW; ++q) p[q] = m.p1[q];
      } else {
        motion_state<DW>(m, j * g.dt, p, vv);
      }
      ok = point_free_culled<DW>(ws, cull, p);
    }
  }
  valid[c] = ok ? 1 : 0;
  nsteps[c] = ok ? L : 0;
}

template <int DW>
__global__ void k_emit_edges(GraphArgs g, const int64_t* __restrict__ d_ncand, int64_t* __restrict__ d_E,
                             const int64_t* __restrict__ cand_off,
                             const int32_t* __restrict__ c_v, const int32_t* __restrict__ c_u,
                             const double* __restrict__ c_tau, const double* __restrict__ c_cost,
                             const uint8_t* __restrict__ valid, const int32_t* __restrict__ nsteps,
                             const int64_t* __restrict__ eoff, int32_t* __restrict__ e_from, int32_t* __restrict__ e_to,
                             double* __restrict__ e_cost, double* __restrict__ e_tau, double* __restrict__ e_acc0,
                             double* __restrict__ e_jerk, int32_t* __restrict__ e_nsteps,
                             int64_t* __restrict__ row_ptr) {
  const int64_t c = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const int64_t n_cand = *d_ncand;
  if (c < g.n + 1) row_ptr[c] = eoff[cand_off[c]];  // valid candidates before row c
  if (c == n_cand) *d_E = eoff[c];                  // the edge count
  if (c >= n_cand || !valid[c]) return;
  const int64_t e = eoff[c];
  const int v = c_v[c], u = c_u[c];
  const double tau = c_tau[c];
  e_from[e] = v;
  e_to[e] = u;
  e_cost[e] = c_cost[c];
  e_tau[e] = tau;
  e_nsteps[e] = nsteps[c];
  double a0[DW], j0[DW];
  coeffs_dev<DW>(g.pos + v * DW, g.vel + v * DW, g.pos + u * DW, g.vel + u * DW, tau, a0, j0);
#pragma unroll
  for (int k = 0; k < DW; ++k) {
    e_acc0[e * DW + k] = a0[k];
    e_jerk[e * DW + k] = j0[k];
  }
}

// Single pass: each waypoint computes its half-spaces once and reserves
// output space with one warp-aggregated atomicAdd.  Waypoint w owns
// [hs_off[w], hs_off[w] + hs_cnt[w]) (not in waypoint order; export rebuilds
// the CSR).  If the reserved total exceeds cap nothing past cap is written and
// the host reruns with the exact size (the counter returns it).  KW = 0 (at
// most 16 boxes): convex_region_fused, per-box squared distances computed
// once into shared memory, the half-spaces kept in registers.  KW > 0 (up to
// 32 KW boxes): convex_region_scan, the first kRegLocal half-spaces kept per
// thread; a waypoint with more recomputes its region straight into its
// reserved range.  Each waypoint finds its edge in the k_wp_edge map.
constexpr int kOnceMaxObs = 16;
constexpr int kRegLocal = 8;
constexpr int kLbsMaxObs = 1024;  // per-warp distance bounds in shared memory up to this many boxes
constexpr int kOrdMeta = (33 + 32 + 32) * 4 + 12;  // per-warp bucket offsets, cursors, minima (+ pad to 16 B)
constexpr int kBucketMaxObs = 512;  // bucket order for the first search up to this many boxes (1000: measured slower)

// waypoint -> owning edge (one thread per edge fills its waypoint range)
__global__ void k_wp_edge(int64_t n_edges, const int64_t* __restrict__ wp_off, int32_t* __restrict__ wp_edge) {
  const int64_t e = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (e >= n_edges) return;
  for (int64_t x = wp_off[e]; x < wp_off[e + 1]; ++x) wp_edge[x] = static_cast<int32_t>(e);
}
// waypoint x of the edge CSR: (y, yd) at its time j dt (motion_waypoints,
// steer.hpp:185-212; the last waypoint is the edge's end state)
template <int DW>
__device__ __forceinline__ void wp_state(const GraphArgs& g, int64_t x, const int64_t* __restrict__ wp_off,
                                         const int32_t* __restrict__ e_from, const int32_t* __restrict__ e_to,
                                         const double* __restrict__ e_tau, const double* __restrict__ e_acc0,
                                         const double* __restrict__ e_jerk, const int32_t* __restrict__ e_nsteps,
                                         const int32_t* __restrict__ wp_edge, double* y, double* yd) {
  const int64_t e = wp_edge[x];
  const int j = static_cast<int>(x - wp_off[e]) + 1;
  const int L = e_nsteps[e];
  const int v = e_from[e], u = e_to[e];
  MotionD<DW> m;
  m.tau = e_tau[e];
#pragma unroll
  for (int k = 0; k < DW; ++k) {
    m.p0[k] = g.pos[v * DW + k];
    m.v0[k] = g.vel[v * DW + k];
    m.p1[k] = g.pos[u * DW + k];
    m.v1[k] = g.vel[u * DW + k];
    m.a[k] = e_acc0[e * DW + k];
    m.j[k] = e_jerk[e * DW + k];
  }
  if (j == L) {
#pragma unroll
    for (int k = 0; k < DW; ++k) {
      y[k] = m.p1[k];
      yd[k] = m.v1[k];
    }
  } else {
    motion_state<DW>(m, j * g.dt, y, yd);
  }
}

// Spatial order of the waypoints for the region pass: state into ys
// ([x][y, yd]), a row-major cell id of a grid over the workspace bounds, and
// the cell histogram.  k_wp_scatter then lists the waypoints cell by cell.
// An edge's end waypoint is its end node's state (wp_state), so its region is
// the node's: the pass takes the n nodes as items n_wp + u instead of the E end
// waypoints (key -1: not listed), and k_wp_end_link points each end waypoint at
// its node's records.
struct WpCells {
  double lo[3], inv[3];
  int dim[3];
};
template <int DW>
__global__ void k_wp_prep(GraphArgs g, int64_t n_wp, const int64_t* __restrict__ wp_off,
                          const int32_t* __restrict__ e_from, const int32_t* __restrict__ e_to,
                          const double* __restrict__ e_tau, const double* __restrict__ e_acc0,
                          const double* __restrict__ e_jerk, const int32_t* __restrict__ e_nsteps,
                          const int32_t* __restrict__ wp_edge, WpCells cg, double* __restrict__ ys,
                          int32_t* __restrict__ key, int32_t* __restrict__ hist) {
  const int64_t x = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (x >= n_wp + g.n) return;
  double y[DW], yd[DW];
  if (x >= n_wp) {  // node u = x - n_wp
#pragma unroll
    for (int k = 0; k < DW; ++k) {
      y[k] = g.pos[(x - n_wp) * DW + k];
      yd[k] = g.vel[(x - n_wp) * DW + k];
    }
  } else {
    const int e = wp_edge[x];
    if (x == wp_off[e + 1] - 1) {  // the end waypoint: its node's region
      key[x] = -1;
      return;
    }
    wp_state<DW>(g, x, wp_off, e_from, e_to, e_tau, e_acc0, e_jerk, e_nsteps, wp_edge, y, yd);
  }
  int id = 0;
#pragma unroll
  for (int k = DW - 1; k >= 0; --k) {
    ys[x * 2 * DW + k] = y[k];
    ys[x * 2 * DW + DW + k] = yd[k];
    double c = (y[k] - cg.lo[k]) * cg.inv[k];
    int ci = c > 0 ? static_cast<int>(c) : 0;  // (NaN-safe: > 0 fails)
    ci = ci < cg.dim[k] ? ci : cg.dim[k] - 1;
    id = id * cg.dim[k] + ci;
  }
  key[x] = id;
  atomicAdd(hist + id, 1);
}
__global__ void k_wp_scatter(int64_t n_wp, const int32_t* __restrict__ key, const int64_t* __restrict__ cell_off,
                             int32_t* __restrict__ cursor, int32_t* __restrict__ perm) {
  const int64_t x = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (x >= n_wp) return;
  const int c = key[x];
  if (c < 0) return;
  perm[cell_off[c] + atomicAdd(cursor + c, 1)] = static_cast<int32_t>(x);
}
// an edge's end waypoint -> its end node's records (items n_wp + u of the
// region pass); *delta += (shared records - the nodes' own records), so the
// waypoint total H = stored + delta
__global__ void k_wp_end_link(int64_t n_edges, int n_nodes, int64_t n_wp, const int64_t* __restrict__ wp_off,
                              const int32_t* __restrict__ e_to, int64_t* __restrict__ hs_off,
                              int32_t* __restrict__ hs_cnt, unsigned long long* __restrict__ delta) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  long long d = 0;
  if (i < n_edges && wp_off[i + 1] > wp_off[i]) {
    const int64_t x = wp_off[i + 1] - 1, src = n_wp + e_to[i];
    hs_off[x] = hs_off[src];
    hs_cnt[x] = hs_cnt[src];
    d += hs_cnt[src];
  }
  if (i < n_nodes) d -= hs_cnt[n_wp + i];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) d += __shfl_xor_sync(0xffffffffu, d, o);
  if ((threadIdx.x & 31) == 0 && d != 0) atomicAdd(delta, static_cast<unsigned long long>(d));
}

// blocks of 128 threads, 512 above 256 boxes (the staged boxes are shared by
// more warps: forest1000 regions at 12 -> 32 resident warps per SM)
__host__ __device__ constexpr int regions_block(int kw) { return kw >= 32 ? 512 : 128; }
template <int DW, int KW>
__global__ void __launch_bounds__(regions_block(KW)) k_regions_once(GraphArgs g, WorldD w, int64_t n_wp, int64_t n_edges,
                                                      const int64_t* __restrict__ wp_off,
                                                      const int32_t* __restrict__ e_from,
                                                      const int32_t* __restrict__ e_to, const double* __restrict__ e_tau,
                                                      const double* __restrict__ e_acc0,
                                                      const double* __restrict__ e_jerk,
                                                      const int32_t* __restrict__ e_nsteps,
                                                      const int32_t* __restrict__ wp_edge, int64_t cap,
                                                      unsigned long long* __restrict__ counter,
                                                      int64_t* __restrict__ hs_off, int32_t* __restrict__ hs_cnt,
                                                      double* __restrict__ hs_pk, uint8_t* __restrict__ hs_fb,
                                                      int* __restrict__ err, unsigned long long* __restrict__ work,
                                                      const int32_t* __restrict__ perm, const double* __restrict__ ys,
                                                      const int64_t* __restrict__ n_list) {
  extern __shared__ double smem[];
  // sorted pass: n_list = the listed items (perm entries), on the device
  const int64_t n_act = n_list ? *n_list : n_wp;
  if (static_cast<int64_t>(blockIdx.x) * blockDim.x >= n_act) return;  // (block-uniform)
  const WorldD ws = stage_world<DW>(w, smem);
  const int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const int lane = threadIdx.x & 31;
  const bool active = t < n_act;
  // spatially ordered pass (perm given): thread t takes waypoint perm[t] with
  // its state precomputed by k_wp_prep, so a warp holds nearby waypoints
  const int64_t x = !active ? t : perm ? perm[t] : t;
  constexpr int kLoc = KW == 0 ? kOnceMaxObs : kRegLocal;
  double la[kLoc * DW], lb[kLoc];
  uint8_t lf[kLoc];
  int n = 0;
  double y[DW], yd[DW];
  if (active) {
    if (perm) {
#pragma unroll
      for (int k = 0; k < DW; ++k) {
        y[k] = ys[x * 2 * DW + k];
        yd[k] = ys[x * 2 * DW + DW + k];
      }
    } else {
      wp_state<DW>(g, x, wp_off, e_from, e_to, e_tau, e_acc0, e_jerk, e_nsteps, wp_edge, y, yd);
    }
  }
  // KW > 0: the warp's waypoint bounding box W; per box a lower bound of its
  // squared distance to W (lbs, shrunk by 2e-9) and the warp minimum over the
  // boxes of the largest squared distance from W (ub): convex_region_scan
  // skips the distances these bounds prove cannot be the nearest
  float* lbs = nullptr;
  double ub = __builtin_inf();
  BoxOrder box_order{};
  const BoxOrder* bord = nullptr;
  if (KW > 0 && w.n_obs <= kLbsMaxObs) {
    lbs = reinterpret_cast<float*>(smem + 2 * w.n_obs * DW) + (threadIdx.x >> 5) * w.n_obs;
    double wlo[DW], whi[DW];
#pragma unroll
    for (int k = 0; k < DW; ++k) {
      wlo[k] = active ? y[k] : __builtin_inf();
      whi[k] = active ? y[k] : -__builtin_inf();
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const double a = __shfl_xor_sync(0xffffffffu, wlo[k], o), b = __shfl_xor_sync(0xffffffffu, whi[k], o);
        wlo[k] = a < wlo[k] ? a : wlo[k];
        whi[k] = b > whi[k] ? b : whi[k];
      }
    }
    if (wlo[0] <= whi[0]) {  // any waypoint in this warp
      for (int o = lane; o < w.n_obs; o += 32) {
        double lb = 0.0, far = 0.0;
#pragma unroll
        for (int k = 0; k < DW; ++k) {
          const double lo = ws.lo[o * DW + k], hi = ws.hi[o * DW + k];
          const double g1 = lo - whi[k], g2 = wlo[k] - hi;  // gap between W and the box on axis k
          const double gap = g1 > 0 ? g1 : (g2 > 0 ? g2 : 0.0);
          lb = lb + gap * gap;
          // farthest 1-D distance to [lo, hi] over W's extent: at an end of W
          const double e1 = wlo[k] < lo ? lo - wlo[k] : (wlo[k] > hi ? wlo[k] - hi : 0.0);
          const double e2 = whi[k] < lo ? lo - whi[k] : (whi[k] > hi ? whi[k] - hi : 0.0);
          const double e = e1 > e2 ? e1 : e2;
          far = far + e * e;
        }
        lbs[o] = __double2float_rd(lb * (1.0 - 2e-9));  // rounded down: still a lower bound
        ub = far < ub ? far : ub;
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const double t = __shfl_xor_sync(0xffffffffu, ub, o);
        ub = t < ub ? t : ub;
      }
      __syncwarp();
    }
    if (wlo[0] <= whi[0] && w.n_obs <= kBucketMaxObs) {
      // the boxes in 32 buckets of ascending bound (counting sort by the
      // monotone map lbs -> floor(lbs * 31 / ub), bounds above ub last)
      char* wbase = reinterpret_cast<char*>(smem + 2 * w.n_obs * DW) +
                    static_cast<size_t>(blockDim.x / 32) * w.n_obs * 4 +
                    static_cast<size_t>(threadIdx.x >> 5) * (kOrdMeta + ((2 * w.n_obs + 15) & ~15));
      int* bstart = reinterpret_cast<int*>(wbase);               // 33 counts -> offsets
      int* bcur = bstart + 33;                                    // 32 cursors
      unsigned* bminu = reinterpret_cast<unsigned*>(bcur + 32);  // 32 smallest bounds (float bits)
      uint16_t* order = reinterpret_cast<uint16_t*>(wbase + kOrdMeta);
      const float scale = ub > 0.0 ? static_cast<float>(31.0 / ub) : 0.0f;
      auto bucket_of = [&](float l) -> int {
        if (static_cast<double>(l) > ub) return 31;
        const int b = static_cast<int>(l * scale);
        return b < 30 ? b : 30;
      };
      bstart[lane] = 0;
      if (lane == 0) bstart[32] = 0;
      bminu[lane] = 0x7f800000u;
      __syncwarp();
      for (int o = lane; o < w.n_obs; o += 32) {
        const int b = bucket_of(lbs[o]);
        atomicAdd(&bstart[b], 1);
        atomicMin(&bminu[b], __float_as_uint(lbs[o]));
      }
      __syncwarp();
      const int cnt = bstart[lane];
      int inc = cnt;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int t = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc += t;
      }
      __syncwarp();
      bstart[lane] = inc - cnt;
      bcur[lane] = inc - cnt;
      if (lane == 31) bstart[32] = inc;
      __syncwarp();
      for (int o = lane; o < w.n_obs; o += 32) order[atomicAdd(&bcur[bucket_of(lbs[o])], 1)] = static_cast<uint16_t>(o);
      __syncwarp();
      box_order = BoxOrder{order, bstart, reinterpret_cast<const float*>(bminu)};
      bord = &box_order;
    }
    __syncwarp();
  }
  unsigned n_clamp = 0, n_prune = 0;
  auto region = [&](double* ao, double* bo, uint8_t* fo, int as, int bst, int ocap) {
    if constexpr (KW == 0) {
      return convex_region_fused<DW>(ws, y, yd, smem + 2 * w.n_obs * DW + threadIdx.x, blockDim.x, ao, bo, fo,
                                     n_clamp, n_prune);
    } else {
      return convex_region_scan<DW, KW>(ws, y, yd, ao, bo, fo, as, bst, ocap, n_clamp, n_prune, lbs, ub, bord);
    }
  };
  if (active) {
    n = region(la, lb, lf, DW, 1, kLoc);
    if (n < 0) {
      atomicExch(err, 1);
      n = 0;
    }
  }
  // algorithmic work of the region loop (distance evaluations, prune tests)
  unsigned long long wc = n_clamp, wp = n_prune;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    wc += __shfl_xor_sync(0xffffffffu, wc, o);
    wp += __shfl_xor_sync(0xffffffffu, wp, o);
  }
  if (lane == 0 && work) {  // spread over 128 slot pairs: one address per warp would serialize at L2
    const unsigned slot = static_cast<unsigned>((x >> 5) & 127);
    atomicAdd(work + 2 * slot, wc);
    atomicAdd(work + 2 * slot + 1, wp);
  }
  // warp-aggregated reservation
  int incl = n;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int yy = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += yy;
  }
  const int total = __shfl_sync(0xffffffffu, incl, 31);
  unsigned long long base = 0;
  if (lane == 31 && total > 0) base = atomicAdd(counter, static_cast<unsigned long long>(total));
  base = __shfl_sync(0xffffffffu, base, 31);
  if (!active) return;
  const int64_t start = static_cast<int64_t>(base) + (incl - n);
  hs_off[x] = start;
  hs_cnt[x] = n;
  if (start + n <= cap) {
    if constexpr (KW > 0) {
      if (n > kLoc) {  // rare: recompute straight into the reserved range
        region(hs_pk + start * 4, hs_pk + start * 4 + 3, hs_fb + start, 4, 4, n);
        return;
      }
    }
    for (int h = 0; h < n; ++h) {
#pragma unroll
      for (int k = 0; k < DW; ++k) hs_pk[(start + h) * 4 + k] = la[h * DW + k];
      hs_pk[(start + h) * 4 + 3] = lb[h];
      hs_fb[start + h] = lf[h];
    }
  }
}

// ------------------------------------------------------------------ host
static inline size_t al(size_t x) { return (x + 255) & ~size_t(255); }

void build_graph_device(DevGraph& G, Ctx& c, int n, int dw, const double* h_pos, const double* h_vel,
                        const DevWorld& w, double r_n, double dt, double eps_cc, double tau_max, double ratio,
                        int row_lo, int row_hi, bool gather) {
  if (row_hi < 0) row_hi = n;
  if (row_lo < 0 || row_lo > row_hi || row_hi > n) throw std::invalid_argument("build_graph: bad row range");
  if (r_n <= 0) throw std::invalid_argument("build_graph: r_n must be positive");
  if (dt <= 0) throw std::invalid_argument("motion_waypoints: dt must be positive");
  if (w.n_obs > 4096) throw std::invalid_argument("build_graph: more than 4096 obstacles");
  static const bool dbg_t = std::getenv("PUMP_DEBUG_TIMING") != nullptr;
  const auto t_start = std::chrono::steady_clock::now();
  auto mark = [&](const char* what) {
    if (dbg_t)
      std::fprintf(stderr, "[pump g] %-24s %8.3f ms\n", what,
                   1e3 * std::chrono::duration<double>(std::chrono::steady_clock::now() - t_start).count());
  };
  G.n = n;
  G.dw = dw;
  G.r_n = r_n;
  G.dt = dt;
  cudaStream_t st = c.stream;
  if (h_pos) {  // else the caller already placed the nodes in G.pos / G.vel (device sampler)
    G.pos.ensure(al(n * dw * 8));
    G.vel.ensure(al(n * dw * 8));
    c.h2d(G.pos.p, h_pos, n * dw * 8);
    c.h2d(G.vel.p, h_vel, n * dw * 8);
  }
  GraphArgs ga{n, G.pos.as<double>(), G.vel.as<double>(), r_n, dt, eps_cc, tau_max, ratio};
  const LbGrid lbg = make_lb_grid(r_n);
  {  // k_pair_filter_grid reads the table from device memory (uploaded when r_n changes)
    DBuf& lbb = c.buf("g_lbgrid", sizeof(LbGrid));
    if (c.lbgrid_rn != r_n) {
      c.h2d(lbb.p, &lbg, sizeof(LbGrid));
      c.lbgrid_rn = r_n;
    }
  }
  WorldD wd;
  wd.n_obs = w.n_obs;
  wd.lo = w.d_lo;
  wd.hi = w.d_hi;
  for (int k = 0; k < 6; ++k) {
    wd.blo[k] = w.blo[k];
    wd.bhi[k] = w.bhi[k];
  }
  const size_t wsmem = 2 * static_cast<size_t>(w.n_obs) * dw * sizeof(double);
  int cap = 1024;
  DBuf& rcnt = c.buf("g_rowcnt", al((n + 8) * 4));
  PUMP_CUDA(cudaMemsetAsync(rcnt.p, 0, (n + 8) * 4, st));  // rows outside [row_lo, row_hi) stay empty
  DBuf& soff = c.buf("g_soff", al((n + 2) * 8));
  DBuf& stmp = c.buf("g_scantmp", scan_temp_bytes(static_cast<int64_t>(n) * n + 16));
  // ---- cell grid of the nodes for the exact spatial cull (k_pair_filter_grid)
  const size_t bits_bytes = static_cast<size_t>((n + 31) / 32) * 4;
  const bool use_grid = n > 0 && row_hi > row_lo && bits_bytes <= 160 * 1024;
  CellGrid cg{};
  SausTab sz{};
  if (use_grid) {
    KScope ks(st, F_PAIR);
    DBuf& stats = c.buf("g_nstats", 256);
    PUMP_CUDA(cudaMemsetAsync(stats.p, 0xff, 24, st));
    PUMP_CUDA(cudaMemsetAsync(stats.as<char>() + 24, 0, 32, st));
    dispatch_dw(dw, [&]<int DW>() {
      k_node_stats<DW><<<std::min(64, (n + 255) / 256), 256, 0, st>>>(n, G.pos.as<double>(), G.vel.as<double>(),
                                                                      stats.as<unsigned long long>());
    });
    ++c.launches;
    PUMP_CUDA(cudaGetLastError());
    unsigned long long hs[7];
    c.d2h(hs, stats.p, 56);
    c.sync();
    double lo[3] = {0, 0, 0}, hi[3] = {0, 0, 0};
    for (int k = 0; k < dw; ++k) {
      lo[k] = dbl_of(hs[k]);
      hi[k] = dbl_of(hs[3 + k]);
    }
    const double V = std::sqrt(dbl_of(hs[6])) * (1.0 + 1e-12);
    const double thr = r_n * (1.0 + 1e-6);
    // velocity-aware reach intervals (SausTab, k_pair_filter_grid)
    for (int i = 0; i < kSaus; ++i) {
      sz.tl[i] = i == 0 ? 0.0 : i == 1 ? thr / 64 : thr * (i - 1) / 32;
      sz.th[i] = i == 0 ? thr / 64 : thr * i / 32;
      const double rho = V * sz.th[i] * 0.5 + std::sqrt((thr - sz.tl[i]) * sz.th[i] * sz.th[i] * sz.th[i] / 12.0);
      const double r = rho * (1.0 + 1e-9) + 1e-12;
      sz.rho2[i] = r * r;
      sz.ext = std::max(sz.ext, r + V * sz.th[i] * 0.5 * (1.0 + 1e-9));
    }
    for (int q = 0; q < kSausGroups; ++q)
      for (int i = saus_g0(q); i < saus_g0(q + 1); ++i) sz.grho2[q] = std::max(sz.grho2[q], sz.rho2[i]);
    // cells of ~ext / 2.8 (A/B on the forest: 3.5 and 2.2 slower; ~500 candidates per row vs
    // 2249 with the position-only reach), grown until a row's cell range fits
    // kCellMaxList and the grid 2^22 cells
    double h = sz.ext / 2.8;
    bool finite = std::isfinite(sz.ext) && sz.ext > 0;
    for (int k = 0; k < dw; ++k) finite = finite && std::isfinite(lo[k]) && std::isfinite(hi[k]);
    if (finite) {
      for (;;) {
        int64_t cells = 1, range = 1;
        for (int k = 0; k < dw; ++k) {
          cg.dims[k] = static_cast<int>(std::min(1024.0, std::floor((hi[k] - lo[k]) / h) + 1.0));
          cells *= cg.dims[k];
          range *= std::min<int64_t>(cg.dims[k], static_cast<int64_t>(std::floor(2.0 * sz.ext / h)) + 2);
        }
        if (cells <= (int64_t(1) << 22) && range <= kCellMaxList) break;
        h *= 1.03;
      }
      for (int k = 0; k < dw; ++k) cg.lo[k] = lo[k];
      cg.inv_h = 1.0 / h;
    } else {
      cg.dims[0] = cg.dims[1] = cg.dims[2] = 1;  // one cell: every node is visited
      cg.inv_h = 0.0;
      for (int i = 0; i < kSaus; ++i) sz.rho2[i] = INFINITY;
      for (int q = 0; q < kSausGroups; ++q) sz.grho2[q] = INFINITY;
      sz.ext = INFINITY;
    }
    int n_cells = 1;
    for (int k = 0; k < dw; ++k) n_cells *= cg.dims[k];
    DBuf& ccnt = c.buf("g_ccnt", al((n_cells + 8) * 4));
    DBuf& cbox = c.buf("g_cbox", al(static_cast<size_t>(n_cells) * 48 + 64));
    DBuf& cst = c.buf("g_cstart", al((n_cells + 2) * 8));
    DBuf& nci = c.buf("g_ncell", al((n + 8) * 4));
    DBuf& nrk = c.buf("g_nrank", al((n + 8) * 4));
    DBuf& sidx = c.buf("g_sidx", al((n + 8) * 4));
    DBuf& spos = c.buf("g_spos", al(static_cast<size_t>(n) * dw * 8 + 64));
    DBuf& svel = c.buf("g_svel", al(static_cast<size_t>(n) * dw * 8 + 64));
    DBuf& ctmp = c.buf("g_cscantmp", scan_temp_bytes(n_cells + 16));
    PUMP_CUDA(cudaMemsetAsync(ccnt.p, 0, static_cast<size_t>(n_cells) * 4, st));
    dispatch_dw(dw, [&]<int DW>() {
      k_cell_box_init<<<grid_for(static_cast<int64_t>(n_cells) * 6, 256), 256, 0, st>>>(n_cells, cbox.as<unsigned long long>());
      k_cell_count<DW><<<grid_for(n, 256), 256, 0, st>>>(n, G.pos.as<double>(), cg, ccnt.as<int32_t>(),
                                                         cbox.as<unsigned long long>(), nci.as<int32_t>(),
                                                         nrk.as<int32_t>());
    });
    c.launches += 2;
    exclusive_scan<int32_t>(ccnt.as<int32_t>(), cst.as<int64_t>(), n_cells, ctmp.p, st, &c.launches);
    dispatch_dw(dw, [&]<int DW>() {
      k_cell_scatter<DW><<<grid_for(n, 256), 256, 0, st>>>(n, G.pos.as<double>(), G.vel.as<double>(), nci.as<int32_t>(),
                                                           nrk.as<int32_t>(), cst.as<int64_t>(), sidx.as<int32_t>(),
                                                           spos.as<double>(), svel.as<double>());
    });
    ++c.launches;
    PUMP_CUDA(cudaGetLastError());
  }
  int64_t n_surv = 0;
  for (;;) {  // pass 1 with an exact per-row refit if a row overflows the slab
    DBuf& suB = c.buf("g_su", al(static_cast<size_t>(n) * cap * 4));
    {
      KScope ks(st, F_PAIR);
      dispatch_dw(dw, [&]<int DW>() {
        constexpr int refill = 16;  // lane-refill threshold of the filter walks
        if (use_grid) {
          const int sm = static_cast<int>(bits_bytes);
          if (sm > 32 * 1024)
            PUMP_CUDA(cudaFuncSetAttribute(k_pair_filter_grid<DW>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm));
          k_pair_filter_grid<DW><<<row_hi - row_lo, kGridBlock, sm, st>>>(
              ga, c.scratch["g_lbgrid"].as<LbGrid>(), cg, sz, cap, row_lo, refill, c.scratch["g_ccnt"].as<int32_t>(), c.scratch["g_cstart"].as<int64_t>(),
              c.scratch["g_cbox"].as<unsigned long long>(), c.scratch["g_sidx"].as<int32_t>(),
              c.scratch["g_spos"].as<double>(), c.scratch["g_svel"].as<double>(), rcnt.as<int32_t>(),
              suB.as<int32_t>(), 1);
        } else if (row_hi > row_lo)  // more nodes than the row bitmask holds
          k_pair_filter_q<DW><<<row_hi - row_lo, kRowBlock, 0, st>>>(ga, lbg, cap, row_lo, refill, rcnt.as<int32_t>(),
                                                                     suB.as<int32_t>());
      });
      ++c.launches;
      PUMP_CUDA(cudaGetLastError());
    }
    // the slab check and the survivor total in one round trip
    DBuf& mx = c.buf("g_maxcnt", 256);
    PUMP_CUDA(cudaMemsetAsync(mx.p, 0, 4, st));
    k_max_count<<<std::min(148, (n + 255) / 256 + 1), 256, 0, st>>>(n, rcnt.as<int32_t>(), mx.as<int>());
    exclusive_scan<int32_t>(rcnt.as<int32_t>(), soff.as<int64_t>(), n, stmp.p, st, &c.launches);
    c.launches += 1;
    int max_cnt = 0;
    c.d2h(&max_cnt, mx.p, 4);
    c.d2h(&n_surv, soff.as<int64_t>() + n, 8);
    c.sync();
    mark("pair_filter + survivor scan");
    if (max_cnt <= cap) break;
    cap = max_cnt;
  }
  kprof_work(F_CONNECT, static_cast<int64_t>(n) * (n - 1));
  int32_t* su = c.scratch["g_su"].as<int32_t>();
  G.n_connect = n_surv;
  DBuf& skeep = c.buf("g_skeep", al(n_surv + 1));
  DBuf& sv = c.buf("g_sv", al((n_surv + 1) * 4));
  DBuf& suu = c.buf("g_suu", al((n_surv + 1) * 4));
  DBuf& stau = c.buf("g_stau", al((n_surv + 1) * 8));
  DBuf& scost = c.buf("g_scost", al((n_surv + 1) * 8));
  DBuf& cpos = c.buf("g_cpos", al((n_surv + 2) * 8));
  if (n_surv > 0) {
    KScope ks(st, F_CONNECT);
    dispatch_dw(dw, [&]<int DW>() {
      k_connect<DW><<<grid_for(n_surv, 128), 128, 0, st>>>(ga, cap, n_surv, soff.as<int64_t>(), su,
                                                           skeep.as<uint8_t>(), sv.as<int32_t>(), suu.as<int32_t>(),
                                                           stau.as<double>(), scost.as<double>());
    });
    ++c.launches;
    PUMP_CUDA(cudaGetLastError());
  }
  DBuf& stmpc = c.buf("g_scantmpc", scan_temp_bytes(n_surv + 16));
  exclusive_scan<uint8_t>(skeep.as<uint8_t>(), cpos.as<int64_t>(), n_surv, stmpc.p, st, &c.launches);
  // the candidate count stays on the device (cpos[n_surv]); the candidate and
  // edge arrays are sized by its bound n_surv, so no round trip until the
  // waypoint count is needed
  const int64_t n_cand = n_surv;  // bound
  const int64_t* d_ncand = cpos.as<int64_t>() + n_surv;
  DBuf& cv = c.buf("g_cv", al((n_cand + 1) * 4));
  DBuf& cuu = c.buf("g_cuu", al((n_cand + 1) * 4));
  DBuf& ctau = c.buf("g_ctau2", al((n_cand + 1) * 8));
  DBuf& ccost = c.buf("g_ccost2", al((n_cand + 1) * 8));
  DBuf& coff = c.buf("g_candoff", al((n + 2) * 8));
  {
    const int64_t items = std::max<int64_t>(n_surv, n + 1);
    KScope ks(st, F_EMIT);
    k_cand_compact<<<grid_for(items, 256), 256, 0, st>>>(n, n_surv, skeep.as<uint8_t>(), cpos.as<int64_t>(),
                                                          soff.as<int64_t>(), sv.as<int32_t>(), suu.as<int32_t>(),
                                                          stau.as<double>(), scost.as<double>(), cv.as<int32_t>(),
                                                          cuu.as<int32_t>(), ctau.as<double>(), ccost.as<double>(),
                                                          coff.as<int64_t>());
    ++c.launches;
    PUMP_CUDA(cudaGetLastError());
  }
  DBuf& valid = c.buf("g_valid", al(n_cand + 1));
  DBuf& nst = c.buf("g_nsteps", al((n_cand + 1) * 4));
  DBuf& eoff = c.buf("g_eoff", al((n_cand + 2) * 8));
  DBuf& stmp2 = c.buf("g_scantmp2", scan_temp_bytes(n_cand + 16));
  if (n_cand > 0) {
    KScope ks(st, F_COLLIDE);
    dispatch_dw(dw, [&]<int DW>() {
      auto kern = w.n_obs <= 64 * kCullWords ? k_collide<DW, 0> : k_collide<DW, kCullList>;
      if (wsmem > 48 * 1024)
        PUMP_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)wsmem));
      kern<<<grid_for(n_cand, 128), 128, wsmem, st>>>(ga, wd, d_ncand, cv.as<int32_t>(), cuu.as<int32_t>(),
                                                      ctau.as<double>(), valid.as<uint8_t>(), nst.as<int32_t>());
    });
    ++c.launches;
    PUMP_CUDA(cudaGetLastError());
  }
  exclusive_scan<uint8_t>(valid.as<uint8_t>(), eoff.as<int64_t>(), n_cand, stmp2.p, st, &c.launches, d_ncand);
  int64_t E = n_cand;  // bound until the totals come back
  DBuf& d_tot = c.buf("g_totals", 256);
  int64_t* d_E = d_tot.as<int64_t>() + 4;
  G.e_from.ensure(al((E + 1) * 4));
  G.e_to.ensure(al((E + 1) * 4));
  G.e_cost.ensure(al((E + 1) * 8));
  G.e_tau.ensure(al((E + 1) * 8));
  G.e_acc0.ensure(al((E + 1) * dw * 8));
  G.e_jerk.ensure(al((E + 1) * dw * 8));
  G.e_nsteps.ensure(al((E + 1) * 4));
  G.row_ptr.ensure(al((n + 1) * 8));
  G.wp_off.ensure(al((E + 2) * 8));
  {
    KScope ks(st, F_EMIT);
    dispatch_dw(dw, [&]<int DW>() {
      const int64_t items = std::max<int64_t>(n_cand + 1, n + 1);  // c == n_cand writes the edge count
      k_emit_edges<DW><<<grid_for(items, 256), 256, 0, st>>>(
          ga, d_ncand, d_E, coff.as<int64_t>(), cv.as<int32_t>(), cuu.as<int32_t>(), ctau.as<double>(), ccost.as<double>(),
          valid.as<uint8_t>(), nst.as<int32_t>(), eoff.as<int64_t>(), G.e_from.as<int32_t>(), G.e_to.as<int32_t>(),
          G.e_cost.as<double>(), G.e_tau.as<double>(), G.e_acc0.as<double>(), G.e_jerk.as<double>(),
          G.e_nsteps.as<int32_t>(), G.row_ptr.as<int64_t>());
    });
    ++c.launches;
    PUMP_CUDA(cudaGetLastError());
  }
  const bool multi = gather && c.world > 1;
  if (multi) {  // the gather needs this rank's edge count on the host
    int64_t nc = 0;
    c.d2h(&nc, d_ncand, 8);
    c.d2h(&E, d_E, 8);
    c.sync();
    G.n_cand = nc;
  }
  if (multi) {
    // ---- concatenate the ranks' row slices (graph sharded by source row)
    DBuf& cnts = c.buf("g_rank_edges", al(static_cast<size_t>(c.world) * 8 + 8));
    PUMP_CUDA(cudaMemsetAsync(cnts.p, 0, static_cast<size_t>(c.world) * 8, st));
    c.h2d(cnts.as<int64_t>() + c.rank, &E, 8);
    allreduce_sum_i64(c, cnts.as<int64_t>(), c.world);
    std::vector<int64_t> per(c.world);
    c.d2h(per.data(), cnts.p, static_cast<size_t>(c.world) * 8);
    c.sync();
    std::vector<int64_t> off(c.world + 1, 0);
    for (int r = 0; r < c.world; ++r) off[r + 1] = off[r] + per[r];
    const int64_t Et = off[c.world];
    auto gather_array = [&](DBuf& local, size_t elem) {
      DBuf& glob = c.buf("g_gather_tmp", al((Et + 1) * elem));
      std::vector<int64_t> bo(c.world), bl(c.world);
      for (int r = 0; r < c.world; ++r) {
        bo[r] = off[r] * static_cast<int64_t>(elem);
        bl[r] = per[r] * static_cast<int64_t>(elem);
      }
      gather_segments(c, local.p, glob.p, bo, bl);
      local.ensure(al((Et + 1) * elem));  // (reallocates only when growing; content replaced below)
      PUMP_CUDA(cudaMemcpyAsync(local.p, glob.p, Et * elem, cudaMemcpyDeviceToDevice, st));
    };
    gather_array(G.e_from, 4);
    gather_array(G.e_to, 4);
    gather_array(G.e_cost, 8);
    gather_array(G.e_tau, 8);
    gather_array(G.e_acc0, static_cast<size_t>(dw) * 8);
    gather_array(G.e_jerk, static_cast<size_t>(dw) * 8);
    gather_array(G.e_nsteps, 4);
    // a row's local row_ptr is 0 before the rank's slice and E_r after it, so
    // the global row_ptr is the element-wise sum over the ranks
    allreduce_sum_i64(c, G.row_ptr.as<int64_t>(), n + 1);
    E = Et;
    G.E = E;
    G.wp_off.ensure(al((E + 2) * 8));
    mark("gather");
  }
  DBuf& stmp3 = c.buf("g_scantmp3", scan_temp_bytes(E + 16));
  int64_t NW = 0;
  if (multi) {
    exclusive_scan<int32_t>(G.e_nsteps.as<int32_t>(), G.wp_off.as<int64_t>(), E, stmp3.p, st, &c.launches);
    c.d2h(&NW, G.wp_off.as<int64_t>() + E, 8);
    c.sync();
  } else {
    // waypoint offsets over the device edge count, then candidate / edge /
    // waypoint totals in one copy
    exclusive_scan<int32_t>(G.e_nsteps.as<int32_t>(), G.wp_off.as<int64_t>(), E, stmp3.p, st, &c.launches, d_E);
    k_graph_totals<<<1, 1, 0, st>>>(d_ncand, d_E, G.wp_off.as<int64_t>(), d_tot.as<int64_t>());
    ++c.launches;
    int64_t tot[3];
    c.d2h(tot, d_tot.p, 24);
    c.sync();
    G.n_cand = tot[0];
    E = tot[1];
    NW = tot[2];
    G.E = E;
  }
  mark("connect .. waypoint scan");
  G.NW = NW;
  DBuf& err = c.buf("g_err", 256);
  G.hs_off.ensure(al((NW + n + 2) * 8));  // (+ n: the nodes' regions, sorted pass)
  G.hs_cnt.ensure(al((NW + n + 2) * 4));
  PUMP_CUDA(cudaMemsetAsync(err.p, 0, 4, st));
  {
    DBuf& wpe = c.buf("g_wp_edge", al((NW + 8) * 4));
    if (E > 0) {
      KScope ks(st, F_REGIONS);
      k_wp_edge<<<grid_for(E, 256), 256, 0, st>>>(E, G.wp_off.as<int64_t>(), wpe.as<int32_t>());
      ++c.launches;
    }
    // more than 16 boxes: the region pass visits the waypoints cell by cell
    // (k_wp_prep, scan, k_wp_scatter), so a warp's waypoints are neighbours:
    // coherent branches and tight per-warp distance bounds (for <= 16 boxes
    // the fused region is cheaper than the ordering: indoor 0.79 vs 1.30 ms)
    const bool sorted = w.n_obs > kOnceMaxObs && NW > 0;
    const int32_t* d_perm = nullptr;
    const double* d_ys = nullptr;
    const int64_t* d_nlist = nullptr;
    int64_t n_items = NW;
    if (sorted) {
      WpCells cg{};
      double vol = 1.0;
      for (int k = 0; k < dw; ++k) vol *= std::max(w.bhi[k] - w.blo[k], 1e-9);
      // ~16 waypoints per cell on average, <= 2^21 cells
      const double h = std::pow(vol * 16.0 / static_cast<double>(NW), 1.0 / dw);
      int64_t ncell = 1;
      for (int k = 0; k < dw; ++k) {
        const double ext = std::max(w.bhi[k] - w.blo[k], 1e-9);
        cg.lo[k] = w.blo[k];
        cg.dim[k] = static_cast<int>(std::min(128.0, std::max(1.0, std::ceil(ext / h))));
        cg.inv[k] = cg.dim[k] / ext;
        ncell *= cg.dim[k];
      }
      // items: the waypoints but the edges' end waypoints, then the n nodes
      const int64_t NI = NW + n;
      DBuf& ysb = c.buf("g_wp_ys", al(NI * 2 * dw * 8 + 64));
      DBuf& keyb = c.buf("g_wp_key", al(NI * 4 + 64));
      DBuf& permb = c.buf("g_wp_perm", al(NI * 4 + 64));
      DBuf& hist = c.buf("g_wp_hist", al((ncell + 2) * 4));
      DBuf& hoff = c.buf("g_wp_hoff", al((ncell + 2) * 8));
      DBuf& htmp = c.buf("g_wp_htmp", scan_temp_bytes(ncell + 2));
      PUMP_CUDA(cudaMemsetAsync(hist.p, 0, (ncell + 1) * 4, st));
      KScope ks(st, F_REGIONS);
      dispatch_dw(dw, [&]<int DW>() {
        k_wp_prep<DW><<<grid_for(NI, 256), 256, 0, st>>>(
            ga, NW, G.wp_off.as<int64_t>(), G.e_from.as<int32_t>(), G.e_to.as<int32_t>(), G.e_tau.as<double>(),
            G.e_acc0.as<double>(), G.e_jerk.as<double>(), G.e_nsteps.as<int32_t>(), wpe.as<int32_t>(), cg,
            ysb.as<double>(), keyb.as<int32_t>(), hist.as<int32_t>());
      });
      exclusive_scan<int32_t>(hist.as<int32_t>(), hoff.as<int64_t>(), ncell, htmp.p, st, &c.launches);
      PUMP_CUDA(cudaMemsetAsync(hist.p, 0, (ncell + 1) * 4, st));
      k_wp_scatter<<<grid_for(NI, 256), 256, 0, st>>>(NI, keyb.as<int32_t>(), hoff.as<int64_t>(), hist.as<int32_t>(),
                                                     permb.as<int32_t>());
      c.launches += 2;
      d_perm = permb.as<int32_t>();
      d_ys = ysb.as<double>();
      d_nlist = hoff.as<int64_t>() + ncell;  // the listed items (the scan total)
      n_items = NI;
    }
    DBuf& ctr = c.buf("g_hs_counter", 256);
    int64_t cap = std::max<int64_t>(G.hs_cap, NW * 4 + 16);
    // the first pass counts even what does not fit (the exact rerun below), so
    // its buffer never needs more than the free memory
    auto room = [&]() {
      size_t free_b = 0, total_b = 0;
      PUMP_CUDA(cudaMemGetInfo(&free_b, &total_b));
      const size_t mine = G.hs_pk.cap + G.hs_fb.cap, keep = size_t(1) << 30;
      return static_cast<int64_t>((free_b + mine > keep ? free_b + mine - keep : 0) / 33);
    };
    // (only when the buffer must grow: cudaMemGetInfo is not free)
    if (static_cast<size_t>(cap + 1) * 32 > G.hs_pk.cap) cap = std::max<int64_t>(16, std::min(cap, room()));
    for (int attempt = 0; attempt < 2; ++attempt) {
      G.hs_pk.ensure(al((cap + 1) * 32));
      G.hs_fb.ensure(al(cap + 1));
      G.hs_cap = cap;
      PUMP_CUDA(cudaMemsetAsync(ctr.p, 0, 16, st));  // stored records, end-waypoint delta
      // work counters only while the per-kernel profiler is on (bench.py's second pass)
      KProf* kp = kprof_current();
      const bool count = kp && kp->on;
      DBuf& wk = c.buf("g_reg_work", 256 * 8 + 256);
      if (count) PUMP_CUDA(cudaMemsetAsync(wk.p, 0, 256 * 8, st));
      if (NW > 0) {
        KScope ks(st, F_REGIONS);
        dispatch_dw(dw, [&]<int DW>() {
          auto kern = w.n_obs <= kOnceMaxObs ? k_regions_once<DW, 0>
                      : w.n_obs <= 256      ? k_regions_once<DW, 8>
                      : w.n_obs <= 1024     ? k_regions_once<DW, 32>
                                            : k_regions_once<DW, 128>;
          const int blk = w.n_obs <= 256 ? 128 : regions_block(w.n_obs <= 1024 ? 32 : 128);
          const size_t sm = wsmem + (w.n_obs <= kOnceMaxObs ? static_cast<size_t>(w.n_obs) * 128 * 8
                                     : w.n_obs <= kLbsMaxObs
                                         ? static_cast<size_t>(w.n_obs) * (blk / 32) * 4  // lbs
                                               + (w.n_obs <= kBucketMaxObs
                                                      ? static_cast<size_t>(blk / 32) * (kOrdMeta + ((2 * w.n_obs + 15) & ~15))
                                                      : 0)
                                         : 0);
          if (sm > 48 * 1024)
            PUMP_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
          kern<<<grid_for(n_items, blk), blk, sm, st>>>(
              ga, wd, NW, E, G.wp_off.as<int64_t>(), G.e_from.as<int32_t>(), G.e_to.as<int32_t>(),
              G.e_tau.as<double>(), G.e_acc0.as<double>(), G.e_jerk.as<double>(), G.e_nsteps.as<int32_t>(),
              c.scratch["g_wp_edge"].as<int32_t>(), cap,
              ctr.as<unsigned long long>(), G.hs_off.as<int64_t>(), G.hs_cnt.as<int32_t>(), G.hs_pk.as<double>(),
              G.hs_fb.as<uint8_t>(), err.as<int>(), count ? wk.as<unsigned long long>() : nullptr, d_perm, d_ys,
              d_nlist);
        });
        ++c.launches;
        PUMP_CUDA(cudaGetLastError());
        if (sorted) {
          k_wp_end_link<<<grid_for(std::max<int64_t>(E, n), 256), 256, 0, st>>>(
              E, n, NW, G.wp_off.as<int64_t>(), G.e_to.as<int32_t>(), G.hs_off.as<int64_t>(), G.hs_cnt.as<int32_t>(),
              ctr.as<unsigned long long>() + 1);
          ++c.launches;
        }
      }
      int64_t Hd[2] = {0, 0};
      int herr = 0;
      std::vector<int64_t> wv(count ? 256 : 0);
      c.d2h(Hd, ctr.p, 16);
      if (count) c.d2h(wv.data(), wk.p, 256 * 8);
      c.d2h(&herr, err.p, 4);
      c.sync();
      const int64_t H = Hd[0];  // stored records (the capacity check)
      int64_t Hw[3] = {H, 0, 0};
      for (int q = 0; q < 128 && count; ++q) {
        Hw[1] += wv[2 * q];
        Hw[2] += wv[2 * q + 1];
      }
      // FP64-pipe ops of the region loop: a box distance |clamp(y) - y|^2 is
      // 6 compares + 3 sub + 3 mul + 2 add, a prune test 3 sub + 3 mul + 3 add
      // + 1 compare (the fraction in bench.py's roofline)
      kprof_work(F_REGIONS, 14 * Hw[1] + 10 * Hw[2]);
      mark("regions");
      if (herr) throw std::runtime_error("local_convex_region: pruning loop failed to make progress");
      G.H_pk = H;
      G.H = H + Hd[1];  // every waypoint's half-spaces
      if (H <= cap && std::getenv("PUMP_DEBUG_GRAPH"))
        std::fprintf(stderr, "[pump graph] n=%d pairs=%lld survivors=%lld candidates=%lld edges=%lld waypoints=%lld "
                     "halfspaces=%lld stored=%lld\n", n, (long long)n * (n - 1), (long long)G.n_connect,
                     (long long)G.n_cand, (long long)G.E, (long long)NW, (long long)G.H, (long long)H);
      if (H <= cap) break;
      cap = H + H / 8;  // rerun with room to spare (per-waypoint content is deterministic)
      if (H > room())
        throw CudaError("build_graph: the convex regions of " + std::to_string(NW) + " edge waypoints hold " +
                        std::to_string(H) + " half-spaces (" + std::to_string(static_cast<long long>(H * 33 / 1e9)) +
                        " GB), more than the free device memory");
      cap = std::min(cap, room());
    }
    c.sync();
    return;
  }
}

}  // namespace pumpg
