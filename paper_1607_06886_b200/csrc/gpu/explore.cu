// Explore wavefront (planner.hpp:74-267) on one B200.
//
// One round = one group B of open plans (sorted by (bucket, id)) expanded
// along every outgoing edge.  Device pipeline per round, one host sync:
//   k_expand      warp per (plan, edge) task: cost/t_end, horizon discard,
//                 HSMC over the edge's waypoints (ballot kill masks), keep =
//                 cp < alpha_max                         (planner.hpp:154-177)
//   scan + k_commit   kept candidates get arena ids in task order; goal
//                 bookkeeping; newcomers counted per head (planner.hpp:180-196)
//   k_relayout / k_place_new   per-node Pareto member segments rebuilt
//   k_dom         CTA per touched node: drop newcomers dominated by any member
//                 (old or new), evict old members (!= root) dominated by a
//                 surviving newcomer                     (planner.hpp:198-242)
//   scan + k_pool_append  surviving newcomers enter the open pool in id order
//   k_pool_min / k_round_i   next threshold i (skipping empty thresholds)
//   k_select + multisplit    next group = open pool entries with bucket <=
//                 min(i, nb-1), stably ordered by (bucket, id) (:248-261)
//   k_group_post + scan      task offsets (degree prefix sum) of the group
// The arena, member segments, pool and group stay resident in HBM.
#include <algorithm>
#include <climits>
#include <cstdio>
#include <cstdlib>
#include <utility>

#include "dispatch.cuh"
#include <cooperative_groups.h>

#include "explore.h"
#include "scan.cuh"

namespace pumpg {

constexpr int kOpen = 1;

DevExplore::~DevExplore() {
  if (status_h) cudaFreeHost(status_h);
  for (cudaEvent_t e : status_ev)
    if (e) cudaEventDestroy(e);
}

struct ExpandArgs {
  const int32_t* group;
  const int64_t* task_off;
  const int32_t* task_pid;
  const int64_t* task_e;
  const int64_t* d_G;
  const int64_t* d_T;
  const int64_t* row_ptr;
  const int32_t* e_to;
  const double* e_cost;
  const int32_t* e_nsteps;
  const int64_t* wp_off;
  const int64_t* hs_off;
  const int32_t* hs_cnt;
  const double* hs_pk;  // H x 4 {a, (pad), b}
  const int32_t* head;
  const double* cost;
  const int32_t* t_end;
  const uint64_t* mask;
  const double* dy;
  const double* bank_box;  // per bank row: particle box lo[DW], hi[DW]
  int N, horizon, W;
  int count_hs;  // accumulate st->hs_read (profiled pass only)
  double alpha_max;
  uint8_t* keep;
  int32_t* c_head;
  int32_t* c_src;
  int32_t* c_tend;
  double* c_cost;
  double* c_cp;
  uint64_t* c_mask;
  ExploreStatus* st;
  // a kept candidate's slot among its node's newcomers, the per-node newcomer
  // counts and the touched-node list (before: assigned in commit_one; here the
  // round tail's commit scan and node-size scan need not wait for each other)
  int32_t* new_cnt;
  int32_t* new_slot;  // per task
  int32_t* touched;
};

// The particle test of one half-space (cp.hpp:197-201): s = 0 + a0 p0 + ...
// evaluated without the leading "0 +" (it can only turn a -0 partial sum
// into +0, and the verdict s > b is identical for both zeros).
template <int DW, int CH>
__device__ __forceinline__ void hs_test(const double2 q0, const double2 q1, const double (&p)[CH][DW],
                                        bool (&kill)[CH]) {
  const double av[3] = {q0.x, q0.y, q1.x};  // {a0, a1}, {a2 | pad, b}
  const double b = q1.y;
#pragma unroll
  for (int c = 0; c < CH; ++c) {
    double s = av[0] * p[c][0];
#pragma unroll
    for (int k = 1; k < DW; ++k) s += av[k] * p[c][k];
    kill[c] = kill[c] || (s > b);
  }
}

template <int DW, int CH>
__device__ __forceinline__ void load_row(const double* row, int N, int lane, double (&p)[CH][DW], int pb = 0) {
#pragma unroll
  for (int c = 0; c < CH; ++c) {
    const int i = pb + c * 32 + lane;
#pragma unroll
    for (int k = 0; k < DW; ++k) p[c][k] = (i < N) ? row[i * DW + k] : 0.0;
  }
}

constexpr int kExpBlock = 256;

// Programmatic dependent launch: the per-round chain (gate, task map, expand,
// cooperative tail) is enqueued with programmatic stream serialization, so a
// kernel's launch and block ramp overlap its predecessor's last blocks; each
// of them waits here for its predecessor's completion (and memory) before it
// reads anything.  A no-op for a kernel launched without the attribute.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
constexpr int kExpStage = 64;  // half-spaces staged per warp (2 KB of shared memory)

// One warp per task (planner.hpp:140-176): the parent plan's particle mask is
// extended along the edge's waypoints with their half-spaces.  For edges of
// <= 32 waypoints whose half-spaces fit kExpStage, the warp first copies them
// into shared memory (every lane its own waypoint's, all loads in flight at
// once) and prefetches each next waypoint's bank row while testing the
// current one, so the loop does not wait on a chain of global round trips.
template <int DW, int CH>
__device__ __forceinline__ void expand_task(const ExpandArgs& a, int64_t task, int lane, int wib,
                                            double2 (*s_hs)[kExpStage][2]) {
  const int pid = a.task_pid[task];  // the task's plan and edge (k_task_map)
  const int64_t e = a.task_e[task];
  const double cc = a.cost[pid] + a.e_cost[e];
  const int pt = a.t_end[pid];
  const int ns = a.e_nsteps[e];
  const int te = pt + ns;
  if (lane == 0) {
    a.c_head[task] = a.e_to[e];
    a.c_src[task] = pid;
    a.c_cost[task] = cc;
    a.c_tend[task] = te;
  }
  if (te > a.horizon) {  // planner.hpp:164-168
    if (lane == 0) {
      a.keep[task] = 0;
      a.c_cp[task] = 2.0;
      atomicAdd(reinterpret_cast<unsigned long long*>(&a.st->disc_hor), 1ull);
    }
    return;
  }
  const int64_t w0 = a.wp_off[e];
  const double2* hpk = reinterpret_cast<const double2*>(a.hs_pk);
  int64_t tests = 0;
  // waypoint metadata of the first 32 waypoints in one parallel load
  int64_t my_h0 = 0;
  int my_cnt = 0;
  if (lane < ns) {
    my_h0 = a.hs_off[w0 + lane];
    my_cnt = a.hs_cnt[w0 + lane];
  }
  int incl = my_cnt;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += y;
  }
  const int total = __shfl_sync(0xffffffffu, incl, 31);
  int64_t hs_sum = total;  // the edge's half-spaces (first 32 waypoints; the rest below)
  // particles are independent (survival is an AND of per-particle tests), so
  // plans of more than 32 * CH particles run the same steps slab by slab
  constexpr int kSlab = 32 * CH;
  const int n_slab = CH == 16 ? (a.N + kSlab - 1) / kSlab : 1;  // (N <= 32 CH below 16 chunks)
  int pop = 0;
  for (int slab = 0; slab < n_slab; ++slab) {
  const int pb = slab * kSlab;
  bool kill[CH];
#pragma unroll
  for (int c = 0; c < CH; ++c) kill[c] = false;
  if (ns <= 32 && total <= kExpStage) {
    const int my_pre = incl - my_cnt;
    // Each lane stages its waypoint's half-spaces and decides which of them
    // can kill any particle of the bank row the waypoint reads: with the
    // row's per-axis particle box [lo, hi], fl(a_k p_k) <= M_k =
    // max(fl(a_k lo_k), fl(a_k hi_k)) by monotone rounding, and the sum is
    // formed in the test's order, so bound <= b proves s <= b (no kill) for
    // every particle of the row, bit-exactly.  Waypoints without such a
    // half-space skip the row load and the tests.
    uint64_t my_need = 0;
    const double* box = my_cnt > 0 ? a.bank_box + static_cast<int64_t>(pt + lane + 1) * 2 * DW : nullptr;
    double blo[DW], bhi[DW];
    if (my_cnt > 0) {
#pragma unroll
      for (int k = 0; k < DW; ++k) {
        blo[k] = box[k];
        bhi[k] = box[DW + k];
      }
    }
    for (int q = 0; q < my_cnt; ++q) {
      const double2 q0 = hpk[(my_h0 + q) * 2], q1 = hpk[(my_h0 + q) * 2 + 1];
      s_hs[wib][my_pre + q][0] = q0;
      s_hs[wib][my_pre + q][1] = q1;
      const double av[3] = {q0.x, q0.y, q1.x};
      double bound = 0;
#pragma unroll
      for (int k = 0; k < DW; ++k) {
        const double m1 = av[k] * blo[k], m2 = av[k] * bhi[k];
        const double mk = m1 > m2 ? m1 : m2;
        bound = k == 0 ? mk : bound + mk;
      }
      if (bound > q1.y) my_need |= 1ull << q;
    }
    __syncwarp();
    unsigned live = __ballot_sync(0xffffffffu, my_need != 0);  // waypoints whose row can lose a particle
    if (slab == 0) {
      tests = __popcll(my_need);
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) tests += __shfl_xor_sync(0xffffffffu, tests, o);
    }
    double p[CH][DW], pn[CH][DW];
    int j = live ? __ffs(live) - 1 : -1;
    if (j >= 0) load_row<DW, CH>(a.dy + static_cast<int64_t>(pt + j + 1) * a.N * DW, a.N, lane, p, pb);
    while (j >= 0) {
      live &= ~(1u << j);
      const int jn = live ? __ffs(live) - 1 : -1;
      if (jn >= 0) load_row<DW, CH>(a.dy + static_cast<int64_t>(pt + jn + 1) * a.N * DW, a.N, lane, pn, pb);
      const int cnt = __shfl_sync(0xffffffffu, my_cnt, j);
      const int pre = __shfl_sync(0xffffffffu, incl, j) - cnt;
      const uint64_t need = __shfl_sync(0xffffffffu, my_need, j);
      for (int h = 0; h < cnt; ++h)
        if ((need >> h) & 1ull) hs_test<DW, CH>(s_hs[wib][pre + h][0], s_hs[wib][pre + h][1], p, kill);
      if (jn >= 0) {
#pragma unroll
        for (int c = 0; c < CH; ++c)
#pragma unroll
          for (int k = 0; k < DW; ++k) p[c][k] = pn[c][k];
      }
      j = jn;
    }
  } else {
    // long edges / many half-spaces: 32 waypoints at a time, each lane its
    // waypoint's harmless-half-space filter (as above; past 64 half-spaces a
    // waypoint tests all), then the rows that can lose a particle in order,
    // the next one prefetched
    for (int jb = 0; jb < ns; jb += 32) {
      const int jj = jb + lane;
      int64_t h0 = 0;
      int cnt = 0;
      if (jj < ns) {
        if (jb == 0) {
          h0 = my_h0;
          cnt = my_cnt;
        } else {
          h0 = a.hs_off[w0 + jj];
          cnt = a.hs_cnt[w0 + jj];
        }
      }
      uint64_t need = 0;
      const bool all = cnt > 64;
      if (cnt > 0 && !all) {
        const double* box = a.bank_box + static_cast<int64_t>(pt + jj + 1) * 2 * DW;
        double blo[DW], bhi[DW];
#pragma unroll
        for (int k = 0; k < DW; ++k) {
          blo[k] = box[k];
          bhi[k] = box[DW + k];
        }
        for (int q = 0; q < cnt; ++q) {
          const double2 q0 = hpk[(h0 + q) * 2], q1 = hpk[(h0 + q) * 2 + 1];
          const double av[3] = {q0.x, q0.y, q1.x};
          double bound = 0;
#pragma unroll
          for (int k = 0; k < DW; ++k) {
            const double m1 = av[k] * blo[k], m2 = av[k] * bhi[k];
            const double mk = m1 > m2 ? m1 : m2;
            bound = k == 0 ? mk : bound + mk;
          }
          if (bound > q1.y) need |= 1ull << q;
        }
      }
      unsigned live = __ballot_sync(0xffffffffu, need != 0 || all);
      int64_t t_l = all ? cnt : __popcll(need);
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) t_l += __shfl_xor_sync(0xffffffffu, t_l, o);
      if (slab == 0) {
        tests += t_l;
        if (jb > 0) {
          int c_l = cnt;
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) c_l += __shfl_xor_sync(0xffffffffu, c_l, o);
          hs_sum += c_l;
        }
      }
      double p[CH][DW], pn[CH][DW];
      int j = live ? __ffs(live) - 1 : -1;
      if (j >= 0) load_row<DW, CH>(a.dy + static_cast<int64_t>(pt + jb + j + 1) * a.N * DW, a.N, lane, p, pb);
      while (j >= 0) {
        live &= ~(1u << j);
        const int jn = live ? __ffs(live) - 1 : -1;
        if (jn >= 0) load_row<DW, CH>(a.dy + static_cast<int64_t>(pt + jb + jn + 1) * a.N * DW, a.N, lane, pn, pb);
        const int64_t hj = __shfl_sync(0xffffffffu, h0, j);
        const int cj = __shfl_sync(0xffffffffu, cnt, j);
        const uint64_t nj = __shfl_sync(0xffffffffu, need, j);
        const bool aj = cj > 64;
        for (int h = 0; h < cj; ++h)
          if (aj || ((nj >> h) & 1ull)) hs_test<DW, CH>(hpk[(hj + h) * 2], hpk[(hj + h) * 2 + 1], p, kill);
        if (jn >= 0) {
#pragma unroll
          for (int c = 0; c < CH; ++c)
#pragma unroll
            for (int k = 0; k < DW; ++k) p[c][k] = pn[c][k];
        }
        j = jn;
      }
    }
  }
#pragma unroll
  for (int w = 0; w < (CH + 1) / 2; ++w) {
    const unsigned lo32 = __ballot_sync(0xffffffffu, kill[2 * w]);
    const unsigned hi32 = (2 * w + 1 < CH) ? __ballot_sync(0xffffffffu, kill[2 * w + 1]) : 0u;
    const int gw = slab * (kSlab / 64) + w;
    if (gw < a.W) {
      const uint64_t m = a.mask[static_cast<int64_t>(pid) * a.W + gw] & ~((static_cast<uint64_t>(hi32) << 32) | lo32);
      pop += __popcll(m);
      if (lane == 0) a.c_mask[task * a.W + gw] = m;
    }
  }
  }  // slab
  if (lane == 0 && a.count_hs) {
    // the roofline's work counts: only in the profiled pass (a same-address
    // atomic per task costs ~0.2 ms per solve)
    atomicAdd(reinterpret_cast<unsigned long long*>(&a.st->hs_tests), static_cast<unsigned long long>(tests));
    atomicAdd(reinterpret_cast<unsigned long long*>(&a.st->hs_read), static_cast<unsigned long long>(hs_sum));
  }
  if (lane == 0) {
    const double cp = 1.0 - static_cast<double>(pop) / a.N;  // ParticleMask::cp (cp.hpp:42)
    a.c_cp[task] = cp;
    const bool keep = cp < a.alpha_max;
    a.keep[task] = keep ? 1 : 0;
    if (!keep) {
      atomicAdd(reinterpret_cast<unsigned long long*>(&a.st->disc_cp), 1ull);
    } else {
      const int hv = a.e_to[e];
      const int slot = atomicAdd(&a.new_cnt[hv], 1);
      a.new_slot[task] = slot;
      if (slot == 0) a.touched[atomicAdd(reinterpret_cast<unsigned long long*>(&a.st->touched), 1ull)] = hv;
    }
  }
}

template <int DW, int CH>
__global__ void __launch_bounds__(kExpBlock, (CH <= 2 ? 4 : 2)) k_expand(const ExpandArgs a) {
  __shared__ double2 s_hs[kExpBlock / 32][kExpStage][2];
  const int64_t task = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  pdl_wait();
  // (a pipelined round's grid covers its task capacity; a halted round has none)
  if (task >= *a.d_T || a.st->halt) return;
  expand_task<DW, CH>(a, task, lane, wib, s_hs);
}

struct CommitArgs {
  const int64_t* d_T;
  const uint8_t* keep;
  const int64_t* rank;
  const int32_t* c_head;
  const int32_t* c_src;
  const int32_t* c_tend;
  const double* c_cost;
  const double* c_cp;
  const uint64_t* c_mask;
  int W;
  double width, alpha_min;
  const uint8_t* is_goal;
  int32_t* head;
  int32_t* parent;
  double* cost;
  double* cp;
  int32_t* t_end;
  uint64_t* mask;
  int32_t* bucket;
  uint8_t* flags;
  int32_t* new_cnt;
  int32_t* new_slot;
  int32_t* touched;
  ExploreStatus* st;
};

// commit candidate t (kept) as arena plan n_plans + r (r = its rank)
__device__ __forceinline__ void commit_one(const CommitArgs& a, int64_t t, int64_t r) {
  const int64_t P0 = a.st->n_plans;
  const int64_t id = P0 + r;
  const int hv = a.c_head[t];
  const double c = a.c_cost[t];
  const double q = a.c_cp[t];
  a.head[id] = hv;
  a.parent[id] = a.c_src[t];
  a.cost[id] = c;
  a.cp[id] = q;
  a.t_end[id] = a.c_tend[t];
  for (int w = 0; w < a.W; ++w) a.mask[id * a.W + w] = a.c_mask[t * a.W + w];
  int b = static_cast<int>(ceil(c / a.width - 1e-12));  // planner.hpp:86
  a.bucket[id] = b < 0 ? 0 : b;
  a.flags[id] = 0;
  if (a.is_goal[hv]) {
    if (q < a.alpha_min)  // note_goal (planner.hpp:95-98)
      atomicMin(&a.st->best_goal_bits, __double_as_longlong(c));
    atomicMax(&a.st->max_goal_tend, static_cast<long long>(a.c_tend[t]));
  }
}

__global__ void k_commit(const CommitArgs a) {
  const int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (t >= *a.d_T || !a.keep[t]) return;
  commit_one(a, t, a.rank[t]);
}

// node sizes for the member relayout; thread 0 also publishes K = kept
// candidates (rank[T]) and resets min_bucket for this round's k_pool_min
__global__ void k_node_sizes(int n, const int32_t* mem_cnt, const int32_t* new_cnt, int32_t* sz, ExploreStatus* st,
                             const int64_t* rank_total, int64_t* d_K) {
  const int v = blockIdx.x * blockDim.x + threadIdx.x;
  if (v == 0) {
    const int64_t K = *rank_total;
    st->K = K;
    *d_K = K;
    st->min_bucket = LLONG_MAX;
  }
  if (v < n) sz[v] = mem_cnt[v] + new_cnt[v];
}

__global__ void k_relayout(int n, const int64_t* old_off, const int32_t* mem_cnt, const int32_t* old_ids,
                           const int64_t* new_off, int32_t* new_ids) {
  const int64_t gw = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (gw >= n) return;
  const int v = static_cast<int>(gw);
  const int m = mem_cnt[v];
  const int64_t a = old_off[v], b = new_off[v];
  for (int k = lane; k < m; k += 32) new_ids[b + k] = old_ids[a + k];
}

__global__ void k_place_new(const int64_t* d_T, const ExploreStatus* st, const uint8_t* keep, const int64_t* rank,
                            const int32_t* c_head, const int64_t* new_off, const int32_t* mem_cnt,
                            const int32_t* new_slot, int32_t* new_ids) {
  const int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (t >= *d_T || !keep[t]) return;
  const int64_t id = st->n_plans + rank[t];
  const int hv = c_head[t];
  new_ids[new_off[hv] + mem_cnt[hv] + new_slot[t]] = static_cast<int32_t>(id);
}

// RemoveDominated, both directions, for one touched node per CTA.
// Segment layout on entry: [old members (ascending ids) | newcomers (any
// order)].  On exit: [old survivors | surviving newcomers by id].
constexpr int kDomCap = 1024;
struct DomShared {
  int old_surv, new_surv, drop, evict, evict_open;
  int32_t id[kDomCap];
  double c[kDomCap], p[kDomCap];
  uint8_t dr[kDomCap];
};
struct DomArgs {
  const int32_t* touched;
  const int64_t* new_off;
  int32_t* mem_cnt;
  int32_t* new_cnt;
  int32_t* ids;
  const double* cost;
  const double* cp;
  uint8_t* flags;
  uint8_t* drop;
  uint8_t* surv;
  int32_t* fpos;
  ExploreStatus* stw;
};

// one touched node b; all threads of the block call it together
__device__ void dom_node(const DomArgs& A, DomShared& sh, int64_t b, int64_t P0) {
  int32_t* ids = A.ids;
  const double* cost = A.cost;
  const double* cp = A.cp;
  uint8_t* drop = A.drop;
  constexpr int kMaxLocal = 64;
  {
    const int v = A.touched[b];
    const int64_t base = A.new_off[v];
    const int m_old = A.mem_cnt[v];
    const int m_new = A.new_cnt[v];
    const int m = m_old + m_new;
    const bool staged = m <= kDomCap;
    if (threadIdx.x == 0) {
      sh.old_surv = 0;
      sh.new_surv = 0;
      sh.drop = 0;
      sh.evict = 0;
      sh.evict_open = 0;
    }
    if (staged) {
      for (int x = threadIdx.x; x < m; x += blockDim.x) {
        const int id = ids[base + x];
        sh.id[x] = id;
        sh.c[x] = cost[id];
        sh.p[x] = cp[id];
      }
    }
    __syncthreads();
    auto ID = [&](int x) { return staged ? sh.id[x] : ids[base + x]; };
    auto CO = [&](int x) { return staged ? sh.c[x] : cost[ids[base + x]]; };
    auto CP = [&](int x) { return staged ? sh.p[x] : cp[ids[base + x]]; };
    // (1) drop newcomers dominated by any member of the pre-removal set,
    //     old or new (planner.hpp:200-211); dominates(o, q) = q.cost > o.cost
    //     && q.cp >= o.cp (planner.hpp:58-60)
    for (int qi = threadIdx.x; qi < m_new; qi += blockDim.x) {
      const int q = ID(m_old + qi);
      const double qc = CO(m_old + qi), qp = CP(m_old + qi);
      bool d = false;
      for (int x = 0; x < m && !d; ++x) d = (qc > CO(x)) && (qp >= CP(x));
      drop[q - P0] = d ? 1 : 0;
      A.surv[q - P0] = d ? 0 : 1;
      if (staged) sh.dr[m_old + qi] = d ? 1 : 0;
      if (d) atomicAdd(&sh.drop, 1);
    }
    __syncthreads();
    auto DROPPED = [&](int qi) { return staged ? sh.dr[m_old + qi] != 0 : drop[ids[base + m_old + qi] - P0] != 0; };
    // (2) evict old members other than the root that a surviving newcomer
    //     dominates (planner.hpp:219-238); evicted slots become -1 - id
    for (int pi = threadIdx.x; pi < m_old; pi += blockDim.x) {
      const int p = ID(pi);
      if (p == 0) continue;
      const double pc = CO(pi), pp = CP(pi);
      bool ev = false;
      for (int qi = 0; qi < m_new && !ev; ++qi) {
        if (DROPPED(qi)) continue;
        ev = (pc > CO(m_old + qi)) && (pp >= CP(m_old + qi));
      }
      if (ev) {
        atomicAdd(&sh.evict, 1);
        if (A.flags[p] & kOpen) {  // waiting in a bucket: skipped at collection
          A.flags[p] &= static_cast<uint8_t>(~kOpen);
          atomicAdd(&sh.evict_open, 1);
        }
        if (staged)
          sh.id[pi] = -1 - p;
        else
          ids[base + pi] = -1 - p;
      }
    }
    __syncthreads();
    // (3) rank surviving newcomers by id; compact old survivors in order
    for (int qi = threadIdx.x; qi < m_new; qi += blockDim.x) {
      if (DROPPED(qi)) continue;
      const int q = ID(m_old + qi);
      int r = 0;
      for (int xi = 0; xi < m_new; ++xi) r += (!DROPPED(xi) && ID(m_old + xi) < q) ? 1 : 0;
      A.fpos[q - P0] = r;
      atomicAdd(&sh.new_surv, 1);
    }
    if (threadIdx.x == 0) {
      int w = 0;
      for (int pi = 0; pi < m_old; ++pi) {
        const int p = ID(pi);
        if (p >= 0) ids[base + w++] = p;
      }
      sh.old_surv = w;
    }
    if (staged) {
      __syncthreads();
      // (4) surviving newcomers after the old survivors, in id order (their
      //     ids are still in shared memory)
      for (int qi = threadIdx.x; qi < m_new; qi += blockDim.x) {
        if (DROPPED(qi)) continue;
        const int q = sh.id[m_old + qi];
        ids[base + sh.old_surv + A.fpos[q - P0]] = q;
      }
    } else {
      // (4) gather surviving newcomers before overwriting their slots
      int my_q[kMaxLocal];
      int my_n = 0;
      for (int qi = threadIdx.x; qi < m_new; qi += blockDim.x) {
        const int q = ids[base + m_old + qi];
        if (!drop[q - P0] && my_n < kMaxLocal) my_q[my_n++] = q;
      }
      __syncthreads();
      if (m_new > kMaxLocal * static_cast<int>(blockDim.x)) {
        if (threadIdx.x == 0) atomicExch(reinterpret_cast<unsigned long long*>(&A.stw->err), 2ull);
      } else {
        for (int k = 0; k < my_n; ++k) ids[base + sh.old_surv + A.fpos[my_q[k] - P0]] = my_q[k];
      }
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      A.mem_cnt[v] = sh.old_surv + sh.new_surv;
      A.new_cnt[v] = 0;
      atomicAdd(reinterpret_cast<unsigned long long*>(&A.stw->removed),
                static_cast<unsigned long long>(sh.drop + sh.evict));
      atomicAdd(reinterpret_cast<unsigned long long*>(&A.stw->evicted_open),
                static_cast<unsigned long long>(sh.evict_open));
    }
    __syncthreads();
  }
}

// The same RemoveDominated steps for a node of <= kDomWarpCap members, one
// warp per node (the cooperative round's dom phase: thousands of small
// nodes, so a warp each keeps many in flight); members staged per warp.
constexpr int kDomWarpCap = 128;
struct DomWarpShared {
  int32_t id[kDomWarpCap];
  double c[kDomWarpCap], p[kDomWarpCap];
  uint8_t dr[kDomWarpCap];
};

__device__ void dom_node_warp(const DomArgs& A, DomWarpShared& sh, int v, int64_t P0, int lane) {
  int32_t* ids = A.ids;
  const int64_t base = A.new_off[v];
  const int m_old = A.mem_cnt[v];
  const int m_new = A.new_cnt[v];
  const int m = m_old + m_new;
  for (int x = lane; x < m; x += 32) {
    const int id = ids[base + x];
    sh.id[x] = id;
    sh.c[x] = A.cost[id];
    sh.p[x] = A.cp[id];
  }
  __syncwarp();
  // (1) drop newcomers dominated by any member (old or new)
  unsigned n_drop = 0;
  for (int qi = lane; qi < m_new; qi += 32) {
    const int q = sh.id[m_old + qi];
    const double qc = sh.c[m_old + qi], qp = sh.p[m_old + qi];
    bool d = false;
    for (int x = 0; x < m && !d; ++x) d = (qc > sh.c[x]) && (qp >= sh.p[x]);
    A.drop[q - P0] = d ? 1 : 0;
    A.surv[q - P0] = d ? 0 : 1;
    sh.dr[m_old + qi] = d ? 1 : 0;
    n_drop += d ? 1u : 0u;
  }
  __syncwarp();
  // (2) evict old members (not the root) a surviving newcomer dominates
  unsigned n_ev = 0, n_ev_open = 0;
  for (int pi = lane; pi < m_old; pi += 32) {
    const int p = sh.id[pi];
    if (p == 0) continue;
    const double pc = sh.c[pi], pp = sh.p[pi];
    bool ev = false;
    for (int qi = 0; qi < m_new && !ev; ++qi) {
      if (sh.dr[m_old + qi]) continue;
      ev = (pc > sh.c[m_old + qi]) && (pp >= sh.p[m_old + qi]);
    }
    if (ev) {
      ++n_ev;
      if (A.flags[p] & kOpen) {
        A.flags[p] &= static_cast<uint8_t>(~kOpen);
        ++n_ev_open;
      }
      sh.id[pi] = -1 - p;
    }
  }
  __syncwarp();
  // (3) surviving newcomers ranked by id; old survivors compacted in order
  unsigned n_new_surv = 0;
  for (int qi = lane; qi < m_new; qi += 32) {
    if (sh.dr[m_old + qi]) continue;
    const int q = sh.id[m_old + qi];
    int r = 0;
    for (int xi = 0; xi < m_new; ++xi) r += (!sh.dr[m_old + xi] && sh.id[m_old + xi] < q) ? 1 : 0;
    A.fpos[q - P0] = r;
    ++n_new_surv;
  }
  int w = 0;
  const unsigned lt = (1u << lane) - 1u;
  for (int c0 = 0; c0 < m_old; c0 += 32) {
    const int pi = c0 + lane;
    const int p = pi < m_old ? sh.id[pi] : -1;
    const unsigned keepm = __ballot_sync(0xffffffffu, p >= 0);
    if (p >= 0) ids[base + w + __popc(keepm & lt)] = p;
    w += __popc(keepm);
  }
  __syncwarp();
  // (4) surviving newcomers after the old survivors, in id order
  for (int qi = lane; qi < m_new; qi += 32) {
    if (sh.dr[m_old + qi]) continue;
    const int q = sh.id[m_old + qi];
    ids[base + w + A.fpos[q - P0]] = q;
  }
  n_drop = __reduce_add_sync(0xffffffffu, n_drop);
  n_ev = __reduce_add_sync(0xffffffffu, n_ev);
  n_ev_open = __reduce_add_sync(0xffffffffu, n_ev_open);
  n_new_surv = __reduce_add_sync(0xffffffffu, n_new_surv);
  if (lane == 0) {
    A.new_cnt[v] = 0;
    A.mem_cnt[v] = w + static_cast<int>(n_new_surv);
    atomicAdd(reinterpret_cast<unsigned long long*>(&A.stw->removed), static_cast<unsigned long long>(n_drop + n_ev));
    atomicAdd(reinterpret_cast<unsigned long long*>(&A.stw->evicted_open), static_cast<unsigned long long>(n_ev_open));
  }
  __syncwarp();
}

// RemoveDominated at one touched node per CTA (planner.hpp:200-238).  The
// node's members (ids, cost, cp) are first staged in shared memory with one
// batch of independent loads, so the O(m_new * m) dominance scans read shared
// memory instead of chasing ids through global memory; nodes with more than
// kDomCap members take the same steps on global memory.
__global__ void __launch_bounds__(128) k_dom(const ExploreStatus* st, const int32_t* touched,
                                             const int64_t* new_off, int32_t* mem_cnt, int32_t* new_cnt,
                                             int32_t* ids, const double* cost, const double* cp, uint8_t* flags,
                                             uint8_t* drop, uint8_t* surv, int32_t* fpos, ExploreStatus* stw) {
  __shared__ DomShared sh;
  const DomArgs A{touched, new_off, mem_cnt, new_cnt, ids, cost, cp, flags, drop, surv, fpos, stw};
  const int64_t P0 = st->n_plans;
  for (int64_t b = blockIdx.x; b < st->touched; b += gridDim.x) dom_node(A, sh, b, P0);
}

__global__ void k_pool_append(const int64_t* d_K, const ExploreStatus* st, const uint8_t* surv, const int64_t* spos,
                              const int32_t* bucket, uint8_t* flags, int32_t* pool, ExploreStatus* stw) {
  const int64_t r = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (r >= *d_K || !surv[r]) return;
  const int64_t id = st->n_plans + r;
  pool[st->pool_n + spos[r]] = static_cast<int32_t>(id);
  flags[id] |= kOpen;
  atomicMax(&stw->max_bucket, static_cast<long long>(bucket[id]));
}

// lowest open bucket of the pool after this round's appends (spos[K] =
// surviving newcomers appended behind the st->pool_n carried in)
__global__ void k_pool_min(const ExploreStatus* st, const int64_t* d_K, const int64_t* spos, const int32_t* pool,
                           const uint8_t* flags, const int32_t* bucket, ExploreStatus* stw) {
  const int64_t x = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (x >= st->pool_n + spos[*d_K]) return;
  const int id = pool[x];
  if (flags[id] & kOpen) atomicMin(&stw->min_bucket, static_cast<long long>(bucket[id]));
}

// End of round bookkeeping, then i <- max(i + 1, lowest open bucket): the
// reference's `continue` over empty thresholds (planner.hpp:250-261)
// collapsed into one step.  Single thread.
__global__ void k_round_i(ExploreStatus* st, const int64_t* d_K, const int64_t* spos, int64_t* d_pool_n,
                          int64_t* limits) {
  {
    const int64_t K = *d_K;
    const int64_t ns = spos[K];
    st->n_surv = ns;
    st->pool_n += ns;
    st->open_count += ns - st->evicted_open - st->G;
    st->n_plans += K;
  }
  long long i = st->i + 1;
  if (st->min_bucket != LLONG_MAX && st->min_bucket > i) i = st->min_bucket;
  st->i = i;
  const long long limit = i < st->max_bucket ? i : st->max_bucket;
  limits[0] = limit;
  limits[1] = st->min_bucket == LLONG_MAX ? 0 : st->min_bucket;
  *d_pool_n = st->pool_n;
  st->G = 0;
  st->T = 0;
  st->min_group_bits = 0x7ff0000000000000ll;
  st->touched = 0;
  st->evicted_open = 0;
}

__global__ void k_select(const int64_t* d_pool_n, const int64_t* limits, const int32_t* pool, const uint8_t* flags,
                         const int32_t* bucket, int32_t* keys, uint8_t* stay, int64_t n_keys, ExploreStatus* st) {
  const int64_t x = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (x >= *d_pool_n) return;
  const int id = pool[x];
  const bool open = flags[id] & kOpen;
  const int b = bucket[id];
  const bool sel = open && b <= limits[0];
  const int64_t key = b - limits[1];
  if (sel && key >= n_keys) atomicExch(reinterpret_cast<unsigned long long*>(&st->err), 3ull);  // bound violated
  keys[x] = sel ? static_cast<int32_t>(key) : -1;
  stay[x] = (open && !sel) ? 1 : 0;
}

__global__ void k_pool_compact(const int64_t* d_pool_n, const int32_t* pool, const uint8_t* stay, const int64_t* pos,
                               int32_t* out) {
  const int64_t x = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (x >= *d_pool_n || !stay[x]) return;
  out[pos[x]] = pool[x];
}

__global__ void k_group_post(const int64_t* d_G, const int32_t* group, const int32_t* head, const double* cost,
                             const int64_t* row_ptr, uint8_t* flags, int32_t* deg, ExploreStatus* st) {
  const int64_t g = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (g >= *d_G) return;
  const int id = group[g];
  flags[id] &= static_cast<uint8_t>(~kOpen);
  const int hv = head[id];
  deg[g] = static_cast<int32_t>(row_ptr[hv + 1] - row_ptr[hv]);
  atomicMin(&st->min_group_bits, __double_as_longlong(cost[id]));
}

// task -> group entry (warp per group), so k_expand starts without a search
// per task: its plan and edge (warp per group entry), so k_expand starts
// from two independent loads instead of a chain group -> plan -> head -> row
__global__ void k_task_map(const int64_t* d_G, const int64_t* task_off, const int32_t* group, const int32_t* head,
                           const int64_t* row_ptr, int32_t* task_pid, int64_t* task_e, const ExploreStatus* st) {
  const int lane = threadIdx.x & 31;
  pdl_wait();
  if (st->halt) return;
  const int64_t Gn = *d_G;
  const int64_t stride = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
  for (int64_t g = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5; g < Gn; g += stride) {
    const int64_t t0 = task_off[g], t1 = task_off[g + 1];
    const int pid = group[g];
    const int64_t e0 = row_ptr[head[pid]];
    for (int64_t t = t0 + lane; t < t1; t += 32) {
      task_pid[t] = pid;
      task_e[t] = e0 + (t - t0);
    }
  }
}

// Pipelined rounds: the loop-top decisions of run_explore_device made on the
// device before each enqueued round (planner.hpp:126-138 termination, the
// cooperative path's key-range and buffer-capacity conditions).  A round that
// may not run sets halt; every later kernel of it, and every later round,
// then exits at once, and the host takes over from the status it reads.
struct GateCaps {
  long long T, arena, pool;
};
__global__ void k_round_gate(ExploreStatus* S, GateCaps cap) {
  pdl_wait();
  if (S->halt) return;
  const double best_goal = __longlong_as_double(S->best_goal_bits);
  const double min_group = __longlong_as_double(S->min_group_bits);
  if ((S->G > 0 && best_goal != __builtin_inf() && best_goal <= min_group) || (S->G == 0 && S->open_count == 0)) {
    S->halt = 1;
    return;
  }
  const long long T = S->T;
  // (as the host's n_keys_r: with no open plan yet the newcomers' minimum
  // bucket is unknown but >= 0, so i + 2 bounds the key range)
  long long nk = 1 << 18;
  const long long mb = S->min_bucket == LLONG_MAX ? 0 : S->min_bucket;
  if (S->i + 2 - mb <= 512) nk = S->i + 2 - mb > 1 ? S->i + 2 - mb : 1;
  if (T <= 0 || nk > 512 || T + 1 > cap.T || S->n_plans + T + 1 > cap.arena || S->pool_n + T + 1 > cap.pool) {
    S->halt = 2;
    return;
  }
  S->n_keys = nk;
  S->rounds += 1;
  S->partial_plans += T;
}

// group size, its task count (task_off[G]) and the compacted pool size
__global__ void k_group_final(ExploreStatus* st, const int64_t* d_G, const int64_t* task_off,
                              const int64_t* stay_pos, const int64_t* d_pool_n, int64_t* d_T) {
  const int64_t G = *d_G;
  st->G = G;
  st->T = task_off[G];
  *d_T = task_off[G];
  st->pool_n = stay_pos[*d_pool_n];
}

// ======================================================================
// Cooperative round: one persistent launch per explore round.  Every phase
// after the expand (merge, relayout, RemoveDominated, pool append, bucket
// selection, frontier compaction and multisplit, task offsets) and the next
// round's task map run as grid-stride phases of one kernel separated by grid
// barriers, instead of ~25 launches of tiny kernels.  The phases are the
// per-item bodies of the kernels above (shared device functions where they
// are non-trivial), so both paths compute the same records.
struct GridBar {
  unsigned int count;
  unsigned int gen;
};

// all blocks are co-resident (cooperative launch): cooperative_groups' grid
// barrier (measured ~5% faster over a round than the sense-reversal barrier
// below, which PUMP_OWN_GRID_BAR builds keep)
__device__ __forceinline__ void grid_sync(GridBar* bar) {
#ifndef PUMP_OWN_GRID_BAR
  (void)bar;
  cooperative_groups::this_grid().sync();
  return;
#endif
  __syncthreads();
  if (threadIdx.x == 0) {
    volatile unsigned int* vgen = &bar->gen;
    const unsigned int g = *vgen;
    __threadfence();
    if (atomicAdd(&bar->count, 1u) == gridDim.x - 1) {
      bar->count = 0;
      __threadfence();
      atomicAdd(&bar->gen, 1u);
    } else {
      while (*vgen == g) __nanosleep(32);
    }
    __threadfence();
  }
  __syncthreads();
}

constexpr int kCoopBlock = kExpBlock;  // 256 (512 measured no faster: the phases are dependent-latency bound)
__device__ __forceinline__ int64_t block_sum(int64_t v, int64_t* red) {
  v = warp_sum(v);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) red[w] = v;
  __syncthreads();
  int64_t t = 0;
  for (int k = 0; k < kCoopBlock / 32; ++k) t += red[k];
  return t;
}

// exclusive scan across the block; *tot = block total
__device__ __forceinline__ int64_t block_excl(int64_t v, int64_t* red, int64_t* tot) {
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  const int64_t inc = warp_incl_scan(v);
  __syncthreads();
  if (l == 31) red[w] = inc;
  __syncthreads();
  int64_t before = 0, all = 0;
  for (int k = 0; k < kCoopBlock / 32; ++k) {
    const int64_t x = red[k];
    before += k < w ? x : 0;
    all += x;
  }
  *tot = all;
  return before + inc - v;
}

// Grid-wide exclusive scan of val(i) for i < n into out[0..n] (out[n] =
// total, written by the last block); post(i, excl, v) runs for every i.
// val(i, pass) is evaluated twice (pass 0: block reduce, pass 1: scan).
// Decoupled look-back across the co-resident blocks instead of a barrier:
// block b publishes its aggregate in status[b] tagged with the scan's epoch
// (every block writes its entry in every scan, so an entry with the current
// epoch is this scan's), then sums predecessors back to the nearest
// inclusive prefix.  The caller syncs the grid before reading out[] of
// other blocks.  Returns the total on the last block only (others: -1).
#ifndef PUMP_SCAN_ALLAGG
#define PUMP_SCAN_ALLAGG 1
#endif
#ifndef PUMP_SCAN_DIRECT
#define PUMP_SCAN_DIRECT 8192
#endif
constexpr int64_t kCoopScanDirect = PUMP_SCAN_DIRECT;  // scans up to this many items skip the look-back
template <class Val, class Post>
__device__ int64_t coop_scan(int64_t n, Val val, Post post, int64_t* out, unsigned long long* status, unsigned epoch,
                             int64_t* red, int64_t* s_pre) {
  constexpr unsigned long long kAgg = 1ull << 46, kInc = 2ull << 46, kVal = (1ull << 46) - 1;
  const unsigned long long tag = static_cast<unsigned long long>(epoch & 0xffffu) << 48;
  const int64_t nb = gridDim.x, b = blockIdx.x;
  const int64_t chunk = (n + nb - 1) / nb;
  const int64_t lo = min(n, b * chunk), hi = min(n, lo + chunk);
  // small scans: every block sums its predecessors' items itself (one batch
  // of independent loads) instead of waiting on the look-back chain
  const bool direct = n <= kCoopScanDirect;
  int64_t s = 0, pre_direct = 0;
  if (direct) {
    for (int64_t i = threadIdx.x; i < hi; i += blockDim.x) {
      const int64_t v = val(i, 0);
      if (i < lo) pre_direct += v;
      else s += v;
    }
    pre_direct = block_sum(pre_direct, red);
  } else {
    for (int64_t i = lo + threadIdx.x; i < hi; i += blockDim.x) s += val(i, 0);
  }
  s = block_sum(s, red);
  volatile unsigned long long* vs = status;
  // (a direct scan still writes its entry: every scan tags every entry, so a
  // stale entry can never carry the current epoch)
  if (direct && threadIdx.x == 0) vs[b] = tag | kInc | static_cast<unsigned long long>(pre_direct + s);
#if PUMP_SCAN_ALLAGG
  // all predecessors' aggregates at once, a thread per block (the grid is
  // co-resident and about one block per SM, so one wave of polling loads
  // replaces the look-back's chain of 32-wide windows)
  int64_t pre_all = 0;
  if (!direct) {
    if (threadIdx.x == 0) vs[b] = tag | kAgg | static_cast<unsigned long long>(s);
    int64_t acc = 0;
    for (int64_t j = threadIdx.x; j < b; j += blockDim.x) {
      unsigned long long w = vs[j];
      while ((w & (0xffffull << 48)) != tag || (w & (3ull << 46)) == 0) w = vs[j];
      acc += static_cast<int64_t>(w & kVal);
    }
    pre_all = block_sum(acc, red);
  }
#else
  const int64_t pre_all = 0;
  if (!direct && threadIdx.x < 32) {
    const int lane = threadIdx.x;
    int64_t pre = 0;
    if (b == 0) {
      if (lane == 0) vs[0] = tag | kInc | static_cast<unsigned long long>(s);
    } else {
      if (lane == 0) vs[b] = tag | kAgg | static_cast<unsigned long long>(s);
      int64_t j = b - 1 - lane;
      while (true) {
        unsigned long long w = j >= 0 ? vs[j] : (tag | kInc);
        auto ready = [&](unsigned long long x) { return (x & (0xffffull << 48)) == tag && (x & (3ull << 46)) != 0; };
        while (__any_sync(0xffffffffu, !ready(w))) {
          if (!ready(w)) w = vs[j];
        }
        const unsigned incm = __ballot_sync(0xffffffffu, (w & (3ull << 46)) == kInc);
        const int stop = incm ? __ffs(incm) - 1 : 31;
        int64_t v = lane <= stop ? static_cast<int64_t>(w & kVal) : 0;
        pre += warp_sum(v);
        if (incm) break;
        j -= 32;
      }
      if (lane == 0) vs[b] = tag | kInc | static_cast<unsigned long long>(pre + s);
    }
    if (lane == 0) *s_pre = pre;
  }
#endif
  __syncthreads();
  int64_t pre = direct ? pre_direct : PUMP_SCAN_ALLAGG ? pre_all : *s_pre;
  const int64_t total = pre + s;  // meaningful on the last block
  for (int64_t base = lo; base < hi; base += blockDim.x) {
    const int64_t i = base + threadIdx.x;
    const int64_t v = i < hi ? val(i, 1) : 0;
    int64_t tile = 0;
    const int64_t ex = block_excl(v, red, &tile);
    if (i < hi) {
      out[i] = pre + ex;
      post(i, pre + ex, v);
    }
    pre += tile;
  }
  if (b == nb - 1) {
    if (threadIdx.x == 0) out[n] = total;
    return total;
  }
  return -1;
}

struct CoopArgs {
  ExpandArgs ex;
  CommitArgs cm;
  int n;
  GridBar* bar;
  unsigned long long* scan_status;  // gridDim.x look-back words
  unsigned epoch;                   // per launch (tags the scans' status words)
  ExploreStatus* S;
  int64_t *d_K, *d_pool_n, *d_G, *d_T, *limits;
  // members: old layout (mem_off, old_ids) -> new layout (off2, new_ids)
  const int64_t* mem_off;
  int32_t* mem_cnt;
  int32_t* new_cnt;
  const int32_t* old_ids;
  int64_t* off2;
  int32_t* new_ids;
  const int32_t* new_slot;
  int32_t* touched;
  uint8_t *drop, *surv;
  int32_t* fpos;
  int64_t* spos;
  // pool and frontier
  int32_t* pool_cur;
  int32_t* pool_nxt;
  int32_t* keys;
  int64_t* stay_pos;
  int64_t n_keys;  // <= kCoopKeys
  int32_t* ms_counts;
  int64_t* ms_offs;
  int32_t* group;
  int64_t* task_off;
  int32_t* task_grp;
  int64_t* task_e;
  // > 0: the next round's task map (k_task_map's records) is written here for
  // every group entry whose tasks end below map_cap (the host skips
  // k_task_map when the next round runs gated with this capacity)
  int64_t map_cap;
  const int64_t* row_ptr;
  unsigned long long* stamps;  // optional phase timestamps (PUMP_DEBUG_COOP)
};
constexpr int kCoopKeys = 512;

union DomSmem {  // the warp pass and the block pass of the dom phase run one after the other
  DomShared blk;
  DomWarpShared warp[kCoopBlock / 32];
};

__global__ void __launch_bounds__(kCoopBlock, 2) k_round_tail(const CoopArgs A) {
  // the dom phase's staging and the multisplit's histograms never live at once
  __shared__ union {
    DomSmem dom;
    struct {
      int hist[kCoopKeys];
      int64_t run[kCoopKeys];
    } ms;
  } csm;
  DomSmem& dsm = csm.dom;
  DomShared& dsh = dsm.blk;
  DomWarpShared* wsh = dsm.warp;
  int* s_hist = csm.ms.hist;
  int64_t* s_run = csm.ms.run;
  __shared__ int64_t red[kCoopBlock / 32];
  __shared__ int64_t s_pre;
  __shared__ int64_t s_big[kCoopBlock];
  __shared__ int s_big_n;
  ExploreStatus* S = A.S;
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const int64_t gtid = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const int64_t gthreads = static_cast<int64_t>(gridDim.x) * blockDim.x;
  const int64_t gwarp = gtid >> 5, gwarps = gthreads >> 5;
  const int nb = gridDim.x;
  int stamp_i = 0;
  auto STAMP = [&]() {
    if (A.stamps && gtid == 0) {
      unsigned long long t;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      A.stamps[stamp_i] = t;
    }
    ++stamp_i;
  };
  pdl_wait();
  STAMP();
  if (S->halt) return;  // pipelined round that does not run (uniform: the gate ran before this launch)
  const int64_t n_keys = A.n_keys > 0 ? A.n_keys : S->n_keys;

  // (k_task_map and k_expand ran as their own launches before this one)
  const int64_t T = *A.d_T;
  (void)wib;
  // keep -> rank, commit as plan n_plans + rank
  const int64_t P0 = S->n_plans;
  const uint8_t* keep = A.cm.keep;
  unsigned ep = A.epoch * 8u;
  int64_t* rank = const_cast<int64_t*>(A.cm.rank);
  // and, in the same phase (expand already counted each node's newcomers),
  // the member relayout's new offsets: the second scan keeps its look-back
  // words in the upper half of scan_status (a block's entry for one scan may
  // still be polled while it posts the other)
  coop_scan(
      T, [&](int64_t i, int) -> int64_t { return keep[i]; },
      [&](int64_t i, int64_t ex, int64_t v) {
        if (v) commit_one(A.cm, i, ex);
      },
      rank, A.scan_status, ep++, red, &s_pre);
  const int n = A.n;
  coop_scan(
      n, [&](int64_t v, int) -> int64_t { return A.mem_cnt[v] + A.new_cnt[v]; }, [](int64_t, int64_t, int64_t) {},
      A.off2, A.scan_status + nb + 2, ep++, red, &s_pre);
  grid_sync(A.bar);
  const int64_t K = rank[T];
  if (gtid == 0) {
    S->K = K;
    *A.d_K = K;
    S->min_bucket = LLONG_MAX;
  }
  STAMP();
  STAMP();
  // a warp takes 32 consecutive nodes: each lane loads its node's segment
  // (one round trip for all 32) and copies a short segment itself; segments of
  // more than 8 members are then copied by the whole warp, one after another
  for (int64_t v0 = gwarp * 32; v0 < n; v0 += gwarps * 32) {
    const int64_t v = v0 + lane;
    int m = 0;
    int64_t a0 = 0, b0 = 0;
    if (v < n) {
      m = A.mem_cnt[v];
      a0 = A.mem_off[v];
      b0 = A.off2[v];
    }
    const bool small = m <= 8;
    if (small)
      for (int k = 0; k < m; ++k) A.new_ids[b0 + k] = A.old_ids[a0 + k];
    for (unsigned big = __ballot_sync(0xffffffffu, !small); big; big &= big - 1) {
      const int src = __ffs(big) - 1;
      const int mb = __shfl_sync(0xffffffffu, m, src);
      const int64_t ab = __shfl_sync(0xffffffffu, a0, src), bb = __shfl_sync(0xffffffffu, b0, src);
      for (int k = lane; k < mb; k += 32) A.new_ids[bb + k] = A.old_ids[ab + k];
    }
  }
  for (int64_t t = gtid; t < T; t += gthreads) {
    if (!keep[t]) continue;
    const int hv = A.cm.c_head[t];
    A.new_ids[A.off2[hv] + A.mem_cnt[hv] + A.new_slot[t]] = static_cast<int32_t>(P0 + rank[t]);
  }
  grid_sync(A.bar);
  STAMP();
  // RemoveDominated, block per touched node
  {
    const DomArgs D{A.touched, A.off2, A.mem_cnt, A.new_cnt, A.new_ids, A.cm.cost, A.cm.cp, A.cm.flags,
                    A.drop, A.surv, A.fpos, S};
    const int64_t nt = S->touched;
    // small nodes: a warp each; then nodes over kDomWarpCap: a block each
    for (int64_t b = gwarp; b < nt; b += gwarps) {
      const int v = A.touched[b];
      // classify by the pre-removal size off2[v+1] - off2[v]: it does not
      // change during this phase (mem_cnt / new_cnt of other warps' nodes do)
      if (A.off2[v + 1] - A.off2[v] <= kDomWarpCap) dom_node_warp(D, wsh[threadIdx.x >> 5], v, P0, lane);
    }
    __syncthreads();  // the block pass reuses the warps' shared memory
    // this block's touched nodes (b = blockIdx.x + k * nb) are classified by
    // all its threads at once and the big ones listed in shared memory: a
    // serial scan paid two dependent L2 round trips per touched node
    for (int64_t b0 = blockIdx.x; b0 < nt; b0 += static_cast<int64_t>(nb) * blockDim.x) {
      if (threadIdx.x == 0) s_big_n = 0;
      __syncthreads();
      const int64_t b = b0 + static_cast<int64_t>(threadIdx.x) * nb;
      if (b < nt) {
        const int v = A.touched[b];
        if (A.off2[v + 1] - A.off2[v] > kDomWarpCap) s_big[atomicAdd(&s_big_n, 1)] = b;
      }
      __syncthreads();
      const int nbig = s_big_n;
      for (int k = 0; k < nbig; ++k) dom_node(D, dsh, s_big[k], P0);  // nodes are independent: any order
      __syncthreads();
    }
  }
  grid_sync(A.bar);
  STAMP();
  // surviving newcomers -> open pool (id order); lowest open bucket
  const int64_t pool_old = S->pool_n;
  const int32_t* bucket = A.cm.bucket;
  uint8_t* flags = A.cm.flags;
  // (bucket extremes reduced per thread, then per warp: one atomic per warp
  // instead of one per plan on a single address)
  int b_min = INT_MAX, b_max = INT_MIN;
  coop_scan(
      K, [&](int64_t r, int) -> int64_t { return A.surv[r]; },
      [&](int64_t r, int64_t ex, int64_t v) {
        if (v) {
          const int64_t id = P0 + r;
          A.pool_cur[pool_old + ex] = static_cast<int32_t>(id);
          flags[id] |= kOpen;
          b_max = max(b_max, bucket[id]);
          b_min = min(b_min, bucket[id]);
        }
      },
      A.spos, A.scan_status, ep++, red, &s_pre);
  for (int64_t x = gtid; x < pool_old; x += gthreads) {
    const int id = A.pool_cur[x];
    if (flags[id] & kOpen) b_min = min(b_min, bucket[id]);
  }
  b_min = __reduce_min_sync(0xffffffffu, b_min);
  b_max = __reduce_max_sync(0xffffffffu, b_max);
  if (lane == 0) {
    if (b_min != INT_MAX) atomicMin(&S->min_bucket, static_cast<long long>(b_min));
    if (b_max != INT_MIN) atomicMax(&S->max_bucket, static_cast<long long>(b_max));
  }
  grid_sync(A.bar);
  STAMP();
  // end-of-round bookkeeping and the next threshold (k_round_i): every
  // thread derives the values the selection needs from the status (final
  // after the barrier above); thread 0 records them after the next barrier,
  // when no block reads the old ones any more
  const int64_t NS = A.spos[K];
  const long long pool_n_new = S->pool_n + NS;
  const long long min_b = S->min_bucket, max_b = S->max_bucket;
  long long i_new = S->i + 1;
  if (min_b != LLONG_MAX && min_b > i_new) i_new = min_b;
  const long long lim0 = i_new < max_b ? i_new : max_b, lim1 = min_b == LLONG_MAX ? 0 : min_b;
  const long long open_new = S->open_count + NS - S->evicted_open - S->G, n_plans_new = S->n_plans + K;
  STAMP();
  // bucket selection (k_select) fused into the stay scan; stayers compacted;
  // the multisplit's per-block key histogram over the scan's own chunk
  const int64_t m = pool_n_new;
  const int nk = static_cast<int>(n_keys);
  for (int k = threadIdx.x; k < nk; k += blockDim.x) s_hist[k] = 0;
  __syncthreads();
  coop_scan(
      m,
      [&](int64_t x, int pass) -> int64_t {
        const int id = A.pool_cur[x];
        const bool open = flags[id] & kOpen;
        const int b = bucket[id];
        const bool sel = open && b <= lim0;
        if (pass) {
          const int64_t key = b - lim1;
          if (sel && key >= n_keys) atomicExch(reinterpret_cast<unsigned long long*>(&S->err), 3ull);
          A.keys[x] = sel ? static_cast<int32_t>(key) : -1;
          if (sel && key < n_keys) atomicAdd(&s_hist[key], 1);
        }
        return (open && !sel) ? 1 : 0;
      },
      [&](int64_t x, int64_t ex, int64_t v) {
        if (v) A.pool_nxt[ex] = A.pool_cur[x];
      },
      A.stay_pos, A.scan_status, ep++, red, &s_pre);
  __syncthreads();
  for (int k = threadIdx.x; k < nk; k += blockDim.x) A.ms_counts[static_cast<int64_t>(k) * nb + blockIdx.x] = s_hist[k];
  grid_sync(A.bar);
  const int64_t stay_n = A.stay_pos[m];
  if (gtid == 0) {
    S->n_surv = NS;
    S->pool_n = pool_n_new;
    S->open_count = open_new;
    S->n_plans = n_plans_new;
    S->i = i_new;
    A.limits[0] = lim0;
    A.limits[1] = lim1;
    *A.d_pool_n = pool_n_new;
    S->G = 0;
    S->T = 0;
    S->min_group_bits = 0x7ff0000000000000ll;
    S->touched = 0;
    S->evicted_open = 0;
  }
  STAMP();
  // stable multisplit by key (one radix pass, keys < n_keys <= 512): the
  // per-block histograms (above, over the scan's contiguous chunks), key-major
  // scan, ordered scatter
  const int64_t chunk = (m + nb - 1) / nb;
  const int64_t lo = min(m, static_cast<int64_t>(blockIdx.x) * chunk), hi = min(m, lo + chunk);
  STAMP();
  int64_t Gn = 0;
  if (nk <= 32) {
    // few keys: each block derives its own run starts (key k's total over the
    // blocks and the part before this block, then the keys' exclusive scan)
    // from the counts directly, with no grid-wide scan and barrier
    __shared__ int64_t s_ktot[32], s_kpre[32], s_gn;
    for (int k = wib; k < nk; k += kCoopBlock / 32) {
      int64_t tot = 0, pre = 0;
      for (int b2 = lane; b2 < nb; b2 += 32) {
        const int cnt = A.ms_counts[static_cast<int64_t>(k) * nb + b2];
        tot += cnt;
        pre += b2 < static_cast<int>(blockIdx.x) ? cnt : 0;
      }
      tot = warp_sum(tot);
      pre = warp_sum(pre);
      if (lane == 0) {
        s_ktot[k] = tot;
        s_kpre[k] = pre;
      }
    }
    __syncthreads();
    if (wib == 0) {
      const int64_t t = lane < nk ? s_ktot[lane] : 0;
      const int64_t inc = warp_incl_scan(t);
      if (lane < nk) s_run[lane] = inc - t + s_kpre[lane];
      if (lane == 31) s_gn = inc;
    }
    __syncthreads();
    Gn = s_gn;
  } else {
    coop_scan(
        static_cast<int64_t>(nk) * nb, [&](int64_t i, int) -> int64_t { return A.ms_counts[i]; },
        [](int64_t, int64_t, int64_t) {}, A.ms_offs, A.scan_status, ep++, red, &s_pre);
    grid_sync(A.bar);
    Gn = A.ms_offs[static_cast<int64_t>(nk) * nb];
    for (int k = threadIdx.x; k < nk; k += blockDim.x) s_run[k] = A.ms_offs[static_cast<int64_t>(k) * nb + blockIdx.x];
    __syncthreads();
  }
  STAMP();
  if (wib == 0) {
    const unsigned lt = (1u << lane) - 1u;
    for (int64_t base = lo; base < hi; base += 32) {
      const int64_t x = base + lane;
      const int key = x < hi ? A.keys[x] : -1;
      const unsigned peers = __match_any_sync(0xffffffffu, key);
      const int rank = __popc(peers & lt);
      if (key >= 0) A.group[s_run[key] + rank] = A.pool_cur[x];
      __syncwarp();
      if (key >= 0 && rank == __popc(peers) - 1) s_run[key] += __popc(peers);
      __syncwarp();
    }
  }
  if (gtid == 0) *A.d_G = Gn;
  grid_sync(A.bar);
  STAMP();
  // the new group: close it, its degrees -> task offsets, cheapest cost
  long long g_min = LLONG_MAX;  // (the costs are non-negative: their bits order like the values)
  const int64_t Tn_last = coop_scan(
      Gn,
      [&](int64_t g, int pass) -> int64_t {
        const int id = A.group[g];
        const int hv = A.ex.head[id];
        if (pass) {
          flags[id] &= static_cast<uint8_t>(~kOpen);
          const long long cb = __double_as_longlong(A.cm.cost[id]);
          g_min = cb < g_min ? cb : g_min;
        }
        return A.row_ptr[hv + 1] - A.row_ptr[hv];
      },
      [&](int64_t g, int64_t t0, int64_t deg) {
        // the next round's task map (as k_task_map): task t of entry g is
        // (its plan, the edge row_ptr[head] + t - t0)
        if (t0 + deg + 1 > A.map_cap) return;
        const int id = A.group[g];
        const int64_t e0 = A.row_ptr[A.ex.head[id]];
        for (int64_t k = 0; k < deg; ++k) {
          A.task_grp[t0 + k] = id;
          A.task_e[t0 + k] = e0 + k;
        }
      },
      A.task_off, A.scan_status, ep++, red, &s_pre);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const long long t = __shfl_xor_sync(0xffffffffu, g_min, o);
    g_min = t < g_min ? t : g_min;
  }
  if (lane == 0 && g_min != LLONG_MAX) atomicMin(&S->min_group_bits, g_min);
  if (blockIdx.x == gridDim.x - 1 && threadIdx.x == 0) {  // the scan's last block holds the total
    S->G = Gn;
    S->T = Tn_last;
    *A.d_T = Tn_last;
    S->pool_n = stay_n;
    // algorithmic bytes of the round (see the host's per-round formula)
    const long long Wd = A.cm.W;
    S->commit_bytes += T * (37 + 8 * Wd) + K * (33 + 8 * Wd) + static_cast<long long>(n) * 16 + (pool_old + K) * 9 +
                       Gn * 28;
  }
  STAMP();
}

// per bank row t: the particles' per-axis box lo[DW], hi[DW] (expand's no-kill test)
__global__ void __launch_bounds__(128) k_bank_box(const double* __restrict__ dy, int n, int dw,
                                                  double* __restrict__ box) {
  const int t = blockIdx.x;
  __shared__ double s_lo[128][3], s_hi[128][3];
  double lo[3] = {__builtin_inf(), __builtin_inf(), __builtin_inf()}, hi[3] = {-lo[0], -lo[1], -lo[2]};
  for (int i = threadIdx.x; i < n; i += blockDim.x)
    for (int k = 0; k < dw; ++k) {
      const double v = dy[(static_cast<int64_t>(t) * n + i) * dw + k];
      lo[k] = v < lo[k] ? v : lo[k];
      hi[k] = v > hi[k] ? v : hi[k];
    }
  for (int k = 0; k < 3; ++k) {
    s_lo[threadIdx.x][k] = lo[k];
    s_hi[threadIdx.x][k] = hi[k];
  }
  __syncthreads();
  if (threadIdx.x < dw) {
    const int k = threadIdx.x;
    double a = __builtin_inf(), b = -__builtin_inf();
    for (int x = 0; x < static_cast<int>(blockDim.x); ++x) {
      a = s_lo[x][k] < a ? s_lo[x][k] : a;
      b = s_hi[x][k] > b ? s_hi[x][k] : b;
    }
    box[static_cast<int64_t>(t) * 2 * dw + k] = a;
    box[static_cast<int64_t>(t) * 2 * dw + dw + k] = b;
  }
}

static void swap_buf(DBuf& a, DBuf& b) {
  std::swap(a.p, b.p);
  std::swap(a.cap, b.cap);
}

// ------------------------------------------------------------------ host
static inline size_t al(size_t x) { return (x + 255) & ~size_t(255); }

// keep_all: a round in flight may commit plans past X.n_plans, keep them all
static void ensure_arena(DevExplore& X, int64_t need, cudaStream_t st, bool keep_all = false) {
  if (need <= X.cap) return;
  int64_t cap = X.cap ? X.cap : 1 << 16;
  while (cap < need) cap += cap / 2 + 1024;
  const int64_t old = keep_all ? X.cap : X.n_plans;
  X.head.grow(al(cap * 4), old * 4, st);
  X.parent.grow(al(cap * 4), old * 4, st);
  X.cost.grow(al(cap * 8), old * 8, st);
  X.cp.grow(al(cap * 8), old * 8, st);
  X.t_end.grow(al(cap * 4), old * 4, st);
  X.mask.grow(al(cap * X.W * 8), old * X.W * 8, st);
  X.bucket.grow(al(cap * 4), old * 4, st);
  X.flags.grow(al(cap), old, st);
  // member segments and the pool hold at most every plan once
  X.mem_a.grow(al((cap + 16) * 4), X.mem_a.cap, st);
  X.mem_b.grow(al((cap + 16) * 4), X.mem_b.cap, st);
  X.pool_a.grow(al((cap + 16) * 4), X.pool_a.cap, st);
  X.pool_b.grow(al((cap + 16) * 4), X.pool_b.cap, st);
  X.cap = cap;
}

template <class T>
static T* ptr(DBuf& b) {
  return b.as<T>();
}

__global__ void k_explore_init(int n, int W, int N, int ng, const int32_t* __restrict__ goal_sorted,
                               int64_t* __restrict__ mem_off, int32_t* __restrict__ mem_cnt, int32_t* __restrict__ new_cnt,
                               uint8_t* __restrict__ is_goal, int32_t* head, int32_t* parent, double* cost, double* cp,
                               int32_t* t_end, int32_t* bucket, uint64_t* mask, uint8_t* flags, int32_t* mem_a,
                               int32_t* group, const int64_t* __restrict__ row_ptr, ExploreStatus h0,
                               ExploreStatus* S, int64_t* d_scal, int64_t* task_off) {
  const int v = blockIdx.x * blockDim.x + threadIdx.x;
  if (v <= n) mem_off[v] = v == 0 ? 0 : 1;  // pareto[0] = {0}: node 0's segment holds one entry
  if (v < n) {
    mem_cnt[v] = v == 0 ? 1 : 0;
    new_cnt[v] = 0;
    int lo = 0, hi = ng;  // v in the ascending goal list?
    while (lo < hi) {
      const int mid = (lo + hi) >> 1;
      if (goal_sorted[mid] < v)
        lo = mid + 1;
      else
        hi = mid;
    }
    is_goal[v] = (lo < ng && goal_sorted[lo] == v) ? 1 : 0;
  }
  if (v == 0) {
    head[0] = 0;
    parent[0] = -1;
    cost[0] = 0.0;
    cp[0] = 0.0;
    t_end[0] = 0;
    bucket[0] = 0;
    for (int w = 0; w < W; ++w)
      mask[w] = (w == W - 1 && N % 64) ? (1ull << (N % 64)) - 1 : ~0ull;
    flags[0] = 0;
    mem_a[0] = 0;
    group[0] = 0;
    const int64_t T0 = row_ptr[1] - row_ptr[0];
    h0.T = T0;
    *S = h0;
    task_off[0] = 0;
    task_off[1] = T0;
    d_scal[0] = 0;
    d_scal[1] = 0;
    d_scal[2] = 1;
    d_scal[3] = T0;
  }
}

// a round's kernels after the first: programmatic stream serialization (see
// pdl_wait), plus the cooperative attribute for the round tail
template <class... KArgs, class... Args>
static void launch_round(void (*k)(KArgs...), dim3 grid, dim3 block, cudaStream_t st, bool coop, Args&&... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = 0;
  cfg.stream = st;
  cudaLaunchAttribute at[2];
  int na = 0;
#ifndef PUMP_NO_PDL
  at[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[na].val.programmaticStreamSerializationAllowed = 1;
  ++na;
#endif
  if (coop) {
    at[na].id = cudaLaunchAttributeCooperative;
    at[na].val.cooperative = 1;
    ++na;
  }
  cfg.attrs = at;
  cfg.numAttrs = na;
  PUMP_CUDA(cudaLaunchKernelEx(&cfg, k, std::forward<Args>(args)...));
}

void run_explore_device(DevExplore& X, Ctx& c, const DevGraph& G, const ExploreArgs& prm) {
  if (!c.bank.p) throw std::invalid_argument("explore: no particle bank in this context");
  if (c.bank_dw != G.dw) throw std::invalid_argument("explore: bank / graph dimension mismatch");
  cudaStream_t st = c.stream;
  const int n = G.n, N = c.bank_n, W = (N + 63) / 64;
  X.n = n;
  X.N = N;
  X.W = W;
  // lanes hold CH chunks of 32 particles; above 512 particles a warp runs
  // its task slab by slab (expand_task)
  const int ch = [&] {
    int q = (N + 31) / 32, p = 1;
    while (p < q && p < 16) p <<= 1;
    return p;
  }();
  // particle box of every bank row (k_expand skips rows no half-space can cut)
  DBuf& box = c.buf("x_bank_box", al(static_cast<size_t>(c.bank_horizon + 2) * 2 * G.dw * 8));
  k_bank_box<<<c.bank_horizon + 1, 128, 0, st>>>(c.bank.as<double>(), N, G.dw, box.as<double>());
  ++c.launches;
  X.n_plans = 0;  // buffers (and their capacity) persist across solves
  const int count_hs = (kprof_current() && kprof_current()->on) ? 1 : 0;
  ensure_arena(X, 1 << 16, st);
  if (!X.status_h) PUMP_CUDA(cudaMallocHost(&X.status_h, 3 * sizeof(ExploreStatus)));
  for (cudaEvent_t& e : X.status_ev)
    if (!e) PUMP_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  X.status_d.ensure(al(sizeof(ExploreStatus)) + 256);
  ExploreStatus* S = X.status_d.as<ExploreStatus>();
  int64_t* d_scal = reinterpret_cast<int64_t*>(reinterpret_cast<char*>(X.status_d.p) + al(sizeof(ExploreStatus)));
  // d_scal: [0] K, [1] pool_n, [2] G, [3] T, [4..5] limits
  int64_t* d_K = d_scal + 0;
  int64_t* d_pool_n = d_scal + 1;
  int64_t* d_G = d_scal + 2;
  int64_t* d_T = d_scal + 3;
  int64_t* d_limits = d_scal + 4;

  // per-node state
  X.mem_off.ensure(al((n + 1) * 8));
  X.mem_cnt.ensure(al(n * 4));
  X.new_cnt.ensure(al(n * 4));
  X.is_goal.ensure(al(n));
  X.touched.ensure(al(n * 4));
  DBuf& node_sz = c.buf("x_node_sz", al(n * 4));
  DBuf& off2 = c.buf("x_off2", al((n + 1) * 8));
  std::vector<int32_t> goal_sorted(G.goal_nodes);  // (an uploaded graph's list may come in any order)
  std::sort(goal_sorted.begin(), goal_sorted.end());
  const bool root_goal = n > 0 && !goal_sorted.empty() && goal_sorted[0] == 0;
  ExploreStatus h{};
  h.G = 1;
  h.n_plans = 1;
  h.open_count = 1;
  h.i = 0;
  h.max_bucket = 0;
  h.min_bucket = LLONG_MAX;
  h.pool_n = 0;
  h.best_goal_bits = root_goal && 0.0 < prm.alpha_min ? 0ll : 0x7ff0000000000000ll;
  h.min_group_bits = 0;  // root cost 0
  // the initial state in one kernel (root plan, planner.hpp:100-103; node 0's
  // member segment {0}; is_goal; group [0]; the first round's task count)
  X.group.ensure(al(64 * 4));
  X.task_off.ensure(al(64 * 8));
  X.mem_flip = false;
  {
    const int ng = static_cast<int>(goal_sorted.size());
    DBuf& gl = c.buf("x_goal_list", al((ng + 1) * 4));
    if (ng) c.h2d(gl.p, goal_sorted.data(), ng * 4);
    k_explore_init<<<grid_for(n + 1, 256), 256, 0, st>>>(
        n, W, N, ng, gl.as<int32_t>(), X.mem_off.as<int64_t>(), X.mem_cnt.as<int32_t>(), X.new_cnt.as<int32_t>(),
        X.is_goal.as<uint8_t>(), X.head.as<int32_t>(), X.parent.as<int32_t>(), X.cost.as<double>(),
        X.cp.as<double>(), X.t_end.as<int32_t>(), X.bucket.as<int32_t>(), X.mask.as<uint64_t>(),
        X.flags.as<uint8_t>(), X.mem_a.as<int32_t>(), X.group.as<int32_t>(), G.row_ptr.as<int64_t>(), h, S, d_scal,
        X.task_off.as<int64_t>());
    ++c.launches;
  }
  int64_t T0 = 0;  // the host sizes the first round by it
  c.d2h(&T0, d_scal + 3, 8);
  c.sync();
  h.T = T0;
  X.partial_plans = 0;
  X.rounds = 0;
  X.pool_flip = false;
  const double width = prm.lambda * prm.r_n;

  // cooperative round kernel for this (dw, particle-words) instance
  const void* coop_fn = reinterpret_cast<const void*>(&k_round_tail);
  int coop_blocks = 0;
  {
    int per_sm = 0, sms = 0, coop_attr = 0;
    PUMP_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, coop_fn, kCoopBlock, 0));
    per_sm = std::min(per_sm, 1);  // one block per SM: cheaper grid barriers (2 per SM measured within noise)
    PUMP_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, c.device));
    PUMP_CUDA(cudaDeviceGetAttribute(&coop_attr, cudaDevAttrCooperativeLaunch, c.device));
    coop_blocks = coop_attr ? per_sm * sms : 0;
  }
  const bool coop_ok = coop_blocks > 0;
  if (coop_ok) {  // look-back status words start untagged
    DBuf& scan_st = c.buf("x_coop_scan_status", al((2 * coop_blocks + 4) * 8));
    PUMP_CUDA(cudaMemsetAsync(scan_st.p, 0, (2 * coop_blocks + 4) * 8, st));
  }
  // Pipelined rounds: with the cooperative path and no round hook, batches of
  // kBatch rounds are enqueued behind device-side gates (k_round_gate) and the
  // status is read once per batch; buffers are sized for Tcap tasks per round
  // and a round that does not fit (or needs the per-kernel path) halts the
  // batch, after which the host runs that round synchronously.
  constexpr int kBatch = 8;
  bool force_sync = false;
  int64_t max_T = 0;
  long long commit_bytes_legacy = 0;
  c.tic();
  ExploreStatus h_hook{};
  bool hook_pending = false;
  // Window (per-round hook, run_pump): gated rounds as in a batch, but the
  // host keeps one round in flight and consumes the status of the round
  // before it (copied into a pinned slot behind that round), so the device
  // never idles while the host reads a status, runs the hook and enqueues the
  // next round.  A halt (termination or capacity) stops the window: the round
  // in flight halts too and is drained before the host goes on.
  const bool window = coop_ok && kBatch > 1 && prm.on_round && !prm.on_round_batched && !prm.on_round_state;
  bool inflight = false;
  int in_slot = 0, next_slot = 0;
  // a gated round's status: rounds that ran, undo the flips of one that did
  // not, clear a halt; true when the round (or an earlier one) halted
  auto win_consume = [&](const ExploreStatus& hs) {
    const ExploreStatus hp = h;
    h = hs;
    X.n_plans = h.n_plans;
    if (h.err) throw std::runtime_error("explore: device error " + std::to_string(h.err));
    const long long ran = h.rounds - hp.rounds;
    if (ran == 0) {
      swap_buf(X.mem_off, off2);
      X.mem_flip = !X.mem_flip;
      X.pool_flip = !X.pool_flip;
    }
    X.rounds += static_cast<int>(ran);
    X.partial_plans += h.partial_plans - hp.partial_plans;
    bool halted = false;
    if (h.halt) {
      static const bool dbg_w = std::getenv("PUMP_DEBUG_TIMING") != nullptr;
      if (dbg_w) std::fprintf(stderr, "[pump w] window halt %lld after round %lld\n", h.halt, h.rounds);
      if (h.halt == 2) force_sync = true;
      h.halt = 0;
      const long long zero = 0;
      c.h2d(&S->halt, &zero, 8);
      halted = true;
    }
    prm.on_round(h);
    return halted;
  };
  struct MapPrev {
    int64_t cap;
    const void* grp;
    const void* e;
  };
  MapPrev map_prev{0, nullptr, nullptr};  // the last cooperative launch's task-map capacity and buffers
  auto win_drain = [&]() {
    PUMP_CUDA(cudaEventSynchronize(X.status_ev[in_slot]));
    win_consume(X.status_h[1 + in_slot]);
    inflight = false;
  };
  for (;;) {
    // loop-top termination (planner.hpp:126-138); h is the status after the
    // previous collection
    const double best_goal = __builtin_bit_cast(double, h.best_goal_bits);
    const double min_group = __builtin_bit_cast(double, h.min_group_bits);
    if (h.G > 0 && best_goal != __builtin_inf() && best_goal <= min_group) {
      if (inflight) {  // (its gate halts it: drain, then decide on its status)
        win_drain();
        continue;
      }
      X.termination = 0;
      break;
    }
    if (h.G == 0 && h.open_count == 0) {
      if (inflight) {
        win_drain();
        continue;
      }
      X.termination = best_goal == __builtin_inf() ? 1 : 0;
      break;
    }
    const int64_t Th = h.T;
    max_T = std::max<int64_t>(max_T, Th);
    const bool pipe = coop_ok && kBatch > 1 && (!prm.on_round || prm.on_round_batched || window) &&
                      !prm.on_round_state && !force_sync;
    const bool win = window && pipe;
    std::vector<int32_t> expanded;  // (round hook) this round's group
    if (prm.on_round_state) {
      expanded.resize(h.G);
      if (h.G > 0) c.d2h(expanded.data(), X.group.p, h.G * 4);
      c.sync();
    }
    force_sync = false;
    // buffer sizes: this round's T, or a per-round capacity for a batch
    const int64_t T = pipe ? std::max<int64_t>({Th, 2 * max_T, 4096}) : Th;
    const int64_t nrounds = win ? 1 : pipe ? kBatch : 1;
    const int64_t ahead = win ? 2 : nrounds;  // rounds past the status h the buffers must hold
    if (!pipe) {
      X.rounds++;
      X.partial_plans += Th;
    }
    ensure_arena(X, X.n_plans + (win ? 2 * T : pipe ? kBatch * T / 2 : T) + 1, st, inflight);
    // candidate buffers
    X.cand_keep.ensure(al(T + 1));
    X.cand_head.ensure(al((T + 1) * 4));
    X.cand_src.ensure(al((T + 1) * 4));
    X.cand_tend.ensure(al((T + 1) * 4));
    X.cand_cost.ensure(al((T + 1) * 8));
    X.cand_cp.ensure(al((T + 1) * 8));
    X.cand_mask.ensure(al((T + 1) * W * 8));
    X.cand_rank.ensure(al((T + 2) * 8));
    X.new_slot.ensure(al((T + 1) * 4));
    X.drop.ensure(al(T + 1));
    X.surv.ensure(al(T + 1));
    X.fpos.ensure(al((T + 1) * 4));
    DBuf& spos = c.buf("x_spos", al((T + 2) * 8));
    DBuf& stmp = c.buf("x_scan_tmp", scan_temp_bytes(std::max<int64_t>({T, n, X.cap}) + 16));

    // distinct bucket keys of the next selection (see k_select): <= i + 2 -
    // min_bucket; with no open plan yet (the first round) the newcomers'
    // minimum is unknown but >= 0 (buckets are clamped at 0), so i + 2 bounds it
    int64_t n_keys_r = 1 << 18;
    const long long mb = h.min_bucket == LLONG_MAX ? 0 : h.min_bucket;
    if (h.i + 2 - mb <= 512) n_keys_r = std::max<int64_t>(1, h.i + 2 - mb);
    bool ran_coop = false;
    if (pipe || (coop_ok && T > 0 && n_keys_r <= kCoopKeys)) {
     ran_coop = true;
     const long long rounds0 = h.rounds;  // (pipelined: the status counts the rounds that ran)
     const int64_t pool_ub = h.pool_n + (pipe ? ahead * T : T) + 1;
     for (int64_t rr = 0; rr < nrounds; ++rr) {
      // ---- one cooperative launch for the whole round
      if (pipe) {
        const GateCaps caps{T, X.cap, pool_ub};
        launch_round(k_round_gate, dim3(1), dim3(1), st, false, S, caps);
        ++c.launches;
      }
      X.task_grp.ensure(al((T + 1) * 4));
      X.task_e.ensure(al((T + 1) * 8));
      // (a round in flight may be writing the next group: keep everything)
      X.group.grow(al((pool_ub + 1) * 4), inflight ? X.group.cap : static_cast<size_t>(h.G) * 4, st);
      X.task_off.grow(al((pool_ub + 2) * 8), inflight ? X.task_off.cap : static_cast<size_t>(h.G + 1) * 8, st);
      DBuf& keys = c.buf("x_sel_keys", al((pool_ub + 1) * 4));
      DBuf& stay_pos = c.buf("x_stay_pos", al((pool_ub + 2) * 8));
      DBuf& msc = c.buf("x_coop_counts", al(static_cast<size_t>(kCoopKeys) * coop_blocks * 4));
      DBuf& mso = c.buf("x_coop_offs", al((static_cast<size_t>(kCoopKeys) * coop_blocks + 2) * 8));
      DBuf& scan_st = c.buf("x_coop_scan_status", al((2 * coop_blocks + 4) * 8));
      DBuf& bar = c.buf("x_coop_bar", 256);
      DBuf& old_ids = X.mem_flip ? X.mem_b : X.mem_a;
      DBuf& new_ids = X.mem_flip ? X.mem_a : X.mem_b;
      DBuf& pool_cur = X.pool_flip ? X.pool_b : X.pool_a;
      DBuf& pool_nxt = X.pool_flip ? X.pool_a : X.pool_b;
#ifdef PUMP_OWN_GRID_BAR
      PUMP_CUDA(cudaMemsetAsync(bar.p, 0, 8, st));  // (the cooperative-groups barrier needs no state)
#endif
      CoopArgs A{};
      A.ex = ExpandArgs{X.group.as<int32_t>(), X.task_off.as<int64_t>(), X.task_grp.as<int32_t>(), X.task_e.as<int64_t>(), d_G, d_T,
                        G.row_ptr.as<int64_t>(), G.e_to.as<int32_t>(), G.e_cost.as<double>(),
                        G.e_nsteps.as<int32_t>(), G.wp_off.as<int64_t>(), G.hs_off.as<int64_t>(),
                        G.hs_cnt.as<int32_t>(), G.hs_pk.as<double>(), X.head.as<int32_t>(), X.cost.as<double>(),
                        X.t_end.as<int32_t>(), X.mask.as<uint64_t>(), c.bank.as<double>(), box.as<double>(), N,
                        c.bank_horizon, W, count_hs,
                        prm.alpha_max, X.cand_keep.as<uint8_t>(), X.cand_head.as<int32_t>(),
                        X.cand_src.as<int32_t>(), X.cand_tend.as<int32_t>(), X.cand_cost.as<double>(),
                        X.cand_cp.as<double>(), X.cand_mask.as<uint64_t>(), S,
                        X.new_cnt.as<int32_t>(), X.new_slot.as<int32_t>(), X.touched.as<int32_t>()};
      A.cm = CommitArgs{d_T, X.cand_keep.as<uint8_t>(), X.cand_rank.as<int64_t>(), X.cand_head.as<int32_t>(),
                        X.cand_src.as<int32_t>(), X.cand_tend.as<int32_t>(), X.cand_cost.as<double>(),
                        X.cand_cp.as<double>(), X.cand_mask.as<uint64_t>(), W, width, prm.alpha_min,
                        X.is_goal.as<uint8_t>(), X.head.as<int32_t>(), X.parent.as<int32_t>(), X.cost.as<double>(),
                        X.cp.as<double>(), X.t_end.as<int32_t>(), X.mask.as<uint64_t>(), X.bucket.as<int32_t>(),
                        X.flags.as<uint8_t>(), X.new_cnt.as<int32_t>(), X.new_slot.as<int32_t>(),
                        X.touched.as<int32_t>(), S};
      A.n = n;
      A.bar = bar.as<GridBar>();
      A.scan_status = scan_st.as<unsigned long long>();
      A.epoch = ++X.coop_epoch;
      A.S = S;
      A.d_K = d_K;
      A.d_pool_n = d_pool_n;
      A.d_G = d_G;
      A.d_T = d_T;
      A.limits = d_limits;
      A.mem_off = X.mem_off.as<int64_t>();
      A.mem_cnt = X.mem_cnt.as<int32_t>();
      A.new_cnt = X.new_cnt.as<int32_t>();
      A.old_ids = old_ids.as<int32_t>();
      A.off2 = off2.as<int64_t>();
      A.new_ids = new_ids.as<int32_t>();
      A.new_slot = X.new_slot.as<int32_t>();
      A.touched = X.touched.as<int32_t>();
      A.drop = X.drop.as<uint8_t>();
      A.surv = X.surv.as<uint8_t>();
      A.fpos = X.fpos.as<int32_t>();
      A.spos = spos.as<int64_t>();
      A.pool_cur = pool_cur.as<int32_t>();
      A.pool_nxt = pool_nxt.as<int32_t>();
      A.keys = keys.as<int32_t>();
      A.stay_pos = stay_pos.as<int64_t>();
      A.n_keys = pipe ? 0 : n_keys_r;  // pipelined: the gate's value in the status
      A.ms_counts = msc.as<int32_t>();
      A.ms_offs = mso.as<int64_t>();
      A.group = X.group.as<int32_t>();
      A.task_off = X.task_off.as<int64_t>();
      A.task_grp = X.task_grp.as<int32_t>();
      A.task_e = X.task_e.as<int64_t>();
      A.map_cap = T;
      A.row_ptr = G.row_ptr.as<int64_t>();
      static const bool dbg_coop = std::getenv("PUMP_DEBUG_COOP") != nullptr;
      DBuf& stamps = c.buf("x_coop_stamps", 64 * 8);
      A.stamps = dbg_coop ? stamps.as<unsigned long long>() : nullptr;
      const int64_t grid_cap = static_cast<int64_t>(coop_blocks) * 8;
      // the previous cooperative round wrote this round's task map when it
      // fit its capacity; a gated round with that same capacity (and the same
      // buffers) either fits it or halts at its gate
      const bool map_ready = pipe && map_prev.cap == T && map_prev.grp == X.task_grp.p && map_prev.e == X.task_e.p;
      map_prev = MapPrev{T, X.task_grp.p, X.task_e.p};
      if (!map_ready) launch_round(k_task_map,
                   dim3(pipe ? static_cast<unsigned>(std::min<int64_t>(grid_for(pool_ub * 32, 256), grid_cap))
                             : grid_for(h.G * 32, 256)),
                   dim3(256), st, false, static_cast<const int64_t*>(d_G), X.task_off.as<int64_t>(),
                   X.group.as<int32_t>(), X.head.as<int32_t>(), G.row_ptr.as<int64_t>(), X.task_grp.as<int32_t>(),
                   X.task_e.as<int64_t>(), static_cast<const ExploreStatus*>(S));
      if (!map_ready) ++c.launches;
      {
        const unsigned grid = grid_for(T * 32, 256);  // pipelined: T is the per-round task capacity
        KScope ks(st, F_EXPAND);
        dispatch_dw(G.dw, [&]<int DW>() {
          switch (ch) {
            case 1: launch_round(k_expand<DW, 1>, dim3(grid), dim3(256), st, false, A.ex); break;
            case 2: launch_round(k_expand<DW, 2>, dim3(grid), dim3(256), st, false, A.ex); break;
            case 4: launch_round(k_expand<DW, 4>, dim3(grid), dim3(256), st, false, A.ex); break;
            case 8: launch_round(k_expand<DW, 8>, dim3(grid), dim3(256), st, false, A.ex); break;
            default: launch_round(k_expand<DW, 16>, dim3(grid), dim3(256), st, false, A.ex); break;
          }
        });
        ++c.launches;
      }
      {
        KScope ks(st, F_COMMIT);
        launch_round(k_round_tail, dim3(coop_blocks), dim3(kCoopBlock), st, true, A);
      }
      ++c.launches;
      PUMP_CUDA(cudaGetLastError());
      if (dbg_coop) {
        unsigned long long ts[32];
        c.d2h(ts, stamps.p, sizeof(ts));
        c.sync();
        std::fprintf(stderr, "[coop] T=%lld", (long long)T);
        for (int q = 1; q < 16; ++q) std::fprintf(stderr, " %.1f", (ts[q] - ts[q - 1]) * 1e-3);
        std::fprintf(stderr, "\n");
      }
      swap_buf(X.mem_off, off2);  // new offsets become current
      X.mem_flip = !X.mem_flip;
      X.pool_flip = !X.pool_flip;
     }
     (void)rounds0;
    } else {
      map_prev = MapPrev{0, nullptr, nullptr};  // (no task map written for the next round)
      if (T > 0) {
        X.task_grp.ensure(al((T + 1) * 4));
        X.task_e.ensure(al((T + 1) * 8));
        k_task_map<<<grid_for(h.G * 32, 256), 256, 0, st>>>(d_G, X.task_off.as<int64_t>(), X.group.as<int32_t>(),
                                                              X.head.as<int32_t>(), G.row_ptr.as<int64_t>(),
                                                              X.task_grp.as<int32_t>(), X.task_e.as<int64_t>(), S);
        ++c.launches;
        ExpandArgs ea{X.group.as<int32_t>(), X.task_off.as<int64_t>(), X.task_grp.as<int32_t>(), X.task_e.as<int64_t>(), d_G, d_T,
                      G.row_ptr.as<int64_t>(),
                      G.e_to.as<int32_t>(), G.e_cost.as<double>(), G.e_nsteps.as<int32_t>(), G.wp_off.as<int64_t>(),
                      G.hs_off.as<int64_t>(), G.hs_cnt.as<int32_t>(), G.hs_pk.as<double>(),
                      X.head.as<int32_t>(),
                      X.cost.as<double>(), X.t_end.as<int32_t>(), X.mask.as<uint64_t>(), c.bank.as<double>(),
                    box.as<double>(), N,
                      c.bank_horizon, W, count_hs, prm.alpha_max, X.cand_keep.as<uint8_t>(), X.cand_head.as<int32_t>(),
                      X.cand_src.as<int32_t>(), X.cand_tend.as<int32_t>(), X.cand_cost.as<double>(),
                      X.cand_cp.as<double>(), X.cand_mask.as<uint64_t>(), S,
                        X.new_cnt.as<int32_t>(), X.new_slot.as<int32_t>(), X.touched.as<int32_t>()};
        const unsigned grid = grid_for(T * 32, 256);
        KScope ks(st, F_EXPAND);
        dispatch_dw(G.dw, [&]<int DW>() {
          switch (ch) {
            case 1: k_expand<DW, 1><<<grid, 256, 0, st>>>(ea); break;
            case 2: k_expand<DW, 2><<<grid, 256, 0, st>>>(ea); break;
            case 4: k_expand<DW, 4><<<grid, 256, 0, st>>>(ea); break;
            case 8: k_expand<DW, 8><<<grid, 256, 0, st>>>(ea); break;
            default: k_expand<DW, 16><<<grid, 256, 0, st>>>(ea); break;
          }
        });
        ++c.launches;
        PUMP_CUDA(cudaGetLastError());
      }
      exclusive_scan<uint8_t>(X.cand_keep.as<uint8_t>(), X.cand_rank.as<int64_t>(), T, stmp.p, st, &c.launches, d_T);
      if (T == 0) PUMP_CUDA(cudaMemsetAsync(X.cand_rank.p, 0, 8, st));
      CommitArgs ca{d_T, X.cand_keep.as<uint8_t>(), X.cand_rank.as<int64_t>(), X.cand_head.as<int32_t>(),
                    X.cand_src.as<int32_t>(), X.cand_tend.as<int32_t>(), X.cand_cost.as<double>(),
                    X.cand_cp.as<double>(), X.cand_mask.as<uint64_t>(), W, width, prm.alpha_min,
                    X.is_goal.as<uint8_t>(), X.head.as<int32_t>(), X.parent.as<int32_t>(), X.cost.as<double>(),
                    X.cp.as<double>(), X.t_end.as<int32_t>(), X.mask.as<uint64_t>(), X.bucket.as<int32_t>(),
                    X.flags.as<uint8_t>(), X.new_cnt.as<int32_t>(), X.new_slot.as<int32_t>(),
                    X.touched.as<int32_t>(), S};
      if (T > 0) {
        KScope ks(st, F_COMMIT);
        k_commit<<<grid_for(T, 256), 256, 0, st>>>(ca);
        ++c.launches;
      }
      // member relayout; K = total kept (rank[T], T from host) published on the way
      DBuf& old_ids = X.mem_flip ? X.mem_b : X.mem_a;
      DBuf& new_ids = X.mem_flip ? X.mem_a : X.mem_b;
      k_node_sizes<<<grid_for(std::max(n, 1), 256), 256, 0, st>>>(n, X.mem_cnt.as<int32_t>(), X.new_cnt.as<int32_t>(),
                                                                   node_sz.as<int32_t>(), S,
                                                                   X.cand_rank.as<int64_t>() + T, d_K);
      exclusive_scan<int32_t>(node_sz.as<int32_t>(), off2.as<int64_t>(), n, stmp.p, st, &c.launches);
      k_relayout<<<grid_for(static_cast<int64_t>(n) * 32, 256), 256, 0, st>>>(
          n, X.mem_off.as<int64_t>(), X.mem_cnt.as<int32_t>(), old_ids.as<int32_t>(), off2.as<int64_t>(),
          new_ids.as<int32_t>());
      c.launches += 2;
      if (T > 0) {
        k_place_new<<<grid_for(T, 256), 256, 0, st>>>(d_T, S, X.cand_keep.as<uint8_t>(), X.cand_rank.as<int64_t>(),
                                                        X.cand_head.as<int32_t>(), off2.as<int64_t>(),
                                                        X.mem_cnt.as<int32_t>(), X.new_slot.as<int32_t>(),
                                                        new_ids.as<int32_t>());
        const unsigned gd = static_cast<unsigned>(std::min<int64_t>(std::max<int64_t>(T, 1), 148 * 16));
        KScope ks(st, F_DOM);
        k_dom<<<gd, 128, 0, st>>>(S, X.touched.as<int32_t>(), off2.as<int64_t>(), X.mem_cnt.as<int32_t>(),
                                  X.new_cnt.as<int32_t>(), new_ids.as<int32_t>(), X.cost.as<double>(),
                                  X.cp.as<double>(), X.flags.as<uint8_t>(), X.drop.as<uint8_t>(),
                                  X.surv.as<uint8_t>(), X.fpos.as<int32_t>(), S);
        c.launches += 2;
      }
      swap_buf(X.mem_off, off2);  // new offsets become current
      X.mem_flip = !X.mem_flip;
      // surviving newcomers -> open pool in id order
      exclusive_scan<uint8_t>(X.surv.as<uint8_t>(), spos.as<int64_t>(), std::max<int64_t>(T, 1), stmp.p, st,
                              &c.launches, d_K);
      DBuf& pool_cur = X.pool_flip ? X.pool_b : X.pool_a;
      DBuf& pool_nxt = X.pool_flip ? X.pool_a : X.pool_b;
      if (T > 0) {
        k_pool_append<<<grid_for(T, 256), 256, 0, st>>>(d_K, S, X.surv.as<uint8_t>(), spos.as<int64_t>(),
                                                          X.bucket.as<int32_t>(), X.flags.as<uint8_t>(),
                                                          pool_cur.as<int32_t>(), S);
        ++c.launches;
      }
      // next group
      const int64_t pool_ub = h.pool_n + T + 1;
      k_pool_min<<<grid_for(pool_ub, 256), 256, 0, st>>>(S, d_K, spos.as<int64_t>(), pool_cur.as<int32_t>(),
                                                           X.flags.as<uint8_t>(), X.bucket.as<int32_t>(), S);
      k_round_i<<<1, 1, 0, st>>>(S, d_K, spos.as<int64_t>(), d_pool_n, d_limits);
      c.launches += 2;
      DBuf& keys = c.buf("x_sel_keys", al((pool_ub + 1) * 4));
      DBuf& stay = c.buf("x_sel_stay", al(pool_ub + 1));
      DBuf& stay_pos = c.buf("x_stay_pos", al((pool_ub + 2) * 8));
      // Distinct selection keys this round: the group takes buckets in
      // [min_bucket, min(i, max_bucket)].  Costs only grow along a plan, so the
      // new min_bucket >= the previous one, and i = max(i_prev + 1, min_bucket):
      // at most i_prev + 2 - min_bucket_prev keys (1 when i jumps to min_bucket).
      // Within 512 the stable multisplit needs one radix pass instead of two;
      // k_select flags a violated bound (never expected) as a device error.
      int64_t n_keys = 1 << 18;
      if (h.min_bucket != LLONG_MAX && h.i + 2 - h.min_bucket <= 512) n_keys = std::max<int64_t>(1, h.i + 2 - h.min_bucket);
      k_select<<<grid_for(pool_ub, 256), 256, 0, st>>>(d_pool_n, d_limits, pool_cur.as<int32_t>(),
                                                         X.flags.as<uint8_t>(), X.bucket.as<int32_t>(),
                                                         keys.as<int32_t>(), stay.as<uint8_t>(), n_keys, S);
      ++c.launches;
      DBuf& stmp2 = c.buf("x_scan_tmp2", scan_temp_bytes(pool_ub + 16));
      exclusive_scan<uint8_t>(stay.as<uint8_t>(), stay_pos.as<int64_t>(), pool_ub, stmp2.p, st, &c.launches,
                              d_pool_n);
      k_pool_compact<<<grid_for(pool_ub, 256), 256, 0, st>>>(d_pool_n, pool_cur.as<int32_t>(), stay.as<uint8_t>(),
                                                               stay_pos.as<int64_t>(), pool_nxt.as<int32_t>());
      ++c.launches;
      X.group.ensure(al((pool_ub + 1) * 4));
      DBuf& mtmp = c.buf("x_ms_tmp", multisplit_temp_bytes(pool_ub, 1 << 18));
      stable_multisplit(keys.as<int32_t>(), pool_cur.as<int32_t>(), pool_ub, static_cast<int>(n_keys), X.group.as<int32_t>(), d_G,
                        mtmp.p, st, &c.launches, d_pool_n);
      DBuf& deg = c.buf("x_deg", al((pool_ub + 1) * 4));
      X.task_off.ensure(al((pool_ub + 2) * 8));
      k_group_post<<<grid_for(pool_ub, 256), 256, 0, st>>>(d_G, X.group.as<int32_t>(), X.head.as<int32_t>(),
                                                             X.cost.as<double>(), G.row_ptr.as<int64_t>(),
                                                             X.flags.as<uint8_t>(), deg.as<int32_t>(), S);
      ++c.launches;
      DBuf& stmp3 = c.buf("x_scan_tmp3", scan_temp_bytes(pool_ub + 16));
      exclusive_scan<int32_t>(deg.as<int32_t>(), X.task_off.as<int64_t>(), pool_ub, stmp3.p, st, &c.launches, d_G);
      k_group_final<<<1, 1, 0, st>>>(S, d_G, X.task_off.as<int64_t>(), stay_pos.as<int64_t>(), d_pool_n, d_T);
      ++c.launches;
      X.pool_flip = !X.pool_flip;
      PUMP_CUDA(cudaGetLastError());
    }
    // the previous round's hook (side-stream launches) runs here, while the
    // device works on this round, instead of between the rounds
    if (hook_pending) {
      prm.on_round(h_hook);
      hook_pending = false;
    }
    if (win) {
      const int sl = next_slot;
      next_slot ^= 1;
      c.d2h(X.status_h + 1 + sl, S, sizeof(ExploreStatus));
      PUMP_CUDA(cudaEventRecord(X.status_ev[sl], st));
      if (inflight) {
        const int prev = in_slot;
        in_slot = sl;
        PUMP_CUDA(cudaEventSynchronize(X.status_ev[prev]));
        if (win_consume(X.status_h[1 + prev])) win_drain();  // the round just enqueued halts too
      } else {
        in_slot = sl;
        inflight = true;
      }
      continue;
    }
    c.d2h(X.status_h, S, sizeof(ExploreStatus));
    c.sync();
    const ExploreStatus hp = h;
    h = *X.status_h;
    X.n_plans = h.n_plans;
    if (h.err) throw std::runtime_error("explore: device error " + std::to_string(h.err));
    if (pipe) {
      // rounds that did not run left the buffers as they were: undo their flips
      const long long ran = h.rounds - hp.rounds;
      for (long long q = ran; q < nrounds; ++q) {
        swap_buf(X.mem_off, off2);
        X.mem_flip = !X.mem_flip;
        X.pool_flip = !X.pool_flip;
      }
      X.rounds += static_cast<int>(ran);
      X.partial_plans += h.partial_plans - hp.partial_plans;
      if (h.halt) {
        if (h.halt == 2) force_sync = true;  // the next round runs synchronously
        h.halt = 0;
        const long long zero = 0;
        c.h2d(&S->halt, &zero, 8);
      }
    }
    if (!ran_coop) {
      // algorithmic bytes of the round after expand (SURVEY §8d K_merge/K_dom/
      // K_bucket): candidate records read and ranked, kept plans written to the
      // arena, node sizes, the pool scanned, the new group read
      const int64_t Tr = hp.T, Kr = h.K;
      commit_bytes_legacy += Tr * (37 + 8 * W) + Kr * (33 + 8 * W) + static_cast<int64_t>(n) * 16 +
                             (hp.pool_n + Kr) * 9 + h.G * 28;
    }
    if (prm.on_round) {
      h_hook = h;
      hook_pending = true;
    }
    if (prm.on_round_state) {
      X.disc_cp = h.disc_cp;
      X.disc_hor = h.disc_hor;
      X.removed = h.removed;
      prm.on_round_state(X.rounds, expanded);
    }
  }
  if (hook_pending) prm.on_round(h_hook);  // the last round's
  X.kernel_ms = c.toc();
  kprof_work(F_COMMIT, commit_bytes_legacy + h.commit_bytes);  // (the cooperative rounds count on the device)
  kprof_work(F_EXPAND, h.hs_tests * N);
  X.hs_tests = h.hs_tests;
  X.hs_read = h.hs_read;
  X.n_plans = h.n_plans;
  X.disc_cp = h.disc_cp;
  X.disc_hor = h.disc_hor;
  X.removed = h.removed;
}

// Latency floor of the cooperative round: microseconds per grid barrier
// (the kernel's own grid_sync, the round's grid) and per dependent L2 load
// chain step, measured with the round kernel's launch shape.
__global__ void __launch_bounds__(kCoopBlock, 2) k_probe_barrier(GridBar* bar, int iters) {
  for (int k = 0; k < iters; ++k) grid_sync(bar);
}
__global__ void k_probe_chain(const int32_t* __restrict__ next, int steps, int32_t* __restrict__ out) {
  int x = 0;
  for (int k = 0; k < steps; ++k) x = next[x];
  out[0] = x;
}
void probe_round_latency(Ctx& c, double* us_barrier, double* us_load) {
  int per_sm = 0, sms = 0;
  PUMP_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, reinterpret_cast<const void*>(&k_probe_barrier),
                                                          kCoopBlock, 0));
  PUMP_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, c.device));
  const int blocks = std::min(per_sm, 1) * sms;  // the round kernel's grid (one block per SM)
  DBuf& bar = c.buf("probe_bar", 256);
  PUMP_CUDA(cudaMemsetAsync(bar.p, 0, 8, c.stream));
  GridBar* b = bar.as<GridBar>();
  int iters = 8;
  void* args[] = {&b, &iters};
  PUMP_CUDA(cudaLaunchCooperativeKernel(reinterpret_cast<const void*>(&k_probe_barrier), dim3(blocks),
                                        dim3(kCoopBlock), args, 0, c.stream));  // warm-up
  iters = 2000;
  c.tic();
  PUMP_CUDA(cudaLaunchCooperativeKernel(reinterpret_cast<const void*>(&k_probe_barrier), dim3(blocks),
                                        dim3(kCoopBlock), args, 0, c.stream));
  *us_barrier = c.toc() * 1e3 / iters;
  // dependent loads over a 64 MiB permutation (L2-missing pointer chase would be
  // HBM latency; 1 MiB stays L2-resident: the round's working set)
  const int n = 1 << 18;  // 1 MiB of int32
  std::vector<int32_t> h(n);
  for (int k = 0; k < n; ++k) h[k] = static_cast<int32_t>((static_cast<int64_t>(k) * 40503 + 12345) % n);
  DBuf& nx = c.buf("probe_next", n * 4 + 256);
  DBuf& o = c.buf("probe_out", 256);
  c.h2d(nx.p, h.data(), n * 4);
  k_probe_chain<<<1, 1, 0, c.stream>>>(nx.as<int32_t>(), 1000, o.as<int32_t>());
  const int steps = 20000;
  c.tic();
  k_probe_chain<<<1, 1, 0, c.stream>>>(nx.as<int32_t>(), steps, o.as<int32_t>());
  *us_load = c.toc() * 1e3 / steps;
  c.launches += 4;
}

}  // namespace pumpg
