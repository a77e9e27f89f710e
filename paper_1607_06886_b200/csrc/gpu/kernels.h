// Host-callable launchers of the sm_100a kernels (implemented in *.cu).
// All launchers are stream-ordered; none synchronizes.
#pragma once

#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <stdexcept>
#include <string>
#include <vector>

#include <cuda_runtime.h>

#include "../../../include/pump_gpu.h"

namespace pumpg {

struct CudaError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

inline void cuda_check(cudaError_t e, const char* what) {
  if (e != cudaSuccess) {
    // clear a non-sticky error (e.g. an allocation that did not fit) so the
    // next call of the context does not report it again
    (void)cudaGetLastError();
    throw CudaError(std::string(what) + ": " + cudaGetErrorString(e));
  }
}
#define PUMP_CUDA(x) ::pumpg::cuda_check((x), #x)

// cudaMalloc calls made by DBuf (a steady-state solve should make none)
inline int64_t g_dev_allocs = 0;

// Grow-only device buffer.
struct DBuf {
  void* p = nullptr;
  size_t cap = 0;
  void ensure(size_t bytes) {
    if (bytes <= cap) return;
    if (p) cudaFree(p);
    p = nullptr;
    cap = 0;
    size_t want = bytes < 256 ? 256 : bytes;
    PUMP_CUDA(cudaMalloc(&p, want));
    ++g_dev_allocs;
    if (std::getenv("PUMP_DEBUG_ALLOC")) std::fprintf(stderr, "[pump alloc] ensure %zu\n", want);
    cap = want;
  }
  // grow keeping the first `keep` bytes
  void grow(size_t bytes, size_t keep, cudaStream_t st) {
    if (bytes <= cap) return;
    void* q = nullptr;
    size_t want = bytes + bytes / 2;
    PUMP_CUDA(cudaMalloc(&q, want));
    ++g_dev_allocs;
    if (std::getenv("PUMP_DEBUG_ALLOC")) std::fprintf(stderr, "[pump alloc] grow %zu\n", want);
    if (p && keep) PUMP_CUDA(cudaMemcpyAsync(q, p, keep, cudaMemcpyDeviceToDevice, st));
    if (p) {
      PUMP_CUDA(cudaStreamSynchronize(st));
      cudaFree(p);
    }
    p = q;
    cap = want;
  }
  template <class T>
  T* as() const {
    return static_cast<T*>(p);
  }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    cap = 0;
  }
  ~DBuf() { release(); }
  DBuf() = default;
  DBuf(const DBuf&) = delete;
  DBuf& operator=(const DBuf&) = delete;
};

// ------------------------------------------------------- kernel profiler
// Kernel families timed with CUDA events on the launching stream when a
// profiler is active on this host thread (pump_ctx_profile).
// same order as PUMP_FAM_* in pump_gpu.h
enum KFam {
  F_BANK_NOISE, F_BANK_REC, F_HSMC, F_MC, F_CONNECT, F_COLLIDE, F_EMIT, F_REGIONS,
  F_EXPAND, F_COMMIT, F_DOM, F_SCAN, F_SPLIT, F_MISC, F_PAIR, F_MC_TABLE, F_COUNT
};

struct KProf {
  bool on = false;
  struct Rec {
    int fam;
    cudaEvent_t a, b;
  };
  std::vector<Rec> recs;
  std::vector<cudaEvent_t> pool;
  double ms[F_COUNT] = {0};
  int64_t count[F_COUNT] = {0};
  // algorithmic work units per family (e.g. MC rollout-steps, steer_cost evals)
  int64_t work[F_COUNT] = {0};
  cudaEvent_t get() {
    if (pool.empty()) {
      cudaEvent_t e;
      cuda_check(cudaEventCreate(&e), "cudaEventCreate");
      return e;
    }
    cudaEvent_t e = pool.back();
    pool.pop_back();
    return e;
  }
  void resolve() {  // caller synchronized the stream
    for (auto& r : recs) {
      float x = 0;
      cuda_check(cudaEventElapsedTime(&x, r.a, r.b), "cudaEventElapsedTime");
      ms[r.fam] += x;
      count[r.fam] += 1;
      pool.push_back(r.a);
      pool.push_back(r.b);
    }
    recs.clear();
  }
};

KProf*& kprof_current();

struct KScope {
  KProf* p;
  int fam;
  cudaStream_t st;
  cudaEvent_t a = nullptr;
  KScope(cudaStream_t s, int f) : p(kprof_current()), fam(f), st(s) {
    if (p && p->on) {
      a = p->get();
      cuda_check(cudaEventRecord(a, st), "cudaEventRecord");
    }
  }
  ~KScope() {
    if (p && p->on && a) {
      cudaEvent_t b = p->get();
      cudaEventRecord(b, st);
      p->recs.push_back({fam, a, b});
    }
  }
};

inline void kprof_work(int fam, int64_t units) {
  KProf* p = kprof_current();
  if (p && p->on) p->work[fam] += units;
}

// Host copy of a ClosedLoop (row-major), dims checked.
struct HostLoop {
  int d = 0, dw = 0;
  std::vector<double> F, Gv, Gw, Sv, Sw, S0, C;
};
HostLoop host_loop(const pump_closed_loop* cl);

// Workspace on the device: obstacles packed lo[o*dw+k], hi[o*dw+k].
struct DevWorld {
  int dw = 0, n_obs = 0;
  double blo[6] = {0}, bhi[6] = {0};
  double* d_lo = nullptr;
  double* d_hi = nullptr;
};

// ------------------------------------------------------------------ bank
// presample_bank (lti.hpp:257-292) into d_dy [(T+1) x n x dw].
// scratch must hold bank_scratch_bytes(...) bytes.
size_t bank_scratch_bytes(const HostLoop& L, int n, int T);
void launch_bank(const HostLoop& L, int n, int T, uint64_t seed, double* d_dy, void* d_scratch, cudaStream_t st,
                 int64_t* launches);

// ------------------------------------------------------------------ hsmc
// Batched hsmc_extend (cp.hpp:180-208); d_err set to 1 on a step outside
// [0, horizon].
void launch_hsmc_batch(int dw, int n, int horizon, const double* d_dy, int64_t n_tasks, int n_words,
                       const uint64_t* d_in, const int64_t* d_step_off, const int32_t* d_step_t,
                       const int64_t* d_step_hs_off, const double* d_hs_a, const double* d_hs_b, uint64_t* d_out,
                       int32_t* d_pop, int* d_err, cudaStream_t st, int64_t* launches);

// --------------------------------------------------------------------- mc
// Batched mc_certify (cp.hpp:214-268) over trajectories and the rollout
// range [r0, r1); d_hits[j] += colliding rollouts of trajectory j.
// Axis-separable closed loop (mc.cu): per axis k the 4 z entries
// g(rho) = {k, dw+k, d+k, d+dw+k} couple only among themselves.
struct SepBlocks {
  double F[3][16], Gv[3][8], Gw[3][4], Sv[3][4], Sw[3], S0[3][4], C[3][2];
};
bool separable(const HostLoop& L);
SepBlocks sep_blocks(const HostLoop& L);

// Common-random-number table of the MC rollouts.  The deviation of rollout i
// from ANY nominal trajectory, dy_t = C z_t, depends only on (closed loop,
// seed, i, t): z_t is driven by the counter-hash noise alone.  The table
// holds dy[t][i][k] for the rollouts [r0, r1) and t <= t_done, in HBM, so
// every trajectory certified against the same (loop, seed) reads its
// realizations instead of re-drawing ~9 normals per rollout-step.  Extended
// in place (z_{t_done} kept per rollout) when a longer trajectory arrives.
struct McTable {
  DBuf dy;  // [t][i][k], t < t_cap
  DBuf z;   // z_{t_done} per rollout
  DBuf flags;  // per (trajectory, rollout) hit flags of one certification
  DBuf maxdev;  // [t][k]: max over rollouts of |dy| (bits of a non-negative double)
  DBuf nz;      // build scratch: per (t, rollout, axis) the Sv / Sw products of the step's normals
  DBuf step_list, step_nl, step_skip;  // per (trajectory, step) candidate obstacles (k_mc_steps)
  int64_t r0 = 0, r1 = 0;
  int t_done = -1, t_cap = 0;
  uint64_t seed = 0;
  HostLoop L;
  bool valid = false;
  bool sep = false;
  void invalidate() { valid = false; }
};

// Build / extend the table for rollouts [r0, r1) and steps t <= T on `st`
// (launch_mc then finds it ready); no-op when the table would not fit.
void mc_table_prepare(McTable& tab, const HostLoop& L, int64_t r0, int64_t r1, uint64_t seed, int T,
                      cudaStream_t st, int64_t* launches);
// the table already holds rollouts [r0, r1), steps t <= T of this closed loop and seed
bool mc_table_covers(const McTable& tab, const HostLoop& L, int64_t r0, int64_t r1, uint64_t seed, int T);
// candidate obstacles listed per (trajectory, step) for the table path (more: nl = -1, test all)
constexpr int kStepCap = 64;
// rollouts per table certification (larger ones go in chunks)
constexpr int64_t kTabRollouts = int64_t(1) << 19;
// the table's per-(trajectory, step) list buffers for n_traj x max_points rows
void mc_step_buffers(McTable& tab, int n_traj, int max_points);
void launch_mc(const HostLoop& L, const DevWorld& w, int n_traj, const int64_t* d_traj_off, const double* d_ynom,
               int max_points, int64_t r0, int64_t r1, uint64_t seed, double eps_cc, unsigned long long* d_hits,
               cudaStream_t st, int64_t* launches, unsigned long long* d_steps = nullptr, McTable* table = nullptr,
               const int32_t* d_live = nullptr,  // d_live[j] == 0: skip trajectory j (table path; hits stay 0)
               bool lists_ready = false);  // the caller wrote the table's step lists (mc_step_row)

}  // namespace pumpg
