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
#include "dispatch.cuh"

namespace pumpg {

constexpr int kMcBlock = 128;

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

void launch_mc(const HostLoop& HL, const DevWorld& w, int n_traj, const int64_t* d_traj_off, const double* d_ynom,
               int max_points, int64_t r0, int64_t r1, uint64_t seed, double eps_cc, unsigned long long* d_hits,
               cudaStream_t st, int64_t* launches, unsigned long long* d_steps) {
  if (r1 <= r0 || n_traj <= 0) return;
  if (HL.dw != w.dw) throw std::invalid_argument("mc_certify: workspace / model dimension mismatch");
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
