// K_hsmc (batched API form): hsmc_extend (cp.hpp:180-208) for many tasks.
//
// One warp per task; lane l owns particles l, l+32, ... (CH = ceil(N/32)
// chunks).  Per step the lane loads its particles' bank rows once (the warp
// reads the whole [t][0..N)[0..dw) row: coalesced), then tests every
// half-space of the step: s = ((0 + a0 p0) + a1 p1) + a2 p2 > b, exactly the
// reference's sequential dot.  Kills are OR-accumulated per chunk and turned
// into mask words with one ballot per chunk; popcount via __popcll.
// Survival is an AND over all (step, half-space) tests, so evaluating dead
// particles too (the reference skips them) cannot change any bit.
#include "dispatch.cuh"

namespace pumpg {

template <int DW, int CH>
__global__ void __launch_bounds__(256) k_hsmc_batch(const double* __restrict__ dy, int n, int horizon,
                                                    int64_t n_tasks, int n_words, const uint64_t* __restrict__ in,
                                                    const int64_t* __restrict__ step_off,
                                                    const int32_t* __restrict__ step_t,
                                                    const int64_t* __restrict__ step_hs_off,
                                                    const double* __restrict__ hs_a, const double* __restrict__ hs_b,
                                                    uint64_t* __restrict__ out, int32_t* __restrict__ pop,
                                                    int* __restrict__ err) {
  const int64_t task = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (task >= n_tasks) return;
  bool kill[CH];
#pragma unroll
  for (int c = 0; c < CH; ++c) kill[c] = false;
  const int64_t s0 = step_off[task], s1 = step_off[task + 1];
  for (int64_t s = s0; s < s1; ++s) {
    const int t = step_t[s];
    if (t < 0 || t > horizon) {  // cp.hpp:186-187, checked before the empty-region skip
      if (lane == 0) atomicExch(err, 1);
      return;
    }
    const int64_t h0 = step_hs_off[s], h1 = step_hs_off[s + 1];
    if (h0 == h1) continue;
    double p[CH][DW];
    const double* row = dy + static_cast<int64_t>(t) * n * DW;
#pragma unroll
    for (int c = 0; c < CH; ++c) {
      const int i = c * 32 + lane;
#pragma unroll
      for (int k = 0; k < DW; ++k) p[c][k] = (i < n) ? row[i * DW + k] : 0.0;
    }
    for (int64_t h = h0; h < h1; ++h) {
      double a[DW];
#pragma unroll
      for (int k = 0; k < DW; ++k) a[k] = hs_a[h * DW + k];
      const double b = hs_b[h];
#pragma unroll
      for (int c = 0; c < CH; ++c) {
        double sdot = 0;
#pragma unroll
        for (int k = 0; k < DW; ++k) sdot += a[k] * p[c][k];
        kill[c] = kill[c] || (sdot > b);
      }
    }
  }
  int total = 0;
#pragma unroll
  for (int w = 0; w < (CH + 1) / 2; ++w) {
    const unsigned lo = __ballot_sync(0xffffffffu, kill[2 * w]);
    const unsigned hi = (2 * w + 1 < CH) ? __ballot_sync(0xffffffffu, kill[2 * w + 1]) : 0u;
    if (w < n_words) {
      const uint64_t k = (static_cast<uint64_t>(hi) << 32) | lo;
      const uint64_t m = in[task * n_words + w] & ~k;
      total += __popcll(m);
      if (lane == 0) out[task * n_words + w] = m;
    }
  }
  if (lane == 0) pop[task] = total;
}

// Plans of more than 512 particles: a warp per (task, 64-particle mask word),
// lane l owning particles 64w + l and 64w + 32 + l, the same tests in the
// same order; the survivor count is summed per task with one atomic per word.
template <int DW>
__global__ void __launch_bounds__(256) k_hsmc_wide(const double* __restrict__ dy, int n, int horizon, int64_t n_tasks,
                                                   int n_words, const uint64_t* __restrict__ in,
                                                   const int64_t* __restrict__ step_off,
                                                   const int32_t* __restrict__ step_t,
                                                   const int64_t* __restrict__ step_hs_off,
                                                   const double* __restrict__ hs_a, const double* __restrict__ hs_b,
                                                   uint64_t* __restrict__ out, int32_t* __restrict__ pop,
                                                   int* __restrict__ err) {
  const int64_t gw = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (gw >= n_tasks * n_words) return;
  const int64_t task = gw / n_words;
  const int w = static_cast<int>(gw % n_words);
  const int i0 = 64 * w + lane, i1 = i0 + 32;
  const uint64_t m_in = in[task * n_words + w];
  bool k0 = false, k1 = false;
  const int64_t s0 = step_off[task], s1 = step_off[task + 1];
  for (int64_t s = s0; s < s1; ++s) {
    const int t = step_t[s];
    if (t < 0 || t > horizon) {  // cp.hpp:186-187, checked before the empty-region skip
      if (lane == 0) atomicExch(err, 1);
      return;
    }
    const int64_t h0 = step_hs_off[s], h1 = step_hs_off[s + 1];
    if (h0 == h1 || m_in == 0) continue;
    const double* row = dy + static_cast<int64_t>(t) * n * DW;
    double p0[DW], p1[DW];
#pragma unroll
    for (int k = 0; k < DW; ++k) {
      p0[k] = i0 < n ? row[static_cast<int64_t>(i0) * DW + k] : 0.0;
      p1[k] = i1 < n ? row[static_cast<int64_t>(i1) * DW + k] : 0.0;
    }
    for (int64_t h = h0; h < h1; ++h) {
      const double b = hs_b[h];
      double sa = 0, sb = 0;
#pragma unroll
      for (int k = 0; k < DW; ++k) {
        const double ak = hs_a[h * DW + k];
        sa += ak * p0[k];
        sb += ak * p1[k];
      }
      k0 = k0 || (sa > b);
      k1 = k1 || (sb > b);
    }
  }
  const unsigned lo = __ballot_sync(0xffffffffu, k0), hi = __ballot_sync(0xffffffffu, k1);
  if (lane == 0) {
    const uint64_t m = m_in & ~((static_cast<uint64_t>(hi) << 32) | lo);
    out[task * n_words + w] = m;
    atomicAdd(&pop[task], __popcll(m));
  }
}

template <int DW>
static void hsmc_dispatch_ch(int ch, dim3 g, cudaStream_t st, const double* d_dy, int n, int horizon,
                             int64_t n_tasks, int n_words, const uint64_t* d_in, const int64_t* a, const int32_t* b,
                             const int64_t* c, const double* ha, const double* hb, uint64_t* o, int32_t* p, int* e) {
#define PUMP_HSMC_CASE(X)                                                                              \
  case X:                                                                                              \
    k_hsmc_batch<DW, X><<<g, 256, 0, st>>>(d_dy, n, horizon, n_tasks, n_words, d_in, a, b, c, ha, hb, o, p, e); \
    break;
  switch (ch) {
    PUMP_HSMC_CASE(1)
    PUMP_HSMC_CASE(2)
    PUMP_HSMC_CASE(4)
    PUMP_HSMC_CASE(8)
    PUMP_HSMC_CASE(16)
    default:
      throw std::invalid_argument("hsmc_extend: particle count must be <= 512");
  }
#undef PUMP_HSMC_CASE
}

int chunks_for(int n) {
  int ch = (n + 31) / 32;
  int p = 1;
  while (p < ch) p <<= 1;
  return p;
}

void launch_hsmc_batch(int dw, int n, int horizon, const double* d_dy, int64_t n_tasks, int n_words,
                       const uint64_t* d_in, const int64_t* d_step_off, const int32_t* d_step_t,
                       const int64_t* d_step_hs_off, const double* d_hs_a, const double* d_hs_b, uint64_t* d_out,
                       int32_t* d_pop, int* d_err, cudaStream_t st, int64_t* launches) {
  if (n_tasks <= 0) return;
  if (n_words != (n + 63) / 64) throw std::invalid_argument("hsmc_extend: mask word count does not match the bank");
  const int ch = chunks_for(n);
  dim3 g(grid_for(n_tasks * 32, 256));
  KScope ks(st, F_HSMC);
  if (ch > 16) {
    PUMP_CUDA(cudaMemsetAsync(d_pop, 0, static_cast<size_t>(n_tasks) * sizeof(int32_t), st));
    dispatch_dw(dw, [&]<int DW>() {
      k_hsmc_wide<DW><<<grid_for(n_tasks * n_words * 32, 256), 256, 0, st>>>(
          d_dy, n, horizon, n_tasks, n_words, d_in, d_step_off, d_step_t, d_step_hs_off, d_hs_a, d_hs_b, d_out, d_pop,
          d_err);
    });
    ++*launches;
    PUMP_CUDA(cudaGetLastError());
    return;
  }
  dispatch_dw(dw, [&]<int DW>() {
    hsmc_dispatch_ch<DW>(ch, g, st, d_dy, n, horizon, n_tasks, n_words, d_in, d_step_off, d_step_t, d_step_hs_off,
                         d_hs_a, d_hs_b, d_out, d_pop, d_err);
  });
  ++*launches;
  PUMP_CUDA(cudaGetLastError());
}

}  // namespace pumpg
