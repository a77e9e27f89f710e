// K_bank: presample_bank (lti.hpp:257-292) on sm_100a.
//
// The recursion z_{t+1} = F z_t + Gv(Sv nv_t) + Gw(Sw nw_{t+1}) is sequential
// in t per particle, but its noise terms are not: they are pure functions of
// the (seed, particle, timestep, channel) key.  So the bank is built in time
// chunks of kChunk steps:
//   k_bank_noise  — one thread per (t, i): 9 normals (3-D), u = Gv(Sv nv),
//                   w = Gw(Sw nw); massively parallel, issue-bound on the
//                   u64 hash + log/cos.
//   k_bank_rec    — one thread per particle: y_t = C z_t stored, then
//                   z <- ((F z) + u) + w, exactly the reference's rounding.
// Noise is laid out component-major [t][r][i] so the recurrence's loads are
// coalesced across particles.
#include <cstdlib>

#include "dispatch.cuh"

namespace pumpg {

constexpr int kChunk = 256;

template <int D, int DW>
__global__ void __launch_bounds__(128) k_bank_noise(const LoopP<D, DW> L, int n, int t0, int tc, uint64_t seed,
                                                    double* __restrict__ uw) {
  const int64_t idx = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (idx >= static_cast<int64_t>(tc) * n) return;
  const int tl = static_cast<int>(idx / n);
  const int i = static_cast<int>(idx - static_cast<int64_t>(tl) * n);
  const int t = t0 + tl;
  const uint64_t sa = hash_seed_a(seed, static_cast<uint64_t>(i));
  const uint64_t pt = mix64(sa + static_cast<uint64_t>(t));
  const uint64_t pt1 = mix64(sa + static_cast<uint64_t>(t + 1));
  double nv[D], nw[DW], t1[D], t2[DW];
#pragma unroll
  for (int k = 0; k < D; ++k) nv[k] = normal_from_prefix(pt, kProcess + k);
#pragma unroll
  for (int k = 0; k < DW; ++k) nw[k] = normal_from_prefix(pt1, kMeasurement + k);
#pragma unroll
  for (int r = 0; r < D; ++r) t1[r] = row_dot<D>(L.Sv + r * D, nv);
#pragma unroll
  for (int r = 0; r < DW; ++r) t2[r] = row_dot<DW>(L.Sw + r * DW, nw);
  double* base = uw + static_cast<int64_t>(tl) * (4 * D) * n + i;
#pragma unroll
  for (int r = 0; r < 2 * D; ++r) {
    base[static_cast<int64_t>(r) * n] = row_dot<D>(L.Gv + r * D, t1);
    base[static_cast<int64_t>(2 * D + r) * n] = row_dot<DW>(L.Gw + r * DW, t2);
  }
}

template <int D, int DW>
__global__ void __launch_bounds__(32) k_bank_rec(const LoopP<D, DW> L, int n, int T, int t0, int tc, uint64_t seed,
                                                 const double* __restrict__ uw, double* __restrict__ zstate,
                                                 double* __restrict__ dy) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double z[2 * D];
  if (t0 == 0) {
    const uint64_t p0 = mix64(hash_seed_a(seed, static_cast<uint64_t>(i)) + 0ull);
    double nv[D];
#pragma unroll
    for (int k = 0; k < D; ++k) nv[k] = normal_from_prefix(p0, static_cast<uint64_t>(k));  // kInitial + k
#pragma unroll
    for (int r = 0; r < D; ++r) z[r] = row_dot<D>(L.S0 + r * D, nv);
#pragma unroll
    for (int r = D; r < 2 * D; ++r) z[r] = 0.0;
  } else {
#pragma unroll
    for (int r = 0; r < 2 * D; ++r) z[r] = zstate[static_cast<int64_t>(r) * n + i];
  }
  // noise of step tl is prefetched one step ahead (register double buffer)
  double un[4 * D];
  if (tc > 0) {
#pragma unroll
    for (int r = 0; r < 4 * D; ++r) un[r] = uw[static_cast<int64_t>(r) * n + i];
  }
  for (int tl = 0; tl <= tc; ++tl) {
    const int t = t0 + tl;
    if (tl == tc && t != T) break;  // next chunk stores y_t
    double* slot = dy + (static_cast<int64_t>(t) * n + i) * DW;
#pragma unroll
    for (int k = 0; k < DW; ++k) slot[k] = row_dot<D>(L.C + k * D, z);
    if (t == T) break;
    double uc[4 * D];
#pragma unroll
    for (int r = 0; r < 4 * D; ++r) uc[r] = un[r];
    if (tl + 1 < tc) {
      const double* u = uw + static_cast<int64_t>(tl + 1) * (4 * D) * n + i;
#pragma unroll
      for (int r = 0; r < 4 * D; ++r) un[r] = u[static_cast<int64_t>(r) * n];
    }
    double zn[2 * D];
#pragma unroll
    for (int r = 0; r < 2 * D; ++r) {
      double a = row_dot<2 * D>(L.F + r * 2 * D, z);
      zn[r] = (a + uc[r]) + uc[2 * D + r];
    }
#pragma unroll
    for (int r = 0; r < 2 * D; ++r) z[r] = zn[r];
  }
#pragma unroll
  for (int r = 0; r < 2 * D; ++r) zstate[static_cast<int64_t>(r) * n + i] = z[r];
}

// Axis-separable recurrence: one lane per (particle, axis), the 4x4 axis
// block of F and the axis' 4 rows of the (dense, bit-identical) u and w the
// noise kernel wrote.  Dropping F's structural zeros leaves every partial
// sum unchanged (mc.cu, k_mc_sep); y_k = (0 + C_k0 z_k) + C_k1 z_{dw+k}.
// The dense recurrence issues a 2d x 2d gemv per step from ~n/32 warps; this
// one issues 16 products per lane from n * dw lanes.
template <int DW>
__global__ void __launch_bounds__(32) k_bank_rec_sep(const SepBlocks B, int n, int T, int t0, int tc, uint64_t seed,
                                                     const double* __restrict__ uw, double* __restrict__ zstate,
                                                     double* __restrict__ dy) {
  constexpr int D = 2 * DW;
  const int x = blockIdx.x * blockDim.x + threadIdx.x;
  if (x >= n * DW) return;
  const int i = x / DW, k = x - i * DW;
  const double* F = B.F[k];
  const int g[4] = {k, DW + k, D + k, D + DW + k};
  double z[4];
  if (t0 == 0) {
    const uint64_t p0 = mix64(hash_seed_a(seed, static_cast<uint64_t>(i)) + 0ull);
    const double n0 = normal_from_prefix(p0, static_cast<uint64_t>(k));       // kInitial + k
    const double n1 = normal_from_prefix(p0, static_cast<uint64_t>(DW + k));  // kInitial + dw + k
    z[0] = (0.0 + B.S0[k][0] * n0) + B.S0[k][1] * n1;
    z[1] = (0.0 + B.S0[k][2] * n0) + B.S0[k][3] * n1;
    z[2] = 0.0;
    z[3] = 0.0;
  } else {
#pragma unroll
    for (int r = 0; r < 4; ++r) z[r] = zstate[static_cast<int64_t>(x) * 4 + r];
  }
  // only n dw / 32 warps run, so the step loop is bound by the latency of
  // its noise loads: a ring of kRecPf steps in registers, each step's load
  // issued kRecPf steps before it is consumed (the loop unrolled by the ring
  // length so the ring stays in registers)
  constexpr int kRecPf = 4;
  double ring[kRecPf][8];
  auto fetch = [&](int tl, double* dst) {
    const double* u = uw + static_cast<int64_t>(tl) * (4 * D) * n + i;
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      dst[r] = u[static_cast<int64_t>(g[r]) * n];
      dst[4 + r] = u[static_cast<int64_t>(2 * D + g[r]) * n];
    }
  };
#pragma unroll
  for (int q = 0; q < kRecPf; ++q)
    if (q < tc) fetch(q, ring[q]);
  bool done = false;
  for (int tb = 0; tb <= tc && !done; tb += kRecPf) {
#pragma unroll
    for (int q = 0; q < kRecPf; ++q) {
      const int tl = tb + q;
      const int t = t0 + tl;
      if (tl > tc || (tl == tc && t != T)) {  // next chunk stores y_t
        done = true;
        break;
      }
      dy[(static_cast<int64_t>(t) * n + i) * DW + k] = (0.0 + B.C[k][0] * z[0]) + B.C[k][1] * z[1];
      if (t == T) {
        done = true;
        break;
      }
      double uc[8];
#pragma unroll
      for (int r = 0; r < 8; ++r) uc[r] = ring[q][r];
      if (tl + kRecPf < tc) fetch(tl + kRecPf, ring[q]);
      double zn[4];
#pragma unroll
      for (int r = 0; r < 4; ++r) {
        double c = 0.0;
#pragma unroll
        for (int w = 0; w < 4; ++w) c = c + F[r * 4 + w] * z[w];
        zn[r] = (c + uc[r]) + uc[4 + r];
      }
#pragma unroll
      for (int r = 0; r < 4; ++r) z[r] = zn[r];
    }
  }
#pragma unroll
  for (int r = 0; r < 4; ++r) zstate[static_cast<int64_t>(x) * 4 + r] = z[r];
}

size_t bank_scratch_bytes(const HostLoop& L, int n, int T) {
  (void)T;
  const int D = L.d;
  return (static_cast<size_t>(kChunk) * 4 * D * n + static_cast<size_t>(2 * D) * n) * sizeof(double);
}

void launch_bank(const HostLoop& HL, int n, int T, uint64_t seed, double* d_dy, void* d_scratch, cudaStream_t st,
                 int64_t* launches) {
  if (n < 1) throw std::invalid_argument("presample_bank: need at least one particle");
  if (T < 1) throw std::invalid_argument("presample_bank: horizon must be at least 1");
  const bool sep = HL.dw >= 2 && HL.dw <= 3 && separable(HL);
  const SepBlocks B = sep ? sep_blocks(HL) : SepBlocks{};
  dispatch_dims(HL.d, HL.dw, [&]<int D, int DW>() {
    const LoopP<D, DW> L = make_loop<D, DW>(HL);
    double* uw = static_cast<double*>(d_scratch);
    double* zs = uw + static_cast<size_t>(kChunk) * 4 * D * n;
    for (int t0 = 0; t0 <= T; t0 += kChunk) {
      const int tc = std::min(kChunk, T - t0);  // steps advanced in this chunk
      if (tc > 0) {
        const int64_t items = static_cast<int64_t>(tc) * n;
        KScope ks(st, F_BANK_NOISE);
        k_bank_noise<D, DW><<<grid_for(items, 128), 128, 0, st>>>(L, n, t0, tc, seed, uw);
        ++*launches;
        kprof_work(F_BANK_NOISE, items);
      }
      {
        KScope ks(st, F_BANK_REC);
        if constexpr (D == 2 * DW) {
          if (sep)
            k_bank_rec_sep<DW><<<grid_for(static_cast<int64_t>(n) * DW, 32), 32, 0, st>>>(B, n, T, t0, tc, seed, uw,
                                                                                         zs, d_dy);
          else
            k_bank_rec<D, DW><<<grid_for(n, 32), 32, 0, st>>>(L, n, T, t0, tc, seed, uw, zs, d_dy);
        } else {
          k_bank_rec<D, DW><<<grid_for(n, 32), 32, 0, st>>>(L, n, T, t0, tc, seed, uw, zs, d_dy);
        }
        ++*launches;
        kprof_work(F_BANK_REC, static_cast<int64_t>(tc) * n);
      }
      if (tc < kChunk) break;
    }
    PUMP_CUDA(cudaGetLastError());
  });
}

}  // namespace pumpg
