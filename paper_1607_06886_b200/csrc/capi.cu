// C ABI of libpump_gpu.so (include/pump_gpu.h): context, scenario, bank,
// batched HSMC and batched MC certification.  Graph / explore / pipeline
// entry points live in capi_plan.cu.
#include <cstring>
#include <string>

#include "ctx.h"
#include "host/scenario_fast.hpp"
#include "guard.h"

static_assert(static_cast<int>(pumpg::F_COUNT) == PUMP_FAM_COUNT && static_cast<int>(pumpg::F_PAIR) == PUMP_FAM_PAIR,
              "kernel family order must match pump_gpu.h");

using namespace pumpg;

namespace pumpg {

HostLoop host_loop(const pump_closed_loop* cl) {
  if (!cl) throw std::invalid_argument("closed loop: null");
  HostLoop L;
  L.d = cl->d;
  L.dw = cl->dw;
  const int d = cl->d, dw = cl->dw;
  if (d < 1 || dw < 1 || d > 12 || dw > 6) throw std::invalid_argument("closed loop: bad dimensions");
  L.F.assign(cl->F, cl->F + 4 * d * d);
  L.Gv.assign(cl->Gv, cl->Gv + 2 * d * d);
  L.Gw.assign(cl->Gw, cl->Gw + 2 * d * dw);
  L.Sv.assign(cl->Sv, cl->Sv + d * d);
  L.Sw.assign(cl->Sw, cl->Sw + dw * dw);
  L.S0.assign(cl->S0, cl->S0 + d * d);
  L.C.assign(cl->C, cl->C + dw * d);
  return L;
}

DevWorld upload_world(Ctx& c, const pump_workspace* ws, const std::string& prefix) {
  if (!ws) throw std::invalid_argument("workspace: null");
  if (ws->dw < 1 || ws->dw > 6 || ws->n_obs < 0) throw std::invalid_argument("workspace: bad dimensions");
  DevWorld w;
  w.dw = ws->dw;
  w.n_obs = ws->n_obs;
  for (int k = 0; k < ws->dw; ++k) {
    w.blo[k] = ws->bounds_lo[k];
    w.bhi[k] = ws->bounds_hi[k];
  }
  const size_t bytes = static_cast<size_t>(ws->n_obs) * ws->dw * sizeof(double);
  DBuf& lo = c.buf(prefix + "lo", bytes);
  DBuf& hi = c.buf(prefix + "hi", bytes);
  c.h2d(lo.p, ws->obs_lo, bytes);
  c.h2d(hi.p, ws->obs_hi, bytes);
  w.d_lo = lo.as<double>();
  w.d_hi = hi.as<double>();
  return w;
}

}  // namespace pumpg

extern "C" {

const char* pump_last_error(void) { return pumpg::last_error().c_str(); }
int pump_abi_version(void) { return 1; }

int pump_ctx_create(int device, pump_ctx** out) {
  return guard([&] {
    int n = 0;
    PUMP_CUDA(cudaGetDeviceCount(&n));
    if (device < 0 || device >= n) throw CudaError("pump_ctx_create: no such CUDA device");
    cudaDeviceProp prop;
    PUMP_CUDA(cudaGetDeviceProperties(&prop, device));
    if (prop.major != 10) throw CudaError("pump_ctx_create: libpump_gpu.so is built for sm_100a (B200) only");
    PUMP_CUDA(cudaSetDevice(device));
    auto* x = new pump_ctx;
    x->c.device = device;
    // the main chain runs at the highest priority, the side stream (bank, MC
    // table) at the lowest: its blocks fill idle SMs without delaying the
    // latency-critical main-chain kernels queued behind them
    int prio_low = 0, prio_high = 0;
    PUMP_CUDA(cudaDeviceGetStreamPriorityRange(&prio_low, &prio_high));
    PUMP_CUDA(cudaStreamCreateWithPriority(&x->c.stream, cudaStreamNonBlocking, prio_high));
    PUMP_CUDA(cudaStreamCreateWithPriority(&x->c.side, cudaStreamNonBlocking, prio_low));
    PUMP_CUDA(cudaEventCreate(&x->c.ev0));
    PUMP_CUDA(cudaEventCreate(&x->c.ev1));
    PUMP_CUDA(cudaEventCreateWithFlags(&x->c.fork, cudaEventDisableTiming));
    PUMP_CUDA(cudaEventCreateWithFlags(&x->c.join, cudaEventDisableTiming));
    *out = x;
  });
}

int pump_ctx_destroy(pump_ctx* ctx) {
  return guard([&] {
    if (!ctx) return;
    cudaSetDevice(ctx->c.device);
    cudaStreamSynchronize(ctx->c.stream);
    comm_destroy(ctx->c);
    ctx->c.scratch.clear();
    ctx->c.run_graph.reset();
    ctx->c.run_explore.reset();
    ctx->c.bank.release();
    cudaEventDestroy(ctx->c.ev0);
    cudaEventDestroy(ctx->c.ev1);
    cudaEventDestroy(ctx->c.fork);
    cudaEventDestroy(ctx->c.join);
    cudaStreamDestroy(ctx->c.side);
    cudaStreamDestroy(ctx->c.stream);
    delete ctx;
  });
}

double pump_ctx_last_kernel_ms(pump_ctx* ctx) { return ctx ? ctx->c.last_ms : 0.0; }
int64_t pump_ctx_launch_count(pump_ctx* ctx) { return ctx ? ctx->c.launches : 0; }
int pump_ctx_stream(pump_ctx* ctx, void** stream_out) {
  if (!ctx || !stream_out) return PUMP_E_INVALID_ARGUMENT;
  *stream_out = static_cast<void*>(ctx->c.stream);
  return PUMP_OK;
}

// ------------------------------------------------------------- scenario
int pump_scenario_parse(const char* json_text, pump_scenario** out) {
  return guard([&] {
    auto* s = new pump_scenario;
    try {
      const char* t = json_text ? json_text : "";
      auto fast = pumpb::parse_scenario_fast(t);  // the strict fast reader, else the nlohmann path (same errors)
      s->s = fast ? std::move(*fast) : pumpb::parse_scenario_text(t);
    } catch (...) {
      delete s;
      throw;
    }
    *out = s;
  });
}

int pump_scenario_load(const char* path, pump_scenario** out) {
  return guard([&] {
    auto* s = new pump_scenario;
    try {
      s->s = pumpb::load_scenario(path ? path : "");
    } catch (...) {
      delete s;
      throw;
    }
    *out = s;
  });
}

int pump_scenario_free(pump_scenario* s) {
  delete s;
  return PUMP_OK;
}

int pump_scenario_closed_loop(const pump_scenario* s, int32_t* d, int32_t* dw, double* F, double* Gv, double* Gw,
                              double* Sv, double* Sw, double* S0, double* Cm) {
  return guard([&] {
    *dw = s->s.workspace_dim();
    *d = 2 * *dw;
    if (!F) return;
    pumpb::ClosedLoop cl = s->s.models().cl;
    std::memcpy(F, cl.F.a.data(), cl.F.a.size() * 8);
    std::memcpy(Gv, cl.Gv.a.data(), cl.Gv.a.size() * 8);
    std::memcpy(Gw, cl.Gw.a.data(), cl.Gw.a.size() * 8);
    std::memcpy(Sv, cl.Sv.a.data(), cl.Sv.a.size() * 8);
    std::memcpy(Sw, cl.Sw.a.data(), cl.Sw.a.size() * 8);
    std::memcpy(S0, cl.S0.a.data(), cl.S0.a.size() * 8);
    std::memcpy(Cm, cl.C.a.data(), cl.C.a.size() * 8);
  });
}

int pump_scenario_params(const pump_scenario* s, double out[8], int64_t iout[8]) {
  return guard([&] {
    const auto& x = s->s;
    out[0] = x.effective_eps_cc();
    out[1] = x.effective_r_n();
    out[2] = x.effective_tau_max();
    out[3] = x.alpha;
    out[4] = x.effective_eta();
    out[5] = x.lambda;
    out[6] = x.dt;
    out[7] = x.max_speed;
    iout[0] = x.samples;
    iout[1] = x.particles;
    iout[2] = x.mc_samples;
    iout[3] = x.bank_horizon;
    iout[4] = static_cast<int64_t>(x.seeds.bank);
    iout[5] = static_cast<int64_t>(x.seeds.mc);
    iout[6] = static_cast<int64_t>(x.seeds.rrt);
    iout[7] = x.workspace_dim();
  });
}

// ------------------------------------------------------------------ bank
int pump_presample_bank(pump_ctx* ctx, const pump_closed_loop* cl, int32_t t_max, int32_t n, uint64_t seed,
                        double* dy_out) {
  return guard([&] {
    Ctx& c = ctx->c;
    HostLoop L = host_loop(cl);
    if (n < 1) throw std::invalid_argument("presample_bank: need at least one particle");
    if (t_max < 1) throw std::invalid_argument("presample_bank: horizon must be at least 1");
    const size_t bytes = static_cast<size_t>(t_max + 1) * n * L.dw * sizeof(double);
    c.bank.ensure(bytes);
    DBuf& scr = c.buf("bank_scratch", bank_scratch_bytes(L, n, t_max));
    c.tic();
    launch_bank(L, n, t_max, seed, c.bank.as<double>(), scr.p, c.stream, &c.launches);
    c.toc();
    c.bank_n = n;
    c.bank_horizon = t_max;
    c.bank_dw = L.dw;
    if (dy_out) {
      c.d2h(dy_out, c.bank.p, bytes);
      c.sync();
    }
  });
}

int pump_bank_upload(pump_ctx* ctx, int32_t n, int32_t horizon, int32_t dw, const double* dy) {
  return guard([&] {
    Ctx& c = ctx->c;
    if (n < 1 || horizon < 0 || dw < 1) throw std::invalid_argument("bank_upload: bad dimensions");
    const size_t bytes = static_cast<size_t>(horizon + 1) * n * dw * sizeof(double);
    c.bank.ensure(bytes);
    c.h2d(c.bank.p, dy, bytes);
    c.sync();
    c.bank_n = n;
    c.bank_horizon = horizon;
    c.bank_dw = dw;
  });
}

// ------------------------------------------------------------------ hsmc
int pump_hsmc_extend_batch(pump_ctx* ctx, int64_t n_tasks, int32_t n_words, const uint64_t* masks_in,
                           const int64_t* step_off, const int32_t* step_t, const int64_t* step_hs_off,
                           const double* hs_a, const double* hs_b, uint64_t* masks_out, int32_t* popcount_out) {
  return guard([&] {
    Ctx& c = ctx->c;
    if (!c.bank.p) throw std::invalid_argument("hsmc_extend: no particle bank in this context");
    if (n_tasks <= 0) return;
    const int64_t n_steps = step_off[n_tasks];
    const int64_t n_hs = n_steps > 0 ? step_hs_off[n_steps] : 0;
    const int dw = c.bank_dw;
    char* base;
    const size_t b_in = n_tasks * n_words * 8, b_off = (n_tasks + 1) * 8, b_t = n_steps * 4,
                 b_hoff = (n_steps + 1) * 8, b_a = n_hs * dw * 8, b_b = n_hs * 8, b_pop = n_tasks * 4;
    auto al = [](size_t x) { return (x + 255) & ~size_t(255); };
    const size_t total = al(b_in) * 2 + al(b_off) + al(b_t) + al(b_hoff) + al(b_a) + al(b_b) + al(b_pop) + 256;
    DBuf& B = c.buf("hsmc_batch", total);
    base = B.as<char>();
    auto take = [&](size_t bytes) {
      char* p = base;
      base += al(bytes);
      return p;
    };
    uint64_t* d_in = reinterpret_cast<uint64_t*>(take(b_in));
    uint64_t* d_out = reinterpret_cast<uint64_t*>(take(b_in));
    int64_t* d_off = reinterpret_cast<int64_t*>(take(b_off));
    int32_t* d_t = reinterpret_cast<int32_t*>(take(b_t));
    int64_t* d_hoff = reinterpret_cast<int64_t*>(take(b_hoff));
    double* d_a = reinterpret_cast<double*>(take(b_a));
    double* d_b = reinterpret_cast<double*>(take(b_b));
    int32_t* d_pop = reinterpret_cast<int32_t*>(take(b_pop));
    int* d_err = reinterpret_cast<int*>(take(4));
    c.h2d(d_in, masks_in, b_in);
    c.h2d(d_off, step_off, b_off);
    c.h2d(d_t, step_t, b_t);
    c.h2d(d_hoff, step_hs_off, b_hoff);
    c.h2d(d_a, hs_a, b_a);
    c.h2d(d_b, hs_b, b_b);
    PUMP_CUDA(cudaMemsetAsync(d_err, 0, 4, c.stream));
    c.tic();
    launch_hsmc_batch(dw, c.bank_n, c.bank_horizon, c.bank.as<double>(), n_tasks, n_words, d_in, d_off, d_t, d_hoff,
                      d_a, d_b, d_out, d_pop, d_err, c.stream, &c.launches);
    c.toc();
    int err = 0;
    c.d2h(&err, d_err, 4);
    c.d2h(masks_out, d_out, b_in);
    c.d2h(popcount_out, d_pop, b_pop);
    c.sync();
    if (err) throw std::out_of_range("hsmc_extend: plan exceeds bank horizon");
  });
}

// -------------------------------------------------------------------- mc
int pump_mc_certify_batch(pump_ctx* ctx, const pump_closed_loop* cl, const pump_workspace* ws, int32_t n_traj,
                          const int64_t* traj_off, const double* y_nom, int64_t rollout_lo, int64_t rollout_hi,
                          uint64_t seed, double eps_cc, int64_t* hits_out) {
  return guard([&] {
    Ctx& c = ctx->c;
    HostLoop L = host_loop(cl);
    if (n_traj < 0) throw std::invalid_argument("mc_certify: negative trajectory count");
    int max_pts = 0;
    for (int j = 0; j < n_traj; ++j) {
      const int64_t np = traj_off[j + 1] - traj_off[j];
      if (np < 1) throw std::invalid_argument("mc_certify: empty trajectory");
      max_pts = std::max<int>(max_pts, static_cast<int>(np));
    }
    if (n_traj == 0) return;
    DevWorld w = upload_world(c, ws, "mc_ws_");
    const int64_t n_pts = traj_off[n_traj];
    DBuf& off = c.buf("mc_off", (n_traj + 1) * 8);
    DBuf& yn = c.buf("mc_ynom", n_pts * L.dw * 8);
    DBuf& hits = c.buf("mc_hits", (n_traj + 1) * 8);
    c.h2d(off.p, traj_off, (n_traj + 1) * 8);
    c.h2d(yn.p, y_nom, n_pts * L.dw * 8);
    PUMP_CUDA(cudaMemsetAsync(hits.p, 0, (n_traj + 1) * 8, c.stream));
    c.tic();
    // certify against a common-random-number table built within this call
    // (not kept across calls); its parallel noise phase beats the fused
    // kernel even for one trajectory.  PUMP_MC_DIRECT=1 forces the fused
    // kernels (tests/test_gpu_kernels.py checks both paths).
    c.mc_table.invalidate();
    launch_mc(L, w, n_traj, off.as<int64_t>(), yn.as<double>(), max_pts, rollout_lo, rollout_hi, seed, eps_cc,
              hits.as<unsigned long long>(), c.stream, &c.launches, hits.as<unsigned long long>() + n_traj,
              &c.mc_table);
    c.toc();
    std::vector<int64_t> hv(n_traj + 1);
    c.d2h(hv.data(), hits.p, (n_traj + 1) * 8);
    c.sync();
    std::copy(hv.begin(), hv.begin() + n_traj, hits_out);
    kprof_work(F_MC, hv[n_traj]);
    c.mc_rollout_steps += hv[n_traj];
  });
}

int pump_mc_certify(pump_ctx* ctx, const pump_closed_loop* cl, const pump_workspace* ws, int32_t n_points,
                    const double* y_nom, int32_t n_mc, uint64_t seed, double eps_cc, double* value_out) {
  if (n_mc < 1) return fail(PUMP_E_INVALID_ARGUMENT, "mc_certify: need at least one rollout");
  if (n_points < 1) return fail(PUMP_E_INVALID_ARGUMENT, "mc_certify: empty trajectory");
  int64_t off[2] = {0, n_points};
  int64_t hits = 0;
  int rc = pump_mc_certify_batch(ctx, cl, ws, 1, off, y_nom, 0, n_mc, seed, eps_cc, &hits);
  if (rc == PUMP_OK) *value_out = static_cast<double>(hits) / n_mc;
  return rc;
}

}  // extern "C"

// ------------------------------------------------------ measurement hooks
namespace pumpg {

KProf*& kprof_current() {
  static KProf* p = nullptr;
  return p;
}

// FP64 issue-rate microbenchmark: 8 independent DMUL+DADD chains per thread
// (no FMA: --fmad=false), the op mix of the parity-bound kernels.
__global__ void __launch_bounds__(256) k_peak_fp64(double* out, int iters, double a, double b) {
  double x[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) x[k] = threadIdx.x * 1e-3 + k;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int k = 0; k < 8; ++k) x[k] = x[k] * a + b;  // DMUL + DADD (no contraction)
  }
  double s = 0;
#pragma unroll
  for (int k = 0; k < 8; ++k) s += x[k];
  if (s == 12345.678) out[0] = s;  // keep the work alive
}

__global__ void k_flush(uint4* p, size_t n) {
  for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<size_t>(gridDim.x) * blockDim.x)
    p[i] = make_uint4(static_cast<unsigned>(i), 0u, 0u, 0u);
}

}  // namespace pumpg

extern "C" {

int pump_ctx_profile(pump_ctx* ctx, int enable) {
  return guard([&] {
    KProf& p = ctx->c.prof;
    p.on = enable != 0;
    kprof_current() = enable ? &p : nullptr;
    if (enable) {
      for (int f = 0; f < F_COUNT; ++f) {
        p.ms[f] = 0;
        p.count[f] = 0;
        p.work[f] = 0;
      }
    }
  });
}

// per kernel family: total ms, launches, work units (resets the totals)
int pump_ctx_profile_read(pump_ctx* ctx, double* ms, int64_t* counts, int64_t* work) {
  return guard([&] {
    Ctx& c = ctx->c;
    c.sync();
    KProf& p = c.prof;
    p.resolve();
    for (int f = 0; f < F_COUNT; ++f) {
      ms[f] = p.ms[f];
      counts[f] = p.count[f];
      work[f] = p.work[f];
      p.ms[f] = 0;
      p.count[f] = 0;
      p.work[f] = 0;
    }
  });
}

int pump_ctx_io_bytes(pump_ctx* ctx, int64_t* out) {
  out[0] = ctx->c.h2d_bytes;
  out[1] = ctx->c.d2h_bytes;
  out[2] = ctx->c.mc_rollout_steps;
  out[3] = g_dev_allocs;
  out[4] = ctx->c.collectives;
  return PUMP_OK;
}

// Overwrite a buffer larger than the 126 MB L2 (cold-cache timing hygiene).
int pump_ctx_flush_l2(pump_ctx* ctx) {
  return guard([&] {
    Ctx& c = ctx->c;
    const size_t bytes = size_t(256) << 20;
    DBuf& b = c.buf("l2_flush", bytes);
    k_flush<<<148 * 8, 256, 0, c.stream>>>(b.as<uint4>(), bytes / sizeof(uint4));
    ++c.launches;
    PUMP_CUDA(cudaGetLastError());
    c.sync();
  });
}

// Measured FP64 (DMUL/DADD, no FMA) issue rate in Gop/s.
int pump_peak_fp64(pump_ctx* ctx, double* gops) {
  return guard([&] {
    Ctx& c = ctx->c;
    DBuf& o = c.buf("peak_out", 256);
    const int blocks = 148 * 16, threads = 256, iters = 4096;
    k_peak_fp64<<<blocks, threads, 0, c.stream>>>(o.as<double>(), 64, 0.999, 1e-3);  // warm-up
    c.tic();
    k_peak_fp64<<<blocks, threads, 0, c.stream>>>(o.as<double>(), iters, 0.999, 1e-3);
    const double ms = c.toc();
    c.launches += 2;
    const double ops = 2.0 * 8 * iters * static_cast<double>(blocks) * threads;
    *gops = ops / (ms * 1e-3) / 1e9;
  });
}

}  // extern "C"
