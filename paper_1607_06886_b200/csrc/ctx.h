// pump_ctx internals: device, stream, events and grow-only device buffers.
#pragma once

#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <string>

#include "gpu/kernels.h"
#include "host/scenario.hpp"

#include <memory>

namespace pumpg {

struct DevGraph;
struct DevExplore;



struct Ctx {
  int device = 0;
  cudaStream_t stream = nullptr;
  // side stream for work independent of the main chain (the particle bank
  // overlaps the graph build); fork/join events order it against `stream`
  cudaStream_t side = nullptr;
  cudaEvent_t fork = nullptr, join = nullptr;
  bool mc_join_pending = false;  // the MC table was built on `side`: wait before certifying
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  int64_t launches = 0;
  double last_ms = 0;
  int64_t h2d_bytes = 0, d2h_bytes = 0, mc_rollout_steps = 0, collectives = 0;
  // multi-GPU: NCCL communicator for the sharded MC certification
  void* nccl = nullptr;
  int rank = 0, world = 1;
  // or host collectives supplied by the caller (pump_ctx_set_collectives):
  // device data is staged through host memory around each call
  pump_allreduce_i64_fn host_ar = nullptr;
  pump_gather_fn host_gather = nullptr;
  void* host_user = nullptr;
  bool has_comm() const { return world > 1 && (nccl != nullptr || host_ar != nullptr); }
  KProf prof;
  // resident particle bank
  DBuf bank;
  int bank_n = 0, bank_horizon = 0, bank_dw = 0;
  // persistent solve state of run_pump (graph + explore arena stay resident
  // in HBM across solves: no per-solve cudaMalloc/cudaFree)
  std::shared_ptr<DevGraph> run_graph;
  std::shared_ptr<DevExplore> run_explore;
  // common-random-number table of the MC rollouts (kernels.h)
  McTable mc_table;
  // named scratch buffers
  std::map<std::string, DBuf> scratch;
  double lbgrid_rn = -1.0;  // r_n of the interval table in scratch "g_lbgrid" (graph.cu)
  DBuf& buf(const std::string& name, size_t bytes) {
    DBuf& b = scratch[name];
    if (bytes > b.cap && std::getenv("PUMP_DEBUG_ALLOC")) std::fprintf(stderr, "[pump alloc] scratch %s\n", name.c_str());
    b.ensure(bytes);
    return b;
  }
  void sync() { PUMP_CUDA(cudaStreamSynchronize(stream)); }
  void h2d(void* d, const void* h, size_t bytes) {
    if (bytes) PUMP_CUDA(cudaMemcpyAsync(d, h, bytes, cudaMemcpyHostToDevice, stream));
    h2d_bytes += static_cast<int64_t>(bytes);
  }
  void d2h(void* h, const void* d, size_t bytes) {
    if (bytes) PUMP_CUDA(cudaMemcpyAsync(h, d, bytes, cudaMemcpyDeviceToHost, stream));
    d2h_bytes += static_cast<int64_t>(bytes);
  }
  void tic() { PUMP_CUDA(cudaEventRecord(ev0, stream)); }
  double toc() {
    PUMP_CUDA(cudaEventRecord(ev1, stream));
    PUMP_CUDA(cudaEventSynchronize(ev1));
    float ms = 0;
    PUMP_CUDA(cudaEventElapsedTime(&ms, ev0, ev1));
    last_ms = ms;
    return ms;
  }
};

void shard_range(int64_t n, int rank, int world, int64_t* lo, int64_t* hi);
void allreduce_sum_i64(Ctx& c, int64_t* d, size_t count);
void gather_segments(Ctx& c, const void* send, void* recv, const std::vector<int64_t>& off,
                     const std::vector<int64_t>& len);
void comm_destroy(Ctx& c);

// Upload a workspace into ctx scratch buffers named prefix+"lo"/"hi".
DevWorld upload_world(Ctx& c, const pump_workspace* ws, const std::string& prefix);

}  // namespace pumpg

struct pump_ctx {
  pumpg::Ctx c;
};
struct pump_scenario {
  pumpb::Scenario s;
};
