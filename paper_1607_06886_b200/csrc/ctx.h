// pump_ctx internals: device, stream, events and grow-only device buffers.
#pragma once

#include <cstring>
#include <map>
#include <string>

#include "gpu/kernels.h"
#include "host/scenario.hpp"

namespace pumpg {

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
    cap = want;
  }
  // grow keeping the first `keep` bytes
  void grow(size_t bytes, size_t keep, cudaStream_t st) {
    if (bytes <= cap) return;
    void* q = nullptr;
    size_t want = bytes + bytes / 2;
    PUMP_CUDA(cudaMalloc(&q, want));
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

struct Ctx {
  int device = 0;
  cudaStream_t stream = nullptr;
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  int64_t launches = 0;
  double last_ms = 0;
  // resident particle bank
  DBuf bank;
  int bank_n = 0, bank_horizon = 0, bank_dw = 0;
  // named scratch buffers
  std::map<std::string, DBuf> scratch;
  DBuf& buf(const std::string& name, size_t bytes) {
    DBuf& b = scratch[name];
    b.ensure(bytes);
    return b;
  }
  void sync() { PUMP_CUDA(cudaStreamSynchronize(stream)); }
  void h2d(void* d, const void* h, size_t bytes) {
    if (bytes) PUMP_CUDA(cudaMemcpyAsync(d, h, bytes, cudaMemcpyHostToDevice, stream));
  }
  void d2h(void* h, const void* d, size_t bytes) {
    if (bytes) PUMP_CUDA(cudaMemcpyAsync(h, d, bytes, cudaMemcpyDeviceToHost, stream));
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

// Upload a workspace into ctx scratch buffers named prefix+"lo"/"hi".
DevWorld upload_world(Ctx& c, const pump_workspace* ws, const std::string& prefix);

}  // namespace pumpg

struct pump_ctx {
  pumpg::Ctx c;
};
struct pump_scenario {
  pumpb::Scenario s;
};
