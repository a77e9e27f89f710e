// Multi-GPU sharding of the MC certification: rank r owns
// rollouts [n r / W, n (r+1) / W) of every certification batch and the int64
// hit counts are summed with one ncclAllReduce over NVLink.  Integer sums
// make the certified CP bit-identical for any number of ranks.  Everything
// else in the solve (graph, bank, explore) runs replicated on every rank.
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <cstring>
#include <stdexcept>
#include <vector>

#include "ctx.h"
#include "guard.h"

namespace pumpg {

// NCCL is resolved at run time (dlopen of libnccl.so.2) and only when a
// communicator is requested: linking it would bind whichever libnccl loads
// first into the process, and torch needs its own bundled release.  If torch
// already loaded NCCL, dlopen returns that very library.
struct NcclApi {
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
  ncclResult_t (*Broadcast)(const void*, void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
};

static NcclApi& nccl() {
  static NcclApi api;
  static bool loaded = false;
  if (!loaded) {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL | RTLD_NOLOAD);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) throw CudaError(std::string("cannot load libnccl.so.2: ") + dlerror());
    api.GetUniqueId = reinterpret_cast<decltype(api.GetUniqueId)>(dlsym(h, "ncclGetUniqueId"));
    api.CommInitRank = reinterpret_cast<decltype(api.CommInitRank)>(dlsym(h, "ncclCommInitRank"));
    api.AllReduce = reinterpret_cast<decltype(api.AllReduce)>(dlsym(h, "ncclAllReduce"));
    api.CommDestroy = reinterpret_cast<decltype(api.CommDestroy)>(dlsym(h, "ncclCommDestroy"));
    api.GetErrorString = reinterpret_cast<decltype(api.GetErrorString)>(dlsym(h, "ncclGetErrorString"));
    api.Broadcast = reinterpret_cast<decltype(api.Broadcast)>(dlsym(h, "ncclBroadcast"));
    api.GroupStart = reinterpret_cast<decltype(api.GroupStart)>(dlsym(h, "ncclGroupStart"));
    api.GroupEnd = reinterpret_cast<decltype(api.GroupEnd)>(dlsym(h, "ncclGroupEnd"));
    if (!api.GetUniqueId || !api.CommInitRank || !api.AllReduce || !api.CommDestroy || !api.GetErrorString ||
        !api.Broadcast || !api.GroupStart || !api.GroupEnd)
      throw CudaError("libnccl.so.2 lacks a required symbol");
    loaded = true;
  }
  return api;
}

void shard_range(int64_t n, int rank, int world, int64_t* lo, int64_t* hi) {
  *lo = n * rank / world;
  *hi = n * (rank + 1) / world;
}

void allreduce_sum_i64(Ctx& c, int64_t* d, size_t count) {
  if (!c.has_comm()) return;
  if (c.host_ar) {  // caller's host collective: stage through host memory
    std::vector<int64_t> h(count);
    c.d2h(h.data(), d, count * 8);
    c.sync();
    if (c.host_ar(c.host_user, h.data(), static_cast<int64_t>(count)) != 0)
      throw std::runtime_error("host allreduce failed");
    c.h2d(d, h.data(), count * 8);
    c.sync();
    ++c.collectives;
    return;
  }
  const ncclResult_t r = nccl().AllReduce(d, d, count, ncclInt64, ncclSum, static_cast<ncclComm_t>(c.nccl), c.stream);
  if (r != ncclSuccess) throw CudaError(std::string("ncclAllReduce: ") + nccl().GetErrorString(r));
  ++c.collectives;
}

// Concatenate per-rank segments: rank r's `len[r]` bytes at `send` land at
// byte offset off[r] of `recv` on every rank (one grouped ncclBroadcast per
// root; the root's own copy is the broadcast's send -> recv).
void gather_segments(Ctx& c, const void* send, void* recv, const std::vector<int64_t>& off,
                     const std::vector<int64_t>& len) {
  if (!c.has_comm()) throw CudaError("gather_segments: no communicator");
  if (c.host_ar) {
    if (!c.host_gather) throw std::runtime_error("gather_segments: no host gather");
    int64_t total = 0;
    for (int r = 0; r < c.world; ++r) total = std::max(total, off[r] + len[r]);
    std::vector<char> hs(static_cast<size_t>(len[c.rank]) + 1), hr(static_cast<size_t>(total) + 1);
    c.d2h(hs.data(), send, static_cast<size_t>(len[c.rank]));
    c.sync();
    if (c.host_gather(c.host_user, hs.data(), hr.data(), off.data(), len.data(), c.world) != 0)
      throw std::runtime_error("host gather failed");
    for (int r = 0; r < c.world; ++r)
      if (len[r]) c.h2d(static_cast<char*>(recv) + off[r], hr.data() + off[r], static_cast<size_t>(len[r]));
    c.sync();
    ++c.collectives;
    return;
  }
  auto& A = nccl();
  auto chk = [&](ncclResult_t r, const char* what) {
    if (r != ncclSuccess) throw CudaError(std::string(what) + ": " + A.GetErrorString(r));
  };
  chk(A.GroupStart(), "ncclGroupStart");
  for (int r = 0; r < c.world; ++r) {
    if (len[r] == 0) continue;
    chk(A.Broadcast(r == c.rank ? send : nullptr, static_cast<char*>(recv) + off[r], static_cast<size_t>(len[r]),
                    ncclChar, r, static_cast<ncclComm_t>(c.nccl), c.stream),
        "ncclBroadcast");
  }
  chk(A.GroupEnd(), "ncclGroupEnd");
  ++c.collectives;
}

void comm_destroy(Ctx& c) {
  if (c.nccl) nccl().CommDestroy(static_cast<ncclComm_t>(c.nccl));
  c.nccl = nullptr;
  c.host_ar = nullptr;
  c.host_gather = nullptr;
  c.host_user = nullptr;
  c.world = 1;
  c.rank = 0;
}

}  // namespace pumpg

using namespace pumpg;

extern "C" {

int pump_nccl_unique_id(uint8_t* out128) {
  return guard([&] {
    ncclUniqueId id;
    const ncclResult_t r = nccl().GetUniqueId(&id);
    if (r != ncclSuccess) throw CudaError(std::string("ncclGetUniqueId: ") + nccl().GetErrorString(r));
    static_assert(sizeof(id) == 128, "ncclUniqueId size");
    std::memcpy(out128, &id, 128);
  });
}

int pump_ctx_set_comm(pump_ctx* ctx, int rank, int world, const uint8_t* id128) {
  return guard([&] {
    Ctx& c = ctx->c;
    comm_destroy(c);
    if (world <= 1) return;
    if (rank < 0 || rank >= world) throw std::invalid_argument("set_comm: bad rank");
    PUMP_CUDA(cudaSetDevice(c.device));
    ncclUniqueId id;
    std::memcpy(&id, id128, 128);
    ncclComm_t comm;
    const ncclResult_t r = nccl().CommInitRank(&comm, world, id, rank);
    if (r != ncclSuccess) throw CudaError(std::string("ncclCommInitRank: ") + nccl().GetErrorString(r));
    c.nccl = comm;
    c.rank = rank;
    c.world = world;
  });
}

int pump_ctx_set_collectives(pump_ctx* ctx, int rank, int world, pump_allreduce_i64_fn allreduce,
                             pump_gather_fn gather, void* user) {
  return guard([&] {
    Ctx& c = ctx->c;
    comm_destroy(c);
    if (world <= 1 || !allreduce) return;
    if (rank < 0 || rank >= world) throw std::invalid_argument("set_collectives: bad rank");
    c.host_ar = allreduce;
    c.host_gather = gather;
    c.host_user = user;
    c.rank = rank;
    c.world = world;
  });
}

int pump_shard_range(int64_t n, int rank, int world, int64_t* lo, int64_t* hi) {
  if (world < 1 || rank < 0 || rank >= world) return PUMP_E_INVALID_ARGUMENT;
  shard_range(n, rank, world, lo, hi);
  return PUMP_OK;
}

}  // extern "C"
