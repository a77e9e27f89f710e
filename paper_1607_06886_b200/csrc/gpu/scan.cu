// Ordered device primitives (see scan.cuh).
#include <cstdlib>
#include <stdexcept>

#include "kernels.h"
#include "scan.cuh"

namespace pumpg {

// Single-pass scan with decoupled look-back: each CTA takes a ticket (tile
// order independent of block scheduling), publishes its tile aggregate, then
// resolves its exclusive prefix from its predecessors' published words
// (aggregate or inclusive prefix, flag in the top 2 bits of one 64-bit word,
// so a single aligned store publishes both).  The status words and the
// ticket are zeroed by one memset before the launch.  Values are counts:
// non-negative and < 2^62.
constexpr uint64_t kStAgg = 1ull << 62, kStInc = 2ull << 62, kStVal = (1ull << 62) - 1;

template <class InT>
__global__ void __launch_bounds__(kScanBlock) k_scan_lookback(const InT* __restrict__ in, int64_t n,
                                                              int64_t* __restrict__ out, uint64_t* __restrict__ status,
                                                              unsigned* __restrict__ ticket, const int64_t* d_n) {
  __shared__ int64_t tile[kScanTile];
  __shared__ int64_t wsum[kScanBlock / 32];
  __shared__ int64_t s_prefix;
  __shared__ unsigned s_tile;
  if (d_n) n = min(n, *d_n);
  // one tile (ticket == nullptr): no predecessors, no status, no memset
  if (threadIdx.x == 0) s_tile = ticket ? atomicAdd(ticket, 1u) : 0u;
  __syncthreads();
  const unsigned t = s_tile;
  const int64_t base = static_cast<int64_t>(t) * kScanTile;
  if (base >= n && !(n <= 0 && t == 0)) return;  // beyond the device-side count
#pragma unroll
  for (int k = 0; k < kScanItems; ++k) {
    const int64_t i = base + k * kScanBlock + threadIdx.x;
    tile[k * kScanBlock + threadIdx.x] = i < n ? static_cast<int64_t>(in[i]) : 0;
  }
  __syncthreads();
  int64_t v[kScanItems];
  int64_t s = 0;
#pragma unroll
  for (int k = 0; k < kScanItems; ++k) {
    v[k] = tile[threadIdx.x * kScanItems + k];
    s += v[k];
  }
  const int64_t inc = warp_incl_scan(s);
  if ((threadIdx.x & 31) == 31) wsum[threadIdx.x >> 5] = inc;
  __syncthreads();
  if (threadIdx.x < 32) {
    int64_t w = threadIdx.x < kScanBlock / 32 ? wsum[threadIdx.x] : 0;
    const int64_t wi = warp_incl_scan(w);
    if (threadIdx.x < kScanBlock / 32) wsum[threadIdx.x] = wi - w;
    const int64_t agg = __shfl_sync(0xffffffffu, wi, 31);
    // publish, then look back (warp 0)
    volatile uint64_t* vs = status;
    if (t == 0) {
      if (threadIdx.x == 0) {
        if (ticket) vs[0] = kStInc | static_cast<uint64_t>(agg);
        s_prefix = 0;
      }
    } else {
      if (threadIdx.x == 0) vs[t] = kStAgg | static_cast<uint64_t>(agg);
      int64_t prefix = 0;
      int64_t j = static_cast<int64_t>(t) - 1 - threadIdx.x;  // this lane's predecessor
      while (true) {
        uint64_t w2 = j >= 0 ? vs[j] : static_cast<uint64_t>(kStInc);  // before tile 0: inclusive 0
        while (__any_sync(0xffffffffu, (w2 >> 62) == 0)) {
          if ((w2 >> 62) == 0) w2 = vs[j];
        }
        const unsigned incm = __ballot_sync(0xffffffffu, (w2 >> 62) == 2);
        // lanes up to (and including) the nearest inclusive word contribute
        const int stop = incm ? __ffs(incm) - 1 : 31;
        int64_t val = (static_cast<int>(threadIdx.x) <= stop) ? static_cast<int64_t>(w2 & kStVal) : 0;
        val = warp_sum(val);
        prefix += val;
        if (incm) break;
        j -= 32;
      }
      if (threadIdx.x == 0) {
        vs[t] = kStInc | static_cast<uint64_t>(prefix + agg);
        s_prefix = prefix;
      }
    }
    if (threadIdx.x == 0 && base + kScanTile >= n) out[n > 0 ? n : 0] = s_prefix + agg;  // total (last tile)
  }
  __syncthreads();
  int64_t run = s_prefix + wsum[threadIdx.x >> 5] + inc - s;
#pragma unroll
  for (int k = 0; k < kScanItems; ++k) {
    tile[threadIdx.x * kScanItems + k] = run;
    run += v[k];
  }
  __syncthreads();
#pragma unroll
  for (int k = 0; k < kScanItems; ++k) {
    const int64_t i = base + k * kScanBlock + threadIdx.x;
    if (i < n) out[i] = tile[k * kScanBlock + threadIdx.x];
  }
}

size_t scan_temp_bytes(int64_t n) { return static_cast<size_t>((n + kScanTile - 1) / kScanTile + 1) * 8 + 256; }

template <class InT>
void exclusive_scan(const InT* d_in, int64_t* d_out, int64_t n, void* d_temp, cudaStream_t st, int64_t* launches,
                    const int64_t* d_n) {
  if (n <= 0) {
    PUMP_CUDA(cudaMemsetAsync(d_out, 0, sizeof(int64_t), st));
    return;
  }
  const int64_t tiles = (n + kScanTile - 1) / kScanTile;
  uint64_t* status = reinterpret_cast<uint64_t*>(static_cast<char*>(d_temp) + 256);
  unsigned* ticket = static_cast<unsigned*>(d_temp);
  KScope ks(st, F_SCAN);
  if (tiles == 1) {
    k_scan_lookback<InT><<<1, kScanBlock, 0, st>>>(d_in, n, d_out, status, nullptr, d_n);
    *launches += 1;
  } else {
    PUMP_CUDA(cudaMemsetAsync(d_temp, 0, 256 + static_cast<size_t>(tiles) * 8, st));
    k_scan_lookback<InT><<<static_cast<unsigned>(tiles), kScanBlock, 0, st>>>(d_in, n, d_out, status, ticket, d_n);
    *launches += 1;
  }
  PUMP_CUDA(cudaGetLastError());
}

template void exclusive_scan<int32_t>(const int32_t*, int64_t*, int64_t, void*, cudaStream_t, int64_t*,
                                      const int64_t*);
template void exclusive_scan<int64_t>(const int64_t*, int64_t*, int64_t, void*, cudaStream_t, int64_t*,
                                      const int64_t*);
template void exclusive_scan<uint8_t>(const uint8_t*, int64_t*, int64_t, void*, cudaStream_t, int64_t*,
                                      const int64_t*);

// ------------------------------------------------------------ multisplit
constexpr int kMsBlock = 512;
constexpr int kMsItems = 8;
constexpr int kMsTile = kMsBlock * kMsItems;
constexpr int kMsKeys = 512;  // keys per pass
constexpr int kMsWarps = kMsBlock / 32;

__device__ __forceinline__ int ms_digit(int key, int shift) { return key < 0 ? -1 : ((key >> shift) & (kMsKeys - 1)); }

__global__ void __launch_bounds__(kMsBlock) k_ms_hist(const int32_t* __restrict__ keys, int64_t n, int shift,
                                                      int n_tiles, int32_t* __restrict__ counts, const int64_t* d_n) {
  __shared__ int hist[kMsKeys];
  if (d_n) n = min(n, *d_n);
  for (int k = threadIdx.x; k < kMsKeys; k += kMsBlock) hist[k] = 0;
  __syncthreads();
  const int64_t base = static_cast<int64_t>(blockIdx.x) * kMsTile;
  for (int s = 0; s < kMsItems; ++s) {
    const int64_t i = base + s * kMsBlock + threadIdx.x;
    if (i < n) {
      const int d = ms_digit(keys[i], shift);
      if (d >= 0) atomicAdd(&hist[d], 1);
    }
  }
  __syncthreads();
  for (int k = threadIdx.x; k < kMsKeys; k += kMsBlock) counts[static_cast<int64_t>(k) * n_tiles + blockIdx.x] = hist[k];
}

__global__ void __launch_bounds__(kMsBlock) k_ms_scatter(const int32_t* __restrict__ keys,
                                                         const int32_t* __restrict__ vals, int64_t n, int shift,
                                                         int n_tiles, const int64_t* __restrict__ offs,
                                                         int32_t* __restrict__ okeys, int32_t* __restrict__ ovals,
                                                         const int64_t* d_n) {
  __shared__ int wcnt[kMsWarps][kMsKeys];
  if (d_n) n = min(n, *d_n);
  __shared__ int64_t run[kMsKeys];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int k = threadIdx.x; k < kMsKeys; k += kMsBlock) {
    run[k] = offs[static_cast<int64_t>(k) * n_tiles + blockIdx.x];
    for (int w = 0; w < kMsWarps; ++w) wcnt[w][k] = 0;
  }
  __syncthreads();
  const int64_t base = static_cast<int64_t>(blockIdx.x) * kMsTile;
  const unsigned lt = (1u << lane) - 1u;
  for (int s = 0; s < kMsItems; ++s) {
    const int64_t i = base + s * kMsBlock + threadIdx.x;
    const int key = i < n ? keys[i] : -1;
    const int d = ms_digit(key, shift);
    const unsigned peers = __match_any_sync(0xffffffffu, d);
    const int rank = __popc(peers & lt);
    if (d >= 0 && rank == 0) wcnt[warp][d] = __popc(peers);
    __syncthreads();
    if (d >= 0) {
      int64_t pos = run[d] + rank;
      for (int w = 0; w < warp; ++w) pos += wcnt[w][d];
      okeys[pos] = key;
      ovals[pos] = vals[i];
    }
    __syncthreads();
    for (int k = threadIdx.x; k < kMsKeys; k += kMsBlock) {
      int t = 0;
      for (int w = 0; w < kMsWarps; ++w) {
        t += wcnt[w][k];
        wcnt[w][k] = 0;
      }
      run[k] += t;
    }
    __syncthreads();
  }
}

static inline size_t al256(size_t x) { return (x + 255) & ~size_t(255); }

size_t multisplit_temp_bytes(int64_t n, int n_keys) {
  (void)n_keys;
  const int64_t tiles = (n + kMsTile - 1) / kMsTile;
  const int64_t cn = static_cast<int64_t>(kMsKeys) * (tiles > 0 ? tiles : 1);
  return al256(cn * 4) + al256((cn + 1) * 8) + al256(scan_temp_bytes(cn)) + 3 * al256((n + 1) * 4) + 256;
}

// LSD radix over 9-bit digits: one pass for n_keys <= 512, two for <= 2^18.
// Pass 1 drops negative keys; pass 2 only sees the kept items.
void stable_multisplit(const int32_t* d_keys, const int32_t* d_vals, int64_t n, int n_keys, int32_t* d_out,
                       int64_t* d_count, void* d_temp, cudaStream_t st, int64_t* launches, const int64_t* d_n) {
  if (n <= 0) {
    PUMP_CUDA(cudaMemsetAsync(d_count, 0, 8, st));
    return;
  }
  if (n_keys > kMsKeys * kMsKeys) throw std::invalid_argument("multisplit: key range too large");
  const int64_t tiles = (n + kMsTile - 1) / kMsTile;
  const int64_t cn = static_cast<int64_t>(kMsKeys) * tiles;
  char* p = static_cast<char*>(d_temp);
  int32_t* counts = reinterpret_cast<int32_t*>(p);
  p += al256(cn * 4);
  int64_t* offs = reinterpret_cast<int64_t*>(p);
  p += al256((cn + 1) * 8);
  void* stmp = p;
  p += al256(scan_temp_bytes(cn));
  int32_t* kA = reinterpret_cast<int32_t*>(p);
  p += al256((n + 1) * 4);
  int32_t* kB = reinterpret_cast<int32_t*>(p);
  p += al256((n + 1) * 4);
  int32_t* vA = reinterpret_cast<int32_t*>(p);
  const int passes = n_keys <= kMsKeys ? 1 : 2;
  const int32_t* ck = d_keys;
  const int32_t* cv = d_vals;
  const int64_t* cur_n = d_n;
  for (int pass = 0; pass < passes; ++pass) {
    const int shift = 9 * pass;
    const bool last = pass == passes - 1;
    int32_t* ok = pass == 0 ? kA : kB;
    int32_t* ov = last ? d_out : vA;
    KScope ks(st, F_SPLIT);
    k_ms_hist<<<static_cast<unsigned>(tiles), kMsBlock, 0, st>>>(ck, n, shift, static_cast<int>(tiles), counts,
                                                                  cur_n);
    exclusive_scan<int32_t>(counts, offs, cn, stmp, st, launches);
    PUMP_CUDA(cudaMemcpyAsync(d_count, offs + cn, 8, cudaMemcpyDeviceToDevice, st));
    k_ms_scatter<<<static_cast<unsigned>(tiles), kMsBlock, 0, st>>>(ck, cv, n, shift, static_cast<int>(tiles), offs,
                                                                     ok, ov, cur_n);
    *launches += 2;
    ck = ok;
    cv = ov;
    cur_n = d_count;  // pass 2 sees only the kept items
  }
  PUMP_CUDA(cudaGetLastError());
}

}  // namespace pumpg
