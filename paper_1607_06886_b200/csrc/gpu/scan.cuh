// Device-wide ordered primitives used by graph build and the explore
// wavefront: exclusive prefix scan (3 kernels, warp-shuffle scans inside a
// tile) and a stable multisplit by a small key (frontier compaction in
// (bucket, id) order).  Hand-written; no CUB.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace pumpg {

constexpr int kScanBlock = 512;
constexpr int kScanItems = 8;
constexpr int kScanTile = kScanBlock * kScanItems;  // 4096

// Bytes of temporary storage needed by exclusive_scan for n items.
size_t scan_temp_bytes(int64_t n);

// out[0..n] = exclusive prefix sums of in[0..n) (out[n] = total), int64.
// If d_n is given the item count is read on the device (n is then only the
// upper bound used to size the grid).
// InT is int32_t, int64_t or uint8_t.  Stream-ordered, no host sync.
template <class InT>
void exclusive_scan(const InT* d_in, int64_t* d_out, int64_t n, void* d_temp, cudaStream_t st, int64_t* launches,
                    const int64_t* d_n = nullptr);

// Stable multisplit: given n items with keys in [0, n_keys) (key < 0 means
// "drop"), writes the values ordered by (key, original position) into out,
// and the number of kept items to *d_count.  n_keys <= 1024.
size_t multisplit_temp_bytes(int64_t n, int n_keys);
void stable_multisplit(const int32_t* d_keys, const int32_t* d_vals, int64_t n, int n_keys, int32_t* d_out,
                       int64_t* d_count, void* d_temp, cudaStream_t st, int64_t* launches,
                       const int64_t* d_n = nullptr);

// ------------------------------------------------------------ warp helpers
__device__ __forceinline__ int64_t warp_incl_scan(int64_t x) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    int64_t y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  return x;
}

__device__ __forceinline__ int64_t warp_sum(int64_t x) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
  return x;
}

}  // namespace pumpg
