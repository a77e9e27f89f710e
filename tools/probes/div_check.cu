// Empirical check of the shared-reciprocal division used by steer_cost_fast:
// q = RN(a y), r = fma(-b, q, a), q' = fma(r, y, q) with y = RN(1/b) against
// the IEEE quotient a / b, over random operands spanning the magnitudes the
// cost terms take (and integer-ish / power-of-two edge cases).
// nvcc -O3 -gencode arch=compute_100a,code=sm_100a --fmad=false div_check.cu -o div_check
#include <cstdio>
#include <cstdint>
__device__ __forceinline__ uint64_t mix(uint64_t x) {
  x ^= x >> 30; x *= 0xbf58476d1ce4e5b9ULL; x ^= x >> 27; x *= 0x94d049bb133111ebULL; x ^= x >> 31; return x;
}
__global__ void k(uint64_t seed, int64_t n, unsigned long long* bad, unsigned long long* total) {
  unsigned long long nb = 0, nt = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    uint64_t h1 = mix(seed + 2 * i), h2 = mix(seed + 2 * i + 1);
    // mantissas random, exponents in [-80, 80] for b (tau^3, tau^2, tau) and a
    double ma = 1.0 + (h1 >> 12) * 0x1p-52, mb = 1.0 + (h2 >> 12) * 0x1p-52;
    int ea = (int)((h1 & 0xff) % 161) - 80, eb = (int)(((h1 >> 8) & 0xff) % 161) - 80;
    if ((h2 & 7) == 0) mb = 1.0;                       // powers of two
    if ((h2 & 0x38) == 0) ma = (double)((h1 >> 20) & 0xffff);  // small integers
    double a = ldexp(ma, ea) * ((h2 >> 60) & 1 ? -1.0 : 1.0), b = ldexp(mb, eb);
    double y = 1.0 / b;
    double q = a * y;
    double r = fma(-b, q, a);
    double qq = fma(r, y, q);
    double ref = a / b;
    nt++;
    if (__double_as_longlong(qq) != __double_as_longlong(ref)) nb++;
  }
  atomicAdd(bad, nb);
  atomicAdd(total, nt);
}
int main() {
  unsigned long long *d, h[2];
  cudaMalloc(&d, 16);
  for (int rep = 0; rep < 20; ++rep) {
    cudaMemset(d, 0, 16);
    k<<<148 * 16, 256>>>(1234567ull + rep * 1000003ull, 1ll << 28, d, d + 1);
    cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
    printf("rep %d: %llu mismatches of %llu\n", rep, h[0], h[1]);
  }
  return 0;
}
