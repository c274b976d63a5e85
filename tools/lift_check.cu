#include <cstdio>
#include <cstdint>
#include "paper_1810_10121_b200/csrc/hg_device.cuh"
using namespace hg;
__device__ __forceinline__ uint64_t lift_b(int64_t v, const LimbInfo& L) {
  const uint64_t a = v < 0 ? (uint64_t)(-v) : (uint64_t)v;
  uint64_t r = reduce128(a, 0, L);
  r = r >= L.q ? r - L.q : r;
  return (v < 0 && r != 0) ? L.q - r : r;
}
__global__ void k(LimbInfo L, int* bad, unsigned long long seed) {
  unsigned long long s = seed + threadIdx.x + blockIdx.x * 1000003ull;
  for (int i = 0; i < 1000; ++i) {
    s = s * 6364136223846793005ull + 1442695040888963407ull;
    int sh = (int)(s >> 58);
    int64_t v = (int64_t)(s >> (64 - sh - 1));
    if (s & 1) v = -v;
    if (lift_b(v, L) != lift_signed(v, L.q)) { if (atomicAdd(bad, 1) < 5) printf("bad q=%llu v=%lld got %llu want %llu\n", (unsigned long long)L.q, (long long)v, (unsigned long long)lift_b(v, L), (unsigned long long)lift_signed(v, L.q)); }
  }
}
int main() {
  unsigned long long ps[] = {1125899904679937ull, 1073643521ull, 1073479681ull, 68719230977ull, 67043329ull};
  int* bad; cudaMallocManaged(&bad, 4); *bad = 0;
  for (auto q : ps) {
    LimbInfo L{}; L.q = q;
    unsigned __int128 br = (~(unsigned __int128)0) / q;  // floor((2^128-1)/q) == floor(2^128/q) for non-power-of-2 q
    L.br_hi = (uint64_t)(br >> 64); L.br_lo = (uint64_t)br;
    k<<<148, 256>>>(L, bad, q);
    cudaDeviceSynchronize();
  }
  printf("bad=%d\n", *bad);
}
