// Throughput of the sampler's per-position hash filter variants (one B200).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o hp hash_pipes.cu && ./hp
#include <cstdio>
#include <cstdint>
constexpr uint64_t kPhi = 0x9e3779b97f4a7c15ull;
__device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z ^= z >> 30; z *= 0xbf58476d1ce4e5b9ull; z ^= z >> 27; z *= 0x94d049bb133111ebull; z ^= z >> 31; return z;
}
__device__ __forceinline__ uint32_t hi_imad(uint64_t c, uint4 mk) {
  const uint32_t lo = (uint32_t)c, hi = (uint32_t)(c >> 32);
  const uint32_t l1 = lo ^ __funnelshift_r(lo, hi, 30);
  const uint32_t h1 = hi ^ __umulhi(hi, mk.y);
  const uint64_t w = (uint64_t)l1 * 0x1ce4e5b9u;
  const uint32_t h2 = (uint32_t)(w >> 32) + l1 * 0xbf58476du + h1 * 0x1ce4e5b9u;
  const uint32_t l2 = (uint32_t)w;
  const uint32_t l3 = l2 ^ __funnelshift_r(l2, h2, 27);
  const uint32_t h3 = h2 ^ __umulhi(h2, mk.z);
  const uint32_t h4 = __umulhi(l3, 0x133111ebu) + l3 * 0x94d049bbu + h3 * 0x133111ebu;
  return h4 ^ __umulhi(h4, mk.w);
}
__device__ __forceinline__ uint32_t hi_shift(uint64_t c) {
  const uint32_t lo = (uint32_t)c, hi = (uint32_t)(c >> 32);
  const uint32_t l1 = lo ^ __funnelshift_r(lo, hi, 30);
  const uint32_t h1 = hi ^ (hi >> 30);
  const uint64_t w = (uint64_t)l1 * 0x1ce4e5b9u;
  const uint32_t h2 = (uint32_t)(w >> 32) + l1 * 0xbf58476du + h1 * 0x1ce4e5b9u;
  const uint32_t l2 = (uint32_t)w;
  const uint32_t l3 = l2 ^ __funnelshift_r(l2, h2, 27);
  const uint32_t h3 = h2 ^ (h2 >> 27);
  const uint32_t h4 = __umulhi(l3, 0x133111ebu) + l3 * 0x94d049bbu + h3 * 0x133111ebu;
  return h4 ^ (h4 >> 31);
}
__device__ __forceinline__ uint32_t hi_noxor(uint64_t c) {  // h4; x_hi in {h4, h4 ^ 1}
  const uint32_t lo = (uint32_t)c, hi = (uint32_t)(c >> 32);
  const uint32_t l1 = lo ^ __funnelshift_r(lo, hi, 30);
  const uint32_t h1 = hi ^ (hi >> 30);
  const uint64_t w = (uint64_t)l1 * 0x1ce4e5b9u;
  const uint32_t h2 = (uint32_t)(w >> 32) + l1 * 0xbf58476du + h1 * 0x1ce4e5b9u;
  const uint32_t l2 = (uint32_t)w;
  const uint32_t l3 = l2 ^ __funnelshift_r(l2, h2, 27);
  const uint32_t h3 = h2 ^ (h2 >> 27);
  return __umulhi(l3, 0x133111ebu) + l3 * 0x94d049bbu + h3 * 0x133111ebu;
}
__device__ __forceinline__ uint64_t add_fma(uint64_t c, uint64_t d, uint32_t one) {
  uint64_t w;
  asm("mad.wide.u32 %0, %1, %2, %3;" : "=l"(w) : "r"(one), "r"((uint32_t)d), "l"(c));
  uint32_t lo = (uint32_t)w, hi = (uint32_t)(w >> 32);
  asm("mad.lo.u32 %0, %1, %2, %0;" : "+r"(hi) : "r"(one), "r"((uint32_t)(d >> 32)));
  return ((uint64_t)hi << 32) | lo;
}
template <int V>
__global__ void __launch_bounds__(256) k(uint64_t key, uint32_t n, uint64_t thrx, uint4 mk, unsigned* out) {
  uint64_t ctr = key + (blockIdx.x * 256ull + threadIdx.x) * kPhi;
  unsigned cnt = 0;
  const uint32_t thi = (uint32_t)(thrx >> 32);
  for (uint32_t i = 0; i < n; i += 4, ctr += 4 * 0x9e3779b97f4a7c15ull * 37888) {
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const uint64_t c = V >= 4 ? add_fma(ctr, u * kPhi * 9472, mk.x) : ctr + u * kPhi * 9472;
      bool p;
      if (V == 0) p = mix64(c) > thrx;
      else if (V == 1) p = hi_imad(c, mk) >= thi;
      else if (V == 2) p = hi_shift(c) >= thi;
      else p = hi_noxor(c) >= thi - 1;
      cnt += p;
    }
  }
  if (cnt == 12345678) out[0] = cnt;
  atomicAdd(out + 1, cnt);
}
int main() {
  unsigned* d; cudaMalloc(&d, 8);
  const int grid = 148 * 8; const uint32_t n = 1 << 14;
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  uint4 mk = make_uint4(1, 4, 32, 2);
  for (int v = 0; v < 5; ++v) for (int rep = 0; rep < 3; ++rep) {
    cudaMemset(d, 0, 8);
    cudaEventRecord(a);
    if (v == 0) k<0><<<grid, 256>>>(12345, n, 0xfff0000000000000ull, mk, d);
    if (v == 1) k<1><<<grid, 256>>>(12345, n, 0xfff0000000000000ull, mk, d);
    if (v == 2) k<2><<<grid, 256>>>(12345, n, 0xfff0000000000000ull, mk, d);
    if (v == 3) k<3><<<grid, 256>>>(12345, n, 0xfff0000000000000ull, mk, d);
    if (v == 4) k<4><<<grid, 256>>>(12345, n, 0xfff0000000000000ull, mk, d);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    unsigned h[2]; cudaMemcpy(h, d, 8, cudaMemcpyDeviceToHost);
    double pos = (double)grid * 256 * n;
    printf("variant %d: %.3f ms  %.1f Gpos/s  (hits %u)\n", v, ms, pos / ms / 1e6, h[1]);
  }
  return 0;
}
