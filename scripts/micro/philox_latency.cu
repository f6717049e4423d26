// Microbenchmark: dependent-chain latency of one Philox4x32-10 evaluation on
// sm_100a with different 32x32->64 multiply formulations (one warp, clock64).
#include <cstdio>
#include <cstdint>

struct U4 { uint32_t x, y, z, w; };
constexpr uint32_t M0 = 0xD2511F53u, M1 = 0xCD9E8D57u;

template <int V>
__device__ __forceinline__ void mulhilo(uint32_t a, uint32_t m, uint32_t &hi, uint32_t &lo) {
  if (V == 0) { lo = m * a; hi = __umulhi(m, a); }
  else if (V == 1) { const uint64_t p = (uint64_t)a * m; lo = (uint32_t)p; hi = (uint32_t)(p >> 32); }
  else { asm("mul.lo.u32 %0, %2, %3;\n\tmul.hi.u32 %1, %2, %3;" : "=r"(lo), "=r"(hi) : "r"(a), "r"(m)); }
}

template <int V>
__device__ __forceinline__ U4 philox(U4 c, const uint32_t *k0, const uint32_t *k1) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    uint32_t hi0, lo0, hi1, lo1;
    mulhilo<V>(c.x, M0, hi0, lo0);
    mulhilo<V>(c.z, M1, hi1, lo1);
    c = U4{hi1 ^ c.y ^ k0[r], lo1, hi0 ^ c.w ^ k1[r], lo0};
  }
  return c;
}

struct Keys { uint32_t k0[10], k1[10]; };

template <int V>
__global__ void bench(Keys ks, uint32_t seed, unsigned long long *out, uint32_t *sink) {
  U4 c{threadIdx.x ^ seed, 1, 2, 3};
  long long t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < 64; ++i) c = philox<V>(c, ks.k0, ks.k1);  // each call depends on the last
  long long t1 = clock64();
  if (threadIdx.x == 0) out[V] = (t1 - t0) / 64;
  sink[threadIdx.x] = c.x ^ c.y ^ c.z ^ c.w;
}

int main() {
  Keys ks;
  for (int r = 0; r < 10; ++r) { ks.k0[r] = 0x12345 + r * 0x9E3779B9u; ks.k1[r] = 0x6789 + r * 0xBB67AE85u; }
  unsigned long long *out; uint32_t *sink;
  cudaMalloc(&out, 64); cudaMalloc(&sink, 4096);
  for (int rep = 0; rep < 2; ++rep) {
    bench<0><<<1, 32>>>(ks, 7, out, sink);
    bench<1><<<1, 32>>>(ks, 7, out, sink);
    bench<2><<<1, 32>>>(ks, 7, out, sink);
  }
  unsigned long long h[3];
  cudaMemcpy(h, out, sizeof(h), cudaMemcpyDeviceToHost);
  printf("cycles per Philox4x32-10 (dependent chain): umulhi=%llu  u64mul=%llu  ptx=%llu\n", h[0], h[1], h[2]);
  return 0;
}
