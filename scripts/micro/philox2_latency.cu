// Microbenchmark: dependent-chain latency of one Philox2x32-10 block on
// sm_100a for different formulations of the 32x32 -> (hi, lo) product
// (one warp, clock64).  V0: __umulhi + mul (ptxas: IMAD.WIDE), V1: hi and lo
// from separate PTX instructions with the lo product kept off the hi path.
#include <cstdio>
#include <cstdint>

constexpr uint32_t M = 0xD256D193u;

__device__ uint32_t g_zero;

template <int V>
__device__ __forceinline__ void round_(uint32_t &x0, uint32_t &x1, uint32_t k, uint32_t zero) {
  uint32_t hi, lo;
  if (V == 0) {
    hi = __umulhi(M, x0);
    lo = M * x0;
  } else if (V == 1) {
    asm volatile("mul.hi.u32 %0, %1, %2;" : "=r"(hi) : "r"(x0), "r"(M));
    asm volatile("mul.lo.u32 %0, %1, %2;" : "=r"(lo) : "r"(x0), "r"(M));
  } else if (V == 2) {
    uint32_t y;
    asm volatile("mov.b32 %0, %1;" : "=r"(y) : "r"(x0));
    hi = __umulhi(M, x0);
    lo = M * y;
  } else {
    hi = __umulhi(M, x0);
    lo = M * x0 + zero;  // runtime zero: not fusable into the 64-bit product
  }
  x0 = hi ^ k ^ x1;
  x1 = lo;
}

template <int V>
__global__ void bench(const uint32_t *keys, unsigned long long *out, uint32_t *sink) {
  uint32_t x0 = threadIdx.x, x1 = 7;
  const uint32_t zero = g_zero;
  uint32_t kk[10];
  for (int r = 0; r < 10; ++r) kk[r] = keys[r];
  long long t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < 64; ++i) {
#pragma unroll
    for (int r = 0; r < 10; ++r) round_<V>(x0, x1, kk[r], zero);
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) out[V] = (t1 - t0) / 64;
  sink[threadIdx.x] = x0 ^ x1;
}

int main() {
  uint32_t hk[10];
  for (int r = 0; r < 10; ++r) hk[r] = 0x12345u + r * 0x9E3779B9u;
  uint32_t *keys, *sink;
  unsigned long long *out;
  cudaMalloc(&keys, 40);
  cudaMalloc(&out, 32);
  cudaMalloc(&sink, 4096);
  cudaMemcpy(keys, hk, 40, cudaMemcpyHostToDevice);
  for (int rep = 0; rep < 2; ++rep) {
    bench<0><<<1, 32>>>(keys, out, sink);
    bench<1><<<1, 32>>>(keys, out, sink);
    bench<2><<<1, 32>>>(keys, out, sink);
    bench<3><<<1, 32>>>(keys, out, sink);
  }
  unsigned long long h[4];
  cudaMemcpy(h, out, sizeof(h), cudaMemcpyDeviceToHost);
  printf("cycles per Philox2x32-10 block (dependent chain): default=%llu ptx-hi-lo=%llu mov-split=%llu "
         "zero-addend=%llu\n", h[0], h[1], h[2], h[3]);
  return 0;
}
