// Reference-stream replay on the device.
//
// The reference draws, for every construction step, one C-order (m, n) block
// of Exp(1) deviates from Generator(Philox(SeedSequence(seed, spawn_key=(0, it,
// step)))).standard_exponential (rng.py:42-49).  That stream is numpy's
// Philox4x64-10 (counter incremented before each 4-word block) feeding the
// ziggurat of random_standard_exponential (numpy/random/src/distributions):
//   ri = w >> 3; idx = ri & 0xff; ri >>= 8; x = ri * we[idx]
//   accept if ri < ke[idx]; tail (idx 0): r - log1p(-u); wedge: accept if
//   (fe[idx-1] - fe[idx]) u + fe[idx] < exp(-x), else retry with new words,
// u = (next word >> 11) * 2^-53.  ~1.1% of samples take a slow path and consume
// extra words, so the block is one sequential stream.  It is replayed in
// parallel per step:
//   1. k_np_len    every word position p: does a sample starting at p take the
//                  fast path, else how many words L(p) it consumes
//   2. k_np_cover  every slow position: is it a sample start?  (walk from a
//                  provably-unaffected anchor; slow starts mark the positions
//                  they consume as covered)
//   3. exclusive scan of covered-bit counts per 32-position word (CUB)
//   4. k_np_select one warp per ant: locate the ant's first sample by binary
//                  search, decode its row 32 samples at a time (ballot over the
//                  covered bits), and run the reference's log-domain argmax
//                  round (selection.py:143-155, colony.py:143-152).
// The key of each step comes from numpy's SeedSequence on the host.  Values
// match numpy bit for bit except tail samples (log1p: CUDA vs glibc, <= 1
// ulp, ~0.05% of samples, E > 7.69); a wedge comparison closer than 4 ulp (where
// CUDA's exp could flip it) is counted and reported instead of guessed.
#include <cub/device/device_scan.cuh>

#include "numpy_ziggurat_tables.h"
#include "taco_common.cuh"

namespace taco {

constexpr int kMaxSlowLen = 64;  // words one sample may consume (flagged above)
constexpr double kZigExpR = 7.69711747013104972;

struct U64x4 {
  uint64_t x, y, z, w;
};

__device__ __forceinline__ U64x4 philox4x64_10(uint64_t c0, uint64_t k0, uint64_t k1) {
  constexpr uint64_t M0 = 0xD2E7470EE14C6C93ull, M1 = 0xCA5A826395121157ull;
  constexpr uint64_t W0 = 0x9E3779B97F4A7C15ull, W1 = 0xBB67AE8584CAA73Bull;
  uint64_t c1 = 0, c2 = 0, c3 = 0;
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    const uint64_t hi0 = __umul64hi(M0, c0), lo0 = M0 * c0;
    const uint64_t hi1 = __umul64hi(M1, c2), lo1 = M1 * c2;
    const uint64_t n0 = hi1 ^ c1 ^ k0, n2 = hi0 ^ c3 ^ k1;
    c0 = n0;
    c1 = lo1;
    c2 = n2;
    c3 = lo0;
    k0 += W0;
    k1 += W1;
  }
  return U64x4{c0, c1, c2, c3};
}

// word p of the step's stream (block p/4 uses counter p/4 + 1)
__device__ __forceinline__ uint64_t np_word(uint64_t p, uint64_t k0, uint64_t k1) {
  const U64x4 b = philox4x64_10((p >> 2) + 1, k0, k1);
  const uint32_t q = (uint32_t)(p & 3);
  return q == 0 ? b.x : (q == 1 ? b.y : (q == 2 ? b.z : b.w));
}

__device__ __forceinline__ double np_double(uint64_t w) { return (double)(w >> 11) * (1.0 / 9007199254740992.0); }

__device__ __forceinline__ bool np_fast(uint64_t w) {
  const uint64_t ri = (w >> 3) >> 8;
  return ri < kZigKe[(w >> 3) & 0xff];
}

// word source: the step's words materialized by k_np_len (positions < P),
// recomputed from the key past the replay window
struct NpWords {
  const uint64_t *buf;
  uint64_t P, k0, k1;
  __device__ __forceinline__ uint64_t operator()(uint64_t p) const { return p < P ? buf[p] : np_word(p, k0, k1); }
};

// Decode one sample starting at word p (first word w): returns the value,
// writes the number of words consumed; counts wedge tests too close to call.
template <typename Words>
__device__ double np_sample(uint64_t p, uint64_t w, const Words &word, int &len, unsigned *ambiguous) {
  len = 0;
  for (;;) {
    uint64_t ri = w >> 3;
    const int idx = (int)(ri & 0xff);
    ri >>= 8;
    const double x = __dmul_rn((double)ri, __longlong_as_double((long long)kZigWeBits[idx]));
    if (ri < kZigKe[idx]) {
      len += 1;
      return x;
    }
    const double u = np_double(word(p + 1));
    len += 2;
    if (idx == 0) return __dsub_rn(kZigExpR, log1p(-u));
    const double fe_i = __longlong_as_double((long long)kZigFeBits[idx]);
    const double fe_p = __longlong_as_double((long long)kZigFeBits[idx - 1]);
    const double lhs = __dadd_rn(__dmul_rn(__dsub_rn(fe_p, fe_i), u), fe_i);
    const double rhs = exp(-x);
    // |lhs - rhs| within 4 ulp of rhs (ulp(rhs) <= rhs * 2^-52): CUDA's exp
    // and glibc's could order them differently, so count it instead of guessing
    if (ambiguous != nullptr && fabs(lhs - rhs) <= 4.0 * 0x1p-52 * rhs) atomicAdd(ambiguous, 1u);
    if (lhs < rhs) return x;
    p += 2;  // rejected: the retry starts at the next unused word
    w = word(p);
  }
}

struct KeyWords {  // words straight from the key (used while filling the buffer)
  uint64_t k0, k1;
  __device__ __forceinline__ uint64_t operator()(uint64_t p) const { return np_word(p, k0, k1); }
};

struct ReplayWs {
  uint64_t *words;  // [P] the step's Philox4x64 words
  uint32_t *slow;   // [P/32] slow-path bit per position
  uint8_t *lens;    // [P] words consumed by a sample starting at a slow position
  uint32_t *cov;    // [P/32] positions consumed by a previous sample
  uint32_t *before; // [P/32] exclusive prefix of covered counts
  unsigned *flags;  // caller's device words: [0] ambiguous wedge tests, [1] overflow
  void *scan_tmp;
  size_t scan_bytes;
  uint64_t P;       // positions replayed (multiple of 128)
};

__global__ void k_np_len(uint64_t P, uint64_t k0, uint64_t k1, uint64_t *words, uint32_t *slow, uint8_t *lens,
                         unsigned *flags) {
  const uint64_t b = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (4 * b >= P) return;
  const U64x4 blk = philox4x64_10(b + 1, k0, k1);
  const uint64_t ws[4] = {blk.x, blk.y, blk.z, blk.w};
  reinterpret_cast<ulonglong2 *>(words + 4 * b)[0] = make_ulonglong2(blk.x, blk.y);
  reinterpret_cast<ulonglong2 *>(words + 4 * b)[1] = make_ulonglong2(blk.z, blk.w);
  const KeyWords kw{k0, k1};
  uint32_t bits = 0;
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    if (!np_fast(ws[q])) {
      const uint64_t p = 4 * b + q;
      int len;
      np_sample(p, ws[q], kw, len, flags);
      if (len > kMaxSlowLen) atomicOr(flags + 1, 1u);
      lens[p] = (uint8_t)(len > 255 ? 255 : len);
      bits |= 1u << q;
    }
  }
  if (bits) atomicOr(slow + (4 * b >> 5), bits << ((4 * b) & 31));
}

__device__ __forceinline__ bool bit(const uint32_t *v, uint64_t p) { return (v[p >> 5] >> (p & 31)) & 1u; }

__device__ __forceinline__ uint64_t step_len(const uint32_t *slow, const uint8_t *lens, uint64_t s) {
  return bit(slow, s) ? lens[s] : 1;
}

// first slow position >= s (or `limit` if none before it)
__device__ __forceinline__ uint64_t next_slow(const uint32_t *slow, uint64_t s, uint64_t limit) {
  uint64_t w = s >> 5;
  uint32_t bits = slow[w] & (0xffffffffu << (s & 31));
  while (!bits) {
    if (++w * 32 >= limit) return limit;
    bits = slow[w];
  }
  const uint64_t q = w * 32 + (__ffs(bits) - 1);
  return q < limit ? q : limit;
}

// does any slow position q in [lo, a) reach past a (q + L(q) > a)?
__device__ __forceinline__ bool reaches_past(const uint32_t *slow, const uint8_t *lens, uint64_t lo, uint64_t a) {
  for (uint64_t q = next_slow(slow, lo, a); q < a; q = next_slow(slow, q + 1, a))
    if (q + lens[q] > a) return true;
  return false;
}

// thread per 32-position word of the slow bitmap
__global__ void k_np_cover(uint64_t P, const uint32_t *slow, const uint8_t *lens, uint32_t *cov) {
  const uint64_t wi = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (wi >= P / 32) return;
  uint32_t todo = slow[wi];
  while (todo) {
    const int b = __ffs(todo) - 1;
    todo &= todo - 1;
    const uint64_t p = wi * 32 + b;
    // anchor: a position no slow sample before it can reach past is a start
    uint64_t a = p > (uint64_t)kMaxSlowLen ? p - kMaxSlowLen : 0;
    while (a > 0 && reaches_past(slow, lens, a > (uint64_t)kMaxSlowLen ? a - kMaxSlowLen : 0, a))
      a = a > (uint64_t)kMaxSlowLen ? a - kMaxSlowLen : 0;
    // walk the sample starts from the anchor: fast runs are skipped in one
    // jump (each fast position is a start that consumes one word)
    uint64_t s = a;
    while (s < p) s = bit(slow, s) ? s + lens[s] : next_slow(slow, s, p);
    if (s == p)
      for (uint64_t c = p + 1; c < p + lens[p] && c < P; ++c) atomicOr(cov + (c >> 5), 1u << (c & 31));
  }
}

__global__ void k_np_count(uint64_t words, const uint32_t *cov, uint32_t *cnt) {
  const uint64_t w = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (w < words) cnt[w] = __popc(cov[w]);
}

// One warp per ant: the reference's lockstep round on the replayed block.
// Stream position of sample k (the k-th uncovered position): binary search
// over the per-word start counts, then the k-th free bit.
__device__ __forceinline__ uint64_t sample_position(const ReplayWs &ws, uint64_t k) {
  const uint64_t words = ws.P / 32;
  uint64_t lo = 0, hi = words;  // invariant: starts_before(lo) <= k
  while (hi - lo > 1) {
    const uint64_t mid = (lo + hi) / 2;
    const uint64_t sb = 32 * mid - ws.before[mid];
    if (sb <= k) lo = mid; else hi = mid;
  }
  uint32_t freebits = ~ws.cov[lo];
  uint64_t rank = k - (32 * lo - ws.before[lo]);
  while (rank >= (uint64_t)__popc(freebits)) {  // (only past the last word on overflow)
    rank -= __popc(freebits);
    ++lo;
    freebits = lo < words ? ~ws.cov[lo] : 0xffffffffu;
  }
  return lo * 32 + (__fns(freebits, 0, (int)rank + 1));
}

// E[a, 0] of the step's (m, n) block for every ant: the roulette wheel's
// threshold source, u = exp(-E[:, 0]) (rng.step_uniforms rng.py:52-62)
__global__ void k_np_first(int n, int m, uint64_t k0, uint64_t k1, ReplayWs ws, double *e0) {
  const int a = blockIdx.x * blockDim.x + threadIdx.x;
  if (a >= m) return;
  const uint64_t pos = sample_position(ws, (uint64_t)a * n);
  if (pos + 1 > ws.P) atomicOr(ws.flags + 1, 1u);
  int len;
  const NpWords word{ws.words, ws.P, k0, k1};
  e0[a] = np_sample(pos, word(pos), word, len, nullptr);
}

template <int WARPS>
__global__ void __launch_bounds__(WARPS * 32)
    k_np_select(int n, int m, int step, uint64_t k0, uint64_t k1, const double *__restrict__ logw,
                int64_t *current, uint8_t *visited, int64_t *tours, ReplayWs ws, int32_t *status) {
  const int lane = threadIdx.x & 31;
  const int a = blockIdx.x * WARPS + (threadIdx.x >> 5);
  if (a >= m) return;
  uint64_t pos = sample_position(ws, (uint64_t)a * n);

  const int64_t cur = current[a];
  const double *lr = logw + (size_t)cur * n;
  const uint8_t *vr = visited + (size_t)a * n;
  double best = -INFINITY;
  int bj = 0x7fffffff;
  for (int base = 0; base < n; base += 32) {
    // the next 32 sample starts are the first 32 uncovered positions >= pos
    const bool f0 = !(pos + lane < ws.P ? bit(ws.cov, pos + lane) : false);
    const bool f1 = !(pos + 32 + lane < ws.P ? bit(ws.cov, pos + 32 + lane) : false);
    const unsigned m0 = __ballot_sync(0xffffffffu, f0), m1 = __ballot_sync(0xffffffffu, f1);
    const int c0 = __popc(m0);
    if (c0 + __popc(m1) < 32 || pos + 64 > ws.P) atomicOr(ws.flags + 1, 1u);  // replay window too short
    const uint64_t my = lane < c0 ? pos + __fns(m0, 0, lane + 1) : pos + 32 + __fns(m1, 0, lane - c0 + 1);
    const int j = base + lane;
    if (j < n) {
      int len;
      const NpWords word{ws.words, ws.P, k0, k1};
      const double e = np_sample(my, word(my), word, len, nullptr);
      // np.take -> np.subtract -> np.copyto(-inf, where=visited)  (selection.py:152-154)
      const double s = vr[j] ? -INFINITY : __dsub_rn(lr[j], e);
      if (s > best) {
        best = s;
        bj = j;
      }
    }
    pos = __shfl_sync(0xffffffffu, my, 31) + 1;
  }
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    const double ob = __shfl_xor_sync(0xffffffffu, best, off);
    const int oj = __shfl_xor_sync(0xffffffffu, bj, off);
    if (ob > best || (ob == best && oj < bj)) {
      best = ob;
      bj = oj;
    }
  }
  if (lane == 0) {
    const int nxt = (bj == 0x7fffffff) ? 0 : bj;  // argmax of all -inf is 0
    if (visited[(size_t)a * n + nxt]) record_status(status, TACO_NO_CANDIDATE, a);
    visited[(size_t)a * n + nxt] = 1;
    current[a] = nxt;
    tours[(size_t)a * n + step] = nxt;
  }
}

static uint64_t replay_positions(int m, int n) {
  const uint64_t N = (uint64_t)m * n;
  return ((N + N / 16 + 4096) + 127) / 128 * 128;
}

static size_t scan_bytes(uint64_t words) {
  size_t bytes = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, bytes, (const uint32_t *)nullptr, (uint32_t *)nullptr, (int)words);
  return bytes;
}

static size_t al256(size_t x) { return (x + 255) & ~(size_t)255; }

static ReplayWs carve(void *ws, int m, int n) {
  ReplayWs r;
  r.P = replay_positions(m, n);
  const uint64_t words = r.P / 32;
  unsigned char *p = reinterpret_cast<unsigned char *>(ws);
  r.words = reinterpret_cast<uint64_t *>(p);
  p += al256(r.P * 8);
  r.slow = reinterpret_cast<uint32_t *>(p);
  p += al256(words * 4);
  r.cov = reinterpret_cast<uint32_t *>(p);
  p += al256(words * 4);
  r.flags = nullptr;
  r.before = reinterpret_cast<uint32_t *>(p);
  p += al256(words * 4);
  r.lens = p;
  p += al256(r.P);
  r.scan_tmp = p;
  r.scan_bytes = scan_bytes(words);
  return r;
}

}  // namespace taco

using namespace taco;

extern "C" size_t taco_replay_workspace_bytes(int m, int n) {
  if (m < 1 || n < 1) return 0;
  const uint64_t P = replay_positions(m, n), words = P / 32;
  return al256(P * 8) + 3 * al256(words * 4) + al256(P) + al256(scan_bytes(words));
}

// the step's decode pipeline: words, slow-path cover, sample-start counts
static int replay_decode(ReplayWs &r, uint64_t key0, uint64_t key1, unsigned *flags_out, cudaStream_t s) {
  const uint64_t words = r.P / 32;
  if (cudaMemsetAsync(r.slow, 0, words * 4, s) != cudaSuccess ||
      cudaMemsetAsync(r.cov, 0, words * 4, s) != cudaSuccess)
    return TACO_ERR_CUDA;
  k_np_len<<<(unsigned)((r.P / 4 + 255) / 256), 256, 0, s>>>(r.P, key0, key1, r.words, r.slow, r.lens,
                                                              flags_out);
  TACO_CUDA_CHECK_LAUNCH();
  k_np_cover<<<(unsigned)((words + 255) / 256), 256, 0, s>>>(r.P, r.slow, r.lens, r.cov);
  TACO_CUDA_CHECK_LAUNCH();
  k_np_count<<<(unsigned)((words + 255) / 256), 256, 0, s>>>(words, r.cov, r.before);
  TACO_CUDA_CHECK_LAUNCH();
  size_t tb = r.scan_bytes;
  if (cub::DeviceScan::ExclusiveSum(r.scan_tmp, tb, r.before, r.before, (int)words, s) != cudaSuccess)
    return TACO_ERR_CUDA;
  return TACO_OK;
}

extern "C" int taco_select_replay(int n, int m, int step, uint64_t key0, uint64_t key1, const double *logw,
                                  int64_t *current, uint8_t *visited, int64_t *tours, void *workspace,
                                  size_t ws_bytes, unsigned *flags_out, int32_t *status, void *stream) {
  if (n < 2 || m < 1 || step < 1 || step >= n || logw == nullptr || workspace == nullptr) return TACO_ERR_ARG;
  if (flags_out == nullptr || ws_bytes < taco_replay_workspace_bytes(m, n)) return TACO_ERR_ARG;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  ReplayWs r = carve(workspace, m, n);
  r.flags = flags_out;
  const int rc = replay_decode(r, key0, key1, flags_out, s);
  if (rc != TACO_OK) return rc;
  constexpr int WARPS = 8;
  k_np_select<WARPS><<<(m + WARPS - 1) / WARPS, WARPS * 32, 0, s>>>(n, m, step, key0, key1, logw, current,
                                                                   visited, tours, r, status);
  TACO_CUDA_CHECK_LAUNCH();
  return TACO_OK;
}

extern "C" int taco_replay_first_column(int n, int m, uint64_t key0, uint64_t key1, void *workspace,
                                        size_t ws_bytes, double *e0_out, unsigned *flags_out, void *stream) {
  if (n < 2 || m < 1 || workspace == nullptr || e0_out == nullptr || flags_out == nullptr) return TACO_ERR_ARG;
  if (ws_bytes < taco_replay_workspace_bytes(m, n)) return TACO_ERR_ARG;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  ReplayWs r = carve(workspace, m, n);
  r.flags = flags_out;
  const int rc = replay_decode(r, key0, key1, flags_out, s);
  if (rc != TACO_OK) return rc;
  k_np_first<<<(m + 255) / 256, 256, 0, s>>>(n, m, key0, key1, r, e0_out);
  TACO_CUDA_CHECK_LAUNCH();
  return TACO_OK;
}
