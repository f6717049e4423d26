// Tour construction kernels: one warp owns one ant for all n-1 lockstep steps.
//
// Reference: colony.construct_tours colony.py:87-154 (IR / AdaIR branch),
// argmax_select_block selection.py:143-155, start cities rng.py:65-68.
//
// Fast-path rule: next = argmax_j { W[cur, j] * u(step, ant, j) }
// over unvisited j with W[cur, j] > 0, first (lowest j) of ties, where
// W = fp32(P^(1/gamma)) and u is the keyed Philox4x32-10 uniform.  This is the
// product form of the reference's argmax(log P / gamma - E) with E = -log u.
//
// Two variants compute the identical argmax:
//   DENSE  streams the whole fp32 row W[cur, :] with 16-byte loads and draws
//          four uniforms per Philox block (the north-star "row streaming"
//          kernel; HBM/L2-bandwidth + ALU bound).
//   SORTED scans the row's descending (W, j) table and stops as soon as the
//          next table entry satisfies W < best score: since u < 1, no later
//          entry can reach the running best, so the result is bit-identical to
//          the full scan while touching only the head of the row.  Because the
//          uniforms are counter-addressed by city, visiting candidates in
//          sorted order draws exactly the values the full scan would.
#include "taco_common.cuh"

namespace taco {

constexpr unsigned kFull = 0xffffffffu;

struct TourWriter {
  // lane (step & 31) buffers the choice of `step`; every 32 steps the warp
  // writes one coalesced 128-byte segment of the tour row.
  int32_t *row;
  int n;
  int lane;
  int32_t buf;
  __device__ __forceinline__ void put(int step, int32_t city) {
    if (lane == (step & 31)) buf = city;
    if ((step & 31) == 31) row[(step & ~31) + lane] = buf;
  }
  __device__ __forceinline__ void flush() {
    const int last = n - 1;
    if ((last & 31) != 31 && lane <= (last & 31)) row[(last & ~31) + lane] = buf;
  }
};

__device__ __forceinline__ bool is_visited(const uint32_t *vis, uint32_t j) {
  return (vis[j >> 5] >> (j & 31)) & 1u;
}

template <int WARPS>
__global__ void __launch_bounds__(WARPS * 32)
    k_construct_sorted(int n, int m_local, int ant_offset, const float *__restrict__ sw,
                       const uint16_t *__restrict__ si, uint32_t k0, uint32_t k1, uint32_t iteration,
                       int32_t *__restrict__ tours, int32_t *status, int nwords,
                       unsigned long long *scan_count) {
  extern __shared__ uint32_t vis_all[];
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int ant = blockIdx.x * WARPS + warp;
  if (ant >= m_local) return;
  const uint32_t gant = (uint32_t)(ant_offset + ant);
  uint32_t *vis = vis_all + (size_t)warp * nwords;
  for (int w = lane; w < nwords; w += 32) vis[w] = 0u;
  const uint32_t start = start_city((uint32_t)n, gant, iteration, k0, k1);
  __syncwarp();
  if (lane == 0) vis[start >> 5] |= 1u << (start & 31);
  __syncwarp();

  TourWriter tw{tours + (size_t)ant * n, n, lane, 0};
  tw.put(0, (int32_t)start);
  uint32_t cur = start;
  unsigned long long windows = 0;  // 32-entry table windows read (traffic probe)
  for (int step = 1; step < n; ++step) {
    const float *wr = sw + (size_t)cur * n;
    const uint16_t *ir = si + (size_t)cur * n;
    float best = -1.0f;
    uint32_t bestj = 0xffffffffu;
    for (int base = 0; base < n; base += 32) {
      const int e = base + lane;
      float w = 0.0f;
      uint32_t j = 0;
      if (e < n) {
        w = __ldg(wr + e);
        j = __ldg(ir + e);
      }
      uint32_t key = 0u;
      if (w > 0.0f && w >= best && !is_visited(vis, j)) {
        const U4 r = philox4x32_10(U4{j >> 2, (uint32_t)step, gant, iteration}, k0, k1);
        const float s = __fmul_rn(w, bits_to_uniform(word_of(r, j & 3)));
        key = __float_as_uint(s) + 1u;
      }
      const uint32_t mkey = __reduce_max_sync(kFull, key);
      if (mkey != 0u) {
        const uint32_t jmin = __reduce_min_sync(kFull, key == mkey ? j : 0xffffffffu);
        const float sc = __uint_as_float(mkey - 1u);
        if (sc > best || (sc == best && jmin < bestj)) {
          best = sc;
          bestj = jmin;
        }
      }
      ++windows;
      // entries after this window have W <= the window's last W
      const float wl = __shfl_sync(kFull, w, 31);
      if (wl < best || wl <= 0.0f) break;
    }
    if (bestj == 0xffffffffu) {
      if (lane == 0) record_status(status, TACO_NO_CANDIDATE, (int)gant);
      return;
    }
    if (lane == 0) vis[bestj >> 5] |= 1u << (bestj & 31);
    __syncwarp();
    tw.put(step, (int32_t)bestj);
    cur = bestj;
  }
  tw.flush();
  if (scan_count != nullptr && lane == 0) atomicAdd(scan_count, windows);
}

template <int WARPS>
__global__ void __launch_bounds__(WARPS * 32)
    k_construct_dense(int n, int m_local, int ant_offset, const float *__restrict__ w, int ldw,
                      uint32_t k0, uint32_t k1, uint32_t iteration, int32_t *__restrict__ tours,
                      int32_t *status, int nwords) {
  extern __shared__ uint32_t vis_all[];
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int ant = blockIdx.x * WARPS + warp;
  if (ant >= m_local) return;
  const uint32_t gant = (uint32_t)(ant_offset + ant);
  uint32_t *vis = vis_all + (size_t)warp * nwords;
  for (int q = lane; q < nwords; q += 32) vis[q] = 0u;
  const uint32_t start = start_city((uint32_t)n, gant, iteration, k0, k1);
  __syncwarp();
  if (lane == 0) vis[start >> 5] |= 1u << (start & 31);
  __syncwarp();

  TourWriter tw{tours + (size_t)ant * n, n, lane, 0};
  tw.put(0, (int32_t)start);
  uint32_t cur = start;
  const int nq = (n + 3) >> 2;
  for (int step = 1; step < n; ++step) {
    const float4 *row = reinterpret_cast<const float4 *>(w + (size_t)cur * ldw);
    uint32_t lkey = 0u, lj = 0xffffffffu;
#pragma unroll 4
    for (int q = lane; q < nq; q += 32) {
      const float4 wv = __ldg(row + q);
      const uint32_t nib = (vis[q >> 3] >> ((q & 7) * 4)) & 0xfu;
      const bool any = (nib != 0xfu) && (wv.x > 0.0f || wv.y > 0.0f || wv.z > 0.0f || wv.w > 0.0f);
      if (any) {
        const U4 r = philox4x32_10(U4{(uint32_t)q, (uint32_t)step, gant, iteration}, k0, k1);
        const float wc[4] = {wv.x, wv.y, wv.z, wv.w};
        const uint32_t rc[4] = {r.x, r.y, r.z, r.w};
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          const uint32_t j = 4u * q + c;
          if (!((nib >> c) & 1u) && wc[c] > 0.0f && j < (uint32_t)n) {
            const uint32_t key = __float_as_uint(__fmul_rn(wc[c], bits_to_uniform(rc[c]))) + 1u;
            if (key > lkey) {  // strict: the lowest j of this lane's ties stays
              lkey = key;
              lj = j;
            }
          }
        }
      }
    }
    const uint32_t mkey = __reduce_max_sync(kFull, lkey);
    if (mkey == 0u) {
      if (lane == 0) record_status(status, TACO_NO_CANDIDATE, (int)gant);
      return;
    }
    const uint32_t bestj = __reduce_min_sync(kFull, lkey == mkey ? lj : 0xffffffffu);
    if (lane == 0) vis[bestj >> 5] |= 1u << (bestj & 31);
    __syncwarp();
    tw.put(step, (int32_t)bestj);
    cur = bestj;
  }
  tw.flush();
}

__global__ void k_starts(int n, int m_local, int ant_offset, uint32_t k0, uint32_t k1,
                         uint32_t iteration, int32_t *out) {
  const int a = blockIdx.x * blockDim.x + threadIdx.x;
  if (a < m_local) out[a] = (int32_t)start_city((uint32_t)n, (uint32_t)(ant_offset + a), iteration, k0, k1);
}

__global__ void k_uniforms(int count, const uint32_t *step, const uint32_t *ant, const uint32_t *city,
                           uint32_t k0, uint32_t k1, uint32_t iteration, float *out) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= count) return;
  const uint32_t j = city[t];
  const U4 r = philox4x32_10(U4{j >> 2, step[t], ant[t], iteration}, k0, k1);
  out[t] = bits_to_uniform(word_of(r, j & 3));
}

__global__ void k_philox(int count, const uint32_t *ctr, const uint32_t *key, uint32_t *out) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= count) return;
  const U4 r = philox4x32_10(U4{ctr[4 * t], ctr[4 * t + 1], ctr[4 * t + 2], ctr[4 * t + 3]}, key[2 * t],
                             key[2 * t + 1]);
  out[4 * t] = r.x;
  out[4 * t + 1] = r.y;
  out[4 * t + 2] = r.z;
  out[4 * t + 3] = r.w;
}

// One lockstep round of the reference's log-domain selection (parity mode).
template <int WARPS>
__global__ void __launch_bounds__(WARPS * 32)
    k_select_parity(int n, int m, int step, const double *__restrict__ logw,
                    const double *__restrict__ e_block, int64_t *current, uint8_t *visited,
                    int64_t *tours, int32_t *status) {
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int a = blockIdx.x * WARPS + warp;
  if (a >= m) return;
  const int64_t cur = current[a];
  const double *lr = logw + (size_t)cur * n;
  const double *er = e_block + (size_t)a * n;
  const uint8_t *vr = visited + (size_t)a * n;
  double best = -INFINITY;
  int bj = 0x7fffffff;
  for (int j = lane; j < n; j += 32) {
    // np.take -> np.subtract -> np.copyto(-inf, where=visited)  (selection.py:152-154)
    const double s = vr[j] ? -INFINITY : __dsub_rn(lr[j], er[j]);
    if (s > best) {
      best = s;
      bj = j;
    }
  }
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    const double ob = __shfl_xor_sync(kFull, best, off);
    const int oj = __shfl_xor_sync(kFull, bj, off);
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

}  // namespace taco

using namespace taco;

static inline void split_seed(uint64_t seed, uint32_t *k0, uint32_t *k1) {
  *k0 = (uint32_t)(seed & 0xffffffffu);
  *k1 = (uint32_t)(seed >> 32);
}

extern "C" int taco_construct(int n, int m_local, int ant_offset, int variant, const float *w, int ldw,
                              const float *sw, const uint16_t *si, uint64_t seed, uint32_t iteration,
                              int32_t *tours_out, int32_t *status, unsigned long long *scan_count,
                              void *stream) {
  if (n < 3 || n > 65535 || m_local < 0 || ant_offset < 0 || tours_out == nullptr) return TACO_ERR_ARG;
  if (m_local == 0) return TACO_OK;
  uint32_t k0, k1;
  split_seed(seed, &k0, &k1);
  const int nwords = (n + 31) / 32;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  constexpr int WARPS = 4;
  const int grid = (m_local + WARPS - 1) / WARPS;
  const size_t smem = (size_t)WARPS * nwords * sizeof(uint32_t);
  if (variant == TACO_CONSTRUCT_SORTED) {
    if (sw == nullptr || si == nullptr) return TACO_ERR_ARG;
    k_construct_sorted<WARPS><<<grid, WARPS * 32, smem, s>>>(n, m_local, ant_offset, sw, si, k0, k1, iteration,
                                                             tours_out, status, nwords, scan_count);
  } else if (variant == TACO_CONSTRUCT_DENSE) {
    if (w == nullptr || ldw < n || (ldw % 4) != 0) return TACO_ERR_ARG;
    if ((reinterpret_cast<uintptr_t>(w) & 15u) != 0) return TACO_ERR_ARG;
    k_construct_dense<WARPS><<<grid, WARPS * 32, smem, s>>>(n, m_local, ant_offset, w, ldw, k0, k1, iteration,
                                                            tours_out, status, nwords);
  } else {
    return TACO_ERR_ARG;
  }
  TACO_CUDA_CHECK_LAUNCH();
  return TACO_OK;
}

extern "C" int taco_starts(int n, int m_local, int ant_offset, uint64_t seed, uint32_t iteration,
                           int32_t *starts_out, void *stream) {
  if (n < 1 || m_local < 0 || starts_out == nullptr) return TACO_ERR_ARG;
  if (m_local == 0) return TACO_OK;
  uint32_t k0, k1;
  split_seed(seed, &k0, &k1);
  k_starts<<<(m_local + 255) / 256, 256, 0, reinterpret_cast<cudaStream_t>(stream)>>>(
      n, m_local, ant_offset, k0, k1, iteration, starts_out);
  TACO_CUDA_CHECK_LAUNCH();
  return TACO_OK;
}

extern "C" int taco_uniforms(int count, const uint32_t *step, const uint32_t *ant, const uint32_t *city,
                             uint64_t seed, uint32_t iteration, float *u_out, void *stream) {
  if (count < 0) return TACO_ERR_ARG;
  if (count == 0) return TACO_OK;
  uint32_t k0, k1;
  split_seed(seed, &k0, &k1);
  k_uniforms<<<(count + 255) / 256, 256, 0, reinterpret_cast<cudaStream_t>(stream)>>>(count, step, ant, city, k0,
                                                                                     k1, iteration, u_out);
  TACO_CUDA_CHECK_LAUNCH();
  return TACO_OK;
}

extern "C" int taco_philox4x32_10(int count, const uint32_t *ctr4, const uint32_t *key2, uint32_t *out4,
                                  void *stream) {
  if (count < 0) return TACO_ERR_ARG;
  if (count == 0) return TACO_OK;
  k_philox<<<(count + 255) / 256, 256, 0, reinterpret_cast<cudaStream_t>(stream)>>>(count, ctr4, key2, out4);
  TACO_CUDA_CHECK_LAUNCH();
  return TACO_OK;
}

extern "C" int taco_select_parity(int n, int m, int step, const double *logw, const double *e_block,
                                  int64_t *current, uint8_t *visited, int64_t *tours, int32_t *status,
                                  void *stream) {
  if (n < 1 || m < 0 || step < 1 || step >= n) return TACO_ERR_ARG;
  if (m == 0) return TACO_OK;
  constexpr int WARPS = 8;
  k_select_parity<WARPS><<<(m + WARPS - 1) / WARPS, WARPS * 32, 0, reinterpret_cast<cudaStream_t>(stream)>>>(
      n, m, step, logw, e_block, current, visited, tours, status);
  TACO_CUDA_CHECK_LAUNCH();
  return TACO_OK;
}
