// Pieces shared by the tour-construction kernels (k_construct.cu: IR / AdaIR,
// k_roulette.cu: RW): the coalesced tour writer, the fused pairwise tour
// length, per-ant shared scratch and the launch helpers.
#pragma once

#include "taco_common.cuh"

namespace taco {

constexpr unsigned kFull = 0xffffffffu;

// The pairwise-tree leaves of length n, prebuilt once per n and device (the
// head of k_row_update.cu's plan image); null while the stream is being
// captured before that image exists.  Kernels copy them instead of having
// thread 0 walk the tree (a serial, local-memory prologue per CTA).
const int2 *leaves_image(int n, cudaStream_t stream);

__device__ __forceinline__ void load_leaves(int n, int L, int2 *leaves, const int2 *img) {
  if (img != nullptr) {
    for (int q = threadIdx.x; q < L; q += blockDim.x) leaves[q] = img[q];
  } else if (threadIdx.x == 0) {
    pw_leaves(n, leaves);
  }
}

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

// Tour length in numpy's pairwise order, fed one edge at a time in position
// order e = 0..n-1 (edge e joins t[e] and t[(e+1) % n]).  Edge lengths of the
// current pairwise-tree leaf (<= 128 positions, taco_common.cuh) are parked in
// a per-ant shared buffer; when the leaf is complete lane 0 sums it with
// pw_leaf_sum, and the leaf sums are folded at the end — the exact operation
// sequence of ndarray.sum(axis=1), at one shared store per step.
struct LeafCost {
  const double *dist;
  const int2 *leaves;
  double *buf;       // per-ant shared buffer, kPwBlock entries
  double *leaf_sum;  // per-ant shared, n_leaves entries
  int n, lane, L, i, len;
  double pending;
  bool active;

  __device__ __forceinline__ void init(const double *d, const int2 *lv, double *b, double *ls, int n_,
                                       int lane_) {
    dist = d;
    leaves = lv;
    buf = b;
    leaf_sum = ls;
    n = n_;
    lane = lane_;
    active = d != nullptr;
    L = 0;
    i = 0;
    len = active ? leaves[0].y : 0;
    pending = 0.0;
  }
  // lane 0 starts loading the length of edge (a, b); it is parked one step later
  __device__ __forceinline__ void load(uint32_t a, uint32_t b) {
    // 32-bit index: n <= 65535, so a * n + b < 2^32 (one IMAD instead of 64-bit math)
    TACO_DCHECK(!active || (a < (uint32_t)n && b < (uint32_t)n));
    if (active && lane == 0) pending = __ldg(dist + (a * (uint32_t)n + b));
  }
  __device__ __forceinline__ void push() {
    if (!active) return;
    if (lane == 0) buf[i] = pending;
    if (++i == len) {
      if (lane == 0) leaf_sum[L] = pw_leaf_sum(len, [&](int q) { return buf[q]; });
      __syncwarp();
      const bool more = leaves[L].x + len < n;  // leaves tile [0, n) exactly
      ++L;
      if (more) {
        len = leaves[L].y;
        i = 0;
      }
    }
  }
  __device__ __forceinline__ double finish() {
    __syncwarp();
    return pw_fold(n, leaf_sum);  // meaningful in lane 0
  }
};

// Tour length of one finished tour row (int32, global, written by this warp)
// in numpy's pairwise order: lanes sum the leaves in parallel (pw_leaf_sum),
// lane 0 folds them.  Plain loads: the row was written in this kernel.
__device__ __forceinline__ double warp_tour_cost(int n, const int32_t *trow, const double *dist,
                                                 const int2 *leaves, int n_leaves, double *ls, int lane) {
  __syncwarp();
  for (int L = lane; L < n_leaves; L += 32) {
    const int2 lf = leaves[L];
    ls[L] = pw_leaf_sum(lf.y, [&](int q) {
      const int s = lf.x + q;
      const int s1 = (s + 1 == n) ? 0 : s + 1;
      TACO_DCHECK((uint32_t)trow[s] < (uint32_t)n && (uint32_t)trow[s1] < (uint32_t)n);
      return __ldg(dist + ((uint32_t)trow[s] * (uint32_t)n + (uint32_t)trow[s1]));
    });
  }
  __syncwarp();
  return pw_fold(n, ls);  // meaningful in lane 0
}

// ---------------------------------------------------------------------------
// No W > 0 candidate left.  The reference keeps choosing in the log domain
// among every unvisited city with P > 0 (selection.py:143-155), however small
// P^(1/gamma) is; W can be 0 where fp32 cannot hold the ratio to the row's
// best (taco_common.cuh selection_weight: below 2^-126 of it, e.g. gamma < 1).
// The fallback scores those cities in f64, log(v_j) / gamma + log(u_j) with
// v = A[cur, j]^alpha (* B[cur, j]) — P itself, or the row's unnormalized
// tau^alpha eta^beta (same argmax up to rounding: log of the row sum is a
// shared shift) — on the same uniforms u_j, first of ties.  Nothing with
// v > 0 either: numpy's argmax of an all -inf row is city 0 (selection.py:
// 152-155), which is taken when unvisited; otherwise the reference asserts
// (colony.py:149) and 0xffffffff is returned.  Rare (never seen with
// gamma >= 1 on the BASELINE configs), so it is a plain strided scan.
// ---------------------------------------------------------------------------
struct Fallback {
  const double *a;  // n x n, row pitch n (nullable: only the all -inf rule)
  const double *b;  // nullable multiplier
  double alpha;
  double inv_gamma;
};

// G lanes (gl = lane index in the group) pick for one ant; every lane of the
// warp must call (shuffles), `active` marks groups that need the pick.  Kept
// out of line with scalar arguments only (keys rebuilt from the kernel
// parameters): inlined, or given the callers' key registers by reference, it
// raised the register pressure of the step loop it never runs in (C3
// construction 1.57 -> 1.69 ms).  Visited set: byte per city (vis8) or bit
// map word (j >> 5) * stride + offset.
static __device__ __noinline__ uint32_t fallback_pick(const Fallback *f, const PhiloxKeys *ks,
                                               const taco_iter_state *state, uint32_t it, uint32_t gant,
                                               uint32_t n, uint32_t cur, uint32_t step, int G, int gl, int active,
                                               const uint32_t *vis, int vis8, int stride, int offset) {
  auto visited = [&](uint32_t j) -> bool {
    if (vis8) return reinterpret_cast<const uint8_t *>(vis)[j] != 0;
    return (vis[(j >> 5) * (uint32_t)stride + (uint32_t)offset] >> (j & 31)) & 1u;
  };
  const double inv_gamma = state != nullptr ? state->inv_gamma_cur : f->inv_gamma;
  const RoundKeys rk = round_keys(*ks, it);
  const AntKey ak = ant_key(gant, rk);
  double best = -INFINITY;
  uint32_t bj = 0xffffffffu;
  if (active && f->a != nullptr) {
    for (uint32_t j = (uint32_t)gl; j < n; j += (uint32_t)G) {
      if (visited(j)) continue;
      const size_t off = (size_t)cur * n + j;
      double v = numpy_scalar_power(f->a[off], f->alpha);
      if (f->b != nullptr) v = __dmul_rn(v, f->b[off]);
      if (!(v > 0.0)) continue;
      const double u = (double)bits_to_uniform(sel_word(j, step, ak, rk));
      const double sc = __dadd_rn(__dmul_rn(log(v), inv_gamma), log(u));
      if (sc > best || bj == 0xffffffffu) best = sc, bj = j;
    }
  }
  for (int o = G / 2; o > 0; o >>= 1) {
    const double ob = __shfl_xor_sync(0xffffffffu, best, o);
    const uint32_t oj = __shfl_xor_sync(0xffffffffu, bj, o);
    if (oj != 0xffffffffu && (bj == 0xffffffffu || ob > best || (ob == best && oj < bj))) best = ob, bj = oj;
  }
  if (active && bj == 0xffffffffu && !visited(0u)) bj = 0;
  return bj;
}

// Rebuild one ant's whole tour by the warp (the cold path of the fast
// kernels: their step loop leaves as soon as a step has no W > 0 candidate,
// so neither this code nor its call weighs on the loop's registers).  Each
// step scans the ant's FULL row — the same product rule argmax_j W * u over
// unvisited j with W > 0, lowest j on ties, with the uniform of the same slot
// (sorted position, or city for the dense table), so every step the fast loop
// did decide comes out identical — and steps without a candidate go to
// fallback_pick.  vals / idx: the row-sorted table (sw, si) or, idx NULL,
// the dense table; ld: their row pitch.  Visited set as in fallback_pick
// (cleared here: nwords 32-bit words of this ant).  Returns false when the
// reference would assert (colony.py:149).
static __device__ __noinline__ bool rebuild_tour(const float *vals, const uint16_t *idx, int ld, uint32_t n,
                                                 const Fallback *f, const PhiloxKeys *ks,
                                                 const taco_iter_state *state, uint32_t it, uint32_t gant,
                                                 uint32_t *vis, int vis8, int stride, int offset, int nwords,
                                                 int32_t *trow, int lane) {
  const RoundKeys rk = round_keys(*ks, it);
  const AntKey ak = ant_key(gant, rk);
  for (int q = lane; q < nwords; q += 32) vis[q * stride + offset] = 0u;
  __syncwarp();
  auto mark = [&](uint32_t j) {
    if (vis8)
      reinterpret_cast<uint8_t *>(vis)[j] = 1;
    else
      vis[(j >> 5) * (uint32_t)stride + (uint32_t)offset] |= 1u << (j & 31);
  };
  auto seen = [&](uint32_t j) -> bool {
    if (vis8) return reinterpret_cast<const uint8_t *>(vis)[j] != 0;
    return (vis[(j >> 5) * (uint32_t)stride + (uint32_t)offset] >> (j & 31)) & 1u;
  };
  uint32_t cur = start_city(n, ak, rk);
  if (lane == 0) {
    mark(cur);
    trow[0] = (int32_t)cur;
  }
  __syncwarp();
  for (uint32_t step = 1; step < n; ++step) {
    uint32_t bkey = 0u, bj = 0xffffffffu;
    const size_t row = (size_t)cur * (uint32_t)ld;
    for (uint32_t k = (uint32_t)lane; k < n; k += 32) {
      const float w = vals[row + k];
      const uint32_t j = idx != nullptr ? (uint32_t)idx[row + k] : k;
      if (!(w > 0.0f) || seen(j)) continue;
      // slot k: the sorted position (sorted table) or the city (dense table)
      const uint32_t x = idx != nullptr ? pos_word(k, step, ak, rk) : sel_word(k, step, ak, rk);
      const uint32_t key = __float_as_uint(__fmul_rn(w, bits_to_uniform(x))) + 1u;
      if (key > bkey || (key == bkey && j < bj)) bkey = key, bj = j;
    }
    const uint32_t mkey = __reduce_max_sync(0xffffffffu, bkey);
    uint32_t nxt;
    if (mkey != 0u) {
      nxt = __reduce_min_sync(0xffffffffu, bkey == mkey ? bj : 0xffffffffu);
    } else {
      nxt = fallback_pick(f, ks, state, it, gant, n, cur, step, 32, lane, 1, vis, vis8, stride, offset);
      if (nxt == 0xffffffffu) return false;
    }
    TACO_DCHECK(nxt < n && !seen(nxt));
    if (lane == 0) {
      mark(nxt);
      trow[step] = (int32_t)nxt;
    }
    __syncwarp();
    cur = nxt;
  }
  return true;
}

// per-ant shared scratch: leaf buffer, leaf sums, visited bitmask (16-B aligned)
__host__ __device__ __forceinline__ size_t ant_scratch_bytes(int n_leaves, int nwords) {
  return ((size_t)8 * kPwBlock + (size_t)8 * n_leaves + (size_t)4 * nwords + 15) & ~(size_t)15;
}

__device__ __forceinline__ bool is_visited(const uint32_t *vis, uint32_t j) {
  return (vis[j >> 5] >> (j & 31)) & 1u;
}

}  // namespace taco


static inline int sm_count() { return taco::device_sm_count(); }

static inline int set_smem(const void *fn, size_t bytes) {
  if (bytes <= 48 * 1024) return TACO_OK;
  const cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
  if (e != cudaSuccess) {
    taco::note_cuda_error(e);
    return TACO_ERR_CUDA;
  }
  return TACO_OK;
}

