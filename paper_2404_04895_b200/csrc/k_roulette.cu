// Roulette-wheel (RW) tour construction, SURVEY §8f row f3.
//
// Reference: colony.construct_tours colony.py:127-141 (RW branch),
// selection.rw_spin_block selection.py:102-127 (≡ rw_spin :80-99),
// rng.step_uniforms rng.py:52-62.  Per ant and step the reference
//   masks its row of P by the unvisited flags,          x_j = P[cur, j] * unvis
//   takes the sequential running sum (np.cumsum),       c_j = c_{j-1} + x_j
//   divides by the total,                               q_j = c_j / c_{n-1}
//   and picks the first j with q_j > u; if none (u >= 1 with q_{n-1} = 1) the
//   last positive-weight j.
// The pick depends on the rounding of the SEQUENTIAL prefix c_j, so a parallel
// scan alone is not exact.  The warp therefore (1) sums the row in parallel,
// (2) locates the crossing with certified error bounds: any summation order of
// N non-negative terms is within gamma_N * sum of the exact value, so with
// E >= |c_seq - c_par| the conditions
//      c_par(j) > theta_hi(u, T, E)   =>  q_j > u      (surely)
//      c_par(j-1) < theta_lo(u, T, E) =>  q_{j-1} <= u (surely)
// (thresholds evaluated with directed rounding) prove j is the reference's
// pick, because the true q_j is monotone in j.  (3) If the crossing is not
// certified (probability ~ n * 2^-50 per step) the warp recomputes the exact
// sequential cumsum — the bit-exact answer either way.
//
// Layout: one warp per ant; a row is read in tiles of 256 doubles.  Pass A
// streams the row with coalesced 16-B pair loads (lane l: pairs l, l+32, l+64,
// l+96 of each tile, all four in flight before any is used), parks per-lane tile
// partials in shared memory and folds them per tile afterwards, so no
// cross-lane dependency stalls the loads.  Pass B re-reads only the crossing
// tile with lane l owning the 8 contiguous columns [t*256 + 8l, +8).  Device
// stream: one 53-bit uniform per (step, ant) from the Philox2x32-10 counter
// (ant, 0xffff | step << 16) — a low half the IR/AdaIR stream never uses (its
// low half is j >> 1 <= 0x7fff); see taco_common.cuh.
#include "construct_common.cuh"

namespace taco {

constexpr int kRwTile = 256;
constexpr int kRwChunk = 32;  // tiles per pass-A chunk

// per-warp lane partials of one chunk (rows padded to 33 against bank conflicts)
__host__ __device__ __forceinline__ size_t rw_part_bytes(int ntiles) {
  return (size_t)8 * 33 * (ntiles < kRwChunk ? ntiles : kRwChunk);
}

// Symmetric butterfly sum: every lane ends with the same bits (a + b == b + a).
__device__ __forceinline__ double warp_sum_sym(double v) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v = __dadd_rn(v, __shfl_xor_sync(kFull, v, o));
  return v;
}

__device__ __forceinline__ double warp_scan_incl(double v, int lane) {
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const double t = __shfl_up_sync(kFull, v, o);
    if (lane >= o) v = __dadd_rn(v, t);
  }
  return v;
}

// Masked row of the device stream: P row + the ant's visited bitmask (smem).
struct BitmaskRow {
  const double *row;
  const uint32_t *vis;
  int n;
  __device__ __forceinline__ double at(int j) const {
    return ((vis[j >> 5] >> (j & 31)) & 1u) ? 0.0 : __ldg(row + j);
  }
  template <bool VEC>
  __device__ __forceinline__ void load8(int j0, double x[8]) const {
    if (j0 >= n) {
#pragma unroll
      for (int v = 0; v < 8; ++v) x[v] = 0.0;
      return;
    }
    const uint32_t mask = (vis[j0 >> 5] >> (j0 & 31)) & 0xffu;  // j0 % 8 == 0: one word
    if (VEC && j0 + 8 <= n) {
      const double2 *p2 = reinterpret_cast<const double2 *>(row + j0);
#pragma unroll
      for (int h = 0; h < 4; ++h) {
        const double2 d = __ldg(p2 + h);
        x[2 * h] = d.x;
        x[2 * h + 1] = d.y;
      }
    } else {
#pragma unroll
      for (int v = 0; v < 8; ++v) x[v] = (j0 + v < n) ? __ldg(row + j0 + v) : 0.0;
    }
#pragma unroll
    for (int v = 0; v < 8; ++v)
      if ((mask >> v) & 1u) x[v] = 0.0;
  }
  // masked sum of the four column pairs (j, j+1), j = base + 64h (base even):
  // all loads are issued before any is consumed.  FULL: the whole tile lies
  // inside the row (no bounds logic); otherwise addresses are clamped into the
  // row and out-of-row pairs zeroed afterwards.
  template <bool VEC, bool FULL>
  __device__ __forceinline__ double quad_pair_sum(int base) const {
    double x[8];
#pragma unroll
    for (int h = 0; h < 4; ++h) {
      const int j = base + 64 * h;
      const int jc = (FULL || j < n) ? j : 0;
      if (VEC) {  // n even and rows 16-B aligned
        const double2 d = __ldg(reinterpret_cast<const double2 *>(row + jc));
        x[2 * h] = d.x;
        x[2 * h + 1] = d.y;
      } else {
        x[2 * h] = __ldg(row + jc);
        x[2 * h + 1] = __ldg(row + ((FULL || jc + 1 < n) ? jc + 1 : jc));
      }
    }
    double s[2] = {0.0, 0.0};
#pragma unroll
    for (int h = 0; h < 4; ++h) {
      const int j = base + 64 * h;
      const uint32_t bits = (FULL || j < n) ? (vis[j >> 5] >> (j & 31)) & 3u : 3u;  // j even: one word
      const bool tail = !FULL && !VEC && j + 1 >= n;
      const double a0 = (bits & 1u) ? 0.0 : x[2 * h];
      const double a1 = ((bits & 2u) || tail) ? 0.0 : x[2 * h + 1];
      s[h & 1] = __dadd_rn(s[h & 1], __dadd_rn(a0, a1));
    }
    return __dadd_rn(s[0], s[1]);
  }
};

// Masked row of the parity hook: P row + the reference's (m, n) visited bytes.
struct ByteMaskRow {
  const double *row;
  const uint8_t *vis;
  int n;
  __device__ __forceinline__ double at(int j) const { return vis[j] ? 0.0 : row[j]; }
  template <bool VEC>
  __device__ __forceinline__ void load8(int j0, double x[8]) const {
#pragma unroll
    for (int v = 0; v < 8; ++v) x[v] = (j0 + v < n && !vis[j0 + v]) ? row[j0 + v] : 0.0;
  }
  template <bool VEC, bool FULL>
  __device__ __forceinline__ double quad_pair_sum(int base) const {
    double s = 0.0;
    for (int h = 0; h < 4; ++h) {
      const int j = base + 64 * h;
      const double x0 = (j < n && !vis[j]) ? row[j] : 0.0;
      const double x1 = (j + 1 < n && !vis[j + 1]) ? row[j + 1] : 0.0;
      s = __dadd_rn(s, __dadd_rn(x0, x1));
    }
    return s;
  }
};

// Exact sequential spin (rw_spin selection.py:92-98 on the masked row): lane 0
// recomputes np.cumsum's running sum.  Returns -1 when no positive weight
// exists for the u >= 1 fallback (the reference's flatnonzero(...)[-1] fails).
template <class Row>
__device__ int rw_exact(const Row &r, int n, double u, int lane) {
  int pick = 0;
  if (lane == 0) {
    double total = 0.0;
    for (int j = 0; j < n; ++j) total = __dadd_rn(total, r.at(j));
    double c = 0.0;
    int found = -1, last_pos = -1;
    for (int j = 0; j < n; ++j) {
      const double x = r.at(j);
      c = __dadd_rn(c, x);
      if (x > 0.0) last_pos = j;
      if (__ddiv_rn(c, total) > u) {
        found = j;
        break;
      }
    }
    if (found < 0) {
      // (scratch > u).argmax() of an all-False row is 0; rows whose CDF tops
      // out at or below u take the last positive weight (selection.py:121-126)
      const double q_last = __ddiv_rn(total, total);
      found = (q_last <= u) ? last_pos : 0;
    }
    pick = found;
  }
  return __shfl_sync(kFull, pick, 0);
}

// One spin for one ant (warp-uniform result).  tile_tot: per-warp shared
// scratch of ntiles doubles.  *exact is set when the certified fast answer was
// unavailable (or force_exact) and the sequential path ran.
template <bool VEC, class Row>
__device__ int rw_pick(const Row &r, int n, int ntiles, double u, double *tile_tot, double *part, int lane,
                       bool force_exact, bool *exact) {
  // pass A: tile totals.  Each lane sums its four column pairs of a tile
  // (coalesced 16-B loads, 512 B per warp instruction) into part[t][lane];
  // no cross-lane work inside the loop, so the loads of consecutive tiles
  // overlap.  Tiles go in chunks of 32; lane l then folds tile c0 + l.
  for (int c0 = 0; c0 < ntiles; c0 += kRwChunk) {
    const int nt = min(kRwChunk, ntiles - c0);
#pragma unroll 2
    for (int t = 0; t < nt; ++t) {
      const int base = (c0 + t) * kRwTile;
      const double s = base + kRwTile <= n ? r.template quad_pair_sum<VEC, true>(base + 2 * lane)
                                           : r.template quad_pair_sum<VEC, false>(base + 2 * lane);
      part[t * 33 + lane] = s;
    }
    __syncwarp();
    if (lane < nt) {  // four independent accumulators: a short dependent chain
      double acc[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
      for (int i = 0; i < 32; ++i) acc[i & 3] = __dadd_rn(acc[i & 3], part[lane * 33 + i]);
      tile_tot[c0 + lane] = __dadd_rn(__dadd_rn(acc[0], acc[1]), __dadd_rn(acc[2], acc[3]));
    }
    __syncwarp();
  }
  double total = 0.0;
  for (int t = lane; t < ntiles; t += 32) total = __dadd_rn(total, tile_tot[t]);
  total = warp_sum_sym(total);

  int pick = -1;
  if (!force_exact && total > 0.0 && total < INFINITY) {
    // every computed partial sum here and every sequential c_j is within
    // gamma_N * total of its exact value (N = padded term count)
    const double err = __dmul_ru(__dmul_ru(2.1 * (double)(ntiles * kRwTile + kRwTile), 0x1p-53), total);
    const double hi = __dadd_ru(__dmul_ru(__dmul_ru(u, __dadd_ru(total, err)), 1.0 + 0x1p-52), err);
    const double lo = __dsub_rd(__dmul_rd(__dmul_rd(u, __dsub_rd(total, err)), 1.0 - 0x1p-52), err);
    // crossing tile: first tile whose inclusive prefix exceeds hi
    int tstar = -1;
    double before = 0.0, carry = 0.0;
    for (int c0 = 0; c0 < ntiles && tstar < 0; c0 += 32) {
      const bool in = c0 + lane < ntiles;
      const double incl = __dadd_rn(carry, warp_scan_incl(in ? tile_tot[c0 + lane] : 0.0, lane));
      double excl = __shfl_up_sync(kFull, incl, 1);
      if (lane == 0) excl = carry;
      const unsigned hit = __ballot_sync(kFull, in && incl > hi);
      if (hit) {
        const int f = __ffs(hit) - 1;
        tstar = c0 + f;
        before = __shfl_sync(kFull, excl, f);
      }
      carry = __shfl_sync(kFull, incl, 31);
    }
    if (tstar >= 0) {
      // pass B: the crossing tile, exclusive/inclusive prefixes per column
      double x[8];
      r.template load8<VEC>(tstar * kRwTile + lane * 8, x);
      double li[8];
      li[0] = x[0];
#pragma unroll
      for (int v = 1; v < 8; ++v) li[v] = __dadd_rn(li[v - 1], x[v]);
      const double incl = warp_scan_incl(li[7], lane);
      double excl = __shfl_up_sync(kFull, incl, 1);
      if (lane == 0) excl = 0.0;
      const double base = __dadd_rn(before, excl);
      int vj = -1;
      double e_before = 0.0;
#pragma unroll
      for (int v = 7; v >= 0; --v) {  // keep the lowest v whose inclusive prefix exceeds hi
        if (__dadd_rn(base, li[v]) > hi) {
          vj = v;
          e_before = v == 0 ? base : __dadd_rn(base, li[v - 1]);
        }
      }
      const unsigned hit = __ballot_sync(kFull, vj >= 0);
      if (hit) {
        const int f = __ffs(hit) - 1;
        const int v = __shfl_sync(kFull, vj, f);
        const double e = __shfl_sync(kFull, e_before, f);
        if (e < lo) pick = tstar * kRwTile + f * 8 + v;
      }
    }
  }
  if (pick < 0 || pick >= n) {
    *exact = true;
    pick = rw_exact(r, n, u, lane);
  }
  return pick;
}

struct RwArgs {
  int n, m_local, ant_offset, nwords, n_leaves, ntiles;
  const double *p;
  const double *dist;
  uint32_t iteration;
  const taco_iter_state *state;  // nullable: iteration from device memory
  int32_t *tours;
  double *costs;
  int32_t *status;
  unsigned long long *exact_count;
  int force_exact;
  PhiloxKeys ks;
};

__host__ __device__ __forceinline__ size_t rw_warp_bytes(int n_leaves, int nwords, int ntiles) {
  return ant_scratch_bytes(n_leaves, nwords) + (((size_t)8 * ntiles + 15) & ~(size_t)15) + rw_part_bytes(ntiles);
}

// Shared memory: int2 leaves[n_leaves]; per warp (ant): leaf buffer, leaf
// sums, visited bitmask, tile totals.
// __launch_bounds__(128, 7): <= 72 registers, so 28 ants per SM stay resident
// (the headline colony, 4096 ants on 148 SMs, runs in one wave)
template <int WARPS, bool VEC>
__global__ void __launch_bounds__(WARPS * 32, 7) k_construct_rw(const __grid_constant__ RwArgs a) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int n = a.n;
  int2 *leaves = reinterpret_cast<int2 *>(smem);
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  unsigned char *mine = smem + (((size_t)8 * a.n_leaves + 15) & ~(size_t)15) +
                        rw_warp_bytes(a.n_leaves, a.nwords, a.ntiles) * warp;
  double *leaf_buf = reinterpret_cast<double *>(mine);
  double *leaf_sum = leaf_buf + kPwBlock;
  uint32_t *vis = reinterpret_cast<uint32_t *>(leaf_sum + a.n_leaves);
  double *tile_tot = reinterpret_cast<double *>(mine + ant_scratch_bytes(a.n_leaves, a.nwords));
  double *part = tile_tot + ((a.ntiles + 1) & ~1);
  if (threadIdx.x == 0) pw_leaves(n, leaves);
  __syncthreads();
  const int ant = blockIdx.x * WARPS + warp;
  if (ant >= a.m_local) return;
  if (__shfl_sync(kFull, lane == 0 ? (int)chain_stopped_construct(a.status) : 0, 0)) return;  // fail-stop
  const uint32_t gant = (uint32_t)(a.ant_offset + ant);
  const uint32_t it = a.state != nullptr ? a.state->iteration : a.iteration;
  const RoundKeys rk = round_keys(a.ks, it);
  const AntKey ak = ant_key(gant, rk);
  for (int q = lane; q < a.nwords; q += 32) vis[q] = 0u;
  const uint32_t start = start_city((uint32_t)n, ak, rk);
  __syncwarp();
  if (lane == 0) vis[start >> 5] |= 1u << (start & 31);
  __syncwarp();

  TourWriter tw{a.tours + (size_t)ant * n, n, lane, 0};
  tw.put(0, (int32_t)start);
  LeafCost lc;
  lc.init(a.costs != nullptr ? a.dist : nullptr, leaves, leaf_buf, leaf_sum, n, lane);
  uint32_t cur = start;
  unsigned exact_steps = 0;
  for (int step = 1; step < n; ++step) {
    const double u = rw_threshold((uint32_t)step, ak, rk);
    const BitmaskRow row{a.p + (size_t)cur * n, vis, n};
    bool exact = false;
    const int j = rw_pick<VEC>(row, n, a.ntiles, u, tile_tot, part, lane, a.force_exact != 0, &exact);
    exact_steps += exact ? 1u : 0u;
    if (j < 0 || is_visited(vis, (uint32_t)j)) {
      if (lane == 0) record_status(a.status, TACO_NO_CANDIDATE, (int)gant);
      return;
    }
    __syncwarp();
    if (lane == 0) vis[j >> 5] |= 1u << (j & 31);
    if (step > 1) lc.push();
    lc.load(cur, (uint32_t)j);
    __syncwarp();
    tw.put(step, (int32_t)j);
    cur = (uint32_t)j;
  }
  tw.flush();
  if (lc.active) {
    lc.push();
    lc.load(cur, start);
    lc.push();
    const double c = lc.finish();
    if (lane == 0) a.costs[ant] = c;
  }
  if (lane == 0 && a.exact_count != nullptr && exact_steps) atomicAdd(a.exact_count, (unsigned long long)exact_steps);
}

// One lockstep round of the reference's rw_spin_block with the reference's
// thresholds u (parity mode): next = spin(P[cur] * unvisited, u[a]), the
// visited assertion (colony.py:149), then current / visited / tours update.
template <int WARPS>
__global__ void __launch_bounds__(WARPS * 32)
    k_rw_parity(int n, int m, int step, int ntiles, const double *__restrict__ p, const double *__restrict__ u,
                int64_t *current, uint8_t *visited, int64_t *tours, int32_t *status,
                unsigned long long *exact_count, int force_exact) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int a = blockIdx.x * WARPS + warp;
  if (a >= m) return;
  double *tile_tot = reinterpret_cast<double *>(smem + (size_t)warp * (8 * (size_t)ntiles + rw_part_bytes(ntiles)));
  double *part = tile_tot + ntiles;
  const int64_t cur = current[a];
  const ByteMaskRow row{p + (size_t)cur * n, visited + (size_t)a * n, n};
  bool exact = false;
  const int j = rw_pick<false>(row, n, ntiles, u[a], tile_tot, part, lane, force_exact != 0, &exact);
  if (lane == 0) {
    if (exact && exact_count != nullptr) atomicAdd(exact_count, 1ull);
    if (j < 0) {
      record_status(status, TACO_NO_CANDIDATE, a);
      return;
    }
    if (visited[(size_t)a * n + j]) record_status(status, TACO_NO_CANDIDATE, a);
    visited[(size_t)a * n + j] = 1;
    current[a] = j;
    tours[(size_t)a * n + step] = j;
  }
}

__global__ void k_rw_uniforms(int count, const uint32_t *step, const uint32_t *ant, PhiloxKeys ks,
                              uint32_t iteration, double *out) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= count) return;
  const RoundKeys rk = round_keys(ks, iteration);
  out[t] = rw_threshold(step[t], ant_key(ant[t], rk), rk);
}

}  // namespace taco

using namespace taco;

extern "C" int taco_construct_rw(int n, int m_local, int ant_offset, const double *p, uint64_t seed,
                                 uint32_t iteration, const double *dist, int32_t *tours_out, double *costs_out,
                                 int32_t *status, unsigned long long *exact_count, int force_exact,
                                 const taco_iter_state *state, void *stream) {
  if (n < 3 || n > 65535 || m_local < 0 || ant_offset < 0 || p == nullptr || tours_out == nullptr)
    return TACO_ERR_ARG;
  if (costs_out != nullptr && dist == nullptr) return TACO_ERR_ARG;
  if (m_local == 0) return TACO_OK;
  constexpr int WARPS = 4;
  const int nwords = (n + 31) / 32;
  const int n_leaves = pw_num_leaves(n);
  const int ntiles = (n + kRwTile - 1) / kRwTile;
  const size_t smem = (((size_t)8 * n_leaves + 15) & ~(size_t)15) + rw_warp_bytes(n_leaves, nwords, ntiles) * WARPS;
  if (smem > 227 * 1024) return TACO_ERR_UNSUPPORTED;
  RwArgs a{n, m_local, ant_offset, nwords, n_leaves, ntiles, p, dist, iteration, state, tours_out, costs_out,
           status, exact_count, force_exact, philox_keys(seed)};
  const bool vec = (n % 2 == 0) && ((reinterpret_cast<uintptr_t>(p) & 15u) == 0);
  const int grid = (m_local + WARPS - 1) / WARPS;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  if (vec) {
    if (set_smem((const void *)k_construct_rw<WARPS, true>, smem) != TACO_OK) return TACO_ERR_CUDA;
    k_construct_rw<WARPS, true><<<grid, WARPS * 32, smem, s>>>(a);
  } else {
    if (set_smem((const void *)k_construct_rw<WARPS, false>, smem) != TACO_OK) return TACO_ERR_CUDA;
    k_construct_rw<WARPS, false><<<grid, WARPS * 32, smem, s>>>(a);
  }
  TACO_CUDA_CHECK_LAUNCH();
  return TACO_OK;
}

extern "C" int taco_rw_parity(int n, int m, int step, const double *p, const double *u, int64_t *current,
                              uint8_t *visited, int64_t *tours, int32_t *status, unsigned long long *exact_count,
                              int force_exact, void *stream) {
  if (n < 1 || m < 0 || step < 1 || step >= n || p == nullptr || u == nullptr) return TACO_ERR_ARG;
  if (m == 0) return TACO_OK;
  constexpr int WARPS = 8;
  const int ntiles = (n + kRwTile - 1) / kRwTile;
  const size_t smem = ((size_t)8 * ntiles + rw_part_bytes(ntiles)) * WARPS;
  if (set_smem((const void *)k_rw_parity<WARPS>, smem) != TACO_OK) return TACO_ERR_CUDA;
  k_rw_parity<WARPS><<<(m + WARPS - 1) / WARPS, WARPS * 32, smem, reinterpret_cast<cudaStream_t>(stream)>>>(
      n, m, step, ntiles, p, u, current, visited, tours, status, exact_count, force_exact);
  TACO_CUDA_CHECK_LAUNCH();
  return TACO_OK;
}

extern "C" int taco_rw_uniforms(int count, const uint32_t *step, const uint32_t *ant, uint64_t seed,
                                uint32_t iteration, double *u_out, void *stream) {
  if (count < 0) return TACO_ERR_ARG;
  if (count == 0) return TACO_OK;
  k_rw_uniforms<<<(count + 255) / 256, 256, 0, reinterpret_cast<cudaStream_t>(stream)>>>(
      count, step, ant, philox_keys(seed), iteration, u_out);
  TACO_CUDA_CHECK_LAUNCH();
  return TACO_OK;
}
