// Tour lengths, elite ordering, elite edge map, best-so-far tracking and the
// log-weight table.
//
// Reference: model.batch_costs model.py:292-295, pheromone.select_elite
// pheromone.py:17-25, edge_index_matrix pheromone.py:28-38 (edge map feeding
// the fused deposit in k_row_update.cu), selection.scaled_log_weights
// selection.py:62-75.
#include <cub/device/device_radix_sort.cuh>

#include "taco_common.cuh"

namespace taco {

// one warp per ant: lanes sum the pairwise-tree leaves of the gathered edge
// lengths, lane 0 folds them (numpy's (m, n).sum(axis=1) order)
template <int WARPS, typename TourT>
__global__ void __launch_bounds__(WARPS * 32)
    k_tour_cost(int n, int m, const TourT *__restrict__ tours, const double *__restrict__ dist,
                double *__restrict__ costs, int n_leaves) {
  extern __shared__ __align__(16) unsigned char smem[];
  int2 *leaves = reinterpret_cast<int2 *>(smem);
  double *leaf_sum = reinterpret_cast<double *>(smem + 8 * (size_t)n_leaves);
  if (threadIdx.x == 0) pw_leaves(n, leaves);
  __syncthreads();
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int a = blockIdx.x * WARPS + warp;
  if (a >= m) return;
  const TourT *t = tours + (size_t)a * n;
  double *ls = leaf_sum + (size_t)warp * n_leaves;
  for (int L = lane; L < n_leaves; L += 32) {
    const int2 lf = leaves[L];
    ls[L] = pw_leaf_sum(lf.y, [&](int q) {
      const int s = lf.x + q;
      const int s1 = (s + 1 == n) ? 0 : s + 1;
      return __ldg(dist + (size_t)t[s] * n + (size_t)t[s1]);
    });
  }
  __syncwarp();
  if (lane == 0) costs[a] = pw_fold(n, ls);
}

// Stable rank by counting for small colonies: rank(a) = #{b : c_b < c_a} +
// #{b < a : c_b == c_a}; order[rank(a)] = a.  Every CTA stages all m costs in
// shared memory; one thread per ant.  Exact np.argsort(kind="stable").
constexpr int kRankMaxM = 16384;

constexpr int kRankWarps = 8;
constexpr int kRankAntsPerWarp = 4;

// one warp ranks kRankAntsPerWarp ants: lanes split the comparison range,
// redux.sync adds the partial counts
__global__ void __launch_bounds__(kRankWarps * 32)
    k_elite_rank(int m, const double *__restrict__ costs, int32_t *order) {
  extern __shared__ unsigned long long keys[];
  for (int b = threadIdx.x; b < m; b += blockDim.x) keys[b] = (unsigned long long)__double_as_longlong(costs[b]);
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int first = (blockIdx.x * kRankWarps + (threadIdx.x >> 5)) * kRankAntsPerWarp;
  for (int a = first; a < first + kRankAntsPerWarp && a < m; ++a) {
    const unsigned long long ka = keys[a];
    unsigned cnt = 0;
    for (int b = lane; b < m; b += 32) {
      const unsigned long long kb = keys[b];
      cnt += (kb < ka) || (kb == ka && b < a);  // earlier ants win ties
    }
    const unsigned rank = __reduce_add_sync(0xffffffffu, cnt);
    if (lane == 0) order[rank] = a;
  }
}

__global__ void k_cost_keys(int m, const double *costs, unsigned long long *keys, int32_t *vals) {
  const int a = blockIdx.x * blockDim.x + threadIdx.x;
  if (a < m) {
    // non-negative finite doubles order like their bit patterns
    keys[a] = (unsigned long long)__double_as_longlong(costs[a]);
    vals[a] = a;
  }
}

template <typename TourT>
__global__ void k_elite_neighbors(int n, int k, const TourT *__restrict__ tours, const int32_t *order,
                                  const double *costs, int2 *nbr, double *inc) {
  const size_t idx = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= (size_t)k * n) return;
  const int r = (int)(idx / n);
  const int s = (int)(idx % n);
  const int a = order[r];
  const TourT *t = tours + (size_t)a * n;
  const int city = (int)t[s];
  const int prev = (int)t[s == 0 ? n - 1 : s - 1];
  const int next = (int)t[s + 1 == n ? 0 : s + 1];
  // a failed construction leaves partial rows (the iteration's update is then
  // skipped through status[3]): never index with them
  if ((unsigned)city >= (unsigned)n || (unsigned)prev >= (unsigned)n || (unsigned)next >= (unsigned)n) return;
  nbr[(size_t)city * k + r] = make_int2(prev, next);  // city-major: row i reads k contiguous pairs
  if (s == 0) inc[r] = __ddiv_rn(1.0, costs[a]);  // pheromone.py:66 inc = 1.0 / cost
}

// Costs-first exchange, local half: elite row r = this rank's tour of global
// ant order[r] when it owns it, zeros otherwise (a SUM all-reduce over the
// ranks then assembles every elite tour exactly); elite_costs[r] =
// costs_all[order[r]] on every rank.
__global__ void k_shard_elites(int n, int k, const int32_t *__restrict__ order, int ant_offset, int count,
                               const int32_t *__restrict__ tours_local, const double *__restrict__ costs_all,
                               int32_t *elite_tours, double *elite_costs) {
  const int r = blockIdx.x;
  const int a = order[r];
  const bool mine = a >= ant_offset && a < ant_offset + count;
  const int32_t *src = tours_local + (size_t)(mine ? a - ant_offset : 0) * n;
  int32_t *dst = elite_tours + (size_t)r * n;
  for (int s = threadIdx.x; s < n; s += blockDim.x) dst[s] = mine ? src[s] : 0;
  if (threadIdx.x == 0) elite_costs[r] = costs_all[a];
}

__global__ void k_track_best(int n, const int32_t *tours, const double *costs, const int32_t *order,
                             double *best_cost, int32_t *best_tour, int32_t *best_iter, uint32_t iteration,
                             const int32_t *status, const taco_iter_state *state) {
  __shared__ int s_take;
  __shared__ int s_ant;
  if (chain_stopped_update(status)) return;  // a failed construction: no best from its rows
  if (threadIdx.x == 0) {
    const int a = order[0];
    const double c = costs[a];
    s_ant = a;
    s_take = (c < *best_cost);
  }
  __syncthreads();
  if (!s_take) return;
  const int32_t *t = tours + (size_t)s_ant * n;
  for (int s = threadIdx.x; s < n; s += blockDim.x) best_tour[s] = t[s];
  __syncthreads();
  if (threadIdx.x == 0) {
    *best_cost = costs[s_ant];
    *best_iter = (int32_t)(state != nullptr ? state->iteration : iteration);
  }
}

__global__ void k_log_weights(int64_t count, const double *p, double gamma, double *out) {
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < count;
       t += (int64_t)gridDim.x * blockDim.x) {
    const double v = p[t];
    out[t] = (v > 0.0) ? __ddiv_rn(log(v), gamma) : -INFINITY;
  }
}

// dist / eta of an unrounded Euclidean instance from (n, 2) coordinates, with
// numpy's operation order (model.py:124-134 -> _instance_from_dist 82-97):
// d = sqrt(dx*dx + dy*dy) (two products, one sum, IEEE sqrt), eta = 1.0 / d
// off the diagonal (1e-10 stands in for a zero distance when lenient).
// Edge weight of one city pair under the instance builders' conventions:
//   TACO_EDGE_EXACT  sqrt(dx*dx + dy*dy)           euclidean_instance model.py:124-134
//   TACO_EDGE_EUC_2D int(sqrt(..) + 0.5)            tsplib.distance tsplib.py:207-208
//   TACO_EDGE_CEIL_2D ceil(sqrt(..))                tsplib.py:209-210
//   TACO_EDGE_ATT    r = sqrt(../10); t = int(r+.5); t + (t < r)   tsplib.py:211-214
// All roundings explicit (no FMA contraction), so the f64 results are the
// host's bit for bit.  x >= 0 everywhere, so int() truncation == floor.
__device__ __forceinline__ double edge_weight(double dx, double dy, int kind) {
  const double ss = __dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy));
  switch (kind) {
    case TACO_EDGE_EUC_2D:
      return trunc(__dadd_rn(__dsqrt_rn(ss), 0.5));
    case TACO_EDGE_CEIL_2D:
      return ceil(__dsqrt_rn(ss));
    case TACO_EDGE_ATT: {
      const double r = __dsqrt_rn(__ddiv_rn(ss, 10.0));
      const double t = trunc(__dadd_rn(r, 0.5));
      return t < r ? __dadd_rn(t, 1.0) : t;
    }
    default:
      return __dsqrt_rn(ss);
  }
}

// One grid row per city i (blockIdx.y), columns j across x.  dist/eta follow
// _instance_from_dist (model.py:82-97): eta = 1/d off the diagonal, 0 on it;
// a zero off-diagonal distance is DegenerateInstance unless lenient (then
// eta = 1/1e-10).  status[1] = smallest row holding such a zero (the first
// row-major zero lies in that row, so the host finds its column).
__global__ void k_coord_instance(int n, const double *__restrict__ xy, int kind, double *dist, double *eta,
                                 int lenient, int32_t *status) {
  const int i = blockIdx.y;
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= n) return;
  const size_t t = (size_t)i * n + j;
  if (i == j) {
    dist[t] = 0.0;
    eta[t] = 0.0;
    return;
  }
  const double d = edge_weight(__dsub_rn(xy[2 * i], xy[2 * j]), __dsub_rn(xy[2 * i + 1], xy[2 * j + 1]), kind);
  dist[t] = d;
  if (d == 0.0) {
    if (!lenient) record_status(status, TACO_DEGENERATE, i);
    eta[t] = __ddiv_rn(1.0, 1e-10);
  } else {
    eta[t] = __ddiv_rn(1.0, d);
  }
}

static size_t align256(size_t x) { return (x + 255) & ~(size_t)255; }

static size_t cub_temp_bytes(int m) {
  size_t bytes = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, bytes, (const unsigned long long *)nullptr,
                                  (unsigned long long *)nullptr, (const int32_t *)nullptr, (int32_t *)nullptr, m);
  return bytes;
}

}  // namespace taco

using namespace taco;

extern "C" int taco_tour_cost(int n, int m, const void *tours, int tours_is_i64, const double *dist,
                              double *costs_out, void *stream) {
  if (n < 1 || m < 0 || tours == nullptr || dist == nullptr || costs_out == nullptr) return TACO_ERR_ARG;
  if (m == 0) return TACO_OK;
  constexpr int WARPS = 8;
  const int n_leaves = pw_num_leaves(n);
  const size_t smem = 8 * (size_t)n_leaves + 8 * (size_t)WARPS * n_leaves;
  if (smem > 200 * 1024) return TACO_ERR_UNSUPPORTED;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  const int grid = (m + WARPS - 1) / WARPS;
  if (tours_is_i64) {
    if (smem > 48 * 1024)
      cudaFuncSetAttribute(k_tour_cost<WARPS, int64_t>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    k_tour_cost<WARPS, int64_t><<<grid, WARPS * 32, smem, s>>>(n, m, (const int64_t *)tours, dist, costs_out,
                                                               n_leaves);
  } else {
    if (smem > 48 * 1024)
      cudaFuncSetAttribute(k_tour_cost<WARPS, int32_t>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    k_tour_cost<WARPS, int32_t><<<grid, WARPS * 32, smem, s>>>(n, m, (const int32_t *)tours, dist, costs_out,
                                                               n_leaves);
  }
  TACO_CUDA_CHECK_LAUNCH();
  return TACO_OK;
}

extern "C" size_t taco_elite_workspace_bytes(int m) {
  if (m <= kRankMaxM) return 0;  // counting-rank kernel needs no workspace
  return align256((size_t)m * 8) * 2 + align256((size_t)m * 4) + align256(cub_temp_bytes(m));
}

extern "C" int taco_elite_order(int m, const double *costs, int32_t *order_out, void *workspace, size_t ws_bytes,
                                void *stream) {
  if (m < 1 || costs == nullptr || order_out == nullptr) return TACO_ERR_ARG;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  if (m <= kRankMaxM) {
    const size_t smem = (size_t)m * 8;
    if (smem > 48 * 1024 &&
        cudaFuncSetAttribute(k_elite_rank, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
      return TACO_ERR_CUDA;
    constexpr int per_cta = kRankWarps * kRankAntsPerWarp;
    k_elite_rank<<<(m + per_cta - 1) / per_cta, kRankWarps * 32, smem, st>>>(m, costs, order_out);
    TACO_CUDA_CHECK_LAUNCH();
    return TACO_OK;
  }
  if (ws_bytes < taco_elite_workspace_bytes(m) || workspace == nullptr) return TACO_ERR_ARG;
  unsigned char *ws = reinterpret_cast<unsigned char *>(workspace);
  auto *keys_in = reinterpret_cast<unsigned long long *>(ws);
  ws += align256((size_t)m * 8);
  auto *keys_out = reinterpret_cast<unsigned long long *>(ws);
  ws += align256((size_t)m * 8);
  auto *vals_in = reinterpret_cast<int32_t *>(ws);
  ws += align256((size_t)m * 4);
  size_t temp = cub_temp_bytes(m);
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  k_cost_keys<<<(m + 255) / 256, 256, 0, s>>>(m, costs, keys_in, vals_in);
  TACO_CUDA_CHECK_LAUNCH();
  // LSD radix sort is stable: equal costs keep ascending ant order, exactly
  // np.argsort(costs, kind="stable")
  if (cub::DeviceRadixSort::SortPairs(ws, temp, keys_in, keys_out, vals_in, order_out, m, 0, 64, s) !=
      cudaSuccess)
    return TACO_ERR_CUDA;
  TACO_CUDA_CHECK_LAUNCH();
  return TACO_OK;
}

extern "C" int taco_elite_neighbors(int n, int k, const void *tours, int tours_is_i64, const int32_t *order,
                                    const double *costs, int32_t *nbr_out, double *inc_out, void *stream) {
  if (n < 3 || k < 1 || tours == nullptr || order == nullptr || costs == nullptr) return TACO_ERR_ARG;
  const size_t total = (size_t)k * n;
  const int grid = (int)((total + 255) / 256);
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  if (tours_is_i64)
    k_elite_neighbors<int64_t><<<grid, 256, 0, s>>>(n, k, (const int64_t *)tours, order, costs,
                                                    reinterpret_cast<int2 *>(nbr_out), inc_out);
  else
    k_elite_neighbors<int32_t><<<grid, 256, 0, s>>>(n, k, (const int32_t *)tours, order, costs,
                                                    reinterpret_cast<int2 *>(nbr_out), inc_out);
  TACO_CUDA_CHECK_LAUNCH();
  return TACO_OK;
}

extern "C" int taco_shard_elites(int n, int k, const int32_t *order, int ant_offset, int count,
                                 const int32_t *tours_local, const double *costs_all, int32_t *elite_tours,
                                 double *elite_costs, void *stream) {
  if (n < 1 || k < 1 || ant_offset < 0 || count < 0 || order == nullptr || tours_local == nullptr ||
      costs_all == nullptr || elite_tours == nullptr || elite_costs == nullptr)
    return TACO_ERR_ARG;
  k_shard_elites<<<k, 256, 0, reinterpret_cast<cudaStream_t>(stream)>>>(n, k, order, ant_offset, count, tours_local,
                                                                        costs_all, elite_tours, elite_costs);
  TACO_CUDA_CHECK_LAUNCH();
  return TACO_OK;
}

extern "C" int taco_track_best(int n, const int32_t *tours, const double *costs, const int32_t *order,
                               double *best_cost, int32_t *best_tour, int32_t *best_iter, uint32_t iteration,
                               const int32_t *status, const taco_iter_state *state, void *stream) {
  if (n < 1) return TACO_ERR_ARG;
  k_track_best<<<1, 256, 0, reinterpret_cast<cudaStream_t>(stream)>>>(n, tours, costs, order, best_cost,
                                                                      best_tour, best_iter, iteration, status, state);
  TACO_CUDA_CHECK_LAUNCH();
  return TACO_OK;
}

extern "C" int taco_log_weights(int64_t count, const double *p, double gamma, double *logw_out, void *stream) {
  if (count < 0 || !(gamma > 0.0)) return TACO_ERR_ARG;
  if (count == 0) return TACO_OK;
  const int64_t blocks64 = (count + 255) / 256;
  const int grid = (int)(blocks64 < 148 * 16 ? blocks64 : 148 * 16);
  k_log_weights<<<grid, 256, 0, reinterpret_cast<cudaStream_t>(stream)>>>(count, p, gamma, logw_out);
  TACO_CUDA_CHECK_LAUNCH();
  return TACO_OK;
}

namespace taco {
__global__ void k_iter_advance(taco_iter_state *state, const double *inv_gamma_table, int period) {
  const uint32_t next = state->iteration + 1u;
  state->iteration = next;
  state->inv_gamma_cur = state->inv_gamma;
  state->inv_gamma = inv_gamma_table[(next + 1u) % (uint32_t)period];
}
}  // namespace taco

extern "C" int taco_iter_advance(taco_iter_state *state, const double *inv_gamma_table, int period, void *stream) {
  if (state == nullptr || inv_gamma_table == nullptr || period < 1) return TACO_ERR_ARG;
  taco::k_iter_advance<<<1, 1, 0, reinterpret_cast<cudaStream_t>(stream)>>>(state, inv_gamma_table, period);
  TACO_CUDA_CHECK_LAUNCH();
  return TACO_OK;
}

namespace taco {
static thread_local cudaError_t g_last_cuda_error = cudaSuccess;
void note_cuda_error(cudaError_t e) { g_last_cuda_error = e; }
}  // namespace taco

extern "C" const char *taco_last_cuda_error(void) {
  return taco::g_last_cuda_error == cudaSuccess ? "" : cudaGetErrorString(taco::g_last_cuda_error);
}

extern "C" int taco_coord_instance(int n, const double *coords, int edge_weight, double *dist_out,
                                   double *eta_out, int lenient, int32_t *status, void *stream) {
  if (n < 3 || n > 65535 || coords == nullptr || dist_out == nullptr || eta_out == nullptr) return TACO_ERR_ARG;
  if (edge_weight < TACO_EDGE_EXACT || edge_weight > TACO_EDGE_ATT) return TACO_ERR_ARG;
  const dim3 grid((unsigned)((n + 255) / 256), (unsigned)n);
  k_coord_instance<<<grid, 256, 0, reinterpret_cast<cudaStream_t>(stream)>>>(n, coords, edge_weight, dist_out,
                                                                              eta_out, lenient, status);
  TACO_CUDA_CHECK_LAUNCH();
  return TACO_OK;
}

extern "C" int taco_abi_version(void) { return TACO_ABI_VERSION; }

extern "C" const char *taco_status_string(int code) {
  switch (code) {
    case TACO_OK:
      return "ok";
    case TACO_UNDERFLOW:
      return "transition-matrix row normalizer is zero or non-finite";
    case TACO_NO_CANDIDATE:
      return "selector chose a visited city";
    case TACO_DEGENERATE:
      return "two cities are at distance 0";
    case TACO_ERR_ARG:
      return "invalid argument";
    case TACO_ERR_CUDA:
      return "CUDA error";
    case TACO_ERR_UNSUPPORTED:
      return "size outside the compiled kernel variants";
    default:
      return "unknown status";
  }
}
