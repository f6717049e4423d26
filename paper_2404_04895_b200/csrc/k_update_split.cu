// Solver-mode pheromone update as three streaming kernels (no row staged in
// shared memory, no CTA-wide barriers between per-row phases):
//
//   k_deposit_rows     one warp per row: delta[i, :] = 0, then the k elites'
//                      (prev, next) increments folded in rank order
//                      (accumulate_increments pheromone.py:52-68)
//   k_evap_unnorm      elementwise: tau' = max((1 - rho) tau + delta, 1e-12)
//                      (apply_update pheromone.py:71-83) and
//                      unnorm = tau'^alpha eta^beta, zero diagonal
//                      (compute_probability_matrix colony.py:56-62)
//   k_row_normalize    one warp per row: numpy's pairwise row sum of unnorm
//                      (leaves of <= 128 with eight accumulators, then the
//                      pairwise fold), P = unnorm / sum, W = fp32(P^(1/gamma))
//                      (colony.py:63-69, selection.py:62-75)
//
// Same arithmetic, bit for bit, as the fused k_row_update (k_row_update.cu);
// the split trades one extra pass over delta / unnorm (L2-friendly) for full
// row parallelism in every phase.  Fail-stop (status[3]) as in taco_common.cuh.
#include "taco_common.cuh"

namespace taco {

constexpr unsigned kFullMask = 0xffffffffu;

// SMEM: the warp folds into a shared-memory copy of its delta row and writes
// it out once (short rows); otherwise the fold reads / writes global memory.
template <int WARPS, bool SMEM>
__global__ void __launch_bounds__(WARPS * 32)
    k_deposit_rows(int n, int k, const int2 *__restrict__ nbr, const double *__restrict__ inc, double *delta,
                   const int32_t *status) {
  extern __shared__ __align__(16) unsigned char smem_dep[];
  if (chain_stopped_update(status)) return;
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  for (int i = blockIdx.x * WARPS + warp; i < n; i += gridDim.x * WARPS) {
    double *grow = delta + (size_t)i * n;
    double *drow = SMEM ? reinterpret_cast<double *>(smem_dep) + (size_t)warp * n : grow;
    for (int j = lane; j < n; j += 32) drow[j] = 0.0;
    __syncwarp();
    for (int rbase = 0; rbase < k; rbase += 32) {
      // lane l holds elite rbase + l: its (prev, next) of city i and 1/cost
      const bool have = rbase + lane < k;
      const int2 nb = have ? nbr[(size_t)i * k + rbase + lane] : make_int2(-1, -1);
      const double v_e = have ? inc[rbase + lane] : 0.0;
      for (int half = 0; half < 2; ++half) {
        // entries e = 2q + side of elites rbase + 16 half + q, in rank order
        const int q = 16 * half + (lane >> 1);
        const int px = __shfl_sync(kFullMask, nb.x, q);
        const int py = __shfl_sync(kFullMask, nb.y, q);
        const double v = __shfl_sync(kFullMask, v_e, q);
        const int col = (rbase + q < k) ? ((lane & 1) ? py : px) : -1;
        const unsigned peers = __match_any_sync(kFullMask, col);
        const bool leader = col >= 0 && lane == __ffs(peers) - 1;
        if (__any_sync(kFullMask, __popc(peers) > 1)) {
          double acc = leader ? drow[col] : 0.0;
#pragma unroll
          for (int t = 0; t < 32; ++t) {
            const double x = __shfl_sync(kFullMask, v, t);
            if ((peers >> t) & 1u) acc = __dadd_rn(acc, x);
          }
          if (leader) drow[col] = acc;
        } else if (leader) {
          drow[col] = __dadd_rn(drow[col], v);
        }
        __syncwarp();  // orders this window's stores before the next window's loads
      }
    }
    if (SMEM) {
      for (int j = lane; j < n; j += 32) grow[j] = drow[j];
      __syncwarp();  // the shared row is reused by the warp's next row
    }
  }
}

__global__ void k_evap_unnorm(int n, const double *tau_in, double *tau_out, const double *__restrict__ delta,
                              const double *__restrict__ eta_b, int do_evap, double keep, double alpha,
                              double *unnorm, const int32_t *status) {
  if (chain_stopped_update(status)) return;
  for (int i = blockIdx.x; i < n; i += gridDim.x) {  // whole rows per block: no index division
    const size_t off = (size_t)i * n;
#pragma unroll 4
    for (int j = threadIdx.x; j < n; j += blockDim.x) {
      double t = tau_in[off + j];
      if (do_evap) {
        t = __dadd_rn(__dmul_rn(keep, t), delta != nullptr ? delta[off + j] : 0.0);
        t = (t < 1e-12) ? 1e-12 : t;  // np.maximum(new_tau, TAU_MIN), NaN kept
        if (tau_out != nullptr) tau_out[off + j] = t;
      }
      double v = __dmul_rn(numpy_scalar_power(t, alpha), eta_b[off + j]);
      if (i == j) v = 0.0;  // np.fill_diagonal(unnorm, 0.0)
      unnorm[off + j] = v;
    }
  }
}

// Leaf sum of numpy's pairwise base case by eight lanes (one accumulator each):
// lane r accumulates x[r], x[r+8], ... in order; the eight are combined as
// ((a0+a1)+(a2+a3))+((a4+a5)+(a6+a7)) by an xor butterfly (a+b == b+a, so
// every lane of the group ends with the same bits); the len % 8 tail and
// leaves shorter than 8 are added sequentially by the group's lane 0.
__device__ __forceinline__ double leaf_sum8(const double *x, int len, int r, double &mx) {
  double acc = 0.0;
  if (len >= 8) {
    // the <= 16 elements of this accumulator are loaded before the ordered
    // additions, so the leaf costs one memory latency, not sixteen
    const int cnt = len >> 3;  // full groups of eight (leaves hold <= 128)
    double xs[kPwBlock / 8];
#pragma unroll
    for (int q = 0; q < kPwBlock / 8; ++q) xs[q] = q < cnt ? x[8 * q + r] : 0.0;
#pragma unroll
    for (int q = 0; q < kPwBlock / 8; ++q) mx = fmax(mx, xs[q]);
    acc = xs[0];
#pragma unroll
    for (int q = 1; q < kPwBlock / 8; ++q)
      if (q < cnt) acc = __dadd_rn(acc, xs[q]);
  }
#pragma unroll
  for (int o = 1; o < 8; o <<= 1) acc = __dadd_rn(acc, __shfl_xor_sync(kFullMask, acc, o));
  double res = acc;
  if (r == 0) {
    if (len < 8) {
      res = 0.0;
      for (int i = 0; i < len; ++i) res = __dadd_rn(res, x[i]), mx = fmax(mx, x[i]);
    } else {
      for (int i = len - (len % 8); i < len; ++i) res = __dadd_rn(res, x[i]), mx = fmax(mx, x[i]);
    }
  }
  return res;
}

template <int WARPS>
__global__ void __launch_bounds__(WARPS * 32)
    k_row_normalize(int n, int n_leaves, const double *__restrict__ unnorm, double inv_gamma_arg,
                    const taco_iter_state *state, double *p_out, double *rowsum_out, float *w_out, int ldw,
                    int32_t *status) {
  extern __shared__ __align__(16) unsigned char smem[];
  int2 *leaves = reinterpret_cast<int2 *>(smem);
  double *lsum_all = reinterpret_cast<double *>(smem + (((size_t)8 * n_leaves + 15) & ~(size_t)15));
  __shared__ int s_stop;
  if (threadIdx.x == 0) {
    pw_leaves(n, leaves);
    s_stop = chain_stopped_update(status);
  }
  __syncthreads();
  if (s_stop) return;
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  double *lsum = lsum_all + (size_t)warp * n_leaves;
  const double inv_gamma = state != nullptr ? state->inv_gamma : inv_gamma_arg;
  const int grp = lane >> 3, r = lane & 7;
  for (int i = blockIdx.x * WARPS + warp; i < n; i += gridDim.x * WARPS) {
    const double *row = unnorm + (size_t)i * n;
    // leaf sums, four leaves per pass (eight lanes each), and the row maximum
    double mx = 0.0;
    for (int q0 = 0; q0 < n_leaves; q0 += 4) {
      const int q = q0 + grp;
      const int2 lf = q < n_leaves ? leaves[q] : make_int2(0, 0);
      const double s = leaf_sum8(row + lf.x, lf.y, r, mx);
      if (q < n_leaves && r == 0) lsum[q] = s;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(kFullMask, mx, o));
    __syncwarp();
    double sum = 0.0;
    if (lane == 0) sum = pw_fold(n, lsum);
    sum = __shfl_sync(kFullMask, sum, 0);
    if (lane == 0) {
      if (rowsum_out != nullptr) rowsum_out[i] = sum;
      if (!(isfinite(sum) && sum > 0.0)) record_status(status, TACO_UNDERFLOW, i);
    }
    // P = unnorm / sum (colony.py:69) and the selection table (row scale from
    // the largest P, taco_common.cuh selection_weight)
    const double scale = w_out != nullptr ? selection_scale(__ddiv_rn(mx, sum), inv_gamma) : 1.0;
#pragma unroll 4
    for (int j = lane; j < n; j += 32) {
      const double p = __ddiv_rn(row[j], sum);
      if (p_out != nullptr) p_out[(size_t)i * n + j] = p;
      if (w_out != nullptr) w_out[(size_t)i * ldw + j] = selection_weight(p, inv_gamma, scale);
    }
    if (w_out != nullptr)
      for (int j = n + lane; j < ldw; j += 32) w_out[(size_t)i * ldw + j] = 0.0f;
    __syncwarp();  // lsum is reused by the next row
  }
}

static int sm_count_split() { return device_sm_count(); }

int launch_sort_table(int n, int ldw, const float *w, float *sw, uint16_t *si, cudaStream_t s);  // k_row_update.cu

}  // namespace taco

using namespace taco;

extern "C" int taco_update_split(int n, const double *tau_in, double *tau_out, const double *eta_b,
                                 const int32_t *nbr, const double *inc, int k, int do_evap, double keep,
                                 double alpha, double inv_gamma, double *delta_ws, double *unnorm_ws,
                                 double *p_out, double *rowsum_out, float *w_out, int ldw, float *sw_out,
                                 uint16_t *si_out, int32_t *status, const taco_iter_state *state,
                                 void *stream) {
  if (n < 3 || n > 65535 || tau_in == nullptr || eta_b == nullptr || unnorm_ws == nullptr) return TACO_ERR_ARG;
  if (nbr != nullptr && (inc == nullptr || k < 1 || delta_ws == nullptr || !do_evap)) return TACO_ERR_ARG;
  if ((w_out != nullptr || sw_out != nullptr) && (ldw < n || (ldw % 32) != 0)) return TACO_ERR_ARG;
  if ((sw_out == nullptr) != (si_out == nullptr)) return TACO_ERR_ARG;
  if (sw_out != nullptr && w_out == nullptr) return TACO_ERR_ARG;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  const int sms = sm_count_split();
  constexpr int WARPS = 8;
  if (nbr != nullptr) {
    // delta rows in shared memory while 8 warps' rows fit (n <= ~3000)
    const size_t smem = (size_t)8 * n * WARPS;
    const int2 *nb2 = reinterpret_cast<const int2 *>(nbr);
    const int blocks = (n + WARPS - 1) / WARPS;
    if (smem <= 200 * 1024) {
      if (smem > 48 * 1024 && cudaFuncSetAttribute(k_deposit_rows<WARPS, true>,
                                                   cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                   (int)smem) != cudaSuccess)
        return TACO_ERR_CUDA;
      const int grid = blocks < sms ? blocks : sms;
      k_deposit_rows<WARPS, true><<<grid, WARPS * 32, smem, s>>>(n, k, nb2, inc, delta_ws, status);
    } else {
      const int grid = blocks < sms * 8 ? blocks : sms * 8;
      k_deposit_rows<WARPS, false><<<grid, WARPS * 32, 0, s>>>(n, k, nb2, inc, delta_ws, status);
    }
    TACO_CUDA_CHECK_LAUNCH();
  }
  {
    const int grid = n < sms * 16 ? n : sms * 16;
    k_evap_unnorm<<<grid, 256, 0, s>>>(n, tau_in, tau_out, nbr != nullptr ? delta_ws : nullptr, eta_b, do_evap,
                                       keep, alpha, unnorm_ws, status);
    TACO_CUDA_CHECK_LAUNCH();
  }
  {
    const int n_leaves = pw_num_leaves(n);
    const size_t smem = (((size_t)8 * n_leaves + 15) & ~(size_t)15) + (size_t)8 * n_leaves * WARPS;
    if (smem > 227 * 1024) return TACO_ERR_UNSUPPORTED;
    if (smem > 48 * 1024 &&
        cudaFuncSetAttribute(k_row_normalize<WARPS>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) !=
            cudaSuccess)
      return TACO_ERR_CUDA;
    const int blocks = (n + WARPS - 1) / WARPS;
    const int grid = blocks < sms * 8 ? blocks : sms * 8;
    k_row_normalize<WARPS><<<grid, WARPS * 32, smem, s>>>(n, n_leaves, unnorm_ws, inv_gamma, state, p_out,
                                                          rowsum_out, w_out, ldw, status);
    TACO_CUDA_CHECK_LAUNCH();
  }
  if (sw_out != nullptr) return launch_sort_table(n, ldw, w_out, sw_out, si_out, s);
  return TACO_OK;
}
