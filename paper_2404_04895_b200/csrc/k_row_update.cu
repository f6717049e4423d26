// Fused pheromone update + transition matrix + selection table, one row per
// CTA iteration (persistent CTAs stride over the rows).
//
// Replaces, for row i of every n x n matrix (reference file:line):
//   accumulate_increments  pheromone.py:52-68  delta[i, :] in elite rank order
//   apply_update           pheromone.py:71-83  tau' = max((1-rho) tau + delta, 1e-12)
//   compute_probability_matrix colony.py:51-69 P = unnorm / pairwise_rowsum(unnorm)
//   scaled_log_weights     selection.py:62-75  folded into W = fp32(P^(1/gamma))
//
// HBM traffic per row (Solver mode): read tau 8n + eta^beta 8n, write tau 8n,
// write the sorted table 6n, read the row's k elite (prev, next) pairs 8k
// (contiguous: the edge map is city-major).  The row lives in shared memory
// between the phases so tau / unnorm are touched once.
#include <cstdlib>
#include <mutex>
#include <string>

#include <cub/block/block_radix_sort.cuh>

#include "taco_common.cuh"

namespace taco {

struct RowParams {
  int n;
  const double *tau_in;
  double *tau_out;
  const double *eta_b;
  const int2 *nbr;  // [n][k] (prev, next) of city i in elite r
  const double *inc;
  int k;
  const double *delta_in;
  double *delta_out;
  int do_evap;
  double keep;
  int want_p;
  int p_given;  // tau_in holds P itself: no normalization (selection-table mode)
  double alpha;
  double inv_gamma;
  const taco_iter_state *state;  // nullable: inv_gamma from device memory
  double *p_out;
  double *rowsum_out;
  float *w_out;
  int ldw;
  float *sw_out;
  uint16_t *si_out;
  int32_t *status;
  int n_leaves;
  int row_begin, row_end;  // rows [row_begin, row_end) of the n x n matrices (row-partitioned update)
  const unsigned char *plan_image;  // nullable: the pairwise plan prebuilt for n (plan_image_bytes)
};

#ifndef TACO_DEPOSIT_CHUNK
#define TACO_DEPOSIT_CHUNK 512
#endif
constexpr int kDepositChunk = TACO_DEPOSIT_CHUNK;  // elites staged in shared memory per pass
constexpr int kBatch = 4;           // tau / eta^b loads in flight per thread
#ifndef TACO_COLUMNS_MAX
#define TACO_COLUMNS_MAX 256
#endif
constexpr int kColumnsMax = TACO_COLUMNS_MAX;  // column-parallel deposit up to this many distinct columns

// Shared-memory layout (bytes, all regions 16-B aligned):
//   row      double[n]        delta, then unnorm (also the CUB sort workspace)
//   plan     leaves int2[L], left/right/order u16[L], level_start int[42],
//            leaf_sum double[L], ival double[L], hgt u8[L]
//   stage    int2[kDepositChunk], double[kDepositChunk]
//   deposit  column bit map u32[ceil(n/32)], distinct columns int[dcap]
struct RowLayout {
  size_t row_bytes, plan_off, stage_off, bm_off, cols_off, total;
  int dcap;
};

__host__ __device__ inline size_t align16(size_t x) { return (x + 15) & ~(size_t)15; }

// the plan's tables (leaves, left, right, order, level_start) as laid out at
// the start of the plan region, followed by int meta[4] (n_leaves,
// n_internal, height): prebuilt once per n (k_plan_image) and copied by each
// CTA instead of built by one thread (a ~10 us serial prologue per launch)
__host__ __device__ inline size_t plan_tables_bytes(int L) {
  return align16((size_t)8 * L) + 3 * align16((size_t)2 * L) + align16(4 * (kMaxPlanHeight + 2));
}

__host__ __device__ inline RowLayout row_layout(int n, int L, size_t sort_bytes, int dcap = 0) {
  RowLayout l;
  l.row_bytes = align16((size_t)8 * n > sort_bytes ? (size_t)8 * n : sort_bytes);
  l.plan_off = l.row_bytes;
  const size_t plan = align16((size_t)8 * L) + 3 * align16((size_t)2 * L) + align16(4 * (kMaxPlanHeight + 2)) +
                      2 * align16((size_t)8 * L) + align16((size_t)L);
  l.stage_off = l.plan_off + plan;
  l.bm_off = l.stage_off + (size_t)16 * kDepositChunk;
  l.cols_off = l.bm_off + (dcap > 0 ? align16((size_t)4 * ((n + 31) / 32)) : 0);
  l.dcap = dcap;
  l.total = l.cols_off + align16((size_t)4 * dcap);
  return l;
}

template <int BLOCK>
// 1024 threads per SM in flight at <= 64 registers (at 89 registers the 512-thread
// variant ran one CTA per SM: C4 update 2.19 -> 3.25 ms)
__global__ void __launch_bounds__(BLOCK, 1024 / BLOCK) k_row_update(RowParams a, RowLayout lay) {
  extern __shared__ __align__(16) unsigned char smem[];
  double *row = reinterpret_cast<double *>(smem);
  const int L = a.n_leaves > 0 ? a.n_leaves : 1;
  unsigned char *pp = smem + lay.plan_off;
  PwPlan plan;
  plan.leaves = reinterpret_cast<int2 *>(pp);
  pp += align16((size_t)8 * L);
  plan.left = reinterpret_cast<uint16_t *>(pp);
  pp += align16((size_t)2 * L);
  plan.right = reinterpret_cast<uint16_t *>(pp);
  pp += align16((size_t)2 * L);
  plan.order = reinterpret_cast<uint16_t *>(pp);
  pp += align16((size_t)2 * L);
  plan.level_start = reinterpret_cast<int *>(pp);
  pp += align16(4 * (kMaxPlanHeight + 2));
  double *leaf_sum = reinterpret_cast<double *>(pp);
  pp += align16((size_t)8 * L);
  double *ival = reinterpret_cast<double *>(pp);
  pp += align16((size_t)8 * L);
  uint8_t *hgt = pp;
  int2 *nb_stage = reinterpret_cast<int2 *>(smem + lay.stage_off);
  double *inc_stage = reinterpret_cast<double *>(nb_stage + kDepositChunk);
  uint32_t *dep_bm = reinterpret_cast<uint32_t *>(smem + lay.bm_off);
  int *dep_cols = reinterpret_cast<int *>(smem + lay.cols_off);
  __shared__ int s_ndist;
  __shared__ int s_meta[4];  // n_leaves, n_internal, height of the plan; fail-stop flag
  __shared__ double s_wmax[BLOCK / 32];  // per-warp row maxima (selection-table scale)

  const int n = a.n;
  const int tid = threadIdx.x;
  const int lane = tid & 31;
  const bool need_sum = a.want_p && !a.p_given;
  const double inv_gamma = a.state != nullptr ? a.state->inv_gamma : a.inv_gamma;
  const bool have_delta = (a.nbr != nullptr) || (a.delta_in != nullptr);

  // the pairwise tree depends only on n: copied from its prebuilt image, or
  // built once per CTA
  if (need_sum && a.plan_image != nullptr) {
    const int words = (int)(plan_tables_bytes(L) / 16);
    const int4 *src = reinterpret_cast<const int4 *>(a.plan_image);
    int4 *dst = reinterpret_cast<int4 *>(smem + lay.plan_off);
    for (int q = tid; q < words; q += BLOCK) dst[q] = src[q];
    if (tid < 3) s_meta[tid] = reinterpret_cast<const int *>(a.plan_image + plan_tables_bytes(L))[tid];
  } else if (need_sum && tid == 0) {
    pw_plan_build(n, plan, hgt);
    s_meta[0] = plan.n_leaves;
    s_meta[1] = plan.n_internal;
    s_meta[2] = plan.height;
  }
  // fail-stop (taco_common.cuh): tau / P / W untouched after a failed
  // iteration, one decision per CTA
  if (tid == 0) s_meta[3] = chain_stopped_update(a.status);
  __syncthreads();
  if (s_meta[3]) return;
  plan.n_leaves = s_meta[0];
  plan.n_internal = s_meta[1];
  plan.height = s_meta[2];

  for (int i = a.row_begin + blockIdx.x; i < a.row_end; i += gridDim.x) {
    const size_t rowoff = (size_t)i * n;
    // tau / eta^b of this row are loaded kBatch elements per thread at a time;
    // the first batch is issued before the deposit so it lands meanwhile
    double tq[kBatch], eq[kBatch];
    auto load_batch = [&](int jb) {
#pragma unroll
      for (int u = 0; u < kBatch; ++u) {
        const int j = jb + u * BLOCK;
        const bool in = j < n && a.tau_in != nullptr;
        tq[u] = in ? a.tau_in[rowoff + j] : 0.0;
        eq[u] = (in && need_sum) ? a.eta_b[rowoff + j] : 0.0;
      }
    };
    load_batch(tid);

    // ---- delta row ---------------------------------------------------------
    // Column-parallel form (lay.dcap > 0): the row's distinct deposit
    // columns (prev / next of city i in the k elites) are collected first,
    // then each thread owns one of them and walks all k elites in rank
    // order, adding inc_r where the column matches: per column the same
    // sequence ((0 + inc_a) + inc_b) + ... as the reference's per-elite fancy
    // += (pheromone.py:62-67; one cell is hit at most once per elite), with
    // the columns in parallel instead of warp 0 folding 2k entries while the
    // CTA waits (the deposit was 34% of the C3 update, 40% at C4; now half
    // that).  Real colonies have few distinct columns per row (median 42 at
    // C3 from the first iterations, 55 at C4); rows with more than
    // kColumnsMax (random elites) keep the warp fold, which suits them.
    bool dep_done = false;
    if (a.nbr != nullptr && lay.dcap > 0) {
      const int nw = (n + 31) >> 5;
      for (int w = tid; w < nw; w += BLOCK) dep_bm[w] = 0u;
      for (int j = tid; j < n; j += BLOCK) row[j] = 0.0;
      if (tid == 0) s_ndist = 0;
      __syncthreads();
      const int2 *nbi = a.nbr + (size_t)i * a.k;
      for (int r = tid; r < a.k; r += BLOCK) {
        const int2 p = nbi[r];
        TACO_DCHECK((unsigned)p.x < (unsigned)n && (unsigned)p.y < (unsigned)n && p.x != i && p.y != i);
        atomicOr(&dep_bm[p.x >> 5], 1u << (p.x & 31));
        atomicOr(&dep_bm[p.y >> 5], 1u << (p.y & 31));
      }
      __syncthreads();
      for (int w = tid; w < nw; w += BLOCK) {
        uint32_t bits = dep_bm[w];
        if (bits) {
          int at = atomicAdd(&s_ndist, __popc(bits));
          while (bits) {
            const int b = __ffs(bits) - 1;
            if (at < lay.dcap) dep_cols[at] = (w << 5) + b;
            ++at;
            bits &= bits - 1u;
          }
        }
      }
      __syncthreads();
      const int nd = s_ndist;
      if (nd <= lay.dcap && nd <= kColumnsMax && nd <= BLOCK) {  // else the warp fold below
        dep_done = true;
        const int c = tid < nd ? dep_cols[tid] : -2;
        double acc = 0.0;
        for (int rbase = 0; rbase < a.k; rbase += kDepositChunk) {
          const int rcount = min(kDepositChunk, a.k - rbase);
          __syncthreads();
          for (int r = tid; r < rcount; r += BLOCK) {
            nb_stage[r] = nbi[rbase + r];
            inc_stage[r] = a.inc[rbase + r];
          }
          __syncthreads();
          if (tid < nd) {
            for (int r = 0; r < rcount; ++r) {
              const int2 p = nb_stage[r];
              if (p.x == c || p.y == c) acc = __dadd_rn(acc, inc_stage[r]);
            }
          }
        }
        if (c >= 0) row[c] = acc;
      }
    }
    if (a.nbr != nullptr && !dep_done) {
      for (int j = tid; j < n; j += BLOCK) row[j] = 0.0;
      for (int rbase = 0; rbase < a.k; rbase += kDepositChunk) {
        const int rcount = min(kDepositChunk, a.k - rbase);
        __syncthreads();
        for (int r = tid; r < rcount; r += BLOCK) {
          nb_stage[r] = a.nbr[(size_t)i * a.k + rbase + r];  // contiguous per city
          inc_stage[r] = a.inc[rbase + r];
        }
        __syncthreads();
        if (tid < 32) {
          // entries e = 2r + side in rank order; one cell is hit at most once
          // per elite (prev != next for n >= 3), so within a 32-entry window
          // the lanes sharing a column are in rank order and their leader folds
          // them sequentially: ((delta + inc_a) + inc_b) + ... exactly like the
          // reference's per-elite fancy += (pheromone.py:62-67).
          const int total = 2 * rcount;
          for (int base = 0; base < total; base += 32) {
            const int e = base + lane;
            int col = -1;
            double v = 0.0;
            if (e < total) {
              const int2 nb = nb_stage[e >> 1];
              col = (e & 1) ? nb.y : nb.x;
              v = inc_stage[e >> 1];
              TACO_DCHECK((unsigned)col < (unsigned)n && col != i);
            }
            const unsigned peers = __match_any_sync(0xffffffffu, col);
            // every lane folds its column group in lane (= rank) order; the
            // values arrive by shuffle, so the only dependent chain is the
            // group's additions (no shared-memory round trip per element)
            const bool leader = col >= 0 && lane == __ffs(peers) - 1;
            if (__any_sync(0xffffffffu, __popc(peers) > 1)) {
              // leaders walk their group's lanes in increasing (= rank) order;
              // as many rounds as the largest group (not 32)
              unsigned rem = leader ? peers : 0u;
              const int rounds = __reduce_max_sync(0xffffffffu, __popc(rem));
              double acc = leader ? row[col] : 0.0;
#pragma unroll 4
              for (int t = 0; t < rounds; ++t) {
                const int src = rem ? __ffs(rem) - 1 : lane;
                const double x = __shfl_sync(0xffffffffu, v, src);
                if (rem) acc = __dadd_rn(acc, x);
                rem &= rem - 1u;
              }
              if (leader) row[col] = acc;
            } else if (leader) {  // no shared column in this window
              row[col] = __dadd_rn(row[col], v);
            }
            __syncwarp();
          }
        }
      }
    } else if (a.delta_in != nullptr) {
      for (int j = tid; j < n; j += BLOCK) row[j] = a.delta_in[rowoff + j];
    }
    __syncthreads();
    if (a.delta_out != nullptr) {
      for (int j = tid; j < n; j += BLOCK) a.delta_out[rowoff + j] = have_delta ? row[j] : 0.0;
    }
    if (a.tau_in == nullptr) {  // delta-only mode (accumulate_increments)
      __syncthreads();
      continue;
    }

    // ---- tau' and unnormalized weights ---------------------------------------
    double lmax = 0.0;  // the row's largest unnormalized weight (P in selection-table mode)
    for (int jb = tid; jb < n; jb += kBatch * BLOCK) {
      if (jb != tid) load_batch(jb);
#pragma unroll
      for (int u = 0; u < kBatch; ++u) {
        const int j = jb + u * BLOCK;
        if (j >= n) break;
        double t = tq[u];
        if (a.do_evap) {
          const double d = have_delta ? row[j] : 0.0;
          t = __dadd_rn(__dmul_rn(a.keep, t), d);
          t = (t < 1e-12) ? 1e-12 : t;  // np.maximum(new_tau, TAU_MIN), NaN kept
        }
        if (a.tau_out != nullptr) a.tau_out[rowoff + j] = t;
        if (a.p_given) {
          row[j] = t;
          lmax = fmax(lmax, t);
        } else if (a.want_p) {
          double v = __dmul_rn(numpy_scalar_power(t, a.alpha), eq[u]);
          if (j == i) v = 0.0;  // np.fill_diagonal(unnorm, 0.0)
          row[j] = v;
          lmax = fmax(lmax, v);
        }
      }
    }
    if (!a.want_p) {
      __syncthreads();
      continue;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) lmax = fmax(lmax, __shfl_xor_sync(0xffffffffu, lmax, o));
    if (lane == 0) s_wmax[tid >> 5] = lmax;
    __syncthreads();

    // ---- pairwise row sum (numpy order): parallel leaves, parallel fold ----
    double s = 1.0;  // P / 1.0 == P exactly in selection-table mode
    if (need_sum) {
      for (int q = tid; q < plan.n_leaves; q += BLOCK) {
        const int2 lf = plan.leaves[q];
        const double *base = row + lf.x;
        leaf_sum[q] = pw_leaf_sum(lf.y, [&](int x) { return base[x]; });
      }
      __syncthreads();
      s = pw_plan_fold(plan, leaf_sum, ival);
      if (tid == 0) {
        if (a.rowsum_out != nullptr) a.rowsum_out[i] = s;
        if (!(isfinite(s) && s > 0.0)) record_status(a.status, TACO_UNDERFLOW, i);
      }
    }

    // ---- dense outputs (coalesced, striped) ---------------------------------
    if (a.p_out != nullptr || a.w_out != nullptr) {
      // the row's largest P = (largest unnormalized weight) / sum: division
      // is monotone, so this is exactly max_j P[i, j]
      double rmax = s_wmax[0];
#pragma unroll
      for (int q = 1; q < BLOCK / 32; ++q) rmax = fmax(rmax, s_wmax[q]);
      const double scale = a.w_out != nullptr ? selection_scale(__ddiv_rn(rmax, s), inv_gamma) : 1.0;
      for (int j = tid; j < n; j += BLOCK) {
        const double p = __ddiv_rn(row[j], s);
        if (a.p_out != nullptr) a.p_out[rowoff + j] = p;
        if (a.w_out != nullptr) a.w_out[(size_t)i * a.ldw + j] = selection_weight(p, inv_gamma, scale);
      }
      if (a.w_out != nullptr)
        for (int j = n + tid; j < a.ldw; j += BLOCK) a.w_out[(size_t)i * a.ldw + j] = 0.0f;
    }

    __syncthreads();  // row[] is reused by the next row
  }
}

static int sm_count_row() { return device_sm_count(); }

__global__ void k_plan_image(int n, int L, unsigned char *img) {
  PwPlan p;
  unsigned char *q = img;
  p.leaves = reinterpret_cast<int2 *>(q);
  q += align16((size_t)8 * L);
  p.left = reinterpret_cast<uint16_t *>(q);
  q += align16((size_t)2 * L);
  p.right = reinterpret_cast<uint16_t *>(q);
  q += align16((size_t)2 * L);
  p.order = reinterpret_cast<uint16_t *>(q);
  q += align16((size_t)2 * L);
  p.level_start = reinterpret_cast<int *>(q);
  int *meta = reinterpret_cast<int *>(img + plan_tables_bytes(L));
  pw_plan_build(n, p, reinterpret_cast<uint8_t *>(meta + 4));
  meta[0] = p.n_leaves;
  meta[1] = p.n_internal;
  meta[2] = p.height;
}

// the plan image for n on the current device (built on `stream` at first
// use; never freed: a few KB per distinct n).  Null while the stream is being
// captured and no image exists yet (the kernel then builds the plan itself).
static const unsigned char *plan_image(int n, int L, cudaStream_t stream) {
  constexpr int kSlots = 8;
  static int ns[kMaxDevices][kSlots] = {};
  static unsigned char *imgs[kMaxDevices][kSlots] = {};
  static std::mutex mu;  // host threads may launch concurrently (one stream each)
  std::lock_guard<std::mutex> lock(mu);
  const int dev = current_device();
  for (int q = 0; q < kSlots; ++q)
    if (ns[dev][q] == n && imgs[dev][q] != nullptr) return imgs[dev][q];
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  if (cudaStreamIsCapturing(stream, &cs) != cudaSuccess || cs != cudaStreamCaptureStatusNone) return nullptr;
  int slot = -1;
  for (int q = 0; q < kSlots && slot < 0; ++q)
    if (imgs[dev][q] == nullptr) slot = q;
  if (slot < 0) return nullptr;  // many distinct n in one process: build in the kernel
  unsigned char *img = nullptr;
  if (cudaMalloc(&img, plan_tables_bytes(L) + 16 + align16((size_t)L)) != cudaSuccess) {
    (void)cudaGetLastError();
    return nullptr;
  }
  k_plan_image<<<1, 1, 0, stream>>>(n, L, img);
  // once per n and device: complete before any stream can pick the image up
  if (cudaGetLastError() != cudaSuccess || cudaStreamSynchronize(stream) != cudaSuccess) return nullptr;
  ns[dev][slot] = n;
  imgs[dev][slot] = img;
  return img;
}

template <int BLOCK>
static int launch_row_t(const RowParams &a, const RowLayout &lay, cudaStream_t stream) {
  // per device: the shared-memory attribute and the occupancy query
  static size_t configured_[kMaxDevices] = {};
  static int blocks_per_sm_[kMaxDevices] = {};
  static size_t blocks_for_[kMaxDevices] = {};
  const int dev = current_device();
  size_t &configured = configured_[dev], &blocks_for = blocks_for_[dev];
  int &blocks_per_sm = blocks_per_sm_[dev];
  if (lay.total > 48 * 1024 && lay.total > configured) {
    const cudaError_t e =
        cudaFuncSetAttribute(k_row_update<BLOCK>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)lay.total);
    if (e != cudaSuccess) {
      note_cuda_error(e);
      return TACO_ERR_CUDA;
    }
    configured = lay.total;
  }
  if (blocks_for != lay.total) {
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks_per_sm, k_row_update<BLOCK>, BLOCK, lay.total) !=
            cudaSuccess ||
        blocks_per_sm < 1)
      blocks_per_sm = 1;
    blocks_for = lay.total;
  }
  const int sms = sm_count_row();
  const int rows = a.row_end - a.row_begin;
  if (rows <= 0) return TACO_OK;
  const int grid = rows < sms * blocks_per_sm ? rows : sms * blocks_per_sm;
  k_row_update<BLOCK><<<grid, BLOCK, lay.total, stream>>>(a, lay);
  TACO_CUDA_CHECK_LAUNCH();
  return TACO_OK;
}

#ifndef TACO_DEPOSIT_WARP
#define TACO_DEPOSIT_COLUMNS 1
#endif

const int2 *leaves_image(int n, cudaStream_t stream) {
  return reinterpret_cast<const int2 *>(plan_image(n, pw_num_leaves(n), stream));
}

static int launch_row(RowParams a, cudaStream_t stream) {
  a.plan_image = nullptr;
#ifndef TACO_NO_PLAN_IMAGE
  if (a.want_p && !a.p_given && a.n_leaves > 0) a.plan_image = plan_image(a.n, a.n_leaves, stream);
#endif
  int dcap = 0;  // the column-parallel deposit (0: the warp fold)
#ifdef TACO_DEPOSIT_COLUMNS
  if (a.nbr != nullptr && a.k > 0) {
    dcap = 2 * a.k < a.n - 1 ? 2 * a.k : a.n - 1;
    if (dcap > kColumnsMax) dcap = kColumnsMax;  // more distinct columns: the warp fold
  }
#endif
  const RowLayout lay = row_layout(a.n, a.n_leaves > 0 ? a.n_leaves : 1, 0, dcap);
  if (lay.total > 227 * 1024) return TACO_ERR_UNSUPPORTED;
  // CTA width by row length (scripts/row_update_probe.py): 256 threads are
  // best up to n ~ 5000 (n = 2392: 153 us vs 154 / 211 for 128 / 512 with the
  // k = 409 deposit); long rows want 512 (n = 10000: 1565 vs 1832 us)
  if (const char *ev = getenv("TACO_ROW_BLOCK")) {  // tuning knob
    const int b = atoi(ev);
    if (b == 128) return launch_row_t<128>(a, lay, stream);
    if (b == 256) return launch_row_t<256>(a, lay, stream);
    if (b == 512) return launch_row_t<512>(a, lay, stream);
  }
  // re-measured with the prebuilt plan (no per-CTA build): 128 threads at 8
  // CTAs per SM up to n ~ 3000 (n = 2392: 0.157 vs 0.167 ms with the sort,
  // n = 1000: 0.050 vs 0.056; n = 3500: 0.298 vs 0.284)
  if (a.n > 7000) return launch_row_t<512>(a, lay, stream);
  if (a.n > 2800) return launch_row_t<256>(a, lay, stream);
  return launch_row_t<128>(a, lay, stream);
}

// ---------------------------------------------------------------------------
// Row sort of the selection table: sw/si[i, :] = row i of W in descending
// order of the W bits above kSortBit, stable in the column index.  Keys are
// packed (W prefix << 16 | j) so a single 32-bit register per item carries
// both; the exact W is gathered back from a shared copy of the row.  Entries
// past n sort last (prefix 0, larger position) and are not written.
// ---------------------------------------------------------------------------
#ifndef TACO_SORT_RADIX_BITS
#define TACO_SORT_RADIX_BITS 5  // 5-bit digits: -2% at n = 2392, -5% at n = 10000 vs 4 (6: slower; 8: no shared memory)
#endif

template <int BLOCK, int ITEMS, int MINB = 0>
__global__ void __launch_bounds__(BLOCK, MINB) k_row_sort(int n, int row_begin, int row_end, int ldw,
                                                    const float *__restrict__ w, float *__restrict__ sw,
                                                    uint16_t *__restrict__ si) {
  using Sort = cub::BlockRadixSort<uint32_t, BLOCK, ITEMS, cub::NullType, TACO_SORT_RADIX_BITS>;
  extern __shared__ __align__(16) unsigned char smem[];
  auto &ts = *reinterpret_cast<typename Sort::TempStorage *>(smem);
  float *wrow = reinterpret_cast<float *>(smem + ((sizeof(typename Sort::TempStorage) + 15) & ~(size_t)15));
  for (int i = row_begin + blockIdx.x; i < row_end; i += gridDim.x) {
    const float *src = w + (size_t)i * ldw;
    for (int j = threadIdx.x; j < n; j += BLOCK) wrow[j] = src[j];
    __syncthreads();
    uint32_t keys[ITEMS];
#pragma unroll
    for (int q = 0; q < ITEMS; ++q) {
      const int j = threadIdx.x * ITEMS + q;
      keys[q] = j < n ? ((__float_as_uint(wrow[j]) & ~((1u << kSortBit) - 1u)) | (uint32_t)j) : 0xffffu;
    }
    Sort(ts).SortDescendingBlockedToStriped(keys, kSortBit, 31);
#pragma unroll
    for (int q = 0; q < ITEMS; ++q) {
      const int pos = threadIdx.x + q * BLOCK;
      if (pos < n) {
        const uint32_t j = keys[q] & 0xffffu;
        sw[(size_t)i * ldw + pos] = wrow[j];
        si[(size_t)i * ldw + pos] = (uint16_t)j;
      }
    }
    __syncthreads();  // wrow / sort storage reused by the next row
  }
}

template <int BLOCK, int ITEMS, int MINB = 0>
static int launch_sort_t(int n, int r0, int r1, int ldw, const float *w, float *sw, uint16_t *si,
                         cudaStream_t stream) {
  using Sort = cub::BlockRadixSort<uint32_t, BLOCK, ITEMS, cub::NullType, TACO_SORT_RADIX_BITS>;
  const size_t smem = ((sizeof(typename Sort::TempStorage) + 15) & ~(size_t)15) + (size_t)4 * n;
  if (smem > 227 * 1024) return TACO_ERR_UNSUPPORTED;
  static int blocks_per_sm_[kMaxDevices] = {};
  static size_t configured_[kMaxDevices] = {};
  const int dev = current_device();
  int &blocks_per_sm = blocks_per_sm_[dev];
  size_t &configured = configured_[dev];
  if (configured != smem) {
    if (smem > 48 * 1024) {
      const cudaError_t e =
          cudaFuncSetAttribute(k_row_sort<BLOCK, ITEMS, MINB>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      if (e != cudaSuccess) {
        note_cuda_error(e);
        return TACO_ERR_CUDA;
      }
    }
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks_per_sm, k_row_sort<BLOCK, ITEMS, MINB>, BLOCK, smem) !=
            cudaSuccess ||
        blocks_per_sm < 1)
      blocks_per_sm = 1;
    configured = smem;
  }
  const int sms = sm_count_row();
  const int rows = r1 - r0;
  if (rows <= 0) return TACO_OK;
  const int grid = rows < sms * blocks_per_sm ? rows : sms * blocks_per_sm;
  k_row_sort<BLOCK, ITEMS, MINB><<<grid, BLOCK, smem, stream>>>(n, r0, r1, ldw, w, sw, si);
  TACO_CUDA_CHECK_LAUNCH();
  return TACO_OK;
}

static int launch_sort(int n, int r0, int r1, int ldw, const float *w, float *sw, uint16_t *si, cudaStream_t s) {
  if (const char *ev = getenv("TACO_SORT_CFG")) {  // tuning knob: BLOCKxITEMS[xMINB]
    const std::string c(ev);
    if (c == "512x10" && n <= 5120) return launch_sort_t<512, 10>(n, r0, r1, ldw, w, sw, si, s);
    if (c == "512x20x2" && n <= 10240) return launch_sort_t<512, 20, 2>(n, r0, r1, ldw, w, sw, si, s);
    if (c == "1024x10" && n <= 10240) return launch_sort_t<1024, 10>(n, r0, r1, ldw, w, sw, si, s);
    if (c == "256x10x4" && n <= 2560) return launch_sort_t<256, 10, 4>(n, r0, r1, ldw, w, sw, si, s);
    if (c == "256x10" && n <= 2560) return launch_sort_t<256, 10>(n, r0, r1, ldw, w, sw, si, s);
    if (c == "512x5" && n <= 2560) return launch_sort_t<512, 5>(n, r0, r1, ldw, w, sw, si, s);
    if (c == "128x20" && n <= 2560) return launch_sort_t<128, 20>(n, r0, r1, ldw, w, sw, si, s);
    if (c == "128x8" && n <= 1024) return launch_sort_t<128, 8>(n, r0, r1, ldw, w, sw, si, s);
    if (c == "256x20" && n <= 5120) return launch_sort_t<256, 20>(n, r0, r1, ldw, w, sw, si, s);
    if (c == "512x20" && n <= 10240) return launch_sort_t<512, 20>(n, r0, r1, ldw, w, sw, si, s);
  }
  if (n <= 1024) return launch_sort_t<96, 11>(n, r0, r1, ldw, w, sw, si, s);  // vs 128x8: n = 1000 0.046 vs 0.050 ms
  // vs 256x10 and 128x20 at n = 2392: 0.194 / 0.158 / 0.153 ms (row + sort)
  if (n <= 2400) return launch_sort_t<96, 25>(n, r0, r1, ldw, w, sw, si, s);
  if (n <= 2560) return launch_sort_t<128, 20>(n, r0, r1, ldw, w, sw, si, s);
  if (n <= 5120) return launch_sort_t<192, 27>(n, r0, r1, ldw, w, sw, si, s);  // vs 512x10 / 256x20: n = 5000 0.484 / 0.464 / 0.456 ms
  if (n <= 10240) return launch_sort_t<384, 27>(n, r0, r1, ldw, w, sw, si, s);  // vs 512x20: n = 10000 1.96 vs 2.01 ms
  if (n <= 20480) return launch_sort_t<1024, 20>(n, r0, r1, ldw, w, sw, si, s);
  return TACO_ERR_UNSUPPORTED;
}

int launch_sort_table(int n, int ldw, const float *w, float *sw, uint16_t *si, cudaStream_t s) {
  return launch_sort(n, 0, n, ldw, w, sw, si, s);
}

}  // namespace taco

using namespace taco;

extern "C" int taco_max_sorted_n(void) { return 20480; }

static int launch_variant(RowParams &a, bool sorted, cudaStream_t s) {
  const int rc = launch_row(a, s);
  if (rc != TACO_OK || !sorted) return rc;
  return launch_sort(a.n, a.row_begin, a.row_end, a.ldw, a.w_out, a.sw_out, a.si_out, s);
}

static int row_update_impl(int row_begin, int row_end, int n, const double *tau_in, double *tau_out,
                           const double *eta_b, const int32_t *nbr, const double *inc, int k,
                           const double *delta_in, double *delta_out, int do_evap, double keep, int want_p,
                           double alpha, double inv_gamma, double *p_out, double *rowsum_out, float *w_out,
                           int ldw, float *sw_out, uint16_t *si_out, int32_t *status, const taco_iter_state *state,
                           void *stream) {
  if (n < 3 || n > 65535) return TACO_ERR_ARG;
  if (tau_in == nullptr && (do_evap || want_p || tau_out != nullptr)) return TACO_ERR_ARG;
  if (nbr != nullptr && (inc == nullptr || k < 1)) return TACO_ERR_ARG;
  if (nbr != nullptr && delta_in != nullptr) return TACO_ERR_ARG;
  if (want_p && eta_b == nullptr) return TACO_ERR_ARG;
  if ((w_out != nullptr || sw_out != nullptr) && (ldw < n || (ldw % 32) != 0)) return TACO_ERR_ARG;
  if ((sw_out == nullptr) != (si_out == nullptr)) return TACO_ERR_ARG;
  if (sw_out != nullptr && w_out == nullptr) return TACO_ERR_ARG;  // the sort reads the dense table
  if ((sw_out != nullptr || w_out != nullptr || p_out != nullptr) && !want_p) return TACO_ERR_ARG;
  RowParams a;
  a.n = n;
  a.tau_in = tau_in;
  a.tau_out = tau_out;
  a.eta_b = eta_b;
  a.nbr = reinterpret_cast<const int2 *>(nbr);
  a.inc = inc;
  a.k = k;
  a.delta_in = delta_in;
  a.delta_out = delta_out;
  a.do_evap = do_evap;
  a.keep = keep;
  a.want_p = want_p;
  a.p_given = 0;
  a.alpha = alpha;
  a.inv_gamma = inv_gamma;
  a.state = state;
  a.p_out = p_out;
  a.rowsum_out = rowsum_out;
  a.w_out = w_out;
  a.ldw = ldw;
  a.sw_out = sw_out;
  a.si_out = si_out;
  a.status = status;
  a.n_leaves = want_p ? pw_num_leaves(n) : 0;
  a.row_begin = row_begin;
  a.row_end = row_end;
  return launch_variant(a, sw_out != nullptr, reinterpret_cast<cudaStream_t>(stream));
}

extern "C" int taco_row_update(int n, const double *tau_in, double *tau_out, const double *eta_b,
                               const int32_t *nbr, const double *inc, int k, const double *delta_in,
                               double *delta_out, int do_evap, double keep, int want_p, double alpha,
                               double inv_gamma, double *p_out, double *rowsum_out, float *w_out,
                               int ldw, float *sw_out, uint16_t *si_out, int32_t *status,
                               const taco_iter_state *state, void *stream) {
  return row_update_impl(0, n, n, tau_in, tau_out, eta_b, nbr, inc, k, delta_in, delta_out, do_evap, keep, want_p,
                         alpha, inv_gamma, p_out, rowsum_out, w_out, ldw, sw_out, si_out, status, state, stream);
}

// rows [row_begin, row_end) only (row-partitioned multi-GPU update): same
// arguments as taco_row_update; rows outside the range are not touched
extern "C" int taco_row_update_rows(int row_begin, int row_end, int n, const double *tau_in, double *tau_out,
                                    const double *eta_b, const int32_t *nbr, const double *inc, int k,
                                    const double *delta_in, double *delta_out, int do_evap, double keep,
                                    int want_p, double alpha, double inv_gamma, double *p_out, double *rowsum_out,
                                    float *w_out, int ldw, float *sw_out, uint16_t *si_out, int32_t *status,
                                    const taco_iter_state *state, void *stream) {
  if (row_begin < 0 || row_end < row_begin || row_end > n) return TACO_ERR_ARG;
  return row_update_impl(row_begin, row_end, n, tau_in, tau_out, eta_b, nbr, inc, k, delta_in, delta_out, do_evap,
                         keep, want_p, alpha, inv_gamma, p_out, rowsum_out, w_out, ldw, sw_out, si_out, status,
                         state, stream);
}

extern "C" int taco_selection_table(int n, const double *p, double inv_gamma, float *w_out, int ldw,
                                    float *sw_out, uint16_t *si_out, void *stream) {
  if (n < 3 || n > 65535 || p == nullptr) return TACO_ERR_ARG;
  if ((w_out != nullptr || sw_out != nullptr) && (ldw < n || (ldw % 32) != 0)) return TACO_ERR_ARG;
  if ((sw_out == nullptr) != (si_out == nullptr)) return TACO_ERR_ARG;
  if (sw_out != nullptr && w_out == nullptr) return TACO_ERR_ARG;  // the sort reads the dense table
  RowParams a = {};
  a.n = n;
  a.tau_in = p;
  a.want_p = 1;
  a.p_given = 1;
  a.alpha = 1.0;
  a.inv_gamma = inv_gamma;
  a.w_out = w_out;
  a.ldw = ldw;
  a.sw_out = sw_out;
  a.si_out = si_out;
  a.n_leaves = 0;
  a.row_begin = 0;
  a.row_end = n;
  return launch_variant(a, sw_out != nullptr, reinterpret_cast<cudaStream_t>(stream));
}

__global__ void k_eta_power(int64_t count, const double *eta, double beta, double *out) {
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < count;
       t += (int64_t)gridDim.x * blockDim.x)
    out[t] = numpy_scalar_power(eta[t], beta);
}

extern "C" int taco_eta_power(int64_t count, const double *eta, double beta, double *out, void *stream) {
  if (count < 0 || eta == nullptr || out == nullptr) return TACO_ERR_ARG;
  if (count == 0) return TACO_OK;
  const int64_t blocks64 = (count + 255) / 256;
  const int grid = (int)(blocks64 < 148 * 16 ? blocks64 : 148 * 16);
  k_eta_power<<<grid, 256, 0, reinterpret_cast<cudaStream_t>(stream)>>>(count, eta, beta, out);
  TACO_CUDA_CHECK_LAUNCH();
  return TACO_OK;
}
