// Shared device helpers for libtaco: Philox2x32-10, the keyed uniform stream,
// numpy-order pairwise summation, status recording.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

#include "../../include/taco.h"

// Device-side index checks of the debug build (-DTACO_DEBUG_CHECKS,
// scripts/debug_checks.sh): compute-sanitizer is closed on this GPU pool, so
// the GPU suite runs once against a library that traps on any out-of-range
// city / column index the kernels are about to use.  Compiled out otherwise.
#ifdef TACO_DEBUG_CHECKS
#define TACO_DCHECK(cond)                                                                        \
  do {                                                                                          \
    if (!(cond)) {                                                                              \
      printf("TACO_DCHECK failed: %s at %s:%d (block %d thread %d)\n", #cond, __FILE__, __LINE__, \
             (int)blockIdx.x, (int)threadIdx.x);                                                \
      __trap();                                                                                 \
    }                                                                                           \
  } while (0)
#else
#define TACO_DCHECK(cond) \
  do {                    \
  } while (0)
#endif

namespace taco {

// ---------------------------------------------------------------------------
// The device construction stream: Philox2x32-10 (Salmon et
// al., Random123; known-answer vectors pinned in tests/test_oracle_golden.py
// and tests/test_gpu_parity.py).
//   key(seed, it) = H(seed) + it (mod 2^32), H = xor-fold of the MurmurHash3
//                   64-bit finalizer of the seed: distinct iterations of a run
//                   never share a key
//   selection u(step >= 1, ant, slot s):
//                   dense stream, slot s = the city (dense kernel, and the
//                   fallback of steps without a W > 0 city):
//                   counter (ant, (s >> 1) | step << 16), word s & 1
//                   (n <= 65535: s >> 1 <= 0x7fff, step <= 0xfffe);
//                   sorted stream, slot p = the entry's position in the
//                   current row of the row-sorted table (sorted kernels):
//                   counter (ant, p | ((step + 1) >> 1) << 16), word
//                   (step + 1) & 1 (pos_block / pos_word)
//   start city:     counter (ant, 0) (step 0 never selects), word 0, Lemire
//   RW threshold:   counter (ant, 0xffff | step << 16), 53 bits of both words
// Counter word 0 is the ant, so round 1's product is one per ant (AntKey) and
// a window's chain starts at round 2: 9 dependent multiplies per uniform.
//   u = ((x >> 9) + 0.5) * 2^-23 in (0, 1), exact in fp32
// One block is a chain of 10 (IMAD.WIDE, LOP3) pairs: half the instructions
// of a Philox4x32-10 block, of which the sorted scan used one word per lane.
// ---------------------------------------------------------------------------
constexpr uint32_t kPhiloxM = 0xD256D193u;  // Philox2x32 multiplier
constexpr uint32_t kPhiloxW = 0x9E3779B9u;  // key bump (Weyl)
constexpr uint32_t kRwLow = 0xffffu;        // counter low half of the RW thresholds

// per-seed key schedule H(seed) + r*W, r = 0..9 (kernel parameter)
struct PhiloxKeys {
  uint32_t k[10];
};

// round keys of one iteration: k[r] + it (registers, formed once per kernel)
struct RoundKeys {
  uint32_t k[10];
};

inline uint32_t seed_hash32(uint64_t seed) {
  uint64_t f = seed;
  f ^= f >> 33;
  f *= 0xff51afd7ed558ccdull;
  f ^= f >> 33;
  f *= 0xc4ceb9fe1a85ec53ull;
  f ^= f >> 33;
  return (uint32_t)(f ^ (f >> 32));
}

inline PhiloxKeys philox_keys(uint64_t seed) {
  PhiloxKeys s;
  uint32_t a = seed_hash32(seed);
  for (int r = 0; r < 10; ++r) {
    s.k[r] = a;
    a += kPhiloxW;
  }
  return s;
}

__host__ __device__ __forceinline__ RoundKeys round_keys(const PhiloxKeys &ks, uint32_t it) {
  RoundKeys rk;
#pragma unroll
  for (int r = 0; r < 10; ++r) rk.k[r] = ks.k[r] + it;
  return rk;
}

__device__ __forceinline__ uint2 philox2x32_10(uint32_t x0, uint32_t x1, const RoundKeys &rk) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    const uint32_t hi = __umulhi(kPhiloxM, x0);
    const uint32_t lo = kPhiloxM * x0;
    x0 = hi ^ rk.k[r] ^ x1;
    x1 = lo;
  }
  return make_uint2(x0, x1);
}

// plain-key form (known-answer hook)
__device__ __forceinline__ uint2 philox2x32_10(uint32_t x0, uint32_t x1, uint32_t key) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    const uint32_t hi = __umulhi(kPhiloxM, x0);
    const uint32_t lo = kPhiloxM * x0;
    x0 = hi ^ key ^ x1;
    x1 = lo;
    key += kPhiloxW;
  }
  return make_uint2(x0, x1);
}

__device__ __forceinline__ uint32_t sel_counter(uint32_t j, uint32_t step) { return (j >> 1) | (step << 16); }

// round 1 of Philox2x32-10 on counter (ant, c): hi(M ant) ^ k0 ^ c, lo(M ant)
struct AntKey {
  uint32_t hk, lo;  // hi(M * ant) ^ k[0], lo(M * ant)
};

__device__ __forceinline__ AntKey ant_key(uint32_t ant, const RoundKeys &rk) {
  return AntKey{__umulhi(kPhiloxM, ant) ^ rk.k[0], kPhiloxM * ant};
}

// Philox2x32-10 of counter (ant, c), rounds 2..10
__device__ __forceinline__ uint2 philox_ant(uint32_t c, const AntKey &ak, const RoundKeys &rk) {
  uint32_t x0 = ak.hk ^ c, x1 = ak.lo;
#pragma unroll
  for (int r = 1; r < 10; ++r) {
    const uint32_t hi = __umulhi(kPhiloxM, x0);
    const uint32_t lo = kPhiloxM * x0;
    x0 = hi ^ rk.k[r] ^ x1;
    x1 = lo;
  }
  return make_uint2(x0, x1);
}

__device__ __forceinline__ float bits_to_uniform(uint32_t x) {
  // 1 + k 2^-23 (k = x >> 9) built from bits, minus (1 - 2^-24): both steps
  // exact (Sterbenz), so u = (k + 1/2) 2^-23 without an int->float conversion
  // (conversions run on the quarter-rate XU pipe)
  return __fsub_rn(__uint_as_float(0x3f800000u | (x >> 9)), 0x1.fffffep-1f);
}

__device__ __forceinline__ uint32_t lemire_bound(uint32_t x, uint32_t n) {
  return (uint32_t)(((uint64_t)x * (uint64_t)n) >> 32);
}

// selp: a predicated select the compiler cannot turn back into a branch
__device__ __forceinline__ uint32_t select_u32(uint32_t pred, uint32_t a, uint32_t b) {
  uint32_t r;
  asm("{\n\t.reg .pred p;\n\tsetp.ne.u32 p, %1, 0;\n\tselp.b32 %0, %2, %3, p;\n\t}"
      : "=r"(r)
      : "r"(pred), "r"(a), "r"(b));
  return r;
}

// the selection uniform's raw word for slot j (sorted position or city) at (step, ant)
__device__ __forceinline__ uint32_t sel_word(uint32_t j, uint32_t step, const AntKey &ak, const RoundKeys &rk) {
  const uint2 r = philox_ant(sel_counter(j, step), ak, rk);
  return select_u32(j & 1u, r.y, r.x);
}

// the sorted stream's uniforms (slot = sorted position p): counter
// (ant, p | ((step + 1) >> 1) << 16), word (step + 1) & 1 -- one block serves
// position p at steps 2t - 1 (word 0) and 2t (word 1), so the sorted kernels'
// first-window uniforms cost one block per lane every second step
__device__ __forceinline__ uint2 pos_block(uint32_t p, uint32_t step, const AntKey &ak, const RoundKeys &rk) {
  return philox_ant(p | (((step + 1u) >> 1) << 16), ak, rk);
}

__device__ __forceinline__ uint32_t pos_word(uint32_t p, uint32_t step, const AntKey &ak, const RoundKeys &rk) {
  const uint2 r = pos_block(p, step, ak, rk);
  return select_u32(step & 1u, r.x, r.y);
}

__device__ __forceinline__ uint32_t start_city(uint32_t n, const AntKey &ak, const RoundKeys &rk) {
  return lemire_bound(philox_ant(0u, ak, rk).x, n);
}

// RW threshold: ((x >> 5) 2^26 + (y >> 6)) 2^-53, numpy's random() layout
__device__ __forceinline__ double rw_threshold(uint32_t step, const AntKey &ak, const RoundKeys &rk) {
  const uint2 r = philox_ant(kRwLow | (step << 16), ak, rk);
  const uint64_t k = ((uint64_t)(r.x >> 5) << 26) | (uint64_t)(r.y >> 6);
  return (double)k * 0x1p-53;
}

// ---------------------------------------------------------------------------
// Sorted selection table.  Rows are ordered descending by the W bits above
// kSortBit (k_row_update); entries that follow a given entry w therefore have
// W <= bucket_ceiling(w), the largest float sharing w's sorted prefix.  The
// pruned scan stops once bucket_ceiling(last W seen) < best score.
// ---------------------------------------------------------------------------
constexpr int kSortBit = 16;

__device__ __forceinline__ float bucket_ceiling(float w) {
  return __uint_as_float(__float_as_uint(w) | ((1u << kSortBit) - 1u));
}

// np.power(x, e) for a scalar float exponent: numpy dispatches e in
// {-1, 0, 0.5, 1, 2} to reciprocal / ones / sqrt / copy / square (bit-exact
// here); any other exponent uses pow (<= 1 ulp from numpy's SIMD pow).
__device__ __forceinline__ double numpy_scalar_power(double x, double e) {
  if (e == 1.0) return x;
  if (e == 2.0) return __dmul_rn(x, x);
  if (e == 0.0) return 1.0;
  if (e == 0.5) return __dsqrt_rn(x);
  if (e == -1.0) return __ddiv_rn(1.0, x);
  return pow(x, e);
}

// ---------------------------------------------------------------------------
// Selection table entry W[i, j] = fp32(2^-e_i * P[i, j]^(1/gamma)) (DESIGN.md
// §3.1).  The per-row power-of-two scale 2^-e_i puts the row's largest entry
// in [1, 2): a scale shared by a row leaves every step's argmax of W * u
// unchanged (all candidates of a step come from one row, and scaling by 2^-e
// commutes with fp32 rounding), while the row keeps 2^126 of dynamic range
// below its maximum whatever gamma is (gamma < 1 raises P to powers > 1).
// Entries below FLT_MIN after scaling are stored as 0: the construction
// kernels' f64 fallback decides among them exactly if they are all that is
// left (construct_common.cuh).  p^(1/gamma) is exp2(log2(p) / gamma) in f64:
// within ~2^-47 of the exact power, so the fp32 rounding equals that of a
// correctly rounded pow except for ~1 entry in 10^7 (one fp32 ulp), at a
// third of pow's cost; gamma == 1 is the exact conversion.
// ---------------------------------------------------------------------------
__device__ __forceinline__ double selection_power(double p, double inv_gamma) {
  return inv_gamma == 1.0 ? p : exp2(inv_gamma * log2(p));
}

// 2^-e for the row whose largest P is pmax (e = ilogb(pmax^(1/gamma)))
__device__ __forceinline__ double selection_scale(double pmax, double inv_gamma) {
  const double x = selection_power(pmax, inv_gamma);
  int e = (x > 0.0 && x <= 1.7976931348623157e308) ? ilogb(x) : 0;
  e = e < -1000 ? -1000 : (e > 1000 ? 1000 : e);
  return __hiloint2double((1023 - e) << 20, 0);
}

__device__ __forceinline__ float selection_weight(double p, double inv_gamma, double scale) {
  const float w = __double2float_rn(__dmul_rn(selection_power(p, inv_gamma), scale));
  return w < 0x1p-126f ? 0.0f : w;  // NaN kept (the row sum already failed)
}

// ---------------------------------------------------------------------------
// status word: [0] = first failure code, [1] = smallest offending index
// ---------------------------------------------------------------------------
// Fail-stop across Solver iterations: a construction kernel that starts after
// a recorded failure (status[0] != 0) sets status[3] and does nothing; a row
// update that sees status[3] leaves tau / P / W / row sums as they were, so
// a host that checks only after several iterations still reads the state of
// the failing iteration (where the reference raised).  One decision per warp
// (construction) or CTA (row update) keeps barriers uniform.
__device__ __forceinline__ bool chain_stopped_construct(int32_t *status) {
  if (status == nullptr || *reinterpret_cast<volatile int32_t *>(status) == 0) return false;
  reinterpret_cast<volatile int32_t *>(status)[3] = 1;
  return true;
}

__device__ __forceinline__ bool chain_stopped_update(const int32_t *status) {
  return status != nullptr && reinterpret_cast<const volatile int32_t *>(status)[3] != 0;
}

__device__ __forceinline__ void record_status(int32_t *status, int code, int index) {
  if (status == nullptr) return;
  atomicCAS(status, 0, code);
  atomicMin(status + 1, index);
  // a construction failure also stops the rest of its own iteration (best
  // tracking, deposit, evaporation, P / W): tau stays where the reference
  // raised (colony.py:149 fires inside construct_tours)
  if (code == TACO_NO_CANDIDATE) atomicExch(status + 3, 1);
}

// ---------------------------------------------------------------------------
// numpy pairwise summation (numpy/_core/src/umath/loops_utils.h.src,
// pairwise_sum): blocks < 8 sum sequentially from 0.0, blocks <= 128 use eight
// strided accumulators, larger blocks split at n/2 rounded down to a multiple
// of 8.  The split tree depends only on n, so it is enumerated once per CTA
// into a leaf table; lanes/threads sum leaves in parallel and one thread folds
// the leaves in tree order.  Bit-exact with ndarray.sum(axis=-1) on
// contiguous float64 rows (verified in tests/test_oracle_golden.py against
// numpy, and on device in tests/test_gpu_parity.py).
// ---------------------------------------------------------------------------
constexpr int kPwBlock = 128;

__host__ __device__ __forceinline__ int pw_split(int len) {
  int n2 = len / 2;
  return n2 - (n2 % 8);
}

// number of leaves of the pairwise tree for length n
__host__ __device__ inline int pw_num_leaves(int n) {
  // leaves are the maximal blocks of length <= 128 (or the whole array if < 8)
  if (n <= kPwBlock) return 1;
  // iterative count with an explicit stack
  int stack[40];
  int sp = 0, count = 0;
  stack[sp++] = n;
  while (sp) {
    int len = stack[--sp];
    if (len <= kPwBlock) {
      ++count;
    } else {
      int n2 = pw_split(len);
      stack[sp++] = len - n2;
      stack[sp++] = n2;
    }
  }
  return count;
}

// fill leaf (offset, length) pairs in left-to-right order; returns count
__device__ inline int pw_leaves(int n, int2 *leaves) {
  int stack_off[40], stack_len[40];
  int sp = 0, count = 0;
  stack_off[sp] = 0;
  stack_len[sp] = n;
  ++sp;
  while (sp) {
    --sp;
    int off = stack_off[sp], len = stack_len[sp];
    if (len <= kPwBlock) {
      leaves[count++] = make_int2(off, len);
    } else {
      int n2 = pw_split(len);
      // push right first so the left half is processed first
      stack_off[sp] = off + n2;
      stack_len[sp] = len - n2;
      ++sp;
      stack_off[sp] = off;
      stack_len[sp] = n2;
      ++sp;
    }
  }
  return count;
}

// Sum one leaf exactly as numpy's pairwise_sum base cases do.
// `at(i)` returns element i of the leaf.
template <typename F>
__device__ __forceinline__ double pw_leaf_sum(int len, F at) {
  if (len < 8) {
    double res = 0.0;
    for (int i = 0; i < len; ++i) res = __dadd_rn(res, at(i));
    return res;
  }
  double r0 = at(0), r1 = at(1), r2 = at(2), r3 = at(3);
  double r4 = at(4), r5 = at(5), r6 = at(6), r7 = at(7);
  int i = 8;
  const int stop = len - (len % 8);
  for (; i < stop; i += 8) {
    r0 = __dadd_rn(r0, at(i + 0));
    r1 = __dadd_rn(r1, at(i + 1));
    r2 = __dadd_rn(r2, at(i + 2));
    r3 = __dadd_rn(r3, at(i + 3));
    r4 = __dadd_rn(r4, at(i + 4));
    r5 = __dadd_rn(r5, at(i + 5));
    r6 = __dadd_rn(r6, at(i + 6));
    r7 = __dadd_rn(r7, at(i + 7));
  }
  double res = __dadd_rn(__dadd_rn(__dadd_rn(r0, r1), __dadd_rn(r2, r3)),
                         __dadd_rn(__dadd_rn(r4, r5), __dadd_rn(r6, r7)));
  for (; i < len; ++i) res = __dadd_rn(res, at(i));
  return res;
}

// Fold leaf sums (left-to-right order) along the pairwise tree of length n.
__device__ inline double pw_fold(int n, const double *leaf_sum) {
  if (n <= kPwBlock) return leaf_sum[0];
  int lens[40];
  int phase[40];
  double lefts[40];
  int sp = 0, li = 0;
  lens[0] = n;
  phase[0] = 0;
  double ret = 0.0;
  for (;;) {
    int len = lens[sp];
    if (len <= kPwBlock) {
      ret = leaf_sum[li++];
      for (;;) {
        if (sp == 0) return ret;
        --sp;
        if (phase[sp] == 1) {
          lefts[sp] = ret;
          phase[sp] = 2;
          lens[sp + 1] = lens[sp] - pw_split(lens[sp]);
          phase[sp + 1] = 0;
          ++sp;
          break;
        }
        ret = __dadd_rn(lefts[sp], ret);
      }
    } else {
      phase[sp] = 1;
      lens[sp + 1] = pw_split(len);
      phase[sp + 1] = 0;
      ++sp;
    }
  }
}

// ---------------------------------------------------------------------------
// Parallel evaluation of the pairwise tree.  A plan lists the tree's internal
// nodes grouped by height; each level is one round of independent adds
// (left + right, numpy's operand order), so a CTA folds ~L leaves in
// O(log L) barrier rounds instead of a serial walk.  Node ids: leaves are
// 0..L-1, internal node q is kInternal | q.
// ---------------------------------------------------------------------------
constexpr uint16_t kInternal = 0x8000u;
constexpr int kMaxPlanHeight = 40;

struct PwPlan {
  int2 *leaves;        // [L] (offset, length), left to right
  uint16_t *left;      // [L-1] child ids of internal node q
  uint16_t *right;     // [L-1]
  uint16_t *order;     // [L-1] internal nodes sorted by height
  int *level_start;    // [kMaxPlanHeight + 2]
  int n_leaves, n_internal, height;
};

// Build the plan for length n (one thread).  `hgt` is [L-1] scratch.
__device__ inline void pw_plan_build(int n, PwPlan &p, uint8_t *hgt) {
  struct Frame {
    int off, len, state, left_id, left_h;
  };
  Frame st[kMaxPlanHeight];
  int sp = 0, nl = 0, ni = 0, ret_id = 0, ret_h = 0;
  st[sp++] = Frame{0, n, 0, 0, 0};
  while (sp) {
    Frame &f = st[sp - 1];
    if (f.len <= kPwBlock) {
      p.leaves[nl] = make_int2(f.off, f.len);
      ret_id = nl++;
      ret_h = 0;
      --sp;
    } else if (f.state == 0) {
      f.state = 1;
      st[sp++] = Frame{f.off, pw_split(f.len), 0, 0, 0};
    } else if (f.state == 1) {
      f.left_id = ret_id;
      f.left_h = ret_h;
      f.state = 2;
      const int n2 = pw_split(f.len);
      st[sp++] = Frame{f.off + n2, f.len - n2, 0, 0, 0};
    } else {
      p.left[ni] = (uint16_t)f.left_id;
      p.right[ni] = (uint16_t)ret_id;
      const int h = 1 + (f.left_h > ret_h ? f.left_h : ret_h);
      hgt[ni] = (uint8_t)h;
      ret_id = kInternal | ni;
      ret_h = h;
      ++ni;
      --sp;
    }
  }
  p.n_leaves = nl;
  p.n_internal = ni;
  p.height = ret_h;
  // counting sort of the internal nodes by height
  for (int h = 0; h <= kMaxPlanHeight + 1; ++h) p.level_start[h] = 0;
  for (int q = 0; q < ni; ++q) ++p.level_start[hgt[q] + 1];
  for (int h = 1; h <= kMaxPlanHeight + 1; ++h) p.level_start[h] += p.level_start[h - 1];
  int fill[kMaxPlanHeight + 1];
  for (int h = 0; h <= kMaxPlanHeight; ++h) fill[h] = p.level_start[h];
  for (int q = 0; q < ni; ++q) p.order[fill[hgt[q]]++] = (uint16_t)q;
}

// Fold leaf sums into the root with all threads of the CTA; returns the sum
// in every thread.  `ival` is [L-1] scratch.  Contains __syncthreads.
__device__ inline double pw_plan_fold(const PwPlan &p, const double *leaf_sum, double *ival) {
  for (int h = 1; h <= p.height; ++h) {
    const int b = p.level_start[h], e = p.level_start[h + 1];
    for (int t = b + (int)threadIdx.x; t < e; t += blockDim.x) {
      const int q = p.order[t];
      const uint16_t l = p.left[q], r = p.right[q];
      const double lv = (l & kInternal) ? ival[l & ~kInternal] : leaf_sum[l];
      const double rv = (r & kInternal) ? ival[r & ~kInternal] : leaf_sum[r];
      ival[q] = __dadd_rn(lv, rv);
    }
    __syncthreads();
  }
  return p.n_internal == 0 ? leaf_sum[0] : ival[p.n_internal - 1];
}

}  // namespace taco

namespace taco {
// last CUDA error seen by a libtaco entry point (taco_last_cuda_error)
void note_cuda_error(cudaError_t e);

// Host-side caches are per device (a process may drive several GPUs).
constexpr int kMaxDevices = 64;

inline int current_device() {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= kMaxDevices) dev = 0;
  return dev;
}

// SM count of the current device (148 on B200), cached per device
inline int device_sm_count() {
  static int cached[kMaxDevices] = {};
  const int dev = current_device();
  if (cached[dev] == 0) {
    int v = 0;
    if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || v <= 0) v = 148;
    cached[dev] = v;
  }
  return cached[dev];
}
}  // namespace taco

#define TACO_CUDA_CHECK_LAUNCH()                              \
  do {                                                        \
    cudaError_t e_ = cudaGetLastError();                      \
    if (e_ != cudaSuccess) {                                  \
      taco::note_cuda_error(e_);                              \
      return TACO_ERR_CUDA;                                   \
    }                                                         \
  } while (0)
