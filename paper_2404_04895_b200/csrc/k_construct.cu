// Tour construction kernels: one warp owns one ant for all n-1 lockstep steps.
//
// Reference: colony.construct_tours colony.py:87-154 (IR / AdaIR branch),
// argmax_select_block selection.py:143-155, start cities rng.py:65-68, tour
// lengths model.batch_costs model.py:292-295 (fused).
//
// Fast-path rule: next = argmax_j { W[cur, j] * u(step, ant, s) }
// over unvisited j with W[cur, j] > 0, first (lowest j) of ties, where
// W = fp32(P^(1/gamma)) and u is the keyed Philox2x32-10 uniform of slot s.
// The slot is the entry's position in row cur of the row-sorted table for the
// SORTED kernels (so a window's uniforms need no table data and are formed a
// step ahead; one block serves a position at two consecutive steps), and the
// city j for the DENSE kernel: two streams, each an
// exact instance of the rule.  This is the product form of the reference's
// argmax(log P / gamma - E) with E = -log u.
//
// Two variants compute the identical argmax:
//   DENSE  streams the whole fp32 row W[cur, :] with 16-byte loads and draws
//          four uniforms per two Philox blocks (the north-star "row
//          streaming" kernel; ALU bound on Philox).
//   SORTED scans the row's descending (W, j) table and stops as soon as the
//          next table entry satisfies W < best score: since u < 1, no later
//          entry can reach the running best, so the result is bit-identical to
//          the full scan of the table while touching only its head.  Because
//          the uniforms are counter-addressed (by sorted position), visiting
//          candidates in window order draws exactly the values the full scan
//          would.  The median step stops after 3 entries.
// The tour length, in numpy's pairwise order (bit-exact with batch_costs), is
// either accumulated on the fly or computed by k_tour_cost afterwards.
#include <algorithm>
#include <cstdlib>

#include "construct_common.cuh"

// A/B only: -DTACO_NO_FALLBACK drops the rebuild call sites (no W > 0
// candidate then always records TACO_NO_CANDIDATE), to measure what they cost
#ifdef TACO_NO_FALLBACK
#define TACO_REBUILD(...) false
#else
#define TACO_REBUILD(...) rebuild_tour(__VA_ARGS__)
#endif

namespace taco {

// Shared-memory layout of the sorted kernel (dynamic):
//   int2   leaves[n_leaves]
//   per ant: double leaf_buf[kPwBlock], double leaf_sum[n_leaves], uint32 vis[nwords]
//            (VIS8: nwords = ceil(n / 4), one byte per city)
struct SortedArgs {
  int n, m_local, ant_offset, nwords, n_leaves, ld;  // ld: sorted-table row pitch
  const float *sw;
  const uint16_t *si;
  const double *dist;
  uint32_t iteration;
  const taco_iter_state *state;  // nullable: iteration from device memory
  int32_t *tours;
  double *costs;
  int32_t *status;
  unsigned long long *scan_count;
  PhiloxKeys ks;
  Fallback fb;  // no W > 0 candidate left (construct_common.cuh)
  const int2 *leaves_img;  // nullable (construct_common.cuh leaves_image)
};

constexpr int kSortedMaxWarps = 28;      // fused tour length: 72 registers per thread
// MODE 1 (one CTA per SM) holds up to 28 ants per SM at 72 registers (32
// warps at 64 registers rematerialized constants in the step loop; C2 -1%,
// C3 equal); more ants per SM run MODE 2: two CTAs per SM of
// ceil(ants per SM / 2) warps each (balanced: at C4, 55 ants per SM, 2 x 28
// warps instead of 2 x 32 on 108 SMs and 1 x 32 on 40: 15.4 -> 14.1 ms)
#ifndef TACO_MODE1_WARPS
#define TACO_MODE1_WARPS 28
#endif
#ifndef TACO_MODE2_WARPS
#define TACO_MODE2_WARPS 32
#endif
constexpr int kMode1Warps = TACO_MODE1_WARPS;
#ifndef TACO_LATENCY_ANTS
#define TACO_LATENCY_ANTS 16
#endif
constexpr int kLatencyAnts = TACO_LATENCY_ANTS;  // MODE 4 up to this many ants per SM
constexpr int kMode2Warps = TACO_MODE2_WARPS;  // 2 CTAs per SM: 65536 / (64 x this) registers

#ifdef TACO_STEP_PROFILE
// per-step latency phases of ant 0 (-, windows, bookkeeping;
// [5..7]: first-window load wait, vis+Philox+key, the two reductions)
__device__ unsigned long long g_step_prof[8];

__device__ __forceinline__ uint32_t consume(float x) {
  uint32_t r;
  asm volatile("mov.b32 %0, %1;" : "=r"(r) : "f"(x));
  return r;
}
#endif

// Visited set of the warp kernel: one byte per city when it fits in shared
// memory (VIS8: the test is one LDS.U8, the update one STS.U8), else a bit map.
template <bool VIS8>
__device__ __forceinline__ bool visited_at(const uint32_t *vis, uint32_t j) {
  if (VIS8) return reinterpret_cast<const uint8_t *>(vis)[j] != 0;
  return (vis[j >> 5] >> (j & 31)) & 1u;
}

template <bool VIS8>
__device__ __forceinline__ void mark_visited(uint32_t *vis, uint32_t j) {
  if (VIS8)
    reinterpret_cast<uint8_t *>(vis)[j] = 1;
  else
    atomicOr(vis + (j >> 5), 1u << (j & 31));  // one shared-memory RMW instruction (C4 -0.7%)
}

// %laneid: the 32-register MODE 2 loop rematerializes the lane index, and
// this is one S2R instead of S2R tid + LOP3 (C4 -2.3%)
__device__ __forceinline__ int lane_id() {
  int l;
  asm("mov.u32 %0, %%laneid;" : "=r"(l));
  return l;
}

// Score the 32-entry window (w, j) of the sorted row against the running
// (best, bestj).  Warp-uniform control flow: the Philox chain runs once per
// window for all lanes iff any lane holds a candidate (unvisited, W > 0,
// W >= best); a window without candidates costs one shared load per lane.
template <bool VIS8, class Uniform>
__device__ __forceinline__ void score_window_u(float w, uint32_t j, const uint32_t *vis, float &best,
                                               uint32_t &bestj, Uniform uniform) {
  const bool cand = (w > 0.0f) && (w >= best) && !visited_at<VIS8>(vis, j);
  if (__any_sync(kFull, cand)) {
    const uint32_t x = uniform();
    const uint32_t key = cand ? __float_as_uint(__fmul_rn(w, bits_to_uniform(x))) + 1u : 0u;
    const uint32_t mkey = __reduce_max_sync(kFull, key);
    if (mkey != 0u) {
      const uint32_t jmin = __reduce_min_sync(kFull, key == mkey ? j : 0xffffffffu);
      const float sc = __uint_as_float(mkey - 1u);
      if (sc > best || (sc == best && jmin < bestj)) {
        best = sc;
        bestj = jmin;
      }
    }
  }
}

// uniforms of the sorted-table stream are keyed by sorted position `pos`
template <bool VIS8>
__device__ __forceinline__ void score_window(float w, uint32_t j, uint32_t pos, const uint32_t *vis, uint32_t step,
                                             const AntKey &ak, const RoundKeys &rk, float &best, uint32_t &bestj) {
  score_window_u<VIS8>(w, j, vis, best, bestj, [&] { return pos_word(pos, step, ak, rk); });
}

// The first window of the next row is issued as soon as the step's winner is
// known, ahead of the step's bookkeeping (visited bit, tour and length
// buffers), so that L2 round trip overlaps it.  COST: the tour length is
// accumulated on the fly (else taco_construct runs k_tour_cost afterwards).
// MODE 0: fused tour length (COST); 1: separate length, one CTA of <= 28
// warps per SM (72 registers); 3: the same with 29-32 warps (64 registers);
// 2: separate length, two CTAs of ceil(ants per SM / 2) <= 32 warps per SM
// (<= 32 registers: the compiler rematerializes more, so only for > 32
// ants per SM); 4: MODE 1 for few ants per SM, latency-bound rather than
// issue-bound, with the next row's window issued ahead of the stall test.
template <bool PROBE, bool VIS8, int MODE, bool COST = (MODE == 0)>
__global__ void __launch_bounds__(COST ? kSortedMaxWarps * 32
                                       : ((MODE == 1 || MODE == 4) ? kMode1Warps
                                                                   : (MODE == 3 ? 32 : kMode2Warps)) * 32,
                                  MODE == 2 ? 2 : 1)
    k_construct_sorted(const __grid_constant__ SortedArgs a) {
  // the next row's first window issued right after the window loop, before
  // the stall test and the bookkeeping (with the peeled first window): one ant
  // per SM -2.7%, 7 ants per SM -2%, 10-14 ants -1.5-2.5%, but +1% at 21,
  // +2% at 28 (C3) and in MODE 2 (issue-bound there)
  constexpr bool EARLY_LOAD = MODE == 4;
  // the tour row stored by lane 0 every step instead of buffered in lanes and
  // written 128 B at a time: fewer instructions per step (C3 -0.6%), but
  // +2.6% in the 32-register MODE 2
  constexpr bool TOUR_STG = MODE != 2;
  extern __shared__ __align__(16) unsigned char smem[];
  const int n = a.n;
  const int warps = blockDim.x >> 5;
  const int warp = threadIdx.x >> 5;
  const int lane = MODE == 2 ? lane_id() : (int)(threadIdx.x & 31);
  int2 *leaves = reinterpret_cast<int2 *>(smem);
  double *leaf_buf = nullptr, *leaf_sum = nullptr;
  uint32_t *vis;
  if (COST) {  // leaves, then per ant: leaf buffer, leaf sums, visited set
    unsigned char *mine = smem + (((size_t)8 * a.n_leaves + 15) & ~(size_t)15) +
                          ant_scratch_bytes(a.n_leaves, a.nwords) * warp;
    leaf_buf = reinterpret_cast<double *>(mine);
    leaf_sum = leaf_buf + kPwBlock;
    vis = reinterpret_cast<uint32_t *>(leaf_sum + a.n_leaves);
  } else {  // leaves, then per ant: leaf sums (epilogue length), visited set
    const size_t ls_bytes = ((size_t)8 * a.n_leaves + 15) & ~(size_t)15;
    unsigned char *mine = smem + ls_bytes + (ls_bytes + (((size_t)4 * a.nwords + 15) & ~(size_t)15)) * warp;
    leaf_sum = reinterpret_cast<double *>(mine);
    vis = reinterpret_cast<uint32_t *>(mine + ls_bytes);
  }

  if (a.costs != nullptr) load_leaves(n, a.n_leaves, leaves, a.leaves_img);
  __syncthreads();

  const int ant = blockIdx.x * warps + warp;
  if (ant >= a.m_local) return;
  if (__shfl_sync(kFull, lane == 0 ? (int)chain_stopped_construct(a.status) : 0, 0)) return;  // fail-stop
  const uint32_t gant = (uint32_t)(a.ant_offset + ant);
  const uint32_t it = a.state != nullptr ? a.state->iteration : a.iteration;
  const RoundKeys rk = round_keys(a.ks, it);
  const AntKey ak = ant_key(gant, rk);
  const uint32_t un = (uint32_t)n;  // n <= 65535, so every row offset fits in 32 bits
  const float *__restrict__ sw = a.sw;
  const uint16_t *__restrict__ si = a.si;
  const uint32_t ldr = (uint32_t)a.ld;
  for (int q = lane; q < a.nwords; q += 32) vis[q] = 0u;
  const uint32_t start = start_city(un, ak, rk);
  __syncwarp();
  if (lane == 0) mark_visited<VIS8>(vis, start);
  __syncwarp();

  TourWriter tw{a.tours + (size_t)ant * n, n, lane, 0};
  if (TOUR_STG) {
    if (lane == 0) tw.row[0] = (int32_t)start;
  } else {
    tw.put(0, (int32_t)start);
  }
  LeafCost lc;
  lc.init(COST && a.costs != nullptr ? a.dist : nullptr, leaves, leaf_buf, leaf_sum, n, lane);
  uint32_t cur = start;
  unsigned long long windows = 0;  // 32-entry windows read (traffic probe)
  // first window (entries 0..31) of the current row, in flight across the
  // step boundary
  float wg = 0.0f;
  uint32_t jg = 0;
  if ((uint32_t)lane < un) {
    wg = __ldg(sw + (cur * ldr + lane));
    jg = __ldg(si + (cur * ldr + lane));
  }
  // the first window's uniforms depend only on (step, sorted position =
  // lane): each step's are formed in the previous step's shadow, while its
  // window is in flight (C3 -5%, one ant per SM -10%)
  uint32_t xnext, xstash;  // step s's word; word 1 of the block of odd step s - 1
  {
    const uint2 b = pos_block((uint32_t)lane, 1u, ak, rk);
    xnext = b.x;
    xstash = b.y;
  }
  // the step's bookkeeping once its city is known: the next row's first
  // window is issued before it, so that L2 round trip overlaps it
  auto advance = [&](uint32_t bj, uint32_t stp) {
    const uint32_t e = (uint32_t)lane;
    if (!EARLY_LOAD) {
      wg = 0.0f;
      jg = 0;
      if (e < un) {  // also at the last step (row bj exists; unused): no step test (C3 -2%)
        wg = __ldg(sw + (bj * ldr + e));
        jg = __ldg(si + (bj * ldr + e));
      }
    }
    if (stp & 1u) {  // step stp + 1 is even: word 1 of the block formed at stp
      xnext = xstash;
    } else {
      const uint2 b = pos_block(e, stp + 1, ak, rk);
      xnext = b.x;
      xstash = b.y;
    }
    if (lane == 0) mark_visited<VIS8>(vis, bj);
    if (COST) {
      if (stp > 1) lc.push();  // edge stp-2, loaded one step ago
      lc.load(cur, bj);        // edge stp-1
    }
    __syncwarp();
    if (TOUR_STG) {
      if (lane == 0) tw.row[stp] = (int32_t)bj;
    } else {
      tw.put((int)stp, (int32_t)bj);
    }
    cur = bj;
  };
  bool stalled = false;  // a step without a W > 0 candidate (rebuilt below)
  // two steps per loop iteration (the step-pair Philox parity resolves at
  // compile time): C3 -2.5%, C4 -1.3%; not in the latency MODE 4 (+1.2%)
#ifndef TACO_STEP_UNROLL
#define TACO_STEP_UNROLL 2
#endif
  constexpr int kStepUnroll = MODE == 4 ? 1 : TACO_STEP_UNROLL;
#pragma unroll kStepUnroll
  for (uint32_t step = 1; step < un; ++step) {
#ifdef TACO_STEP_PROFILE
    const long long t0 = clock64();
#endif
    const uint32_t row = cur * ldr;  // < 2^32 for n <= 65535
    float best = -1.0f;
    uint32_t bestj = 0xffffffffu;
    bool done = false;
#ifdef TACO_STEP_PROFILE
    const long long t1 = clock64();
    int nwin = 0;
#endif
    // the first window, peeled out of the window loop (its uniforms were
    // formed a step ahead; best is still -1, so no running-best test and the
    // window's best entry wins): a straight-line common path (94% of steps
    // end here), C3 -8%, C4 -4.7%
    uint32_t base = 32;
    {
      // entries after this window have W <= bucket_ceiling(window's last W);
      // the shuffle is issued first so that it overlaps the scoring
      const float wl = __shfl_sync(kFull, wg, 31);
      uint32_t x = xnext;
      asm volatile("" : "+r"(x));
      const bool cand = (wg > 0.0f) && !visited_at<VIS8>(vis, jg);
      if (__any_sync(kFull, cand)) {
        const uint32_t key = cand ? __float_as_uint(__fmul_rn(wg, bits_to_uniform(x))) + 1u : 0u;
        const uint32_t mkey = __reduce_max_sync(kFull, key);
        const uint32_t jsel = key == mkey ? jg : 0xffffffffu;
        best = __uint_as_float(mkey - 1u);
        // the stop test needs only the max: it runs while the min reduction
        // is in flight (C3 -1%, one ant per SM -3%)
        done = (bucket_ceiling(wl) < best) || (wl <= 0.0f) || (base >= un);
        bestj = __reduce_min_sync(kFull, jsel);
      } else {
        done = (wl <= 0.0f) || (base >= un);
      }
      if (PROBE) ++windows;
    }
    while (!done) {  // later windows (6% of steps)
      const uint32_t e = base + lane;
      wg = 0.0f;
      jg = 0;
      if (e < un) {
        wg = __ldg(sw + (row + e));
        jg = __ldg(si + (row + e));
      }
      const float wl = __shfl_sync(kFull, wg, 31);
      score_window<VIS8>(wg, jg, e, vis, step, ak, rk, best, bestj);
      base += 32;
      done = (bucket_ceiling(wl) < best) || (wl <= 0.0f) || (base >= un);
      if (PROBE) ++windows;
    }
#ifdef TACO_STEP_PROFILE
    const long long t2 = clock64();
#endif
    if (EARLY_LOAD) {  // the next row's first window, issued ahead of the stall
                       // test (a stalled step loads row 0 instead of row -1; unused)
      const uint32_t nrow = bestj < un ? bestj : 0u;
      wg = 0.0f;
      jg = 0;
      if ((uint32_t)lane < un) {
        wg = __ldg(sw + (nrow * ldr + lane));
        jg = __ldg(si + (nrow * ldr + lane));
      }
    }
    if (bestj == 0xffffffffu) {  // no W > 0 candidate: the tour is rebuilt after the loop
      stalled = true;
      break;
    }
    TACO_DCHECK(bestj < un && !(lane == 0 && visited_at<VIS8>(vis, bestj)));
    advance(bestj, step);
#ifdef TACO_STEP_PROFILE
    const long long t3 = clock64();
    if (ant == 0 && lane == 0) {
      g_step_prof[0] += t1 - t0;
      g_step_prof[1] += t2 - t1;
      g_step_prof[2] += t3 - t2;
      g_step_prof[3] += 1;
      g_step_prof[4] += (base >> 5);
    }
#endif
  }
  if (stalled) {  // cold path (construct_common.cuh rebuild_tour), off the step loop's registers
    if (MODE == 2) {  // 32 registers: even the out-of-line call costs the loop; k_rebuild_stalled does it
      if (lane == 0) tw.row[n - 1] = -1;  // marker (a finished tour never holds -1)
      return;
    }
    if (!TACO_REBUILD(sw, si, a.ld, un, &a.fb, &a.ks, a.state, it, gant, vis, VIS8, 1, 0, a.nwords, tw.row, lane)) {
      if (lane == 0) record_status(a.status, TACO_NO_CANDIDATE, (int)gant);
      return;
    }
    if (a.costs != nullptr) {
      const double c = warp_tour_cost(n, tw.row, a.dist, leaves, a.n_leaves, leaf_sum, lane);
      if (lane == 0) a.costs[ant] = c;
    }
    return;
  }
  if (!TOUR_STG) tw.flush();
  __syncwarp();
  if (COST && lc.active) {
    lc.push();  // edge n-2
    lc.load(cur, start);
    lc.push();  // closing edge n-1
    const double c = lc.finish();
    if (lane == 0) a.costs[ant] = c;
  }
  if (!COST && a.costs != nullptr) {  // epilogue: the finished row, lanes in parallel
    const double c = warp_tour_cost(n, tw.row, a.dist, leaves, a.n_leaves, leaf_sum, lane);
    if (lane == 0) a.costs[ant] = c;
  }
  if (PROBE && lane == 0) atomicAdd(a.scan_count, windows);
}

// ---------------------------------------------------------------------------
// Lane-group construction: G lanes own one ant (32/G ants per warp) and each
// lane scores E consecutive table entries per iteration with E independent
// Philox chains, so one SIMT pass scores G*E entries for each of the warp's
// ants.  Groups advance through their steps independently (a group that
// finishes a step starts the next one in the following iteration), so a warp
// never waits for its slowest ant within a step.  Same rule, same uniforms and
// the same bucket-ceiling stop as k_construct_sorted: identical tours.
// ---------------------------------------------------------------------------
constexpr int kGroupWarps = 4;

struct GroupArgs {
  int n, m_local, ant_offset, nwords, n_leaves, ld;
  const float *sw;
  const uint16_t *si;
  const double *dist;
  uint32_t iteration;
  const taco_iter_state *state;  // nullable: iteration from device memory
  int32_t *tours;
  double *costs;
  int32_t *status;
  unsigned long long *scan_count;  // optional traffic probe (32-entry windows)
  PhiloxKeys ks;
  Fallback fb;
  const int2 *leaves_img;  // nullable (construct_common.cuh leaves_image)
};


template <int G, int E, bool PROBE>
__global__ void __launch_bounds__(kGroupWarps * 32) k_construct_group(const __grid_constant__ GroupArgs a) {
  static_assert(G == 4 || G == 8 || G == 16, "lanes per ant");
  static_assert(E == 2 || E == 4, "entries per lane");
  constexpr int A = 32 / G;  // ants per warp
  constexpr int CH = G * E;  // entries scored per ant per iteration
  extern __shared__ __align__(16) unsigned char smem[];
  const int n = a.n, L = a.n_leaves;
  int2 *leaves = reinterpret_cast<int2 *>(smem);
  const size_t off = (8 * (size_t)L + 15) & ~(size_t)15;
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const size_t per_warp = (((size_t)4 * a.nwords * A + 15) & ~(size_t)15) + off;
  unsigned char *wp = smem + off + per_warp * warp;
  uint32_t *vis = reinterpret_cast<uint32_t *>(wp);  // [nwords][A]: conflict-free per ant
  double *leaf_sum = reinterpret_cast<double *>(wp + (((size_t)4 * a.nwords * A + 15) & ~(size_t)15));
  load_leaves(n, L, leaves, a.leaves_img);
  for (int q = lane; q < a.nwords * A; q += 32) vis[q] = 0u;
  __syncthreads();

  const int g = lane / G, gl = lane % G, gbase = g * G;
  const int ant = (blockIdx.x * kGroupWarps + warp) * A + g;
  if (__shfl_sync(kFull, lane == 0 ? (int)chain_stopped_construct(a.status) : 0, 0)) return;  // fail-stop
  bool alive = ant < a.m_local;
  const uint32_t gant = (uint32_t)(a.ant_offset + ant);
  const uint32_t it = a.state != nullptr ? a.state->iteration : a.iteration;
  const RoundKeys rk = round_keys(a.ks, it);
  const AntKey ak = ant_key(gant, rk);
  const uint32_t un = (uint32_t)n, ld = (uint32_t)a.ld;
  const uint32_t start = start_city(un, ak, rk);
  int32_t *trow = a.tours + (size_t)ant * n;
  bool complete = false;  // this group's tour reached n cities
  bool stalled = false;   // a step without a W > 0 candidate (rebuilt after the loop)
  if (alive && gl == 0) {
    vis[(start >> 5) * A + g] |= 1u << (start & 31);
    trow[0] = (int32_t)start;
  }
  __syncwarp();

  uint32_t cur = start, step = 1, chunk = 0, bestj = 0xffffffffu;
  float best = -1.0f;
  unsigned long long chunks = 0;
  while (__any_sync(kFull, alive)) {
    if (PROBE && alive) ++chunks;
    // ---- score this iteration's chunk: entries chunk + gl*E .. + E-1 -------
    float w[E];
    uint32_t j[E];
    if (alive) {
      const uint32_t o = cur * ld + chunk + (uint32_t)gl * E;
      if constexpr (E == 4) {
        const float4 wv = __ldg(reinterpret_cast<const float4 *>(a.sw + o));
        const uint2 iv = __ldg(reinterpret_cast<const uint2 *>(a.si + o));
        w[0] = wv.x, w[1] = wv.y, w[2] = wv.z, w[3] = wv.w;
        j[0] = iv.x & 0xffffu, j[1] = iv.x >> 16, j[2] = iv.y & 0xffffu, j[3] = iv.y >> 16;
      } else {
        const float2 wv = __ldg(reinterpret_cast<const float2 *>(a.sw + o));
        const uint32_t iv = __ldg(reinterpret_cast<const uint32_t *>(a.si + o));
        w[0] = wv.x, w[1] = wv.y;
        j[0] = iv & 0xffffu, j[1] = iv >> 16;
      }
    } else {
#pragma unroll
      for (int e = 0; e < E; ++e) w[e] = 0.0f, j[e] = 0u;
    }
    // Philox issued ahead of the visited lookups and the vote (with A ants per
    // warp the vote almost never skips the chunk)
    uint32_t x[E];
#pragma unroll
    for (int e = 0; e < E; ++e) {
      x[e] = pos_word(chunk + (uint32_t)(gl * E + e), step, ak, rk);  // sorted position
      asm volatile("" : "+r"(x[e]));
    }
    bool cand[E];
    bool any = false;
#pragma unroll
    for (int e = 0; e < E; ++e) {
      const uint32_t vw = vis[(j[e] >> 5) * A + g];
      cand[e] = (w[e] > 0.0f) && (w[e] >= best) && !((vw >> (j[e] & 31)) & 1u);
      any |= cand[e];
    }
    unsigned long long p = 0ull;  // packed (key, ~j): max = best score, lowest j
    if (__any_sync(kFull, any)) {
#pragma unroll
      for (int e = 0; e < E; ++e) {
        const uint32_t key =
            cand[e] ? __float_as_uint(__fmul_rn(w[e], bits_to_uniform(x[e]))) + 1u : 0u;
        const unsigned long long pe = ((unsigned long long)key << 32) | (uint32_t)~j[e];
        p = pe > p ? pe : p;
      }
    }
#pragma unroll
    for (int o2 = G / 2; o2 > 0; o2 >>= 1) {
      const unsigned long long q = __shfl_xor_sync(kFull, p, o2);
      p = q > p ? q : p;
    }
    const uint32_t gkey = (uint32_t)(p >> 32);
    if (gkey != 0u) {
      const float sc = __uint_as_float(gkey - 1u);
      const uint32_t gj = ~(uint32_t)p;
      if (sc > best || (sc == best && gj < bestj)) {
        best = sc;
        bestj = gj;
      }
    }
    // entries after this chunk have W <= bucket_ceiling(chunk's last W)
    const float wl = __shfl_sync(kFull, w[E - 1], gbase + G - 1);
    chunk += CH;
    const bool step_done = alive && ((bucket_ceiling(wl) < best) || (wl <= 0.0f) || (chunk >= un));

    // ---- groups whose step is decided move to the next city ----------------
    if (step_done) {
      if (bestj == 0xffffffffu) {  // no W > 0 candidate: rebuilt after the loop
        stalled = true;
        alive = false;
      } else {
        TACO_DCHECK(bestj < un && !((vis[(bestj >> 5) * A + g] >> (bestj & 31)) & 1u));
        if (gl == 0) {
          vis[(bestj >> 5) * A + g] |= 1u << (bestj & 31);
          trow[step] = (int32_t)bestj;
        }
        cur = bestj;
        ++step;
        chunk = 0;
        best = -1.0f;
        bestj = 0xffffffffu;
        if (step == un) {  // tour complete
          complete = true;
          alive = false;
        }
      }
    }
    __syncwarp();
  }
  const int ant0 = (blockIdx.x * kGroupWarps + warp) * A;
  // cold path: tours that met a step without a W > 0 candidate are rebuilt by
  // the whole warp with the fallback (construct_common.cuh rebuild_tour)
#pragma unroll 1
  for (int q = 0; q < A; ++q) {
    if (!__shfl_sync(kFull, (int)stalled, q * G)) continue;
    const bool ok = TACO_REBUILD(a.sw, a.si, a.ld, un, &a.fb, &a.ks, a.state, it,
                                 (uint32_t)(a.ant_offset + ant0 + q), vis, 0, A, q, a.nwords,
                                 a.tours + (size_t)(ant0 + q) * n, lane);
    if (!ok) {
      if (lane == 0) record_status(a.status, TACO_NO_CANDIDATE, a.ant_offset + ant0 + q);
    } else if (g == q) {
      complete = true;
    }
  }
  // tour lengths of the warp's complete tours, the whole warp per tour
  // (pairwise leaves across lanes; the step loop carries no length state)
  if (a.costs != nullptr) {
#pragma unroll 1
    for (int q = 0; q < A; ++q) {
      if (!__shfl_sync(kFull, (int)complete, q * G)) continue;
      const double c = warp_tour_cost(n, a.tours + (size_t)(ant0 + q) * n, a.dist, leaves, L, leaf_sum, lane);
      if (lane == 0) a.costs[ant0 + q] = c;
    }
  }
  if (PROBE && gl == 0 && ant < a.m_local) atomicAdd(a.scan_count, (chunks * CH + 16) / 32);
}

struct DenseArgs {
  int n, m_local, ant_offset, ldw, nwords, n_leaves;
  const float *w;
  const double *dist;
  uint32_t iteration;
  const taco_iter_state *state;  // nullable: iteration from device memory
  int32_t *tours;
  double *costs;
  int32_t *status;
  PhiloxKeys ks;
  Fallback fb;
  const int2 *leaves_img;  // nullable (construct_common.cuh leaves_image)
};

// Shared memory: int2 leaves[n_leaves]; per ant: double leaf_buf[kPwBlock],
// double leaf_sum[n_leaves], uint32 vis[nwords]
template <int WARPS>
__global__ void __launch_bounds__(WARPS * 32) k_construct_dense(const __grid_constant__ DenseArgs a) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int n = a.n;
  int2 *leaves = reinterpret_cast<int2 *>(smem);
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const size_t per_ant = ant_scratch_bytes(a.n_leaves, a.nwords);
  unsigned char *mine = smem + (((size_t)8 * a.n_leaves + 15) & ~(size_t)15) + per_ant * warp;
  double *leaf_buf = reinterpret_cast<double *>(mine);
  double *leaf_sum = leaf_buf + kPwBlock;
  uint32_t *vis = reinterpret_cast<uint32_t *>(leaf_sum + a.n_leaves);
  load_leaves(n, a.n_leaves, leaves, a.leaves_img);
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
  if (lane == 0) mark_visited<false>(vis, start);
  __syncwarp();

  TourWriter tw{a.tours + (size_t)ant * n, n, lane, 0};
  tw.put(0, (int32_t)start);
  LeafCost lc;
  lc.init(a.costs != nullptr ? a.dist : nullptr, leaves, leaf_buf, leaf_sum, n, lane);
  uint32_t cur = start;
  const int nq = (n + 3) >> 2;
  bool stalled = false;
  for (int step = 1; step < n; ++step) {
    const float4 *row = reinterpret_cast<const float4 *>(a.w + (size_t)cur * a.ldw);
    uint32_t lkey = 0u, lj = 0xffffffffu;
    uint32_t wkey = 0u;  // the warp's running best key (refreshed every 32 groups)
    const int rounds = (nq + 31) >> 5;
#pragma unroll 4
    for (int t = 0; t < rounds; ++t) {
      const int q = lane + 32 * t;
      float4 wv = make_float4(0.0f, 0.0f, 0.0f, 0.0f);
      uint32_t nib = 0xfu;
      if (q < nq) {
        wv = __ldg(row + q);
        nib = (vis[q >> 3] >> ((q & 7) * 4)) & 0xfu;
      }
      // a score is w * u < w, so a group whose largest W is below the warp's
      // running best score (key - 1 as float) cannot reach or tie the argmax
      const float wmax = fmaxf(fmaxf(wv.x, wv.y), fmaxf(wv.z, wv.w));
      const uint32_t thr = lkey > wkey ? lkey : wkey;
      const bool any = (nib != 0xfu) && wmax > 0.0f && (thr == 0u || wmax >= __uint_as_float(thr - 1u));
      if (any) {
        // cities 4q..4q+3: the blocks of j >> 1 = 2q and 2q + 1
        const uint2 r0 = philox_ant(sel_counter(4u * q, (uint32_t)step), ak, rk);
        const uint2 r1 = philox_ant(sel_counter(4u * q + 2u, (uint32_t)step), ak, rk);
        const float wc[4] = {wv.x, wv.y, wv.z, wv.w};
        const uint32_t rc[4] = {r0.x, r0.y, r1.x, r1.y};
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
      wkey = __reduce_max_sync(kFull, lkey);
    }
    const uint32_t mkey = __reduce_max_sync(kFull, lkey);
    if (mkey == 0u) {  // no W > 0 candidate: the tour is rebuilt after the loop
      stalled = true;
      break;
    }
    const uint32_t bestj = __reduce_min_sync(kFull, lkey == mkey ? lj : 0xffffffffu);
    TACO_DCHECK(bestj < (uint32_t)n && !is_visited(vis, bestj));
    if (lane == 0) vis[bestj >> 5] |= 1u << (bestj & 31);
    if (step > 1) lc.push();
    lc.load(cur, bestj);
    __syncwarp();
    tw.put(step, (int32_t)bestj);
    cur = bestj;
  }
  if (stalled) {  // cold path (construct_common.cuh rebuild_tour)
    if (!TACO_REBUILD(a.w, nullptr, a.ldw, (uint32_t)n, &a.fb, &a.ks, a.state, it, gant, vis, 0, 1, 0, a.nwords,
                      tw.row, lane)) {
      if (lane == 0) record_status(a.status, TACO_NO_CANDIDATE, (int)gant);
      return;
    }
    if (a.costs != nullptr) {
      const double c = warp_tour_cost(n, tw.row, a.dist, leaves, a.n_leaves, leaf_sum, lane);
      if (lane == 0) a.costs[ant] = c;
    }
    return;
  }
  tw.flush();
  if (lc.active) {
    lc.push();
    lc.load(cur, start);
    lc.push();
    const double c = lc.finish();
    if (lane == 0) a.costs[ant] = c;
  }
}

// Follow-up of the MODE 2 warp kernel: ants whose tour ends in the -1 marker
// met a step without a W > 0 candidate; one warp per ant rebuilds them
// (rebuild_tour) and their lengths.  Every other warp reads one word and
// exits (~µs per launch).  Shared: leaves, then per warp its visited bit map
// and leaf sums.
constexpr int kRebuildWarps = 4;

__global__ void __launch_bounds__(kRebuildWarps * 32) k_rebuild_stalled(const __grid_constant__ SortedArgs a) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int ant = blockIdx.x * kRebuildWarps + warp;
  const bool mine = ant < a.m_local && a.tours[(size_t)ant * a.n + (a.n - 1)] == -1 &&
                    !chain_stopped_update(a.status);
  if (!__syncthreads_or(mine)) return;
  const size_t lb = ((size_t)8 * a.n_leaves + 15) & ~(size_t)15;
  const int nwords = (a.n + 31) / 32;
  const size_t per_warp = ((((size_t)4 * nwords + 15) & ~(size_t)15) + lb);
  int2 *leaves = reinterpret_cast<int2 *>(smem);
  uint32_t *vis = reinterpret_cast<uint32_t *>(smem + lb + per_warp * warp);
  double *leaf_sum = reinterpret_cast<double *>(smem + lb + per_warp * warp + (((size_t)4 * nwords + 15) & ~(size_t)15));
  load_leaves(a.n, a.n_leaves, leaves, a.leaves_img);
  __syncthreads();
  if (!mine) return;
  const uint32_t it = a.state != nullptr ? a.state->iteration : a.iteration;
  const uint32_t gant = (uint32_t)(a.ant_offset + ant);
  int32_t *trow = a.tours + (size_t)ant * a.n;
  if (!rebuild_tour(a.sw, a.si, a.ld, (uint32_t)a.n, &a.fb, &a.ks, a.state, it, gant, vis, 0, 1, 0, nwords, trow,
                    lane)) {
    if (lane == 0) record_status(a.status, TACO_NO_CANDIDATE, (int)gant);
    return;
  }
  if (a.costs != nullptr) {
    const double c = warp_tour_cost(a.n, trow, a.dist, leaves, a.n_leaves, leaf_sum, lane);
    if (lane == 0) a.costs[ant] = c;
  }
}

__global__ void k_starts(int n, int m_local, int ant_offset, PhiloxKeys ks, uint32_t iteration, int32_t *out) {
  const int a = blockIdx.x * blockDim.x + threadIdx.x;
  if (a >= m_local) return;
  const RoundKeys rk = round_keys(ks, iteration);
  out[a] = (int32_t)start_city((uint32_t)n, ant_key((uint32_t)(ant_offset + a), rk), rk);
}

__global__ void k_uniforms(int count, const uint32_t *step, const uint32_t *ant, const uint32_t *city,
                           PhiloxKeys ks, uint32_t iteration, float *out) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= count) return;
  const RoundKeys rk = round_keys(ks, iteration);
  out[t] = bits_to_uniform(sel_word(city[t], step[t], ant_key(ant[t], rk), rk));
}

__global__ void k_philox(int count, const uint32_t *ctr, const uint32_t *key, uint32_t *out) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= count) return;
  const uint2 r = philox2x32_10(ctr[2 * t], ctr[2 * t + 1], key[t]);
  out[2 * t] = r.x;
  out[2 * t + 1] = r.y;
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

// argmax_select_block (selection.py:143-155) as its own drop-in: scores =
// take(logw, current) - e_block, visited := -inf, row argmax (first of ties,
// an all -inf row gives 0).  No visited update and no assertion: those belong
// to construct_tours (colony.py:149-152).
template <int WARPS>
__global__ void __launch_bounds__(WARPS * 32)
    k_argmax_block(int n, int m, const double *__restrict__ logw, const int64_t *__restrict__ current,
                   const double *__restrict__ e_block, const uint8_t *__restrict__ visited, double *scores,
                   int64_t *next_out) {
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int a = blockIdx.x * WARPS + warp;
  if (a >= m) return;
  const double *lr = logw + (size_t)current[a] * n;
  const double *er = e_block + (size_t)a * n;
  const uint8_t *vr = visited + (size_t)a * n;
  double best = -INFINITY;
  int bj = 0x7fffffff;
  for (int j = lane; j < n; j += 32) {
    const double s = vr[j] ? -INFINITY : __dsub_rn(lr[j], er[j]);
    if (scores != nullptr) scores[(size_t)a * n + j] = s;
    if (s > best) best = s, bj = j;
  }
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    const double ob = __shfl_xor_sync(kFull, best, off);
    const int oj = __shfl_xor_sync(kFull, bj, off);
    if (ob > best || (ob == best && oj < bj)) best = ob, bj = oj;
  }
  if (lane == 0) next_out[a] = bj == 0x7fffffff ? 0 : bj;
}

}  // namespace taco

using namespace taco;

extern "C" int taco_argmax_select_block(int n, int m, const double *logw, const int64_t *current,
                                        const double *e_block, const uint8_t *visited, double *scores_out,
                                        int64_t *next_out, void *stream) {
  if (n < 1 || m < 0 || (m > 0 && (logw == nullptr || current == nullptr || e_block == nullptr ||
                                   visited == nullptr || next_out == nullptr)))
    return TACO_ERR_ARG;
  if (m == 0) return TACO_OK;
  constexpr int WARPS = 8;
  k_argmax_block<WARPS><<<(m + WARPS - 1) / WARPS, WARPS * 32, 0, reinterpret_cast<cudaStream_t>(stream)>>>(
      n, m, logw, current, e_block, visited, scores_out, next_out);
  TACO_CUDA_CHECK_LAUNCH();
  return TACO_OK;
}


template <bool PROBE, bool VIS8, int MODE>
static int launch_sorted(const SortedArgs &a, int grid, int threads, size_t smem, cudaStream_t s) {
  if (set_smem((const void *)k_construct_sorted<PROBE, VIS8, MODE>, smem) != TACO_OK) return TACO_ERR_CUDA;
  k_construct_sorted<PROBE, VIS8, MODE><<<grid, threads, smem, s>>>(a);
  return TACO_OK;
}

extern "C" int taco_construct(int n, int m_local, int ant_offset, int variant, const float *w, int ldw,
                              const float *sw, const uint16_t *si, uint64_t seed, uint32_t iteration,
                              const double *dist, int32_t *tours_out, double *costs_out, int32_t *status,
                              unsigned long long *scan_count, const double *fb_a, double fb_alpha,
                              const double *fb_b, double inv_gamma, const taco_iter_state *state, void *stream) {
  if (n < 3 || n > 65535 || m_local < 0 || ant_offset < 0 || tours_out == nullptr) return TACO_ERR_ARG;
  if (fb_b != nullptr && fb_a == nullptr) return TACO_ERR_ARG;
  const Fallback fb{fb_a, fb_b, fb_alpha, inv_gamma};
  if (costs_out != nullptr && dist == nullptr) return TACO_ERR_ARG;
  if (m_local == 0) return TACO_OK;
  const PhiloxKeys ks = philox_keys(seed);
  const int nwords = (n + 31) / 32;
  const int n_leaves = pw_num_leaves(n);
  const size_t per_ant = ant_scratch_bytes(n_leaves, nwords);
  const size_t leaves_bytes = ((size_t)8 * n_leaves + 15) & ~(size_t)15;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  if (variant == TACO_CONSTRUCT_SORTED) {
    if (sw == nullptr || si == nullptr || ldw < n || (ldw % 32) != 0) return TACO_ERR_ARG;
    // kernel choice: lane-group kernel (G lanes x E entries per ant) or the
    // warp-per-ant kernel; TACO_SORTED_KERNEL = warp | g4e4 | g8e4 | g4e2 |
    // g8e2 | g16e2 overrides (tuning knob)
    int G = 0, E = 0;
    // Measured on B200 at n = 2392 (scripts/sweep_kernel_choice.sh): the warp
    // kernel wins up to ~64 ants per SM (m = 8192: 2.93 vs 3.04 ms for g4e4);
    // beyond that the SIMT sharing of the lane-group kernel wins.
    // With position-keyed uniforms (independent of the table loads) four
    // entries per lane win everywhere above 64 ants per SM (round 2, ms, g4e4
    // vs g8e2): n = 5000 m = 12288 8.06 vs 12.02, m = 16384 10.16 vs 12.46,
    // m = 32768 16.39 vs 21.50; n = 2392 m = 16384 4.53 vs 5.70; n = 1000
    // m = 32768 2.95 vs 3.80
    if (m_local > 64 * sm_count()) G = 4, E = 4;
    if (const char *ev = getenv("TACO_SORTED_KERNEL")) {
      G = 0;
      if (ev[0] == 'g') {
        G = atoi(ev + 1);
        const char *pe = ev + 1;
        while (*pe && *pe != 'e') ++pe;
        E = *pe ? atoi(pe + 1) : 4;
      }
    }
    if (G > 0) {
      const size_t A = 32 / G;
      const size_t per_warp = (((size_t)4 * nwords * A + 15) & ~(size_t)15) + leaves_bytes;
      const size_t smem = leaves_bytes + per_warp * kGroupWarps;
      if (smem > 227 * 1024) return TACO_ERR_UNSUPPORTED;
      GroupArgs ga{n, m_local, ant_offset, nwords, n_leaves, ldw, sw, si, dist, iteration, state,
                   tours_out, costs_out, status, scan_count, ks, fb, leaves_image(n, s)};
      const int ants_per_cta = (int)A * kGroupWarps;
      const int grid = (m_local + ants_per_cta - 1) / ants_per_cta;
#define TACO_GROUP_CASE(GG, EE)                                                                         \
  if (G == GG && E == EE) {                                                                             \
    if (scan_count != nullptr) {                                                                        \
      if (set_smem((const void *)k_construct_group<GG, EE, true>, smem) != TACO_OK) return TACO_ERR_CUDA; \
      k_construct_group<GG, EE, true><<<grid, kGroupWarps * 32, smem, s>>>(ga);                         \
    } else {                                                                                            \
      if (set_smem((const void *)k_construct_group<GG, EE, false>, smem) != TACO_OK) return TACO_ERR_CUDA; \
      k_construct_group<GG, EE, false><<<grid, kGroupWarps * 32, smem, s>>>(ga);                        \
    }                                                                                                   \
    TACO_CUDA_CHECK_LAUNCH();                                                                           \
    return TACO_OK;                                                                                     \
  }
      TACO_GROUP_CASE(4, 4)
      TACO_GROUP_CASE(8, 4)
      TACO_GROUP_CASE(4, 2)
      TACO_GROUP_CASE(8, 2)
      TACO_GROUP_CASE(16, 2)
#undef TACO_GROUP_CASE
      return TACO_ERR_ARG;
    }
    // tour length: computed in the kernel's epilogue from the finished tour
    // row, lanes summing pairwise leaves in parallel, so the step loop carries
    // no length state (35 registers in the loop instead of 72) and the random
    // dist reads overlap other warps' construction.  Measured (ms, incl. the
    // length): n = 2392, m = 4096 epilogue 1.755 / separate k_tour_cost pass
    // 1.779 / fused per-step accumulation 1.836; n = 10000, m = 8192 16.3 /
    // 17.2 / 17.7.  TACO_SORTED_COST=fused|separate|epilogue (tuning knob).
    bool fused_cost = false;
    if (const char *ev = getenv("TACO_SORTED_COST")) fused_cost = costs_out != nullptr && ev[0] == 'f';
    const int max_warps = fused_cost ? kSortedMaxWarps : kMode1Warps;  // beyond: MODE 2, 2 x 32 warps
    // warps per CTA: all ants of an SM in one CTA when they fit (one wave);
    // larger colonies run 32-warp CTAs, two per SM.  TACO_SORTED_WARPS
    // overrides (tuning knob).
    const int ants_per_sm = (m_local + sm_count() - 1) / sm_count();
    // MODE 3: 29-32 ants per SM, one 32-warp CTA at 64 registers (MODE 2's
    // 32 registers cost 21% at n = 2392, m = 4400)
    const bool wide = !fused_cost && ants_per_sm > max_warps && ants_per_sm <= 32;
    const bool two_ctas = !fused_cost && ants_per_sm > 32;  // MODE 2
    int warps = ants_per_sm < 1 ? 1 : (ants_per_sm > max_warps ? max_warps : ants_per_sm);
    if (wide) warps = ants_per_sm;
    if (two_ctas) warps = std::min(kMode2Warps, (ants_per_sm + 1) / 2);
    if (const char *ev = getenv("TACO_SORTED_WARPS")) warps = atoi(ev);
    if (warps < 1 || warps > (two_ctas ? kMode2Warps : (wide ? 32 : max_warps))) return TACO_ERR_ARG;
    // (separate: tour lengths by a k_tour_cost launch after the kernel instead
    // of the epilogue; TACO_SORTED_COST=separate, tuning knob)
    const bool separate_cost = !fused_cost && getenv("TACO_SORTED_COST") && getenv("TACO_SORTED_COST")[0] == 's';
    auto scratch = [&](int nw) {
      return fused_cost ? ant_scratch_bytes(n_leaves, nw) : leaves_bytes + (((size_t)4 * nw + 15) & ~(size_t)15);
    };
    const size_t lb = leaves_bytes;
    // visited set: a byte per city when the SM's ants fit with it (VIS8),
    // else the bit map; TACO_SORTED_VIS=bits forces the bit map (tuning knob)
    const int nwords8 = (n + 3) / 4;
    const int resident = two_ctas ? 2 * warps : warps;
    bool vis8 = lb + scratch(nwords8) * (resident > warps ? resident : warps) <= 200 * 1024;
    if (const char *ev = getenv("TACO_SORTED_VIS")) vis8 = vis8 && ev[0] != 'b';
    // (Measured and removed: a shared-memory cache of the first T entries of
    // every row.  Once the next row's first window is issued a step ahead,
    // the separate pass over the cached head only adds work: n = 2392, m = 512
    // 1.39 vs 1.62 ms with T = 12; m = 4096 2.19 vs 2.45.  An L1 prefetch of
    // the top candidates' next windows was slower too, 2.68 vs 2.48 ms.)
    const size_t smem = lb + scratch(vis8 ? nwords8 : nwords) * warps;
    if (smem > 227 * 1024) return TACO_ERR_UNSUPPORTED;
    SortedArgs a{n, m_local, ant_offset, vis8 ? nwords8 : nwords, n_leaves, ldw, sw, si, dist, iteration, state,
                 tours_out, separate_cost ? nullptr : costs_out, status, scan_count, ks, fb,
                 costs_out != nullptr ? leaves_image(n, s) : nullptr};
    const int grid = (m_local + warps - 1) / warps;
    // MODE 4 up to kLatencyAnts ants per SM (latency-bound: few warps to interleave)
    int mode = fused_cost ? 0 : (two_ctas ? 2 : (wide ? 3 : (ants_per_sm <= kLatencyAnts ? 4 : 1)));
    if (const char *ev = getenv("TACO_SORTED_MODE")) {  // tuning knob: 1 <-> 4 where either applies
      const int f = atoi(ev);
      if ((mode == 1 || mode == 4) && (f == 1 || f == 4)) mode = f;
    }
    const int code = mode * 4 + (vis8 ? 2 : 0) + (scan_count ? 1 : 0);
    int rc = TACO_ERR_ARG;
    switch (code) {
#define TACO_SORTED_CASE(MODE, V, P) \
  case MODE * 4 + (V) * 2 + (P): rc = launch_sorted<P, V, MODE>(a, grid, warps * 32, smem, s); break;
      TACO_SORTED_CASE(0, 0, 0) TACO_SORTED_CASE(0, 0, 1) TACO_SORTED_CASE(0, 1, 0) TACO_SORTED_CASE(0, 1, 1)
      TACO_SORTED_CASE(1, 0, 0) TACO_SORTED_CASE(1, 0, 1) TACO_SORTED_CASE(1, 1, 0) TACO_SORTED_CASE(1, 1, 1)
      TACO_SORTED_CASE(2, 0, 0) TACO_SORTED_CASE(2, 0, 1) TACO_SORTED_CASE(2, 1, 0) TACO_SORTED_CASE(2, 1, 1)
      TACO_SORTED_CASE(3, 0, 0) TACO_SORTED_CASE(3, 0, 1) TACO_SORTED_CASE(3, 1, 0) TACO_SORTED_CASE(3, 1, 1)
      TACO_SORTED_CASE(4, 0, 0) TACO_SORTED_CASE(4, 0, 1) TACO_SORTED_CASE(4, 1, 0) TACO_SORTED_CASE(4, 1, 1)
#undef TACO_SORTED_CASE
    }
    if (rc == TACO_OK && mode == 2) {  // tours the MODE 2 kernel left to the rebuild
      const size_t lb2 = leaves_bytes;
      const size_t smem2 = lb2 + ((((size_t)4 * nwords + 15) & ~(size_t)15) + lb2) * kRebuildWarps;
      if (set_smem((const void *)k_rebuild_stalled, smem2) != TACO_OK) return TACO_ERR_CUDA;
      SortedArgs ra = a;
      ra.costs = costs_out;
      k_rebuild_stalled<<<(m_local + kRebuildWarps - 1) / kRebuildWarps, kRebuildWarps * 32, smem2, s>>>(ra);
      TACO_CUDA_CHECK_LAUNCH();
    }
    if (rc == TACO_OK && costs_out != nullptr && separate_cost)
      rc = taco_tour_cost(n, m_local, tours_out, 0, dist, costs_out, stream);
    if (rc != TACO_OK) return rc;
  } else if (variant == TACO_CONSTRUCT_DENSE) {
    if (w == nullptr || ldw < n || (ldw % 4) != 0) return TACO_ERR_ARG;
    if ((reinterpret_cast<uintptr_t>(w) & 15u) != 0) return TACO_ERR_ARG;
    constexpr int WARPS = 4;
    const size_t smem = leaves_bytes + per_ant * WARPS;
    if (smem > 227 * 1024) return TACO_ERR_UNSUPPORTED;
    if (set_smem((const void *)k_construct_dense<WARPS>, smem) != TACO_OK) return TACO_ERR_CUDA;
    DenseArgs a{n, m_local, ant_offset, ldw, nwords, n_leaves, w, dist, iteration, state, tours_out, costs_out,
                status, ks, fb, leaves_image(n, s)};
    k_construct_dense<WARPS><<<(m_local + WARPS - 1) / WARPS, WARPS * 32, smem, s>>>(a);
  } else {
    return TACO_ERR_ARG;
  }
  TACO_CUDA_CHECK_LAUNCH();
  return TACO_OK;
}

#ifdef TACO_STEP_PROFILE
extern "C" int taco_step_profile(unsigned long long *host_out, int reset) {
  if (cudaMemcpyFromSymbol(host_out, g_step_prof, sizeof(unsigned long long) * 8) != cudaSuccess)
    return TACO_ERR_CUDA;
  if (reset) {
    unsigned long long z[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    cudaMemcpyToSymbol(g_step_prof, z, sizeof(z));
  }
  return TACO_OK;
}
#endif

extern "C" int taco_starts(int n, int m_local, int ant_offset, uint64_t seed, uint32_t iteration,
                           int32_t *starts_out, void *stream) {
  if (n < 1 || m_local < 0 || starts_out == nullptr) return TACO_ERR_ARG;
  if (m_local == 0) return TACO_OK;
  k_starts<<<(m_local + 255) / 256, 256, 0, reinterpret_cast<cudaStream_t>(stream)>>>(
      n, m_local, ant_offset, philox_keys(seed), iteration, starts_out);
  TACO_CUDA_CHECK_LAUNCH();
  return TACO_OK;
}

extern "C" int taco_uniforms(int count, const uint32_t *step, const uint32_t *ant, const uint32_t *city,
                             uint64_t seed, uint32_t iteration, float *u_out, void *stream) {
  if (count < 0) return TACO_ERR_ARG;
  if (count == 0) return TACO_OK;
  k_uniforms<<<(count + 255) / 256, 256, 0, reinterpret_cast<cudaStream_t>(stream)>>>(
      count, step, ant, city, philox_keys(seed), iteration, u_out);
  TACO_CUDA_CHECK_LAUNCH();
  return TACO_OK;
}

extern "C" int taco_philox2x32_10(int count, const uint32_t *ctr2, const uint32_t *key, uint32_t *out2,
                                  void *stream) {
  if (count < 0) return TACO_ERR_ARG;
  if (count == 0) return TACO_OK;
  k_philox<<<(count + 255) / 256, 256, 0, reinterpret_cast<cudaStream_t>(stream)>>>(count, ctr2, key, out2);
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
