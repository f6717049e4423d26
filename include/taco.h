/*
 * taco.h — C ABI of libtaco.so, the B200 (sm_100a) engine behind the
 * TensorACO hot path: one ACO iteration with Independent-Roulette (IR) or
 * Adaptive-IR (AdaIR) selection (and the roulette-wheel ablation, RW).
 *
 * The reference (`antbatch`, /root/reference/pkg/src/antbatch) is a pure
 * Python/numpy package and has no FFI of its own; its "plugin boundary" is the
 * set of module-level functions listed below.  Each entry point here names the
 * reference function it replaces (file:line) and is what the Python host layer
 * (paper_2404_04895_b200/) binds through ctypes.
 *
 * Conventions
 *   - Every pointer argument is a DEVICE pointer unless its name ends in _host.
 *     Matrices are row-major (C order), n x n, leading dimension n unless a
 *     separate ld argument is given.
 *   - `stream` is a cudaStream_t passed as void*; every call is asynchronous on
 *     that stream and never allocates memory (callers pass workspaces).
 *   - `status` points to 4 device int32 words the caller initializes to
 *     {0, INT32_MAX, 0, 0}.  Kernels record the first data-dependent failure
 *     there: status[0] = code (TACO_UNDERFLOW / TACO_NO_CANDIDATE /
 *     TACO_DEGENERATE), status[1] = smallest offending row (underflow,
 *     degenerate) or ant (no candidate), kept with atomicMin.  Fail-stop:
 *     a construction call that starts with status[0] != 0 sets status[3] and
 *     builds nothing; a row update that sees status[3] != 0 changes nothing —
 *     iterations queued after a failure leave the failing state in place.
 *   - The return value reports argument / launch errors synchronously:
 *     0 = launched, negative = error (see taco_status_string).
 */
#ifndef TACO_H_
#define TACO_H_

#include <stdint.h>
#include <stddef.h>

#ifdef __cplusplus
extern "C" {
#endif

#define TACO_ABI_VERSION 4

/* status codes (return values and status[0]) */
#define TACO_OK 0
#define TACO_UNDERFLOW 1          /* colony.py:63-68  NumericalUnderflow          */
#define TACO_NO_CANDIDATE 2       /* colony.py:149   "selector chose a visited city" */
#define TACO_DEGENERATE 3         /* model.py:86-91  DegenerateInstance (status[1] = row) */
#define TACO_ERR_ARG (-1)         /* bad argument (ValueError on the Python side)  */
#define TACO_ERR_CUDA (-2)        /* CUDA launch / runtime error                  */
#define TACO_ERR_UNSUPPORTED (-3) /* size outside the compiled kernel variants    */

/* construction variants for taco_construct */
#define TACO_CONSTRUCT_SORTED 0 /* pruned scan of the per-row descending table   */
#define TACO_CONSTRUCT_DENSE 1  /* full-row streaming scan of dense W            */

/*
 * Device-resident iteration scalars (CUDA-graph replay of Solver steps).
 * Entry points taking a `const taco_iter_state *state` read the iteration
 * number / 1/gamma from device memory when state != NULL (ignoring the
 * by-value argument), so one captured iteration replays unchanged;
 * taco_iter_advance moves the state to the next iteration on the stream.
 * inv_gamma is 1/gamma of the selection table built at the END of the
 * iteration, i.e. for iteration + 1 (the W the next construction reads);
 * inv_gamma_cur is 1/gamma of the iteration itself (the table the
 * construction reads; its f64 fallback needs it).
 */
typedef struct taco_iter_state {
  uint32_t iteration;
  uint32_t reserved;
  double inv_gamma;
  double inv_gamma_cur;
  double reserved2;
} taco_iter_state;

int taco_abi_version(void);
const char *taco_status_string(int code);
/* message of the last CUDA error a libtaco call returned TACO_ERR_CUDA for
 * (per host thread; "" if none) */
const char *taco_last_cuda_error(void);
/* largest n the sorted-table (per-row block radix sort) path supports */
int taco_max_sorted_n(void);

/*
 * Fused row kernel: evaporation + index-mapped deposit + P = RowNorm(tau^a eta^b)
 * + the fp32 selection table W = P^(1/gamma) (dense and/or row-sorted).
 * Persistent CTAs, one row at a time.  Replaces, in one pass over tau:
 *   pheromone.accumulate_increments   pheromone.py:52-68   (delta source)
 *   pheromone.apply_update            pheromone.py:71-83   (do_evap != 0)
 *   colony.compute_probability_matrix colony.py:51-69      (p_out / rowsum_out)
 *   selection.scaled_log_weights      selection.py:62-75   (folded into W)
 *
 * Delta source (at most one): nbr+inc (k elites; nbr[i*k + r] = (prev, next)
 * of city i in elite r's tour, inc[r] = 1/cost_r, rank order r = 0..k-1) or a
 * dense delta_in (n x n).  With neither, delta = 0.
 * tau' = max(keep*tau + delta, 1e-12) when do_evap, else tau' = tau_in.
 * eta_b = eta^beta (precomputed once per instance, n x n).
 * Outputs (each nullable): delta_out, tau_out (may alias tau_in), p_out,
 * rowsum_out (n), w_out (n x ldw fp32, pad columns zeroed), sw_out/si_out
 * (n x n fp32 values / uint16 column indices, each row sorted descending by
 * the W bits above bit 16, stable in the column index).
 * eta_b / p outputs are skipped when want_p == 0 (delta/tau-only modes).
 * state (nullable): inv_gamma is read from state->inv_gamma.
 * The row is staged in shared memory: n <= ~27900 (TACO_ERR_UNSUPPORTED above).
 */
int taco_row_update(int n,
                    const double *tau_in, double *tau_out,
                    const double *eta_b,
                    const int32_t *nbr, const double *inc, int k,
                    const double *delta_in, double *delta_out,
                    int do_evap, double keep,
                    int want_p, double alpha, double inv_gamma,
                    double *p_out, double *rowsum_out,
                    float *w_out, int ldw,
                    float *sw_out, uint16_t *si_out,
                    int32_t *status, const taco_iter_state *state,
                    void *stream);

/*
 * taco_row_update restricted to rows [row_begin, row_end) (the row-partitioned
 * multi-GPU update: each rank updates its rows of tau / P / W / the sorted
 * table, then the tables are all-gathered).  Rows outside the range are not
 * touched; all pointers still address the full n-row matrices.
 */
int taco_row_update_rows(int row_begin, int row_end, int n,
                         const double *tau_in, double *tau_out,
                         const double *eta_b, const int32_t *nbr,
                         const double *inc, int k, const double *delta_in,
                         double *delta_out, int do_evap, double keep,
                         int want_p, double alpha, double inv_gamma,
                         double *p_out, double *rowsum_out, float *w_out,
                         int ldw, float *sw_out, uint16_t *si_out,
                         int32_t *status, const taco_iter_state *state,
                         void *stream);

/*
 * The same update as taco_row_update in Solver mode (edge-map deposit,
 * evaporation, P, W / sorted table), as three streaming kernels that need no
 * row in shared memory (any n <= 65535): a warp-per-row deposit into
 * delta_ws (n x n f64), an elementwise evaporation + tau^alpha eta^beta into
 * unnorm_ws (n x n f64), and a warp-per-row pairwise normalization writing P
 * (p_out, nullable), the row sums and W.  Bit-identical results.  nbr / inc
 * (nullable: no deposit) need do_evap; do_evap == 0 leaves tau untouched.
 */
int taco_update_split(int n, const double *tau_in, double *tau_out,
                      const double *eta_b, const int32_t *nbr,
                      const double *inc, int k, int do_evap, double keep,
                      double alpha, double inv_gamma, double *delta_ws,
                      double *unnorm_ws, double *p_out, double *rowsum_out,
                      float *w_out, int ldw, float *sw_out, uint16_t *si_out,
                      int32_t *status, const taco_iter_state *state,
                      void *stream);

/*
 * Selection table from a given P (construct_tours drop-in, colony.py:116):
 * W = fp32(P^(1/gamma)) dense (n x ldw) and/or row-sorted (sw_out/si_out).
 */
int taco_selection_table(int n, const double *p, double inv_gamma,
                         float *w_out, int ldw, float *sw_out,
                         uint16_t *si_out, void *stream);

/*
 * eta^beta with numpy's scalar-exponent dispatch (colony.py:60): exponents
 * 0, 0.5, 1, 2 are exact (ones / sqrt / copy / square), others use pow.
 */
int taco_eta_power(int64_t count, const double *eta, double beta, double *out,
                   void *stream);

/*
 * Tour construction, fast path (device Philox2x32-10 stream; key
 * H(seed) + iteration, counter (ant, (city >> 1) | step << 16), word city & 1).
 * Replaces colony.construct_tours colony.py:87-154 (IR / AdaIR branch) with
 * the deviate block of rng.step_exponentials rng.py:42-49 replaced by the
 * on-chip keyed uniform u(seed, iteration, step, ant, city) and the log-domain
 * rule argmax(log P/gamma - E) by its product form argmax(W * u).
 * Ants [ant_offset, ant_offset + m_local) are built; tours_out is
 * m_local x n int32.  variant: TACO_CONSTRUCT_SORTED (needs sw/si) or
 * TACO_CONSTRUCT_DENSE (needs w, ldw).  When costs_out is given, the tour
 * lengths from dist (n x n f64) are computed in numpy's pairwise order
 * (model.batch_costs model.py:292-295, bit-exact), during construction or by
 * a k_tour_cost pass on the same stream.
 * scan_count (nullable, device u64) is incremented by the number of 32-entry
 * global table windows the SORTED variant read (traffic probe for the
 * roofline report).
 * No W > 0 candidate left (W underflows below 2^-126 of its row's best, e.g.
 * for gamma < 1): the step is decided in f64 among the unvisited cities with
 * v = fb_a[cur, j]^fb_alpha (* fb_b[cur, j]) > 0 by log(v) * inv_gamma +
 * log(u) (fb_a = P, or tau with fb_b = eta^beta; n x n, row pitch n); with
 * none (or fb_a NULL), city 0 if unvisited — numpy's argmax of an all -inf
 * row (selection.py:152-155) — else TACO_NO_CANDIDATE (colony.py:149).
 * state (nullable): iteration from state->iteration, inv_gamma from
 * state->inv_gamma_cur.
 */
int taco_construct(int n, int m_local, int ant_offset, int variant,
                   const float *w, int ldw,
                   const float *sw, const uint16_t *si,
                   uint64_t seed, uint32_t iteration,
                   const double *dist, int32_t *tours_out, double *costs_out,
                   int32_t *status, unsigned long long *scan_count,
                   const double *fb_a, double fb_alpha, const double *fb_b,
                   double inv_gamma,
                   const taco_iter_state *state, void *stream);

/*
 * Roulette-wheel (RW) construction, device stream.
 * Replaces colony.construct_tours colony.py:127-141 (RW branch) with
 * rw_spin_block (selection.py:102-127) evaluated on P (n x n f64, the
 * probability matrix) for ants [ant_offset, ant_offset + m_local): per step
 * the first j with cumsum(P[cur] * unvisited)_j / total > u, bit-exact with
 * the reference's sequential cumsum rule (a certified parallel scan, with an
 * exact sequential recount when the crossing is within rounding distance).
 * u is one 53-bit Philox2x32-10 uniform per (step, ant) (counter
 * (ant, 0xffff | step << 16)) in place of rng.step_uniforms (rng.py:52-62).  Start cities and
 * the fused tour length are as in taco_construct.  exact_count (nullable,
 * device u64) accumulates the steps that took the sequential recount;
 * force_exact != 0 makes every step take it (test hook).  state as in
 * taco_construct.
 */
int taco_construct_rw(int n, int m_local, int ant_offset, const double *p,
                      uint64_t seed, uint32_t iteration, const double *dist,
                      int32_t *tours_out, double *costs_out, int32_t *status,
                      unsigned long long *exact_count, int force_exact,
                      const taco_iter_state *state, void *stream);

/*
 * One lockstep round of rw_spin_block (selection.py:102-127) with the
 * reference's thresholds u (m f64, rng.step_uniforms) — RW parity mode: the
 * visited assert (colony.py:149), then current (m i64) / visited (m x n u8) /
 * tours (m x n i64, column `step`) update.  exact_count / force_exact as in
 * taco_construct_rw.
 */
int taco_rw_parity(int n, int m, int step, const double *p, const double *u,
                   int64_t *current, uint8_t *visited, int64_t *tours,
                   int32_t *status, unsigned long long *exact_count,
                   int force_exact, void *stream);

/* RW device-stream thresholds for given (step, ant) pairs (test hook). */
int taco_rw_uniforms(int count, const uint32_t *step, const uint32_t *ant,
                     uint64_t seed, uint32_t iteration, double *u_out,
                     void *stream);

/* Start cities of the device stream (rng.start_cities rng.py:65-68 analog). */
int taco_starts(int n, int m_local, int ant_offset, uint64_t seed,
                uint32_t iteration, int32_t *starts_out, void *stream);

/* Raw device uniforms for given (step, ant, city) triples (test hook). */
int taco_uniforms(int count, const uint32_t *step, const uint32_t *ant,
                  const uint32_t *city, uint64_t seed, uint32_t iteration,
                  float *u_out, void *stream);

/* Philox2x32-10 (Random123) on `count` (counter[2], key) pairs: the
 * generator of the device stream (KAT hook). */
int taco_philox2x32_10(int count, const uint32_t *ctr2, const uint32_t *key,
                       uint32_t *out2, void *stream);

/*
 * Reference-stream selection step (bit-exact parity mode).  One lockstep
 * round of colony.py:143-152: next = argmax_j(logw[cur, j] - e[a, j]) with
 * visited cities at -inf and first-of-ties (selection.py:143-155), the
 * visited assert (colony.py:149), then current/visited/tours update.
 * logw n x n f64, e_block m x n f64, current m int64, visited m x n uint8,
 * tours m x n int64 (column `step` written).
 */
int taco_select_parity(int n, int m, int step, const double *logw,
                       const double *e_block, int64_t *current,
                       uint8_t *visited, int64_t *tours,
                       int32_t *status, void *stream);

/*
 * argmax_select_block (selection.py:143-155) drop-in: next_out[a] =
 * argmax_j(logw[current[a], j] - e_block[a, j]) with visited (m x n u8) cities
 * at -inf, first of ties, 0 for an all -inf row; scores_out (nullable, m x n
 * f64) receives the masked scores like the reference's scratch buffer.
 * Nothing else is updated (no visited mark, no assertion).
 */
int taco_argmax_select_block(int n, int m, const double *logw,
                             const int64_t *current, const double *e_block,
                             const uint8_t *visited, double *scores_out,
                             int64_t *next_out, void *stream);

/*
 * Reference-stream replay: the same round as
 * taco_select_parity, but the step's (m, n) Exp(1) block of
 * Generator(Philox(SeedSequence(seed, spawn_key=(0, it, step))))
 * .standard_exponential (rng.py:42-49) is regenerated on the device from the
 * step's Philox4x64 key (key0, key1 = SeedSequence.generate_state(2, uint64),
 * computed by the host) with numpy's ziggurat, decoded in parallel.
 * flags_out (2 device words, zeroed by the caller): [0] counts wedge tests
 * closer than 4 ulp (CUDA vs glibc exp could disagree), [1] is set if the
 * replay window overflowed; either makes the round unreliable.
 */
size_t taco_replay_workspace_bytes(int m, int n);
int taco_select_replay(int n, int m, int step, uint64_t key0, uint64_t key1,
                       const double *logw, int64_t *current, uint8_t *visited,
                       int64_t *tours, void *workspace, size_t ws_bytes,
                       unsigned *flags_out, int32_t *status, void *stream);

/* edge-weight conventions for taco_coord_instance */
#define TACO_EDGE_EXACT 0   /* sqrt(dx*dx+dy*dy), unrounded: euclidean_instance model.py:124-134 */
#define TACO_EDGE_EUC_2D 1  /* TSPLIB EUC_2D  int(sqrt+0.5)   tsplib.py:207-208 */
#define TACO_EDGE_CEIL_2D 2 /* TSPLIB CEIL_2D ceil(sqrt)      tsplib.py:209-210 */
#define TACO_EDGE_ATT 3     /* TSPLIB ATT pseudo-Euclidean    tsplib.py:211-214 */

/*
 * Column 0 of the step's reference block, E[a, 0] for every ant (e0_out, m
 * f64), decoded on the device like taco_select_replay: the roulette wheel's
 * thresholds are u = exp(-E[:, 0]) (rng.step_uniforms rng.py:52-62), taken by
 * the host with numpy's own exp for bit parity.  flags_out as above.
 */
int taco_replay_first_column(int n, int m, uint64_t key0, uint64_t key1,
                             void *workspace, size_t ws_bytes, double *e0_out,
                             unsigned *flags_out, void *stream);

/*
 * Instance on the device from (n, 2) f64 coordinates:
 * dist under `edge_weight` and eta = 1/dist off the diagonal, bit-exact with
 * euclidean_instance (model.py:124-134) / build_instance (model.py:98-119)
 * through _instance_from_dist (model.py:82-97).  Replaces the host's n^2
 * Python loop and the 16n^2-byte upload.  A zero off-diagonal distance records
 * TACO_DEGENERATE with status[1] = smallest such row, unless lenient (then
 * eta = 1/1e-10 there).  3 <= n <= 65535.
 */
int taco_coord_instance(int n, const double *coords, int edge_weight,
                        double *dist_out, double *eta_out, int lenient,
                        int32_t *status, void *stream);

/* logw = log(p)/gamma, -inf where p == 0 (selection.py:62-75). */
int taco_log_weights(int64_t count, const double *p, double gamma,
                     double *logw_out, void *stream);

/*
 * Tour lengths: costs[a] = pairwise-sum_s dist[t[s], t[(s+1) % n]] in numpy's
 * pairwise order (model.batch_costs model.py:292-295).  tours int32 or int64
 * (tours_is_i64), m x n.
 */
int taco_tour_cost(int n, int m, const void *tours, int tours_is_i64,
                   const double *dist, double *costs_out, void *stream);

/*
 * Stable ascending argsort of m costs (pheromone.select_elite
 * pheromone.py:17-25 = np.argsort(kind="stable")).  order_out has m entries.
 */
size_t taco_elite_workspace_bytes(int m);
int taco_elite_order(int m, const double *costs, int32_t *order_out,
                     void *workspace, size_t ws_bytes, void *stream);

/*
 * Elite edge map for the fused deposit: nbr[t[s]*k + r] = (t[s-1], t[s+1])
 * and inc[r] = 1.0 / cost of elite r = order[r] (pheromone.py:52-68,
 * edge_index_matrix pheromone.py:28-38).  tours int32 (ld = n) or int64.
 */
int taco_elite_neighbors(int n, int k, const void *tours, int tours_is_i64,
                         const int32_t *order, const double *costs,
                         int32_t *nbr_out, double *inc_out, void *stream);

/*
 * Multi-GPU costs-first exchange, local half.  After the m
 * lengths are all-gathered and ranked (order), elite row r (r < k) receives
 * this rank's tour of global ant order[r] when the rank owns it (ants
 * [ant_offset, ant_offset + count), tours_local count x n), zeros otherwise;
 * a SUM all-reduce of elite_tours (k x n int32) over the ranks then holds every
 * elite tour exactly — k·n instead of m·n exchanged.  elite_costs[r] =
 * costs_all[order[r]].
 */
int taco_shard_elites(int n, int k, const int32_t *order, int ant_offset,
                      int count, const int32_t *tours_local,
                      const double *costs_all, int32_t *elite_tours,
                      double *elite_costs, void *stream);

/*
 * Best-so-far tracking for Solver.step(): if costs[order[0]] < *best_cost,
 * copy that tour to best_tour and update best_cost / best_iter.  Nothing is
 * touched when status (nullable) records a stopped iteration (status[3]).
 */
int taco_track_best(int n, const int32_t *tours, const double *costs,
                    const int32_t *order, double *best_cost,
                    int32_t *best_tour, int32_t *best_iter, uint32_t iteration,
                    const int32_t *status, const taco_iter_state *state,
                    void *stream);

/*
 * End of a graph-replayed iteration: state->iteration += 1 and
 * state->inv_gamma = inv_gamma_table[(state->iteration + 1) % period] (the
 * table holds 1/gamma_at(t) for t = 0..period-1, computed by the host with
 * the reference's arithmetic, selection.py:48-59).
 */
int taco_iter_advance(taco_iter_state *state, const double *inv_gamma_table,
                      int period, void *stream);

#ifdef __cplusplus
}
#endif
#endif /* TACO_H_ */
