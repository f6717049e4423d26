/* ORACLE (test infrastructure only): C restatement of the engine's device
 * stream and product-form selection rule, for parity checks at the BASELINE
 * sizes, where the numpy restatement (oracle/fastpath.py) is too slow.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg load
 * this library (through oracle/fastpath_c.py); the product never does.
 *
 * What it restates (the reference rule it approximates is
 * argmax_j(log P[cur, j] / gamma - E[a, j]) over unvisited j, first of ties,
 * selection.py:143-155 / colony.py:126-152 of /root/reference/pkg/src/antbatch):
 *   - Philox2x32-10 (Random123), key = H(seed) + iteration;
 *     u = ((x >> 9) + 1/2) 2^-23 of the word x of
 *       dense stream (fpo_build_tours; slot s = the city j):
 *         counter (ant, (s >> 1) | step << 16), word s & 1
 *       sorted stream (fpo_build_tours_sorted; slot p = the entry's position
 *       in row cur of the row-sorted table):
 *         counter (ant, p | ((step + 1) >> 1) << 16), word (step + 1) & 1
 *   - start city: Lemire bound of word 0 of counter (ant, 0)
 *   - next = argmax_j fp32(W[cur, j] * u_slot(j)) over unvisited j with W > 0,
 *     lowest j on ties (a FULL scan: no pruning)
 *   - no W > 0 candidate left: the f64 fallback, argmax over unvisited j with
 *     v_j > 0 of log(v_j) * inv_gamma + log(u_j), v = A[cur, j]^alpha (* B[cur, j]),
 *     u_j keyed by the city in both streams;
 *     none either: city 0 when it is unvisited (numpy's argmax of an all -inf
 *     row, selection.py:152-155), else the "selector chose a visited city"
 *     failure (colony.py:149)
 * Compiled without FMA contraction or fast-math so every float operation is
 * one IEEE round-to-nearest, as on the device.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define PHILOX_M 0xD256D193u
#define PHILOX_W 0x9E3779B9u

uint32_t fpo_seed_hash32(uint64_t seed) {
  uint64_t f = seed;
  f ^= f >> 33;
  f *= 0xff51afd7ed558ccdull;
  f ^= f >> 33;
  f *= 0xc4ceb9fe1a85ec53ull;
  f ^= f >> 33;
  return (uint32_t)(f ^ (f >> 32));
}

static inline void philox2x32_10(uint32_t x0, uint32_t x1, uint32_t key, uint32_t out[2]) {
  for (int r = 0; r < 10; ++r) {
    const uint64_t prod = (uint64_t)PHILOX_M * x0;
    const uint32_t hi = (uint32_t)(prod >> 32), lo = (uint32_t)prod;
    x0 = hi ^ key ^ x1;
    x1 = lo;
    key += PHILOX_W;
  }
  out[0] = x0;
  out[1] = x1;
}

void fpo_philox(int count, const uint32_t *ctr2, const uint32_t *key, uint32_t *out2) {
  for (int t = 0; t < count; ++t) philox2x32_10(ctr2[2 * t], ctr2[2 * t + 1], key[t], out2 + 2 * t);
}

static inline float bits_to_uniform(uint32_t x) {
  /* (k + 1/2) 2^-23, k = x >> 9: exact in fp32 */
  return (float)(x >> 9) * 0x1p-23f + 0x1p-24f;
}

static inline uint32_t start_city(uint32_t ant, uint32_t key, uint32_t n) {
  uint32_t r[2];
  philox2x32_10(ant, 0u, key, r);
  return (uint32_t)(((uint64_t)r[0] * n) >> 32);
}

/* the raw words of cities 2q, 2q+1 at (step, ant) */
static inline void pair_words(uint32_t q, uint32_t step, uint32_t ant, uint32_t key, uint32_t r[2]) {
  philox2x32_10(ant, q | (step << 16), key, r);
}

/* the sorted stream's word of position p at (step, ant) */
static inline uint32_t pos_word(uint32_t p, uint32_t step, uint32_t ant, uint32_t key) {
  uint32_t r[2];
  philox2x32_10(ant, p | (((step + 1u) >> 1) << 16), key, r);
  return r[(step + 1u) & 1u];
}

/* the words of slots 2q, 2q+1 of either stream */
static inline void slot_words(int sorted, uint32_t q, uint32_t step, uint32_t ant, uint32_t key, uint32_t r[2]) {
  if (sorted) {
    r[0] = pos_word(2 * q, step, ant, key);
    r[1] = pos_word(2 * q + 1, step, ant, key);
  } else {
    pair_words(q, step, ant, key, r);
  }
}

static inline double fb_value(const double *a, double alpha, const double *b, size_t off) {
  /* numpy's scalar-power dispatch for the exponents the engine uses */
  const double x = a[off];
  double v;
  if (alpha == 1.0)
    v = x;
  else if (alpha == 2.0)
    v = x * x;
  else if (alpha == 0.0)
    v = 1.0;
  else if (alpha == 0.5)
    v = sqrt(x);
  else
    v = pow(x, alpha);
  return b ? v * b[off] : v;
}

/* One ant's tour.  Returns 0, or 2 when the selector is left without a city
 * (the reference's assertion).  scratch: n bytes. */
static int one_tour(const float *w, const uint16_t *idx, int n, int ldw, uint32_t key, uint32_t ant,
                    const double *fb_a, double fb_alpha, const double *fb_b, double inv_gamma, int32_t *tour,
                    uint8_t *seen, int64_t *fallbacks) {
  memset(seen, 0, (size_t)n);
  uint32_t cur = start_city(ant, key, (uint32_t)n);
  seen[cur] = 1;
  tour[0] = (int32_t)cur;
  for (uint32_t step = 1; step < (uint32_t)n; ++step) {
    const float *row = w + (size_t)cur * ldw;
    const uint16_t *irow = idx ? idx + (size_t)cur * ldw : NULL;
    float best = -1.0f;
    int bj = -1;
    /* slots s = 2q, 2q+1: cities (dense) or sorted positions (idx given) */
    for (int q = 0; 2 * q < n; ++q) {
      int c[2], jj[2];
      for (int e = 0; e < 2; ++e) {
        const int slot = 2 * q + e;
        jj[e] = slot < n ? (irow ? (int)irow[slot] : slot) : -1;
        c[e] = slot < n && !seen[jj[e]] && row[slot] > 0.0f;
      }
      if (!c[0] && !c[1]) continue;
      uint32_t r[2];
      slot_words(irow != NULL, (uint32_t)q, step, ant, key, r);
      for (int e = 0; e < 2; ++e) {
        if (!c[e]) continue;
        const float s = row[2 * q + e] * bits_to_uniform(r[e]);
        if (s > best || (s == best && jj[e] < bj)) best = s, bj = jj[e];
      }
    }
    if (bj < 0) { /* f64 fallback, then numpy's all -inf argmax */
      if (fallbacks) ++*fallbacks;
      double fbest = -INFINITY;
      if (fb_a != NULL) {
        for (int j = 0; j < n; ++j) {
          if (seen[j]) continue;
          const double v = fb_value(fb_a, fb_alpha, fb_b, (size_t)cur * n + j);
          if (!(v > 0.0)) continue;
          uint32_t r[2];
          pair_words((uint32_t)j >> 1, step, ant, key, r);
          const double s = log(v) * inv_gamma + log((double)bits_to_uniform(r[j & 1]));
          if (s > fbest) fbest = s, bj = j;
        }
      }
      if (bj < 0) {
        if (seen[0]) return 2;
        bj = 0;
      }
    }
    seen[bj] = 1;
    tour[step] = bj;
    cur = (uint32_t)bj;
  }
  return 0;
}

/* Tours of the given global ant ids.  Returns 0, or 2 and the first failing
 * row index in *fail_row.  fb_a may be NULL (no fallback source). */
static int build_tours_impl(const float *w, const uint16_t *idx, int n, int ldw, uint64_t seed, uint32_t iteration,
                            const int64_t *ants, int count, const double *fb_a, double fb_alpha,
                            const double *fb_b, double inv_gamma, int32_t *tours_out, int64_t *fallbacks,
                            int *fail_row) {
  const uint32_t key = fpo_seed_hash32(seed) + iteration;
  int rc = 0;
  int64_t fb_total = 0;
  *fail_row = -1;
#pragma omp parallel reduction(+ : fb_total)
  {
    uint8_t *seen = (uint8_t *)malloc((size_t)n);
#pragma omp for schedule(dynamic, 1)
    for (int a = 0; a < count; ++a) {
      int64_t fb = 0;
      const int r = one_tour(w, idx, n, ldw, key, (uint32_t)ants[a], fb_a, fb_alpha, fb_b, inv_gamma,
                             tours_out + (size_t)a * n, seen, &fb);
      fb_total += fb;
      if (r != 0) {
#pragma omp critical
        {
          if (rc == 0 || a < *fail_row) *fail_row = a;
          rc = r;
        }
      }
    }
    free(seen);
  }
  if (fallbacks) *fallbacks = fb_total;
  return rc;
}

/* Dense stream: w is the (n, ldw) fp32 table in city order. */
int fpo_build_tours(const float *w, int n, int ldw, uint64_t seed, uint32_t iteration, const int64_t *ants,
                    int count, const double *fb_a, double fb_alpha, const double *fb_b, double inv_gamma,
                    int32_t *tours_out, int64_t *fallbacks, int *fail_row) {
  return build_tours_impl(w, NULL, n, ldw, seed, iteration, ants, count, fb_a, fb_alpha, fb_b, inv_gamma,
                          tours_out, fallbacks, fail_row);
}

/* Sorted stream: (sw, si) is the row-sorted table (W values and their
 * cities, each row in the kernels' order); the uniform of an entry is keyed
 * by its position.  A full scan of every entry — no pruning. */
int fpo_build_tours_sorted(const float *sw, const uint16_t *si, int n, int ld, uint64_t seed, uint32_t iteration,
                           const int64_t *ants, int count, const double *fb_a, double fb_alpha, const double *fb_b,
                           double inv_gamma, int32_t *tours_out, int64_t *fallbacks, int *fail_row) {
  return build_tours_impl(sw, si, n, ld, seed, iteration, ants, count, fb_a, fb_alpha, fb_b, inv_gamma, tours_out,
                          fallbacks, fail_row);
}

/* Selection-level agreement along given tours (the device's): at every step
 * of every ant, with the ant's current city and visited set, compare the
 * recorded choice with
 *   [0] the product rule restated here (must agree everywhere),
 *   [1] the reference's log-domain rule log(P)/gamma + log(u) on the SAME
 *       23-bit uniforms, logw = log(P)/gamma as numpy computes it and
 *       log(u_k) from `logu_table` (numpy's log of the 2^23 values),
 *   [2] the log rule on REFINED uniforms u53 = (k + f) 2^-23, f a 53-bit
 *       fraction from an independent Philox stream (key ^ 0xA5A5A5A5): the
 *       same bin as u, so [2] measures what the 23-bit grid and fp32 W cost
 *       against a ~53-bit-resolution rule like the reference's (E from
 *       numpy's 53-bit ziggurat).
 * out[0] = selections compared, out[1..3] = mismatches of [0], [1], [2];
 * out[4] = steps of [2] where the refined winner had W below 2^-24 of the
 * recorded winner's W (the uniform floor's truncation). */
void fpo_count_mismatches(const float *w, const uint16_t *idx, int n, int ldw, const double *logw,
                          const double *logu_table, uint64_t seed, uint32_t iteration, const int64_t *ants,
                          int count, const int32_t *tours, int64_t *out) {
  const uint32_t key = fpo_seed_hash32(seed) + iteration;
  const uint32_t key2 = key ^ 0xA5A5A5A5u;
  int64_t sel = 0, mm_prod = 0, mm_log = 0, mm_ref = 0, trunc = 0;
#pragma omp parallel reduction(+ : sel, mm_prod, mm_log, mm_ref, trunc)
  {
    uint8_t *seen = (uint8_t *)malloc((size_t)n);
#pragma omp for schedule(dynamic, 1)
    for (int a = 0; a < count; ++a) {
      const uint32_t ant = (uint32_t)ants[a];
      const int32_t *tour = tours + (size_t)a * n;
      memset(seen, 0, (size_t)n);
      uint32_t cur = (uint32_t)tour[0];
      seen[cur] = 1;
      for (uint32_t step = 1; step < (uint32_t)n; ++step) {
        const float *row = w + (size_t)cur * ldw;
        const uint16_t *irow = idx ? idx + (size_t)cur * ldw : NULL;
        const double *lrow = logw + (size_t)cur * n;
        float pbest = -1.0f;
        int pj = -1, lj = 0, rj = 0; /* numpy: an all -inf row's argmax is 0 */
        double lbest = -INFINITY, rbest = -INFINITY;
        for (int q = 0; 2 * q < n; ++q) {
          uint32_t r[2], f[2];
          int any = 0;
          for (int e = 0; e < 2; ++e) {
            const int slot = 2 * q + e;
            any |= slot < n && !seen[irow ? irow[slot] : slot];
          }
          if (!any) continue;
          slot_words(irow != NULL, (uint32_t)q, step, ant, key, r);
          for (int e = 0; e < 2; ++e) {
            const int slot = 2 * q + e;
            if (slot >= n) continue;
            const int j = irow ? (int)irow[slot] : slot;
            if (seen[j]) continue;
            if (row[slot] > 0.0f) {
              const float s = row[slot] * bits_to_uniform(r[e]);
              if (s > pbest || (s == pbest && j < pj)) pbest = s, pj = j;
            }
            /* the log rule visits cities in slot order: first of ties = lowest j */
            const double ls = lrow[j] + logu_table[r[e] >> 9];
            if (ls > lbest || (ls == lbest && j < lj)) lbest = ls, lj = j;
            /* refined uniform: same bin (k = x >> 9), 53-bit position inside it */
            philox2x32_10(ant ^ 0x80000000u, (uint32_t)slot | (step << 16), key2, f);
            const uint64_t frac = (((uint64_t)f[0] << 32) | f[1]) >> 11;
            const double u53 = ((double)(r[e] >> 9) + (double)frac * 0x1p-53) * 0x1p-23;
            const double rs = lrow[j] + log(u53 > 0.0 ? u53 : 0x1p-80);
            if (rs > rbest || (rs == rbest && j < rj)) rbest = rs, rj = j;
          }
        }
        const int got = tour[step];
        ++sel;
        mm_prod += (pj >= 0 ? pj : got) != got;
        mm_log += lj != got;
        if (rj != got) {
          ++mm_ref;
          float wr = 0.0f, wg = 0.0f; /* W of the refined winner and of the recorded one */
          for (int slot = 0; slot < n; ++slot) {
            const int j = irow ? (int)irow[slot] : slot;
            if (j == rj) wr = row[slot];
            if (j == got) wg = row[slot];
          }
          if (wr < wg * 0x1p-24f) ++trunc;
        }
        seen[got] = 1;
        cur = (uint32_t)got;
      }
    }
    free(seen);
  }
  out[0] = sel;
  out[1] = mm_prod;
  out[2] = mm_log;
  out[3] = mm_ref;
  out[4] = trunc;
}

/* Scan-depth profile of the pruned sorted-table scan (k_construct_sorted's
 * stop rule): for the given ants, follow their tours (the same
 * rule as fpo_build_tours) over the row-sorted table (sw, si; rows descending
 * by the W bits above bit 16) and record, per step, how many 32-entry windows
 * the warp kernel reads before `bucket_ceiling(last W) < best`.  hist[w] (w <
 * hist_len - 1) counts steps that read w + 1 windows; the last bin collects
 * the rest.  Test / analysis infrastructure (sizing a head-only table). */
static inline float bucket_ceiling(float w) {
  uint32_t b;
  memcpy(&b, &w, 4);
  b |= 0xffffu;
  float r;
  memcpy(&r, &b, 4);
  return r;
}

void fpo_scan_profile(const float *sw, const uint16_t *si, int n, int ld, uint64_t seed, uint32_t iteration,
                      const int64_t *ants, int count, int64_t *hist, int hist_len) {
  const uint32_t key = fpo_seed_hash32(seed) + iteration;
  memset(hist, 0, sizeof(int64_t) * (size_t)hist_len);
#pragma omp parallel
  {
    uint8_t *seen = (uint8_t *)malloc((size_t)n);
    int64_t *h = (int64_t *)calloc((size_t)hist_len, sizeof(int64_t));
#pragma omp for schedule(dynamic, 1)
    for (int a = 0; a < count; ++a) {
      const uint32_t ant = (uint32_t)ants[a];
      memset(seen, 0, (size_t)n);
      uint32_t cur = start_city(ant, key, (uint32_t)n);
      seen[cur] = 1;
      for (uint32_t step = 1; step < (uint32_t)n; ++step) {
        const float *wr = sw + (size_t)cur * ld;
        const uint16_t *ir = si + (size_t)cur * ld;
        float best = -1.0f;
        int bj = -1, windows = 0;
        for (int base = 0; base < n; base += 32) {
          ++windows;
          float wl = 0.0f;
          for (int e = base; e < base + 32; ++e) {
            const float w = e < n ? wr[e] : 0.0f;
            wl = w;
            if (e >= n || !(w > 0.0f) || seen[ir[e]] || w < best) continue;
            const uint32_t j = ir[e];
            const float s = w * bits_to_uniform(pos_word((uint32_t)e, step, ant, key)); /* sorted position */
            if (s > best || (s == best && (int)j < bj)) best = s, bj = (int)j;
          }
          if (bucket_ceiling(wl) < best || !(wl > 0.0f)) break;
        }
        ++h[windows - 1 < hist_len - 1 ? windows - 1 : hist_len - 1];
        if (bj < 0) break; /* no candidate: the profile stops this ant */
        seen[bj] = 1;
        cur = (uint32_t)bj;
      }
    }
#pragma omp critical
    for (int i = 0; i < hist_len; ++i) hist[i] += h[i];
    free(h);
    free(seen);
  }
}
