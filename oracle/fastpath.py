"""ORACLE (test infrastructure only): numpy restatement of the engine's device
stream and product-form selection rule.

The device rule replaces the reference's per-step Exp(1) block
(rng.py:42-49) with counter-addressed uniforms and evaluates
argmax(log P / gamma - E) (selection.py:143-155) in its product form
argmax(W * u), W = fp32(P^(1/gamma)).  This module restates that rule with
plain numpy so the CUDA kernels can be checked bit for bit, and also
evaluates the reference's log-domain rule on the same uniforms so the
product/log agreement can be counted.
"""

from __future__ import annotations

import numpy as np

PHILOX_M = 0xD256D193  # Random123 PHILOX_M2x32_0
PHILOX_W = 0x9E3779B9  # PHILOX_W32_0
MASK32 = 0xFFFFFFFF
MASK64 = 0xFFFFFFFFFFFFFFFF
RW_LOW = 0xFFFF  # counter low half of the RW thresholds (k_roulette.cu)


def philox2x32_10(ctr: np.ndarray, key) -> np.ndarray:
    """Random123 Philox2x32-10 on (N, 2) counters and (N,) or scalar keys
    (taco_common.cuh philox2x32_10)."""
    x0 = np.asarray(ctr[..., 0], dtype=np.uint64)
    x1 = np.asarray(ctr[..., 1], dtype=np.uint64)
    k = np.broadcast_to(np.asarray(key, dtype=np.uint64), x0.shape).copy()
    for _ in range(10):
        prod = x0 * np.uint64(PHILOX_M)
        hi, lo = prod >> np.uint64(32), prod & np.uint64(MASK32)
        x0, x1 = hi ^ k ^ x1, lo
        k = (k + np.uint64(PHILOX_W)) & np.uint64(MASK32)
    return np.stack([x0, x1], axis=-1).astype(np.uint32)


def seed_hash32(seed: int) -> int:
    """H(seed): xor-fold of the MurmurHash3 64-bit finalizer (taco_common.cuh)."""
    f = seed & MASK64
    f ^= f >> 33
    f = (f * 0xFF51AFD7ED558CCD) & MASK64
    f ^= f >> 33
    f = (f * 0xC4CEB9FE1A85EC53) & MASK64
    f ^= f >> 33
    return (f ^ (f >> 32)) & MASK32


def stream_key(seed: int, iteration: int) -> int:
    """Philox key of one iteration: H(seed) + iteration (mod 2^32)."""
    return (seed_hash32(seed) + iteration) & MASK32


def bits_to_uniform(x: np.ndarray) -> np.ndarray:
    """((x >> 9) + 0.5) * 2^-23 as float32 — exact, in (0, 1)."""
    k = (np.asarray(x, dtype=np.uint32) >> np.uint32(9)).astype(np.float32)
    return k * np.float32(2.0 ** -23) + np.float32(2.0 ** -24)


def uniforms(seed: int, iteration: int, step, ant, city) -> np.ndarray:
    """u(seed, iteration, step, ant, city); arrays broadcast together.
    Counter (ant, (city >> 1) | step << 16), word city & 1."""
    step, ant, city = np.broadcast_arrays(np.asarray(step, dtype=np.uint64),
                                          np.asarray(ant, dtype=np.uint64),
                                          np.asarray(city, dtype=np.uint64))
    ctr = np.stack([ant, ((city >> np.uint64(1)) | (step << np.uint64(16))) & np.uint64(MASK32)], axis=-1)
    words = philox2x32_10(ctr, stream_key(seed, iteration))
    pick = np.where((city & np.uint64(1)) == 1, words[..., 1], words[..., 0])
    return bits_to_uniform(pick)


def position_uniforms(seed: int, iteration: int, step, ant, pos) -> np.ndarray:
    """The sorted stream's u(seed, iteration, step, ant, sorted position).
    Counter (ant, pos | ((step + 1) >> 1) << 16), word (step + 1) & 1: one
    block serves a position at steps 2t - 1 and 2t."""
    step, ant, pos = np.broadcast_arrays(np.asarray(step, dtype=np.uint64),
                                         np.asarray(ant, dtype=np.uint64),
                                         np.asarray(pos, dtype=np.uint64))
    pair = (step + np.uint64(1)) >> np.uint64(1)
    ctr = np.stack([ant, (pos | (pair << np.uint64(16))) & np.uint64(MASK32)], axis=-1)
    words = philox2x32_10(ctr, stream_key(seed, iteration))
    pick = np.where((step & np.uint64(1)) == 1, words[..., 0], words[..., 1])
    return bits_to_uniform(pick)


def starts(seed: int, iteration: int, ants, n: int) -> np.ndarray:
    """Device start cities: Lemire bound of word 0 of counter (ant, 0)."""
    ants = np.asarray(ants, dtype=np.uint64)
    ctr = np.stack([ants, np.zeros_like(ants)], axis=-1)
    x = philox2x32_10(ctr, stream_key(seed, iteration))[..., 0].astype(np.uint64)
    return ((x * np.uint64(n)) >> np.uint64(32)).astype(np.int64)


def rw_uniform(seed: int, iteration: int, step, ant) -> np.ndarray:
    """Device RW threshold: 53 bits of Philox2x32-10 counter
    (ant, 0xffff | step << 16), as numpy's random():
    ((x >> 5) * 2^26 + (y >> 6)) / 2^53."""
    step = np.asarray(step, dtype=np.uint64).ravel()
    ant = np.asarray(ant, dtype=np.uint64).ravel()
    ctr = np.stack([ant, (np.uint64(RW_LOW) | (step << np.uint64(16))) & np.uint64(MASK32)], axis=-1)
    r = philox2x32_10(ctr, stream_key(seed, iteration)).astype(np.uint64)
    k = ((r[:, 0] >> np.uint64(5)) << np.uint64(26)) | (r[:, 1] >> np.uint64(6))
    return k.astype(np.float64) * 2.0**-53


def rw_tours(p: np.ndarray, seed: int, iteration: int, ants) -> np.ndarray:
    """Device-stream roulette-wheel tours: the reference's spin rule
    (rw_spin_block selection.py:102-127 — sequential cumsum, strict >, the
    last-positive fallback) on the device thresholds and start cities."""
    n = p.shape[0]
    ants = np.asarray(ants)
    m = len(ants)
    rows = np.arange(m)
    cur = starts(seed, iteration, ants, n)
    unvisited = np.ones((m, n))
    unvisited[rows, cur] = 0.0
    tours = np.empty((m, n), dtype=np.int64)
    tours[:, 0] = cur
    for step in range(1, n):
        u = rw_uniform(seed, iteration, np.full(m, step), ants)
        cdf = np.cumsum(p[cur] * unvisited, axis=1)
        cdf /= cdf[:, -1:].copy()
        nxt = (cdf > u[:, None]).argmax(axis=1)
        for a in np.flatnonzero(cdf[:, -1] <= u):
            nxt[a] = np.flatnonzero(p[cur[a]] * unvisited[a])[-1]
        unvisited[rows, nxt] = 0.0
        tours[:, step] = nxt
        cur = nxt
    return tours


def selection_table(p: np.ndarray, g: float) -> np.ndarray:
    """W = fp32(2^-e_i P^(1/g)) as the device builds it (taco_common.cuh
    selection_weight): P^(1/g) is the exact value for g == 1, else
    exp2(log2(P)/g) in f64; e_i = ilogb of row i's largest P^(1/g), so the
    row maximum lands in [1, 2); entries below FLT_MIN after scaling are 0.
    numpy's log2/exp2 may differ from CUDA's by an ulp before the fp32
    rounding, so parity tests feed the device-built W to `build_tours`."""
    p = np.asarray(p, dtype=np.float64)
    with np.errstate(divide="ignore"):
        x = p.copy() if g == 1.0 else np.exp2((1.0 / g) * np.log2(p))
        pmax = p.max(axis=1)
        xmax = pmax if g == 1.0 else np.exp2((1.0 / g) * np.log2(pmax))
    e = np.where((xmax > 0) & np.isfinite(xmax), np.frexp(xmax)[1] - 1, 0)
    e = np.clip(e, -1000, 1000)
    w = (x * np.ldexp(1.0, -e)[:, None]).astype(np.float32)
    w[w < np.float32(2.0**-126)] = 0.0
    return w


def _fallback_value(a: np.ndarray, alpha: float, b) -> np.ndarray:
    """v = A^alpha (* B) with numpy's scalar-power dispatch (the kernels'
    numpy_scalar_power)."""
    v = a if alpha == 1.0 else (a * a if alpha == 2.0 else np.power(a, alpha))
    return v if b is None else v * b


def build_tours(w: np.ndarray, seed: int, iteration: int, ants, fallback=None, inv_gamma: float = 1.0) -> np.ndarray:
    """Full-scan product-form construction for the given global ant ids:
    next = argmax_j W[cur, j] * u over unvisited j with W > 0, first of ties.

    No W > 0 candidate left: argmax over unvisited j with v_j > 0 of
    log(v_j) * inv_gamma + log(u_j) in f64, v = A[cur]^alpha (* B[cur]) with
    fallback = (A, alpha, B or None); none either (or no source): city 0
    when unvisited — numpy's argmax of an all -inf row (selection.py:152-155)
    — else the reference's assertion (colony.py:149)."""
    n = w.shape[0]
    ants = np.asarray(ants, dtype=np.int64)
    a = ants.size
    rows = np.arange(a)
    cur = starts(seed, iteration, ants, n)
    seen = np.zeros((a, n), dtype=bool)
    seen[rows, cur] = True
    tours = np.empty((a, n), dtype=np.int64)
    tours[:, 0] = cur
    cities = np.arange(n, dtype=np.uint64)
    for step in range(1, n):
        u = uniforms(seed, iteration, step, ants[:, None], cities[None, :])
        wr = w[cur][:, :n]
        score = wr * u  # float32 x float32, round to nearest
        score[seen | (wr <= 0)] = np.float32(-1.0)
        nxt = score.argmax(axis=1)
        for r in np.flatnonzero(score[rows, nxt] < 0):  # no W > 0 candidate
            pick = -1
            if fallback is not None:
                v = _fallback_value(fallback[0][cur[r]], fallback[1],
                                    None if fallback[2] is None else fallback[2][cur[r]])
                ok = ~seen[r] & (v > 0)
                if ok.any():
                    with np.errstate(divide="ignore"):
                        s = np.log(v) * inv_gamma + np.log(u[r].astype(np.float64))
                    s[~ok] = -np.inf
                    pick = int(s.argmax())
            if pick < 0:
                if seen[r, 0]:
                    raise AssertionError("selector chose a visited city")
                pick = 0
            nxt[r] = pick
        seen[rows, nxt] = True
        tours[:, step] = nxt
        cur = nxt
    return tours


def build_tours_sorted(sw: np.ndarray, si: np.ndarray, seed: int, iteration: int, ants, fallback=None,
                       inv_gamma: float = 1.0) -> np.ndarray:
    """The sorted stream (the kernels that scan the row-sorted table): the
    full-scan product rule over the table entries, the uniform of an entry
    keyed by its POSITION in the current row (slot) instead of its city.
    sw / si: (n, >= n) sorted values and cities; fallback as build_tours
    (its uniforms keyed by city)."""
    n = sw.shape[0]
    ants = np.asarray(ants, dtype=np.int64)
    a = ants.size
    rows = np.arange(a)
    cur = starts(seed, iteration, ants, n)
    seen = np.zeros((a, n), dtype=bool)
    seen[rows, cur] = True
    tours = np.empty((a, n), dtype=np.int64)
    tours[:, 0] = cur
    slots = np.arange(n, dtype=np.uint64)
    for step in range(1, n):
        u = position_uniforms(seed, iteration, step, ants[:, None], slots[None, :])
        wr = sw[cur][:, :n]
        jr = si[cur][:, :n].astype(np.int64)
        score = wr * u
        score[np.take_along_axis(seen, jr, axis=1) | (wr <= 0)] = np.float32(-1.0)
        # argmax over entries; ties to the lowest city
        best = score.max(axis=1)
        jr_masked = np.where(score == best[:, None], jr, n)
        nxt = jr_masked.min(axis=1)
        for r in np.flatnonzero(best < 0):  # no W > 0 candidate: the city-keyed fallback
            pick = -1
            if fallback is not None:
                v = _fallback_value(fallback[0][cur[r]], fallback[1],
                                    None if fallback[2] is None else fallback[2][cur[r]])
                ok = ~seen[r] & (v > 0)
                if ok.any():
                    uc = uniforms(seed, iteration, step, ants[r], np.arange(n, dtype=np.uint64))
                    with np.errstate(divide="ignore"):
                        sc = np.log(v) * inv_gamma + np.log(uc.astype(np.float64))
                    sc[~ok] = -np.inf
                    pick = int(sc.argmax())
            if pick < 0:
                if seen[r, 0]:
                    raise AssertionError("selector chose a visited city")
                pick = 0
            nxt[r] = pick
        seen[rows, nxt] = True
        tours[:, step] = nxt
        cur = nxt
    return tours


def log_rule_tours(p: np.ndarray, g: float, seed: int, iteration: int, ants) -> np.ndarray:
    """The reference's log-domain rule argmax(log P / g - E) (selection.py:
    143-155) driven by the DEVICE uniforms, E = -log(float64(u)).  Counting
    where it differs from `build_tours` measures the product/log agreement."""
    n = p.shape[0]
    logw = np.full(p.shape, -np.inf)
    np.log(p, out=logw, where=p > 0)
    logw /= g
    ants = np.asarray(ants, dtype=np.int64)
    a = ants.size
    rows = np.arange(a)
    cur = starts(seed, iteration, ants, n)
    seen = np.zeros((a, n), dtype=bool)
    seen[rows, cur] = True
    tours = np.empty((a, n), dtype=np.int64)
    tours[:, 0] = cur
    cities = np.arange(n, dtype=np.uint64)
    for step in range(1, n):
        u = uniforms(seed, iteration, step, ants[:, None], cities[None, :]).astype(np.float64)
        s = logw[cur] + np.log(u)
        s[seen] = -np.inf
        nxt = s.argmax(axis=1)
        seen[rows, nxt] = True
        tours[:, step] = nxt
        cur = nxt
    return tours


def pairwise_sum(values) -> float:
    """numpy's pairwise summation order for a contiguous float64 vector
    (numpy/_core/src/umath/loops_utils.h.src: pairwise_sum)."""
    a = [float(v) for v in values]

    def rec(lo: int, n: int) -> float:
        if n < 8:
            res = 0.0
            for i in range(lo, lo + n):
                res += a[i]
            return res
        if n <= 128:
            r = a[lo:lo + 8]
            i = 8
            while i < n - (n % 8):
                for j in range(8):
                    r[j] += a[lo + i + j]
                i += 8
            res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]))
            while i < n:
                res += a[lo + i]
                i += 1
            return res
        n2 = n // 2
        n2 -= n2 % 8
        return rec(lo, n2) + rec(lo + n2, n - n2)

    return rec(0, len(a))
