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
    """W = fp32(P^(1/g)) as the device builds it: exact conversion for g == 1,
    else fp32(exp2(log2(P)/g)) in f64 (k_row_update.cu selection_weight).
    numpy's log2/exp2 may differ from CUDA's by an ulp before the fp32
    rounding, so parity tests feed the device-built W to `build_tours`."""
    if g == 1.0:
        return p.astype(np.float32)
    with np.errstate(divide="ignore"):
        return np.exp2((1.0 / g) * np.log2(p)).astype(np.float32)


def build_tours(w: np.ndarray, seed: int, iteration: int, ants) -> np.ndarray:
    """Full-scan product-form construction for the given global ant ids:
    next = argmax_j W[cur, j] * u over unvisited j with W > 0, first of ties."""
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
        wr = w[cur]
        score = wr * u  # float32 x float32, round to nearest
        score[seen | (wr <= 0)] = np.float32(-1.0)
        nxt = score.argmax(axis=1)
        if (score[rows, nxt] < 0).any():
            raise AssertionError("selector chose a visited city")
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
