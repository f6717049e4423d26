"""ORACLE (test infrastructure only): numpy restatement of the reference hot
path, one ACO iteration with IR / AdaIR selection.

Every function cites the reference code it restates (paths relative to
/root/reference/pkg/src/antbatch/).  It uses the same numpy primitives the
reference uses (Philox + SeedSequence streams, ziggurat standard_exponential,
pairwise sums, stable argsort), so on the same inputs it reproduces the
reference bit for bit; tests/test_oracle_golden.py pins that against the
golden vectors made by running the reference itself (tests/golden/).
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

TAU_MIN = 1e-12  # model.py:18


# ---------------------------------------------------------------------------
# keyed streams (rng.py:26-68)
# ---------------------------------------------------------------------------
def keyed_generator(seed: int, domain: int, *key: int) -> np.random.Generator:
    """Generator addressed by (seed, domain, *key) (rng.py:33-39)."""
    return np.random.Generator(np.random.Philox(
        np.random.SeedSequence(entropy=seed, spawn_key=(domain, *key))))


def exp_block(seed: int, iteration: int, step: int, m: int, n: int) -> np.ndarray:
    """(m, n) Exp(1) deviates of one step, domain 0 (rng.py:42-49)."""
    return keyed_generator(seed, 0, iteration, step).standard_exponential((m, n))


def start_block(seed: int, iteration: int, m: int, n: int) -> np.ndarray:
    """Start city per ant, domain 1 (rng.py:65-68, colony.py:72-78)."""
    return keyed_generator(seed, 1, iteration).integers(0, n, size=m, dtype=np.int64)


# ---------------------------------------------------------------------------
# selection (selection.py:48-75, 143-155)
# ---------------------------------------------------------------------------
def gamma(iteration: int, gamma_max: float = 1.5, gamma_min: float = 1.0, period: int = 1000) -> float:
    """Cosine annealing (selection.py:48-59)."""
    t = iteration % period
    return gamma_min + 0.5 * (gamma_max - gamma_min) * (1.0 + math.cos(math.pi * t / period))


def log_table(p: np.ndarray, g: float) -> np.ndarray:
    """log(p)/g, -inf where p == 0 (selection.py:62-75)."""
    out = np.full(p.shape, -np.inf)
    np.log(p, out=out, where=p > 0)
    return np.divide(out, g, out=out)


def lockstep_round(logw: np.ndarray, cur: np.ndarray, e: np.ndarray, visited: np.ndarray) -> np.ndarray:
    """argmax_j(logw[cur, j] - e[a, j]) with visited at -inf, first of ties
    (selection.py:143-155)."""
    scores = logw[cur] - e
    scores[visited] = -np.inf
    return scores.argmax(axis=1)


# ---------------------------------------------------------------------------
# transition matrix (colony.py:51-69)
# ---------------------------------------------------------------------------
class Underflow(ValueError):
    pass


def transition(tau: np.ndarray, eta: np.ndarray, alpha: float, beta: float) -> np.ndarray:
    """RowNorm(tau^alpha * eta^beta) with a zero diagonal (colony.py:51-69)."""
    with np.errstate(over="ignore", under="ignore", invalid="ignore"):
        w = np.power(tau, alpha) * np.power(eta, beta)
    idx = np.arange(w.shape[0])
    w[idx, idx] = 0.0
    z = w.sum(axis=1, keepdims=True)
    if not np.isfinite(z).all() or (z <= 0.0).any():
        raise Underflow("row normalizer is zero or non-finite")
    return w / z


# ---------------------------------------------------------------------------
# construction (colony.py:87-154)
# ---------------------------------------------------------------------------
def build_tours(p: np.ndarray, m: int, seed: int, iteration: int, g: float) -> np.ndarray:
    """m lockstep tours from the reference streams (colony.py:101-152)."""
    n = p.shape[0]
    logw = log_table(p, g)
    cur = start_block(seed, iteration, m, n)
    rows = np.arange(m)
    seen = np.zeros((m, n), dtype=bool)
    seen[rows, cur] = True
    tours = np.empty((m, n), dtype=np.int64)
    tours[:, 0] = cur
    for step in range(1, n):
        nxt = lockstep_round(logw, cur, exp_block(seed, iteration, step, m, n), seen)
        if seen[rows, nxt].any():  # colony.py:149
            raise AssertionError("selector chose a visited city")
        seen[rows, nxt] = True
        tours[:, step] = nxt
        cur = nxt
    return tours


def spin_round(p: np.ndarray, cur: np.ndarray, unvisited: np.ndarray, u: np.ndarray) -> np.ndarray:
    """Roulette spins of all ants at one step (rw_spin_block selection.py:102-127):
    first j with cumsum(P[cur] * unvisited)_j / total > u, else the last
    positive weight."""
    cdf = np.cumsum(p[cur] * unvisited, axis=1)
    cdf /= cdf[:, -1:].copy()
    nxt = (cdf > u[:, None]).argmax(axis=1)
    for a in np.flatnonzero(cdf[:, -1] <= u):
        nxt[a] = np.flatnonzero(p[cur[a]] * unvisited[a])[-1]
    return nxt


def spin_thresholds(seed: int, iteration: int, step: int, m: int, n: int) -> np.ndarray:
    """u = exp(-E[:, 0]) of the step's block (rng.step_uniforms rng.py:52-62)."""
    return np.exp(-exp_block(seed, iteration, step, m, n)[:, 0])


def build_tours_rw(p: np.ndarray, m: int, seed: int, iteration: int) -> np.ndarray:
    """m lockstep roulette-wheel tours (colony.py:113-141, RW branch)."""
    n = p.shape[0]
    cur = start_block(seed, iteration, m, n)
    rows = np.arange(m)
    unvisited = np.ones((m, n))
    unvisited[rows, cur] = 0.0
    tours = np.empty((m, n), dtype=np.int64)
    tours[:, 0] = cur
    for step in range(1, n):
        nxt = spin_round(p, cur, unvisited, spin_thresholds(seed, iteration, step, m, n))
        if (unvisited[rows, nxt] == 0.0).any():  # colony.py:149
            raise AssertionError("selector chose a visited city")
        unvisited[rows, nxt] = 0.0
        tours[:, step] = nxt
        cur = nxt
    return tours


def lengths(tours: np.ndarray, dist: np.ndarray) -> np.ndarray:
    """Closed-tour lengths, numpy pairwise row sums (model.py:292-295)."""
    return dist[tours, np.roll(tours, -1, axis=1)].sum(axis=1)


# ---------------------------------------------------------------------------
# pheromone update (pheromone.py:17-83)
# ---------------------------------------------------------------------------
def elite_ranks(costs: np.ndarray, k: int) -> np.ndarray:
    """Stable ascending argsort, first k (pheromone.py:17-25)."""
    return np.argsort(costs, kind="stable")[:k]


def deposit(tours: np.ndarray, costs: np.ndarray, n: int) -> np.ndarray:
    """Rank-ordered deposit of 1/cost on both orientations of every edge
    (pheromone.py:52-68)."""
    delta = np.zeros((n, n))
    for t, c in zip(tours, costs):
        inc = 1.0 / float(c)
        back = np.roll(t, 1)
        delta[t, back] += inc
        delta[back, t] += inc
    return delta


def evaporate(tau: np.ndarray, delta: np.ndarray, rho: float) -> np.ndarray:
    """max((1 - rho) tau + delta, TAU_MIN) (pheromone.py:71-83)."""
    return np.maximum((1.0 - rho) * tau + delta, TAU_MIN)


# ---------------------------------------------------------------------------
# one iteration (bench.py:199-206) and a run
# ---------------------------------------------------------------------------
@dataclass
class Config:
    m: int
    k: int
    alpha: float = 1.0
    beta: float = 2.0
    rho: float = 0.1
    q0_tau: float = 1.0
    selection: str = "adair"
    gamma_max: float = 1.5
    gamma_min: float = 1.0
    period: int = 1000
    seed: int = 0

    def gamma(self, iteration: int) -> float:
        if self.selection == "adair":
            return gamma(iteration, self.gamma_max, self.gamma_min, self.period)
        return 1.0


def initial_tau(n: int, q0: float) -> np.ndarray:
    """q0 off the diagonal, 0 on it (model.py:228-232)."""
    tau = np.full((n, n), float(q0))
    np.fill_diagonal(tau, 0.0)
    return tau


def iterate(tau: np.ndarray, p: np.ndarray, dist: np.ndarray, eta: np.ndarray, cfg: Config,
            iteration: int) -> dict:
    """construct -> elite -> deposit -> evaporate -> P (bench.py:199-206)."""
    n = dist.shape[0]
    if cfg.selection == "rw":
        tours = build_tours_rw(p, cfg.m, cfg.seed, iteration)
    else:
        tours = build_tours(p, cfg.m, cfg.seed, iteration, cfg.gamma(iteration))
    costs = lengths(tours, dist)
    order = elite_ranks(costs, cfg.k)
    delta = deposit(tours[order], costs[order], n)
    tau_next = evaporate(tau, delta, cfg.rho)
    p_next = transition(tau_next, eta, cfg.alpha, cfg.beta)
    return {"tours": tours, "costs": costs, "order": order, "delta": delta, "tau": tau_next, "p": p_next}


def run(dist: np.ndarray, eta: np.ndarray, cfg: Config, iterations: int) -> list[float]:
    """Best-so-far trace of a full run (bench.py:189-219)."""
    tau = initial_tau(dist.shape[0], cfg.q0_tau)
    p = transition(tau, eta, cfg.alpha, cfg.beta)
    best, trace = math.inf, []
    for it in range(iterations):
        out = iterate(tau, p, dist, eta, cfg, it)
        tau, p = out["tau"], out["p"]
        best = min(best, float(out["costs"].min()))
        trace.append(best)
    return trace


def instance_arrays(coords: np.ndarray) -> tuple[np.ndarray, np.ndarray]:
    """dist/eta of an unrounded Euclidean instance (model.py:82-97, 124-134)."""
    diff = coords[:, None, :] - coords[None, :, :]
    dist = np.sqrt((diff * diff).sum(axis=2))
    off = ~np.eye(len(coords), dtype=bool)
    eta = np.zeros_like(dist)
    np.divide(1.0, dist, out=eta, where=off)
    return dist, eta


class Degenerate(ValueError):
    """A zero off-diagonal distance (model.py:22-23, raised at model.py:86-91)."""


def _tsplib_weight(dx: float, dy: float, kind: str) -> float:
    """tsplib.distance (tsplib.py:198-215), scalar Python floats."""
    if kind == "EUC_2D":
        return float(int(math.sqrt(dx * dx + dy * dy) + 0.5))
    if kind == "CEIL_2D":
        return float(math.ceil(math.sqrt(dx * dx + dy * dy)))
    if kind == "ATT":
        r = math.sqrt((dx * dx + dy * dy) / 10.0)
        t = int(r + 0.5)
        return float(t + 1 if t < r else t)
    raise ValueError(f"edge weight type {kind!r} not supported")


def coord_instance(coords: np.ndarray, kind: str = "EXACT", lenient: bool = False):
    """dist/eta from coordinates: "EXACT" = euclidean_instance (model.py:124-134),
    else build_instance's pair loop (model.py:110-116) under a TSPLIB rule;
    then _instance_from_dist's eta / zero policy (model.py:82-97)."""
    pts = np.asarray(coords, dtype=np.float64)
    n = len(pts)
    if kind == "EXACT":
        diff = pts[:, None, :] - pts[None, :, :]
        dist = np.sqrt((diff * diff).sum(axis=2))
    else:
        dist = np.zeros((n, n))
        for i in range(n):
            for j in range(i + 1, n):
                dist[i, j] = dist[j, i] = _tsplib_weight(float(pts[i, 0] - pts[j, 0]),
                                                         float(pts[i, 1] - pts[j, 1]), kind)
    off = ~np.eye(n, dtype=bool)
    zero = (dist == 0.0) & off
    if zero.any() and not lenient:
        i, j = np.argwhere(zero)[0]
        raise Degenerate(f"cities {i} and {j} are at distance 0 (duplicate coordinates)")
    eta = np.zeros_like(dist)
    np.divide(1.0, np.where(zero, 1e-10, dist), out=eta, where=off)
    return dist, eta
