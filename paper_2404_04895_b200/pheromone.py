"""Drop-in replacements of the reference's elite pheromone update
(pheromone.py), executed on the B200 through libtaco.

``select_elite`` is a stable device radix argsort (pheromone.py:17-25),
``accumulate_increments`` builds the index-mapped deposit in elite rank order
(pheromone.py:52-68) and ``apply_update`` evaporates, deposits and floors
(pheromone.py:71-83); all three are bit-exact with the reference.  The Solver
fuses the last two with the transition-matrix rebuild in one row kernel.
"""

from __future__ import annotations

import numpy as np
import torch

from . import _device
from .model import TAU_MIN, InvalidPermutation, PheromoneState, check_permutations  # noqa: F401


def select_elite(batch, k: int) -> list[tuple[np.ndarray, float]]:
    """The k cheapest tours, ascending by cost, ties to the lower ant index."""
    if not 1 <= k <= batch.m:
        raise ValueError(f"k must be in [1, m={batch.m}], got {k}")
    dev = _device.device()
    costs = _device.upload(np.asarray(batch.costs, dtype=np.float64), dev)
    ws = _device.EliteWorkspace(costs.numel(), dev)
    order = _device.download(_device.elite_order(costs, ws))[:k]
    return [(batch.tours[a], float(batch.costs[a])) for a in order.tolist()]


def edge_index_matrix(tour) -> np.ndarray:
    """(n, 2) pairs (tour[t], tour[t-1]): the closed tour's n edges
    (pheromone.py:28-38).  Host helper of the tests; the device path builds
    the same pairs inside taco_elite_neighbors."""
    t = np.asarray(tour, dtype=np.int64)
    check_permutations(t, t.size)
    return np.stack((t, np.roll(t, 1)), axis=1)


def increment_matrix(tour, cost: float, n: int) -> np.ndarray:
    """Dense deposit of one tour: 1/cost on both orientations of each edge
    (pheromone.py:41-49); host helper of the tests."""
    idx = edge_index_matrix(tour)
    out = np.zeros((n, n))
    inc = 1.0 / cost
    out[idx[:, 0], idx[:, 1]] = inc
    out[idx[:, 1], idx[:, 0]] = inc
    return out


def _elite_arrays(elites, n: int) -> tuple[np.ndarray, np.ndarray]:
    tours = np.stack([np.asarray(t, dtype=np.int64) for t, _ in elites])
    check_permutations(tours, n)
    costs = np.array([float(c) for _, c in elites], dtype=np.float64)
    return tours, costs


def accumulate_increments(elites, n: int) -> np.ndarray:
    """Sum of the elites' increment matrices, accumulated in rank order from
    0.0 — bitwise equal to the reference's fancy += loop (pheromone.py:52-68)."""
    if not elites:
        raise ValueError("elites must be nonempty")
    tours, costs = _elite_arrays(elites, n)
    k = tours.shape[0]
    dev = _device.device()
    tours_t = _device.upload(tours, dev)
    costs_t = _device.upload(costs, dev)
    order = torch.arange(k, dtype=torch.int32, device=dev)
    nbr = torch.empty((n, k, 2), dtype=torch.int32, device=dev)  # city-major edge map
    inc = torch.empty(k, dtype=torch.float64, device=dev)
    _device.elite_neighbors(tours_t, order, costs_t, k, nbr, inc)
    delta = torch.empty((n, n), dtype=torch.float64, device=dev)
    _device.row_update(n, nbr=nbr, inc=inc, k=k, delta_out=delta)
    return _device.download(delta)


def apply_update(tau, delta, rho: float) -> PheromoneState:
    """tau' = max((1 - rho) * tau + delta, TAU_MIN) elementwise, diagonal
    included; iteration + 1 (pheromone.py:71-83)."""
    if not 0 <= rho < 1:
        raise ValueError(f"rho must be in [0, 1), got {rho}")
    t = np.asarray(tau.tau, dtype=np.float64)
    n = t.shape[0]
    dev = _device.device()
    tau_t = _device.upload(t, dev)
    delta_t = _device.upload(np.asarray(delta, dtype=np.float64), dev)
    out = torch.empty_like(tau_t)
    _device.row_update(n, tau_in=tau_t, tau_out=out, delta_in=delta_t, do_evap=True, keep=1.0 - rho)
    return PheromoneState(tau=_device.download(out), iteration=tau.iteration + 1)
