"""ORACLE (test infrastructure only): sampled CPU timing of the reference
algorithm (oracle.reference_port), used by bench.py as the CPU baseline and
as the `--impl reference` arm.

At the headline size one reference iteration takes ~10 minutes on one core
(n-1 = 2391 lockstep steps of ~240 ms), so the iteration time
is extrapolated from a bounded sample, exactly as BASELINE.md §2 specifies:

    T_iter = (n-1) * T_step + T(P) + T(logw) + T(lengths) + T(elite+deposit+update)

where T_step is the mean over `steps` consecutive construction steps (from
step 3 on) of exp_block + lockstep_round + the visited update
(colony.py:143-152), run on the real construction state of iteration 1.
"""

from __future__ import annotations

import os
import time

import numpy as np

from . import reference_port as ref


def synthetic_coords(n: int, seed: int = 0) -> np.ndarray:
    """U(0, 2000)^2 cities."""
    return np.random.default_rng(seed).uniform(0.0, 2000.0, (n, 2))


def sample_iteration(n: int, m: int, k: int, selection: str = "adair", seed: int = 0,
                     steps: int = 8, period: int = 1000) -> dict:
    """One sampled reference iteration; returns seconds per component and the
    extrapolated iteration time."""
    clock = time.perf_counter
    dist, eta = ref.instance_arrays(synthetic_coords(n, 0))  # the bench instance
    cfg = ref.Config(m=m, k=k, selection=selection, period=period, seed=seed)
    it = 1
    tau = ref.initial_tau(n, 1.0)

    t0 = clock()
    p = ref.transition(tau, eta, cfg.alpha, cfg.beta)
    t_p = clock() - t0

    rw = selection == "rw"
    t0 = clock()
    logw = None if rw else ref.log_table(p, cfg.gamma(it))
    t_logw = clock() - t0

    rows = np.arange(m)
    cur = ref.start_block(seed, it, m, n)
    seen = np.zeros((m, n), dtype=bool)
    seen[rows, cur] = True
    unvisited = (~seen).astype(np.float64)
    first = 3
    steps = max(1, min(steps, n - first))
    step_times = []
    for step in range(1, first + steps):
        t0 = clock()
        if rw:  # colony.py:127-134: thresholds + spins
            nxt = ref.spin_round(p, cur, unvisited, ref.spin_thresholds(seed, it, step, m, n))
            unvisited[rows, nxt] = 0.0
        else:
            e = ref.exp_block(seed, it, step, m, n)
            nxt = ref.lockstep_round(logw, cur, e, seen)
        seen[rows, nxt] = True
        cur = nxt
        dt = clock() - t0
        if step >= first:
            step_times.append(dt)
    t_step = float(np.mean(step_times))

    g = np.random.default_rng(seed + 1)
    tours = np.stack([g.permutation(n) for _ in range(m)])
    t0 = clock()
    costs = ref.lengths(tours, dist)
    t_costs = clock() - t0

    t0 = clock()
    order = ref.elite_ranks(costs, k)
    delta = ref.deposit(tours[order], costs[order], n)
    ref.evaporate(tau, delta, cfg.rho)
    t_update = clock() - t0

    t_iter = (n - 1) * t_step + t_p + t_logw + t_costs + t_update
    return {"t_iter": t_iter, "t_step": t_step, "steps_sampled": len(step_times),
            "t_p": t_p, "t_logw": t_logw, "t_costs": t_costs, "t_update": t_update}


def _worker(args) -> float:
    os.environ.setdefault("OMP_NUM_THREADS", "1")
    n, m, k, selection, seed, steps = args
    return sample_iteration(n, m, k, selection, seed, steps)["t_iter"]


def parallel_samples(n: int, m: int, k: int, selection: str, count: int, procs: int,
                     steps: int = 8) -> list[float]:
    """`count` sampled iteration times, `procs` independent replicas at a time
    (one colony per core: the reference is single-threaded numpy)."""
    import multiprocessing as mp

    ctx = mp.get_context("spawn")
    jobs = [(n, m, k, selection, 1000 + i, steps) for i in range(count)]
    with ctx.Pool(processes=procs) as pool:
        return list(pool.map(_worker, jobs))
