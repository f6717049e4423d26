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
import sys
import time

import numpy as np

from . import reference_port as ref

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
# the UNMODIFIED reference package, installed by
#   pip install --no-index --no-build-isolation --no-deps --target baseline/_ref <copy of /root/reference/pkg>
# (git-ignored; it travels to the GPU box with the repo snapshot)
REF_PATH = os.path.join(ROOT, "baseline", "_ref")


def reference_available() -> bool:
    return os.path.isfile(os.path.join(REF_PATH, "antbatch", "__init__.py"))


def _antbatch():
    """The installed reference package (baseline/_ref/antbatch), never a copy
    in this repo."""
    if REF_PATH not in sys.path:
        sys.path.insert(0, REF_PATH)
    import antbatch

    if not os.path.abspath(antbatch.__file__).startswith(REF_PATH):
        raise ImportError(f"antbatch resolved to {antbatch.__file__}, not {REF_PATH}")
    return antbatch


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


def sample_iteration_reference(n: int, m: int, k: int, selection: str = "adair", seed: int = 0,
                               steps: int = 8, period: int = 1000) -> dict:
    """One sampled iteration of the UNMODIFIED reference (baseline/_ref/antbatch),
    through its own functions and in colony.construct_tours' order
    (colony.py:101-152): compute_probability_matrix, scaled_log_weights, then
    `steps` lockstep rounds of rng.step_exponentials + argmax_select_block +
    the visited assert (rng.step_uniforms + rw_spin_block for RW) on the real
    construction state of iteration 1, then batch_costs, select_elite,
    accumulate_increments and apply_update; extrapolated as in
    sample_iteration."""
    ab = _antbatch()
    from antbatch import colony, model, pheromone, rng
    from antbatch import selection as sel

    clock = time.perf_counter
    inst = model.euclidean_instance(synthetic_coords(n, 0))  # the bench instance
    params = model.AcoParams(m=m, k=k, selection=model.Selection(selection), seed=seed,
                             gamma_schedule=model.GammaSchedule(1.5, 1.0, period))
    it = 1
    tau = model.PheromoneState.initial(n, params.q0_tau)
    t0 = clock()
    prob = colony.compute_probability_matrix(tau, inst, params)
    t_p = clock() - t0
    rw = params.selection is model.Selection.RW
    gamma = sel.gamma_at(it, params.gamma_schedule) if params.selection is model.Selection.ADAIR else 1.0
    t0 = clock()
    logw = None if rw else sel.scaled_log_weights(prob.p, gamma)
    t_logw = clock() - t0

    rows = np.arange(m)
    current = colony.init_starts(m, n, rng.stream(seed, rng.DOMAIN_START, it))
    visited = np.zeros((m, n), dtype=bool)
    visited[rows, current] = True
    unvisited_f = np.ones((m, n))
    unvisited_f[rows, current] = 0.0
    scores = np.empty((m, n))
    first = 3
    steps = max(1, min(steps, n - first))
    step_times = []
    for step in range(1, first + steps):
        t0 = clock()
        if rw:
            u = rng.step_uniforms(seed, it, step, m, n)
            nxt = sel.rw_spin_block(prob.p, current, unvisited_f, u, scores)
            unvisited_f[rows, nxt] = 0.0
        else:
            e_block = rng.step_exponentials(seed, it, step, m, n)
            nxt = sel.argmax_select_block(logw, current, e_block, visited, scores)
        assert not visited[rows, nxt].any(), "selector chose a visited city"
        current = nxt
        visited[rows, current] = True
        dt = clock() - t0
        if step >= first:
            step_times.append(dt)
    t_step = float(np.mean(step_times))

    g = np.random.default_rng(seed + 1)
    tours = np.stack([g.permutation(n) for _ in range(m)])
    t0 = clock()
    costs = model.batch_costs(tours, inst)
    t_costs = clock() - t0
    batch = model.TourBatch(tours=tours, costs=costs)
    t0 = clock()
    elites = pheromone.select_elite(batch, k)
    delta = pheromone.accumulate_increments(elites, n)
    pheromone.apply_update(tau, delta, params.rho)
    t_update = clock() - t0
    t_iter = (n - 1) * t_step + t_p + t_logw + t_costs + t_update
    return {"t_iter": t_iter, "t_step": t_step, "steps_sampled": len(step_times), "t_p": t_p,
            "t_logw": t_logw, "t_costs": t_costs, "t_update": t_update, "antbatch": ab.__version__}


def run_reference_as_is(n: int, m: int, k: int, selection: str, seed: int, iterations: int,
                        period: int) -> dict:
    """The reference's own run_experiment (bench.py:171-238), unmodified, on the
    bench instance: its per-iteration wall clock (the warm-up iteration
    excluded, bench.py:228) — for configs small enough to run whole (C1)."""
    _antbatch()
    from antbatch import bench, model

    inst = model.euclidean_instance(synthetic_coords(n, 0))
    params = model.AcoParams(m=m, k=k, selection=model.Selection(selection), seed=seed, max_iters=iterations,
                             gamma_schedule=model.GammaSchedule(1.5, 1.0, period))
    cfg = bench.ExperimentConfig(params=params, synthetic=bench.SyntheticSpec(n=n, seed=0, kind="uniform"))
    _, summaries = bench.run_experiment(cfg, inst=inst)
    return {"t_iter": summaries[0].mean_ms_per_iter * 1e-3, "iterations": summaries[0].iterations_run,
            "best": summaries[0].final_best_cost}


def _worker(args) -> float:
    os.environ.setdefault("OMP_NUM_THREADS", "1")
    n, m, k, selection, seed, steps, period, kind = args
    if kind == "as-is":
        return run_reference_as_is(n, m, k, selection, seed, steps, period)["t_iter"]
    if kind == "reference":
        return sample_iteration_reference(n, m, k, selection, seed, steps, period)["t_iter"]
    return sample_iteration(n, m, k, selection, seed, steps, period)["t_iter"]


def parallel_samples(n: int, m: int, k: int, selection: str, count: int, procs: int,
                     steps: int = 8, period: int = 1000, kind: str = "port") -> list[float]:
    """`count` iteration times, `procs` independent replicas at a time (one
    colony per core: the reference is single-threaded numpy).  kind: "port"
    (sample_iteration), "reference" (sample_iteration_reference) or "as-is"
    (run_reference_as_is, `steps` = iterations)."""
    import multiprocessing as mp

    ctx = mp.get_context("spawn")
    jobs = [(n, m, k, selection, 1000 + i, steps, period, kind) for i in range(count)]
    with ctx.Pool(processes=procs) as pool:
        return list(pool.map(_worker, jobs))
