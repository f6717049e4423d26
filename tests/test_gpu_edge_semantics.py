"""GPU: the reference's edge semantics through the drop-ins and the Solver.

* argmax_select_block (selection.py:143-155): bit-exact scores and choices,
  including ties (first index) and all -inf rows (index 0).
* scaled_log_weights (selection.py:62-75): CUDA's log is within 1 ulp of
  numpy's SIMD log (they differ on ~3e-5 of inputs), so log / gamma
  is within 2 ulp (measured: 0.5% of entries differ, by 1-2 ulp).
* All-zero candidate rows (P == 0 for every unvisited city): numpy's argmax
  of an all -inf row is city 0, which the reference takes when it is
  unvisited; when city 0 is already visited it asserts (colony.py:149).
* gamma < 1 (AdaIR "greedier than IR"): P^(1/gamma) leaves fp32's range; the
  construction kernels decide such steps by the f64 fallback, exactly as the
  C oracle restates it.
* Fail-stop: a construction failure leaves tau as it was before the failing
  iteration (the reference raises inside construct_tours).
"""

import numpy as np
import pytest
import torch

import paper_2404_04895_b200 as taco
from paper_2404_04895_b200 import _device, _lib
from conftest import euclid
from oracle import fastpath, fastpath_c, reference_port as ref

pytestmark = pytest.mark.gpu


def _ulps(a: np.ndarray, b: np.ndarray) -> np.ndarray:
    """|a - b| in units of the last place (finite, same-sign doubles)."""
    ia, ib = a.view(np.int64), b.view(np.int64)
    return np.abs(ia - ib)


def test_argmax_select_block_is_bit_exact():
    g = np.random.default_rng(5)
    n, m = 300, 97
    logw = np.log(g.uniform(0.0, 1.0, (n, n))) / 1.3
    logw[g.uniform(size=(n, n)) < 0.05] = -np.inf  # P == 0 entries
    cur = g.integers(0, n, m)
    e = g.standard_exponential((m, n))
    vis = g.uniform(size=(m, n)) < 0.4
    vis[3] = True  # all visited: argmax of all -inf is 0
    vis[4] = False
    logw[cur[4]] = -np.inf  # all -inf by weight
    e[5] = 1.0
    logw[cur[5], 10] = logw[cur[5], 20] = 50.0  # an exact tie: the lower index
    vis[5, 10] = vis[5, 20] = False
    scores = np.empty((m, n))
    got = taco.argmax_select_block(logw, cur, e, vis, scores)
    want_scores = np.empty((m, n))
    np.take(logw, cur, axis=0, out=want_scores)
    np.subtract(want_scores, e, out=want_scores)
    np.copyto(want_scores, -np.inf, where=vis)
    assert np.array_equal(scores, want_scores)
    assert np.array_equal(got, want_scores.argmax(axis=1))
    assert np.array_equal(got, ref.lockstep_round(logw, cur, e, vis))
    assert got[3] == 0 and got[4] == 0 and got[5] == 10


def test_scaled_log_weights_within_two_ulp(golden):
    g = np.random.default_rng(2)
    p = golden["int12_adair/s0/it1/p"]
    big = g.uniform(0.0, 1.0, (257, 300))
    big[big < 0.02] = 0.0
    for arr in (p, big, np.array([0.0, 1.0, 1e-300, 5e-324, 0.5])):
        for gamma in (1.0, 1.5, 1.4268, 0.3):
            got = taco.scaled_log_weights(arr, gamma)
            want = ref.log_table(np.asarray(arr, dtype=np.float64), gamma)
            assert np.array_equal(np.isneginf(got), np.isneginf(want))
            fin = np.isfinite(want)
            d = _ulps(got[fin], want[fin])
            assert d.max() <= 2 and (d != 0).mean() < 1e-2
    with pytest.raises(ValueError):
        taco.scaled_log_weights(p, 0.0)


def _two_clusters(n: int = 40):
    """Two clusters at infinite distance: P == 0 between them."""
    pts = np.random.default_rng(3).uniform(0, 100, (n, 2))
    inst = taco.euclidean_instance(pts)
    dist = inst.dist.copy()
    side = np.arange(n) >= n // 2
    dist[side[:, None] != side[None, :]] = np.inf
    return taco.instance_from_distances(dist), side


def _seed_with_starts(n, m, want_side, side, it=0):
    for seed in range(1000):
        st = fastpath.starts(seed, it, np.arange(m), n)
        if (side[st] == want_side).all():
            return seed
    raise AssertionError("no seed")


@pytest.mark.parametrize("variant,env", [("sorted", {}), ("sorted", {"TACO_SORTED_KERNEL": "g8e2"}),
                                         ("dense", {})])
def test_all_zero_candidates_take_city_zero_like_numpy(variant, env, monkeypatch):
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    inst, side = _two_clusters()
    n, m = inst.n, 3
    seed = _seed_with_starts(n, m, True, side)  # every ant starts in the far cluster
    params = taco.AcoParams(m=m, k=1, selection="ir", seed=seed)
    p = taco.compute_probability_matrix(taco.PheromoneState.initial(n, 1.0), inst, params)
    assert (p.p[np.ix_(side, ~side)] == 0).all()
    batch = taco.construct_tours(p, inst, params, 0, variant=variant)
    # the far cluster first, then city 0 (argmax of an all -inf row), then the rest
    half = n // 2
    assert side[batch.tours[:, :half]].all()
    assert (batch.tours[:, half] == 0).all()
    dev = _device.device()
    t = _device.SelectionTables(n, dev, dense=True, sorted_=True)
    _device.selection_table_from_p(_device.upload(p.p, dev), 1.0, t)
    if variant == "sorted":
        want = fastpath_c.build_tours_sorted(t.sw.cpu().numpy(), t.si.cpu().numpy(), seed, 0, np.arange(m), n=n,
                                             fallback=(p.p, 1.0, None))
    else:
        want = fastpath_c.build_tours(t.w.cpu().numpy(), seed, 0, np.arange(m), n=n, fallback=(p.p, 1.0, None))
    assert np.array_equal(batch.tours, want)
    # the reference's own rule and streams agree on the semantics
    ref_tours = ref.build_tours(p.p, m, seed, 0, 1.0) if side[ref.start_block(seed, 0, m, n)].all() else None
    if ref_tours is not None:
        assert (ref_tours[:, half] == 0).all()
    # an ant that starts in city 0's cluster runs out with 0 visited: the assertion
    seed2 = _seed_with_starts(n, m, False, side)
    with pytest.raises(AssertionError, match="selector chose a visited city"):
        taco.construct_tours(p, inst, taco.AcoParams(m=m, k=1, selection="ir", seed=seed2), 0, variant=variant)


def test_solver_construction_failure_leaves_tau_where_the_reference_raised():
    inst, side = _two_clusters()
    n, m = inst.n, 4
    seed = _seed_with_starts(n, m, True, side)  # iteration 0 completes ...
    for it in range(1, 50):  # ... and a later iteration has an ant starting next to city 0
        if not side[fastpath.starts(seed, it, np.arange(m), n)].all():
            break
    params = taco.AcoParams(m=m, k=1, selection="ir", seed=seed)
    s = taco.Solver(inst, params, graph=False)
    for _ in range(it):
        s.step()
    tau_before = s.pheromone().tau
    best_before = s.best()
    with pytest.raises(AssertionError, match="selector chose a visited city"):
        s.step()
    assert np.array_equal(s.pheromone().tau, tau_before)
    assert s.best()[1] == best_before[1] and np.array_equal(s.best()[0], best_before[0])


# (variant, m, env): warp kernel MODE 4 (<= 16 ants per SM, the default at
# m = 64) and MODE 1, each with the byte / bit-map visited set, MODE 2 (> 32
# ants per SM: rebuilt by the follow-up k_rebuild_stalled), the lane-group
# kernels and the dense kernel
FALLBACK_CASES = [
    ("sorted", 64, {}),
    ("sorted", 64, {"TACO_SORTED_VIS": "bits"}),
    ("sorted", 64, {"TACO_SORTED_MODE": "1"}),
    ("sorted", 64, {"TACO_SORTED_MODE": "1", "TACO_SORTED_VIS": "bits"}),
    ("sorted", 6000, {"TACO_SORTED_KERNEL": "warp"}),
    ("sorted", 6000, {"TACO_SORTED_KERNEL": "warp", "TACO_SORTED_VIS": "bits"}),
    ("sorted", 64, {"TACO_SORTED_KERNEL": "g8e2"}),
    ("sorted", 64, {"TACO_SORTED_KERNEL": "g4e4"}),
    ("dense", 64, {}),
]


@pytest.mark.parametrize("variant,m,env", FALLBACK_CASES)
def test_gamma_below_one_uses_the_f64_fallback(variant, m, env, monkeypatch):
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    n, it = 400, 9
    # two clusters 10^4 apart: across them P is ~1e-6 of the row's best, so
    # P^(1/gamma) ~ 1e-50 of it — zero in fp32 — and the first step out of a
    # cluster is decided by the fallback
    g = np.random.default_rng(1)
    pts = g.uniform(0.0, 10.0, (n, 2))
    pts[n // 2:] += 1e4
    inst = taco.euclidean_instance(pts)
    tau = g.uniform(0.05, 3.0, (n, n))
    p = ref.transition((tau + tau.T) / 2, inst.eta, 1.0, 2.0)
    params = taco.AcoParams(m=m, k=4, selection="adair", seed=21,
                            gamma_schedule=taco.GammaSchedule(1.0, 0.1, 10))
    gamma = taco.gamma_at(it, params.gamma_schedule)  # ~0.12: P^(1/gamma) ~ P^8
    assert gamma < 0.15
    batch = taco.construct_tours(taco.ProbabilityMatrix(p), inst, params, it, variant=variant)
    assert (np.sort(batch.tours, axis=1) == np.arange(n)).all()
    # the device table (fp32, row-scaled, zero below 2^-126 of the row's best)
    dev = _device.device()
    t = _device.SelectionTables(n, dev, dense=True, sorted_=True)
    _device.selection_table_from_p(_device.upload(p, dev), 1.0 / gamma, t)
    w = t.w[:, :n].cpu().numpy()
    assert (w == 0).sum() > n  # far outside fp32's range relative to the row best
    assert np.abs(w.astype(np.float64) - fastpath.selection_table(p, gamma)).max() <= 2.0**-22
    ants = np.arange(m) if m <= 64 else np.unique(np.linspace(0, m - 1, 64).astype(np.int64))
    fb = dict(fallback=(p, 1.0, None), inv_gamma=1.0 / gamma)
    if variant == "sorted":
        want = fastpath_c.build_tours_sorted(t.sw.cpu().numpy(), t.si.cpu().numpy(), 21, it, ants, n=n, **fb)
    else:
        want = fastpath_c.build_tours(t.w.cpu().numpy(), 21, it, ants, n=n, **fb)
    assert fastpath_c.build_tours.last_fallbacks > 0  # the fallback really decided steps
    assert np.array_equal(batch.tours[ants], want)
    assert np.array_equal(batch.costs[ants], ref.lengths(want, inst.dist))


def test_solver_runs_gamma_below_one():
    n, m = 200, 48
    inst = euclid(12, n)
    params = taco.AcoParams(m=m, k=5, selection="adair", seed=4,
                            gamma_schedule=taco.GammaSchedule(1.0, 0.1, 6))
    for graph in (False, True):
        s = taco.Solver(inst, params, graph=graph, graph_warmup=1)
        tour, length = s.run(12)
        assert sorted(tour.tolist()) == list(range(n))
        assert length == taco.tour_cost(tour, inst)
        b = s.last_batch()
        assert (np.sort(b.tours, axis=1) == np.arange(n)).all()
    # graph replay (device 1/gamma of the iteration) == eager, bit for bit
    a = taco.Solver(inst, params, graph=False)
    g = taco.Solver(inst, params, graph=True, graph_warmup=1)
    assert a.run(9)[1] == g.run(9)[1]
    assert np.array_equal(a.pheromone().tau, g.pheromone().tau)


def test_row_scaled_table_keeps_tours_of_the_unscaled_rule():
    """gamma >= 1: the power-of-two row scale changes no choice — tours equal
    the full-scan rule on the unscaled fp32(P^(1/gamma)) table."""
    n, m = 500, 40
    inst = euclid(13, n)
    tau = np.random.default_rng(2).uniform(0.05, 3.0, (n, n))
    p = ref.transition((tau + tau.T) / 2, inst.eta, 1.0, 2.0)
    for gamma in (1.0, 1.5):
        params = taco.AcoParams(m=m, k=4, selection="adair", seed=8,
                                gamma_schedule=taco.GammaSchedule(gamma, gamma, 10))
        batch = taco.construct_tours(taco.ProbabilityMatrix(p), inst, params, 2)
        dev = _device.device()
        t = _device.SelectionTables(n, dev, dense=True, sorted_=True)
        _device.selection_table_from_p(_device.upload(p, dev), 1.0 / gamma, t)
        w = t.w[:, :n].cpu().numpy()
        rowmax = w.max(axis=1)
        assert ((rowmax >= 1.0) & (rowmax <= 2.0)).all()
        scale = np.ldexp(1.0, np.frexp(p.max(axis=1) ** (1.0 / gamma))[1] - 1)
        # exact: powers of two (and the sorted order, a function of the W bits
        # above bit 16, is unchanged by them)
        unscaled = (t.sw.cpu().numpy().astype(np.float64) * scale[:, None]).astype(np.float32)
        assert np.array_equal(batch.tours, fastpath_c.build_tours_sorted(unscaled, t.si.cpu().numpy(), 8, 2,
                                                                         np.arange(m), n=n))
