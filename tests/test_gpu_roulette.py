"""GPU: roulette-wheel (RW) selection, SURVEY §8f row f3.

* the reference's spin rule (rw_spin_block selection.py:102-127) on the
  reference's thresholds: taco_rw_parity == oracle spin_round, including
  adversarial rows and thresholds placed exactly on CDF values, where only the
  exact sequential recount can decide;
* the device stream: taco_construct_rw == oracle fastpath.rw_tours;
* the golden pipeline of the reference's RW runs (stream="numpy" and the
  device replay of its stream, drop-ins and full Solver runs);
* the Solver with selection="rw" against the chained drop-ins.
"""

import numpy as np
import pytest
import torch

import paper_2404_04895_b200 as taco
from paper_2404_04895_b200 import _device, _lib
from paper_2404_04895_b200 import rng as trng
from conftest import euclid
from oracle import fastpath, reference_port as ref

pytestmark = pytest.mark.gpu


def _spin_on_device(p, cur, visited, u, force_exact=False):
    dev = _device.device()
    m, n = visited.shape
    p_t = _device.upload(p, dev)
    u_t = _device.upload(u, dev)
    cur_t = _device.upload(cur.astype(np.int64), dev)
    vis_t = _device.upload(visited.astype(np.uint8), dev)
    tours = torch.zeros((m, n), dtype=torch.int64, device=dev)
    status = _device.new_status(dev)
    exact = torch.zeros(1, dtype=torch.int64, device=dev)
    _lib.check(_lib.load().taco_rw_parity(n, m, 1, p_t.data_ptr(), u_t.data_ptr(), cur_t.data_ptr(),
                                          vis_t.data_ptr(), tours.data_ptr(), status.data_ptr(), exact.data_ptr(),
                                          int(force_exact), _device.stream_handle()), "taco_rw_parity")
    code, _ = _device.read_status(status)
    return cur_t.cpu().numpy(), code, int(exact.item())


def _random_p(g, n, spread):
    p = np.exp(g.uniform(-spread, 0.0, (n, n)))
    p[g.uniform(size=(n, n)) < 0.1] = 0.0
    np.fill_diagonal(p, 0.0)
    return p / p.sum(axis=1, keepdims=True)


@pytest.mark.parametrize("n", [3, 7, 256, 257, 700, 2392])
@pytest.mark.parametrize("spread", [1.0, 40.0])
def test_spin_round_matches_reference_rule(n, spread):
    g = np.random.default_rng(n + int(spread))
    m = 64
    p = _random_p(g, n, spread)
    cur = g.integers(0, n, m)
    visited = g.uniform(size=(m, n)) < 0.5
    visited[np.arange(m), cur] = True
    keep = g.integers(0, n, m)
    visited[np.arange(m), keep] = keep == cur  # at least one candidate unless keep == cur
    ok = (p[cur] * ~visited).sum(axis=1) > 0
    cur, visited = cur[ok], visited[ok]
    unvisited = (~visited).astype(np.float64)
    u = g.uniform(size=len(cur))
    want = ref.spin_round(p, cur, unvisited, u)
    for force in (False, True):
        got, code, exact = _spin_on_device(p, cur, visited, u, force)
        assert code == 0 and np.array_equal(got, want)
        assert exact == (len(cur) if force else exact)


def test_spin_thresholds_on_cdf_values_take_the_exact_recount():
    # u equal to a CDF value (and its neighbours) must follow the strict '>' of
    # the sequential cumsum: the certified bounds cannot decide, the recount does
    g = np.random.default_rng(11)
    n = 300
    p = _random_p(g, n, 20.0)
    m = 96
    cur = g.integers(0, n, m)
    visited = g.uniform(size=(m, n)) < 0.3
    visited[np.arange(m), cur] = True
    unvisited = (~visited).astype(np.float64)
    cdf = np.cumsum(p[cur] * unvisited, axis=1)
    cdf /= cdf[:, -1:].copy()
    cols = g.integers(0, n - 1, m)
    u = cdf[np.arange(m), cols]
    u = np.where(np.arange(m) % 3 == 1, np.nextafter(u, 0.0), u)
    u = np.where(np.arange(m) % 3 == 2, np.nextafter(u, 1.0), u)
    want = ref.spin_round(p, cur, unvisited, u)
    got, code, exact = _spin_on_device(p, cur, visited, u)
    assert code == 0 and np.array_equal(got, want)
    assert exact > 0


def test_spin_edges_u_zero_one_and_known_answers(golden):
    for w, u, want in zip(golden["kat/rw_weights"], golden["kat/rw_u"], golden["kat/rw_pick"]):
        p = np.zeros((3, 3))
        p[0] = w
        got, code, _ = _spin_on_device(p, np.array([0]), np.zeros((1, 3), dtype=bool), np.array([u]))
        assert code == 0 and got[0] == want
    # u >= 1 takes the last positive weight, also through the device stream's path
    p = np.array([[0.0, 0.6, 0.4, 0.0], [0.5, 0.0, 0.5, 0.0], [0.2, 0.8, 0.0, 0.0], [0.3, 0.3, 0.4, 0.0]])
    got, code, _ = _spin_on_device(p, np.array([3, 3]), np.array([[False, False, True, True]] * 2),
                                   np.array([1.0, 0.0]))
    assert code == 0 and got.tolist() == [1, 0]


def test_rw_device_uniforms_match_restatement():
    g = np.random.default_rng(2)
    step = g.integers(1, 65535, 5000)  # steps < n <= 65535
    ant = g.integers(0, 2**31, 5000)
    seed = 2**50 + 7
    assert np.array_equal(trng.device_rw_uniforms(seed, 9, step, ant), fastpath.rw_uniform(seed, 9, step, ant))


@pytest.mark.parametrize("n,m", [(3, 5), (12, 10), (64, 40), (257, 33), (300, 70)])
def test_device_rw_tours_match_restatement(n, m):
    inst = euclid(n + 1, n)
    g = np.random.default_rng(n)
    tau = g.uniform(0.1, 2.0, (n, n))
    p = ref.transition((tau + tau.T) / 2, inst.eta, 1.0, 2.0)
    params = taco.AcoParams(m=m, k=1, selection="rw", seed=n)
    for it in (0, 5):
        got = taco.construct_tours(taco.ProbabilityMatrix(p), inst, params, it)
        want = fastpath.rw_tours(p, n, it, np.arange(m))
        assert np.array_equal(got.tours, want)
        assert np.array_equal(got.costs, ref.lengths(want, inst.dist))
    # the exact-recount path alone gives the same tours
    dev = _device.device()
    p_t = _device.upload(p, dev)
    tours = torch.zeros((m, n), dtype=torch.int32, device=dev)
    st = _device.new_status(dev)
    _device.construct_rw(n, m, 0, p_t, n, 5, tours, st, force_exact=True)
    assert np.array_equal(tours.cpu().numpy(), fastpath.rw_tours(p, n, 5, np.arange(m)))


@pytest.mark.parametrize("name", ["int12_rw", "euc29_rw"])
def test_rw_dropin_pipeline_matches_reference_golden(golden, name):
    inst = taco.TspInstance(n=golden[f"{name}/dist"].shape[0], dist=golden[f"{name}/dist"],
                            eta=golden[f"{name}/eta"])
    n, m, k, iters, alpha, beta, rho, period, sel = golden[f"{name}/meta"]
    for seed in golden[f"{name}/seeds"].tolist():
        params = taco.AcoParams(m=int(m), k=int(k), alpha=alpha, beta=beta, rho=rho, selection="rw", seed=seed)
        tau = taco.PheromoneState.initial(inst.n, params.q0_tau)
        prob = taco.compute_probability_matrix(tau, inst, params)
        for it in range(int(iters)):
            key = f"{name}/s{seed}/it{it}"
            assert np.array_equal(prob.p, golden[f"{key}/p"])
            batch = taco.construct_tours(prob, inst, params, it, stream="numpy")
            assert np.array_equal(batch.tours, golden[f"{key}/tours"])
            assert np.array_equal(batch.costs, golden[f"{key}/costs"])
            replayed = taco.construct_tours(prob, inst, params, it, stream="replay")
            assert np.array_equal(replayed.tours, golden[f"{key}/tours"])
            tau = taco.apply_update(tau, taco.accumulate_increments(taco.select_elite(batch, params.k), inst.n),
                                    params.rho)
            assert np.array_equal(tau.tau, golden[f"{key}/tau"])
            prob = taco.compute_probability_matrix(tau, inst, params)
    # full Solver runs on the reference's streams reproduce the golden runs
    for seed in golden[f"{name}/seeds"].tolist():
        params = taco.AcoParams(m=int(m), k=int(k), alpha=alpha, beta=beta, rho=rho, selection="rw", seed=seed)
        s = taco.Solver(inst, params, stream="replay")
        for it in range(int(iters)):
            s.step()
            key = f"{name}/s{seed}/it{it}"
            assert np.array_equal(s.last_batch().tours, golden[f"{key}/tours"])
            assert np.array_equal(s.pheromone().tau, golden[f"{key}/tau"])


def test_rw_solver_matches_chained_dropins():
    n, m = 70, 30
    inst = euclid(21, n)
    params = taco.AcoParams(m=m, k=3, selection="rw", seed=4)
    s = taco.Solver(inst, params)
    tau = taco.PheromoneState.initial(n, 1.0)
    best = np.inf
    for it in range(5):
        prob = taco.compute_probability_matrix(tau, inst, params)
        batch = taco.construct_tours(prob, inst, params, it)
        tau = taco.apply_update(tau, taco.accumulate_increments(taco.select_elite(batch, params.k), n),
                                params.rho)
        tour, length = s.step()
        got = s.last_batch()
        assert np.array_equal(got.tours, batch.tours)
        assert np.array_equal(got.costs, batch.costs)
        assert np.array_equal(s.pheromone().tau, tau.tau)
        best = min(best, batch.costs.min())
        assert length == best


def test_rw_quality_below_ir_like_the_reference():
    # the paper's ablation direction (reference tests/test_acceptance.py:352-360):
    # IR's best tours are not worse than RW's on the same budget
    n, m, iters = 40, 40, 30
    inst = euclid(5, n)
    res = {}
    for mech in ("rw", "ir"):
        res[mech] = np.mean([taco.Solver(inst, taco.AcoParams(m=m, k=3, selection=mech, seed=s)).run(iters)[1]
                             for s in range(4)])
    assert res["ir"] <= res["rw"] * 1.02
