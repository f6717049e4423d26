"""GPU: the reference's acceptance and statistical gates, on the device path.

Mirrors antbatch's tests/test_acceptance.py and tests/test_colony.py gates that
concern the hot path:
  #4  selection closed forms: IR P(first) = 1 - p2/(2 p1); AdaIR
      1 - (p2/p1)^(1/gamma)/2 over gamma in {0.5, 1, 2, 4}; RW p1/(p1+p2)
      (test_acceptance.py:162-183, :244-254), here through the device stream
      and the production kernels (sorted, dense, roulette);
  #7  brute-force optimum found in >= 8/10 seeds at n = 8
      (test_acceptance.py:262-283);
  AdaIR(gamma == 1) == IR bitwise (test_colony.py:132-142);
  beta = 0 gives uniform 1/(n-1) rows (test_colony.py:41-48);
  chunking is bit-invisible (test_colony.py:120-129);
  the device uniforms are in (0, 1) and uniform (KS), the reference's
  stream-contract analog (test_rng.py, test_selection.py:207-237);
  the Solver raises the reference's exceptions (colony.py:63-68, :149).
"""

import itertools
import math

import numpy as np
import pytest
import torch

import paper_2404_04895_b200 as taco
from paper_2404_04895_b200 import _device, _lib
from paper_2404_04895_b200 import rng as trng
from conftest import euclid

pytestmark = pytest.mark.gpu

P1, P2 = 0.6, 0.25  # row 0 of the 3-city table: P(0->1), P(0->2) (renormalized by the rule)


def _three_city_p():
    p = np.array([[0.0, P1, P2], [0.5, 0.0, 0.5], [0.5, 0.5, 0.0]])
    return p


def _first_choice_freq(tours):
    """Among ants starting at city 0, the fraction whose first move goes to city 1."""
    from0 = tours[:, 0] == 0
    return float(np.mean(tours[from0, 1] == 1)), int(from0.sum())


@pytest.mark.parametrize("variant", ["sorted", "dense"])
@pytest.mark.parametrize("gamma", [0.5, 1.0, 2.0, 4.0])
def test_selection_closed_forms_ir_adair(variant, gamma):
    dev = _device.device()
    p = _three_city_p()
    m = 600_000
    t = _device.SelectionTables(3, dev, dense=True, sorted_=(variant == "sorted"))
    _device.selection_table_from_p(_device.upload(p, dev), 1.0 / gamma, t)
    tours = torch.zeros((m, 3), dtype=torch.int32, device=dev)
    st = _device.new_status(dev)
    code = _lib.CONSTRUCT_SORTED if variant == "sorted" else _lib.CONSTRUCT_DENSE
    _device.construct(3, m, 0, code, t, 1234, 7, tours, st)
    freq, trials = _first_choice_freq(tours.cpu().numpy())
    want = 1.0 - (P2 / P1) ** (1.0 / gamma) / 2.0  # argmax(u1 w1, u2 w2), w = p^(1/gamma)
    assert trials > 150_000
    assert abs(freq - want) < 0.005, (freq, want)


def test_selection_closed_form_rw():
    dev = _device.device()
    p = _three_city_p()
    m = 600_000
    tours = torch.zeros((m, 3), dtype=torch.int32, device=dev)
    st = _device.new_status(dev)
    _device.construct_rw(3, m, 0, _device.upload(p, dev), 99, 3, tours, st)
    freq, trials = _first_choice_freq(tours.cpu().numpy())
    assert trials > 150_000
    assert abs(freq - P1 / (P1 + P2)) < 0.005, freq


def _brute_force(dist):
    n = dist.shape[0]
    best = math.inf
    for perm in itertools.permutations(range(1, n)):
        t = (0,) + perm
        c = sum(dist[t[s], t[(s + 1) % n]] for s in range(n))
        best = min(best, c)
    return best


@pytest.mark.parametrize("selection", ["ir", "adair", "rw"])
def test_finds_brute_force_optimum(selection):
    wins = 0
    for seed in range(10):
        inst = euclid(500 + seed, 8)
        opt = _brute_force(inst.dist)
        params = taco.AcoParams(m=16, k=2, selection=selection, seed=seed,
                                gamma_schedule=taco.GammaSchedule(1.5, 1.0, 50))
        _, length = taco.Solver(inst, params).run(50)
        wins += abs(length - opt) <= 1e-9 * opt
    assert wins >= 8, wins


def test_adair_with_gamma_one_is_ir_bitwise():
    inst = euclid(31, 60)
    ir = taco.AcoParams(m=40, k=4, selection="ir", seed=9)
    ad = taco.AcoParams(m=40, k=4, selection="adair", seed=9, gamma_schedule=taco.GammaSchedule(1.0, 1.0, 5))
    a = taco.Solver(inst, ir)
    b = taco.Solver(inst, ad)
    for _ in range(4):
        a.step()
        b.step()
        assert np.array_equal(a.last_batch().tours, b.last_batch().tours)
    assert np.array_equal(a.pheromone().tau, b.pheromone().tau)


def test_beta_zero_gives_uniform_rows():
    inst = euclid(2, 25)
    params = taco.AcoParams(m=4, k=1, beta=0.0)
    p = taco.compute_probability_matrix(taco.PheromoneState.initial(25, 1.0), inst, params).p
    off = ~np.eye(25, dtype=bool)
    assert np.allclose(p[off], 1.0 / 24, rtol=0, atol=1e-15)
    assert np.all(np.diag(p) == 0.0)
    assert np.allclose(p.sum(axis=1), 1.0, rtol=0, atol=1e-12)


def test_chunk_size_is_invisible():
    inst = euclid(4, 50)
    params = taco.AcoParams(m=30, k=3, selection="adair", seed=2)
    prob = taco.compute_probability_matrix(taco.PheromoneState.initial(50, 1.0), inst, params)
    whole = taco.construct_tours(prob, inst, params, 3)
    for chunk in (1, 7, 30, 100):
        part = taco.construct_tours(prob, inst, params, 3, chunk_size=chunk)
        assert np.array_equal(part.tours, whole.tours)
    with pytest.raises(ValueError):
        taco.construct_tours(prob, inst, params, 3, chunk_size=0)


def test_device_uniforms_open_interval_and_uniform():
    from scipy import stats

    g = np.random.default_rng(17)
    count = 400_000
    step = g.integers(1, 3000, count)
    ant = g.integers(0, 100_000, count)
    city = g.integers(0, 3000, count)
    u = trng.device_uniforms(77, 5, step, ant, city).astype(np.float64)
    assert u.min() > 0.0 and u.max() < 1.0
    assert stats.kstest(u, "uniform").pvalue > 1e-4
    # successive cities of one (step, ant) are not correlated
    v = trng.device_uniforms(77, 5, np.full(count, 11), np.full(count, 3), np.arange(count) % 65536)
    assert abs(np.corrcoef(v[:-1], v[1:])[0, 1]) < 0.01
    w = trng.device_rw_uniforms(77, 5, step, ant)
    assert w.min() >= 0.0 and w.max() < 1.0
    assert stats.kstest(w, "uniform").pvalue > 1e-4


def test_starts_cover_every_city():
    starts = trng.device_starts(3, 0, 37, 20_000)
    counts = np.bincount(starts, minlength=37)
    assert counts.min() > 0 and counts.max() < 2 * counts.mean()


BETA = 4.0  # eta^4 underflows to 0 across 1e90, not within 1e75


def _two_far_clusters():
    # cities 0-3 and 4-7 in two clusters 1e90 apart: eta^BETA is exactly 0
    # across the clusters, so P has exact zeros between them
    pts = np.array([[0, 0], [1, 0], [0, 1], [1, 1]], dtype=np.float64)
    coords = np.concatenate([pts, 1e90 + 1e75 * pts])
    return taco.euclidean_instance(coords)


def test_solver_raises_the_reference_exceptions():
    inst = _two_far_clusters()
    # every ant gets stuck in its start cluster: the reference's argmax over an
    # all -inf row picks a visited city and fails its assert (colony.py:149)
    for construct in ("sorted", "dense"):
        with pytest.raises(AssertionError, match="selector chose a visited city"):
            taco.Solver(inst, taco.AcoParams(m=4, k=1, beta=BETA, selection="ir", seed=0),
                        construct=construct).step()
    with pytest.raises(AssertionError, match="selector chose a visited city"):
        taco.Solver(inst, taco.AcoParams(m=4, k=1, beta=BETA, selection="rw", seed=0)).step()
    # the reference's drop-in raises the same
    params = taco.AcoParams(m=4, k=1, beta=BETA, selection="ir")
    prob = taco.compute_probability_matrix(taco.PheromoneState.initial(8, 1.0), inst, params)
    with pytest.raises(AssertionError):
        taco.construct_tours(prob, inst, params, 0)
    # a row whose normalizer underflows: NumericalUnderflow from the Solver's
    # own row update, with the reference's message
    far = taco.euclidean_instance(np.array([[0.0, 0.0], [1e90, 0.0], [0.0, 1e90], [1e90, 1e90]]))
    with pytest.raises(taco.NumericalUnderflow, match="row 0 normalizer"):
        taco.Solver(far, taco.AcoParams(m=4, k=1, beta=BETA)).step()
