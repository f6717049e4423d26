"""CPU: host-side logic of the drop-in (types, validation, gamma schedule,
sharding plan) mirrors the reference's behaviour (antbatch/model.py,
selection.py, pheromone.py)."""

import math

import numpy as np
import pytest

import paper_2404_04895_b200 as taco
from paper_2404_04895_b200 import colony, distributed
from oracle import reference_port as ref


def test_params_validation_matches_reference():
    # model.py:186-203
    for bad in (dict(m=0, k=1), dict(m=4, k=0), dict(m=4, k=5), dict(m=4, k=1, alpha=0.0),
                dict(m=4, k=1, beta=-1.0), dict(m=4, k=1, rho=1.0), dict(m=4, k=1, q0_tau=0.0),
                dict(m=4, k=1, max_iters=0), dict(m=4, k=1, seed=2**64), dict(m=4, k=1, selection="xx")):
        with pytest.raises(ValueError):
            taco.AcoParams(**bad)
    p = taco.AcoParams(m=4, k=2, selection="ir")
    assert p.selection is taco.Selection.IR and p.n_ants == 4


def test_for_instance_sizing_and_n_ants_alias():
    p = taco.AcoParams.for_instance(2392)
    assert (p.m, p.k) == (2392, 239)
    q = taco.AcoParams.for_instance(2392, n_ants=4096, selection="adair")
    assert (q.m, q.k) == (4096, 409)


def test_gamma_schedule_validation_and_values():
    with pytest.raises(ValueError):
        taco.GammaSchedule(gamma_max=0.9)
    with pytest.raises(ValueError):
        taco.GammaSchedule(gamma_min=0.0)
    with pytest.raises(ValueError):
        taco.GammaSchedule(gamma_max=1.2, gamma_min=1.3)
    with pytest.raises(ValueError):
        taco.GammaSchedule(period=0)
    s = taco.GammaSchedule()
    got = [taco.gamma_at(t, s) for t in (0, 250, 500, 999, 1000, 1250)]
    assert got == [ref.gamma(t) for t in (0, 250, 500, 999, 1000, 1250)]
    assert got[0] == 1.5 and abs(got[1] - 1.4268) < 5e-5
    with pytest.raises(ValueError):
        taco.gamma_at(-1, s)


def test_construction_gamma_per_mechanism():
    ir = taco.AcoParams(m=2, k=1, selection="ir")
    ad = taco.AcoParams(m=2, k=1, selection="adair")
    assert colony.construction_gamma(ir, 7) == 1.0
    assert colony.construction_gamma(ad, 0) == 1.5
    assert colony.construction_gamma(taco.AcoParams(m=2, k=1, selection="rw"), 0) == 1.0


def test_instances_frozen_and_degenerate_detection():
    inst = taco.euclidean_instance([[0, 0], [3, 4], [6, 8]])
    assert inst.dist[0, 1] == 5.0 and inst.eta[0, 1] == 0.2 and inst.eta[0, 0] == 0.0
    with pytest.raises(ValueError):
        inst.dist[0, 1] = 1.0
    with pytest.raises(taco.DegenerateInstance):
        taco.euclidean_instance([[0, 0], [0, 0], [1, 1]])
    lenient = taco.euclidean_instance([[0, 0], [0, 0], [1, 1]], lenient=True)
    assert lenient.eta[0, 1] == 1.0 / 1e-10
    with pytest.raises(taco.DegenerateInstance):
        taco.TspInstance(n=2, dist=np.zeros((2, 2)), eta=np.zeros((2, 2)))


def test_value_objects_copy_and_freeze():
    tau = np.ones((3, 3))
    st = taco.PheromoneState(tau=tau)
    tau[0, 0] = 7.0
    assert st.tau[0, 0] == 1.0
    init = taco.PheromoneState.initial(4, 2.0)
    assert np.array_equal(init.tau, ref.initial_tau(4, 2.0)) and init.iteration == 0
    b = taco.TourBatch(tours=[[0, 1, 2]], costs=[3.0])
    assert b.tours.dtype == np.int64 and b.m == 1 and b.n == 3
    with pytest.raises(ValueError):
        b.costs[0] = 1.0


def test_permutation_checks_and_host_helpers():
    with pytest.raises(taco.InvalidPermutation):
        taco.edge_index_matrix(np.array([0, 1, 1]))
    idx = taco.edge_index_matrix(np.array([2, 0, 1]))
    assert idx.tolist() == [[2, 1], [0, 2], [1, 0]]  # reference tests/test_pheromone.py:48-56
    a = taco.increment_matrix(np.array([0, 1, 2]), 4.0, 3)
    assert np.array_equal(a, 0.25 * (1 - np.eye(3)))
    t = np.array([3, 0, 4, 1, 2])
    m5 = taco.increment_matrix(t, 10.0, 5)
    assert np.count_nonzero(m5) == 10 and np.array_equal(m5, m5.T)


def test_underflow_message_matches_reference_choice():
    sums = np.array([1.0, np.inf, 0.0, np.nan])
    err = colony._underflow_from_sums(sums)
    assert isinstance(err, taco.NumericalUnderflow) and str(err).startswith("row 1 ")
    err = colony._underflow_from_sums(np.array([2.0, 0.0, -1.0]))
    assert str(err).startswith("row 2 ")


@pytest.mark.parametrize("m,world", [(4096, 1), (4096, 8), (10, 3), (8192, 8), (7, 7)])
def test_ant_shards_tile_the_colony(m, world):
    shards = [distributed.shard_ants(m, r, world) for r in range(world)]
    assert shards[0].offset == 0
    for a, b in zip(shards, shards[1:]):
        assert b.offset == a.offset + a.count
    assert sum(s.count for s in shards) == m
    assert max(s.count for s in shards) - min(s.count for s in shards) <= 1
    assert all(s.per_rank == math.ceil(m / world) for s in shards)
    idx = distributed.gather_index(m, world)
    if m % world == 0:
        assert idx is None
    else:
        assert len(idx) == m and len(set(idx.tolist())) == m


def test_shard_errors():
    with pytest.raises(ValueError):
        distributed.shard_ants(3, 0, 4)
    with pytest.raises(ValueError):
        distributed.shard_ants(8, 4, 4)


def test_harness_output_formats_match_reference_golden():
    """records CSV and summary JSON are byte-identical to antbatch's writers
    (bench.py:395-462) on the same values (tests/golden/make_harness.py)."""
    import json
    import os
    from types import SimpleNamespace

    from paper_2404_04895_b200 import harness

    here = os.path.join(os.path.dirname(__file__), "golden")
    recs = [harness.IterationRecord(*r) for r in (
        (0, 5, 0, 1.25, 1234.5, 1234.5, 3.1, 1.5, 0.1),
        (0, 5, 1, 0.1 + 0.2, 1200.0, 1200.0, None, 1.4268, 0.1),
        (1, 6, 0, 2.0, 987.654321, 987.654321, None, None, 0.25))]
    sums = [harness.RunSummary(*r) for r in (
        (0, 5, 2, 1200.0, 0.5, 1, 0.30000000000000004, "max_iters"),
        (1, 6, 1, 987.654321, None, 0, 2.0, "time_limit"))]
    assert harness.records_csv_text(recs) == open(os.path.join(here, "harness_records.csv")).read()
    config = harness.ExperimentConfig(
        params=taco.AcoParams(m=8, k=2, alpha=1.0, beta=2.0, rho=0.1, selection="adair",
                              gamma_schedule=taco.GammaSchedule(1.5, 1.0, 7), max_iters=2, seed=5),
        synthetic=harness.SyntheticSpec(n=12, seed=1, kind="uniform"), repetitions=2, best_known=1000.0)
    doc = json.loads(harness.summary_json_text(config, SimpleNamespace(name="rnd12", n=12, best_known=1000.0),
                                               sums))
    assert doc["aggregate"]["cpu_count"] == os.cpu_count()
    doc["aggregate"]["cpu_count"] = None
    assert json.dumps(doc, indent=2, sort_keys=True) + "\n" == open(os.path.join(here, "harness_summary.json")).read()
