"""GPU: the run_experiment-style harness on the Solver."""

import numpy as np
import pytest

import paper_2404_04895_b200 as taco
from paper_2404_04895_b200 import harness
from conftest import euclid

pytestmark = pytest.mark.gpu


def test_run_experiment_records_and_summaries():
    inst = euclid(3, 40)
    params = taco.AcoParams(m=32, k=3, selection="adair", max_iters=12, seed=7,
                            gamma_schedule=taco.GammaSchedule(1.5, 1.0, 12))
    cfg = harness.ExperimentConfig(params=params, repetitions=2, best_known=1000.0)
    records, summaries = harness.run_experiment(cfg, inst)
    assert len(records) == 24 and len(summaries) == 2
    for run_id, summ in enumerate(summaries):
        recs = [r for r in records if r.run_id == run_id]
        assert [r.iteration for r in recs] == list(range(12))
        assert all(r.seed == 7 + run_id for r in recs)
        best = np.minimum.accumulate([r.iteration_best_cost for r in recs])
        assert np.array_equal(best, [r.best_cost_so_far for r in recs])
        assert summ.final_best_cost == best[-1]
        assert summ.terminated_by == "max_iters" and summ.iterations_run == 12
        assert summ.mean_ms_per_iter == pytest.approx(np.mean([r.wall_clock_ms for r in recs[1:]]))
        assert recs[0].gamma == 1.5 and recs[0].rho == 0.1
        assert summ.solution_error_percent == pytest.approx(100.0 * (best[-1] - 1000.0) / 1000.0)
        # the same seed through the Solver gives the same best
        s = taco.Solver(inst, taco.AcoParams(**{**params.__dict__, "seed": 7 + run_id}))
        assert s.run(12)[1] == summ.final_best_cost


def test_time_limit_terminates():
    inst = euclid(4, 30)
    params = taco.AcoParams(m=16, k=2, selection="ir", max_iters=10_000)
    ticks = iter(range(10**6))
    cfg = harness.ExperimentConfig(params=params, time_limit_seconds=5.0)
    records, summaries = harness.run_experiment(cfg, inst, clock=lambda: float(next(ticks)))
    assert summaries[0].terminated_by == "time_limit" and 1 <= len(records) < 10_000


def test_convergence_generation_definition():
    assert harness.convergence_generation([10.0, 5.0, 4.002, 4.0]) == 2
    assert harness.convergence_generation([3.0]) == 0
