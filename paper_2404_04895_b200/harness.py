"""Experiment harness on the device Solver.

Mirrors the reference's ``run_experiment`` (bench.py:171-238) so convergence
studies (IR vs AdaIR, bench.py:162-168) run at GPU scale with the same record
and summary types: run r uses seed base + r, every iteration yields an
``IterationRecord``, and each run a ``RunSummary`` whose mean time excludes
the first (warm-up) iteration.  Iteration times are device times of one full
iteration (CUDA events).  Synthetic instances (bench.py:127-150) are built
on the device (``load_instance``); TSPLIB parsing is outside the accelerated
path, so for ``instance_path`` the caller passes the instance (or
``device_build_instance(raw)``).
"""

from __future__ import annotations

import csv
import io
import json
import os
import time
from dataclasses import asdict, dataclass, replace

import numpy as np
import torch

from ._device import DeviceInstance
from .model import Selection
from .selection import gamma_at
from .solver import Solver

CONVERGENCE_BAND = 1e-3  # bench.py:40

ITER_COLUMNS = [  # bench.py:42-45: the per-iteration CSV, fixed column order
    "run_id", "seed", "iteration", "wall_clock_ms", "iteration_best_cost",
    "best_cost_so_far", "solution_error_percent", "gamma", "rho",
]


@dataclass(frozen=True)
class SyntheticSpec:
    """Deterministic synthetic instance: n cities, layout kind, coordinate
    seed (bench.py:55-69)."""

    n: int
    seed: int = 0
    kind: str = "clustered"
    name: str = ""

    def __post_init__(self):
        if self.kind not in ("clustered", "uniform"):
            raise ValueError(f"kind must be clustered or uniform, got {self.kind!r}")
        if not self.name:
            object.__setattr__(self, "name", f"rnd{self.n}")


def synthetic_coords(spec: SyntheticSpec) -> np.ndarray:
    """The coordinates make_synthetic_instance (bench.py:127-150) writes: the
    same Generator draws, rounded to one decimal; distances are EUC_2D."""
    g = np.random.default_rng(spec.seed)
    if spec.kind == "clustered":
        n_centers = max(2, spec.n // 25)
        centers = g.uniform(0.0, 2000.0, size=(n_centers, 2))
        which = g.integers(0, n_centers, size=spec.n)
        pts = centers[which] + g.normal(0.0, 60.0, size=(spec.n, 2))
    else:
        pts = g.uniform(0.0, 2000.0, size=(spec.n, 2))
    return np.round(pts, 1)


def load_instance(config: "ExperimentConfig") -> DeviceInstance:
    """load_instance (bench.py:152-159) for synthetic specs, built on the
    device (EUC_2D).  TSPLIB files are parsed by the caller."""
    if config.synthetic is None:
        raise NotImplementedError("TSPLIB parsing is outside the accelerated path: parse the file and pass "
                                  "the instance (or device_build_instance(raw)) to run_experiment")
    spec = config.synthetic
    return DeviceInstance.from_coords(synthetic_coords(spec), "EUC_2D", lenient=config.lenient,
                                      best_known=config.best_known, name=spec.name)


@dataclass(frozen=True)
class ExperimentConfig:
    """Run parameters (bench.py:71-98); instance fields are informational."""

    params: object
    instance_path: str | None = None
    synthetic: object | None = None
    repetitions: int = 1
    time_limit_seconds: float | None = None
    output_path: str | None = None
    summary_path: str | None = None
    record_probability_shift: bool = False
    best_known: float | None = None
    lenient: bool = False
    chunk_size: int | None = None

    def __post_init__(self):
        if self.repetitions < 1:
            raise ValueError(f"repetitions must be >= 1, got {self.repetitions}")
        if self.time_limit_seconds is not None and self.time_limit_seconds <= 0:
            raise ValueError("time_limit_seconds must be positive")


@dataclass(frozen=True)
class IterationRecord:
    run_id: int
    seed: int
    iteration: int
    wall_clock_ms: float
    iteration_best_cost: float
    best_cost_so_far: float
    solution_error_percent: float | None
    gamma: float | None
    rho: float


@dataclass(frozen=True)
class RunSummary:
    run_id: int
    seed: int
    iterations_run: int
    final_best_cost: float
    solution_error_percent: float | None
    convergence_generation: int
    mean_ms_per_iter: float
    terminated_by: str


def convergence_generation(best_trace: list[float]) -> int:
    """First iteration whose best-so-far is within 0.1% of the final best."""
    limit = best_trace[-1] * (1.0 + CONVERGENCE_BAND)
    return next(it for it, v in enumerate(best_trace) if v <= limit)


def run_experiment(config: ExperimentConfig, inst=None, clock=time.perf_counter,
                   construct: str = "auto") -> tuple[list[IterationRecord], list[RunSummary]]:
    """construct -> elite -> deposit -> evaporate -> P per iteration on the
    device, `repetitions` runs with seeds base..base+r-1."""
    if inst is None:
        inst = load_instance(config)
    base = config.params
    bk = config.best_known if config.best_known is not None else getattr(inst, "best_known", None)
    records: list[IterationRecord] = []
    summaries: list[RunSummary] = []
    adair = Selection(base.selection) is Selection.ADAIR
    for run_id in range(config.repetitions):
        params = replace(base, seed=base.seed + run_id)
        solver = Solver(inst, params, construct=construct)
        best_so_far = float("inf")
        trace, iter_ms = [], []
        terminated_by = "max_iters"
        run_start = clock()
        for it in range(params.max_iters):
            t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            t0.record()
            solver.step_async()
            t1.record()
            solver.check()  # synchronizes; raises the reference's exceptions
            ms = t0.elapsed_time(t1)
            iteration_best = float(solver.costs_all[solver.order[0]].item())
            best_so_far = min(best_so_far, iteration_best)
            trace.append(best_so_far)
            iter_ms.append(ms)
            records.append(IterationRecord(
                run_id=run_id, seed=params.seed, iteration=it, wall_clock_ms=ms,
                iteration_best_cost=iteration_best, best_cost_so_far=best_so_far,
                solution_error_percent=(100.0 * (best_so_far - bk) / bk) if bk else None,
                gamma=gamma_at(it, params.gamma_schedule) if adair else None, rho=params.rho))
            if config.time_limit_seconds is not None and clock() - run_start >= config.time_limit_seconds:
                terminated_by = "time_limit"
                break
        measured = iter_ms[1:] if len(iter_ms) > 1 else iter_ms
        summaries.append(RunSummary(
            run_id=run_id, seed=params.seed, iterations_run=len(iter_ms), final_best_cost=best_so_far,
            solution_error_percent=(100.0 * (best_so_far - bk) / bk) if bk else None,
            convergence_generation=convergence_generation(trace),
            mean_ms_per_iter=float(np.mean(measured)), terminated_by=terminated_by))
    return records, summaries


# ---------------------------------------------------------------------------
# the reference's output formats (bench.py:395-462): per-iteration CSV and the
# per-experiment summary JSON, byte-identical for the same records
# ---------------------------------------------------------------------------
def _fmt(v) -> str:
    if v is None:
        return ""
    if isinstance(v, float):
        return repr(v)
    return str(v)


def write_records_csv(records: list[IterationRecord], out) -> None:
    """Per-iteration CSV with the fixed ITER_COLUMNS order (bench.py:403-408)."""
    w = csv.writer(out, lineterminator="\n")
    w.writerow(ITER_COLUMNS)
    for r in records:
        w.writerow([_fmt(getattr(r, c)) for c in ITER_COLUMNS])


def records_csv_text(records: list[IterationRecord]) -> str:
    buf = io.StringIO()
    write_records_csv(records, buf)
    return buf.getvalue()


def config_to_dict(config: ExperimentConfig) -> dict:
    """bench.py:424-427: dataclass dict with the selection as its string value."""
    d = asdict(config)
    d["params"]["selection"] = Selection(config.params.selection).value
    return d


def summary_json_text(config: ExperimentConfig, inst, summaries: list[RunSummary]) -> str:
    """One JSON document per experiment: config echo plus aggregates
    (bench.py:441-462)."""
    finals = [s.final_best_cost for s in summaries]
    convs = [s.convergence_generation for s in summaries]
    doc = {
        "config": config_to_dict(config),
        "instance": {
            "name": getattr(inst, "name", ""), "n": int(inst.n), "best_known": getattr(inst, "best_known", None),
            "best_known_source": ("override" if config.best_known is not None else "bundled-table"),
        },
        "runs": [asdict(s) for s in summaries],
        "aggregate": {
            "median_final_best_cost": float(np.median(finals)),
            "median_convergence_generation": float(np.median(convs)),
            "mean_ms_per_iter": float(np.mean([s.mean_ms_per_iter for s in summaries])),
            "cpu_count": os.cpu_count(),
        },
    }
    return json.dumps(doc, indent=2, sort_keys=True) + "\n"
