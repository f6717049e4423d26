"""Generate the golden vectors in tests/golden/ by running the REFERENCE itself.

Run in the build container (the reference is not present on the GPU box):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

It drives the reference's own public API (antbatch: compute_probability_matrix,
construct_tours, select_elite, accumulate_increments, apply_update,
batch_costs, gamma_at) for a few small instances and records every
intermediate, so the oracle restatement (oracle/reference_port.py) and the
device drop-ins can be pinned against reference outputs without the
reference at run time.
"""

from __future__ import annotations

import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
if REF not in sys.path:
    sys.path.insert(0, REF)

import antbatch  # noqa: E402
from antbatch.model import AcoParams, GammaSchedule, PheromoneState, Selection  # noqa: E402
from antbatch.tsplib import RawTspFile  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))


def integer_instance(seed: int, n: int):
    """Distinct integer grid points, EUC_2D rounded distances (exact sums)."""
    g = np.random.default_rng(seed)
    while True:
        pts = g.integers(0, 1000, size=(n, 2))
        if len(np.unique(pts, axis=0)) == n:
            break
    raw = RawTspFile(name="", dimension=n, edge_weight_type="EUC_2D",
                     node_coords=tuple((i + 1, float(x), float(y)) for i, (x, y) in enumerate(pts)))
    return antbatch.build_instance(raw)


def euclid_instance(seed: int, n: int):
    g = np.random.default_rng(seed)
    return antbatch.euclidean_instance(g.uniform(0.0, 1000.0, size=(n, 2)))


CASES = [
    # name, instance factory, n, m, k, selection, seeds, iterations, alpha, beta, rho, period
    ("int12_ir", lambda: integer_instance(2024, 12), 12, 10, 2, "ir", (0, 1, 2), 4, 1.0, 2.0, 0.1, 4),
    ("int12_adair", lambda: integer_instance(2024, 12), 12, 10, 2, "adair", (0, 1, 2), 4, 1.0, 2.0, 0.1, 4),
    ("euc23_adair", lambda: euclid_instance(7, 23), 23, 16, 3, "adair", (5,), 3, 1.0, 2.0, 0.2, 3),
    ("euc17_ab", lambda: euclid_instance(11, 17), 17, 8, 2, "ir", (3,), 2, 1.5, 3.0, 0.3, 10),
    ("int12_rw", lambda: integer_instance(2024, 12), 12, 10, 2, "rw", (0, 1), 3, 1.0, 2.0, 0.1, 4),
    ("euc29_rw", lambda: euclid_instance(13, 29), 29, 16, 3, "rw", (4,), 3, 1.0, 2.0, 0.2, 4),
]

SELECTION_CODE = {"ir": 0, "adair": 1, "rw": 2}  # meta[8]


def main() -> None:
    out = {}
    for name, make, n, m, k, sel, seeds, iters, alpha, beta, rho, period in CASES:
        inst = make()
        out[f"{name}/dist"] = inst.dist
        out[f"{name}/eta"] = inst.eta
        out[f"{name}/meta"] = np.array([n, m, k, iters, alpha, beta, rho, period, SELECTION_CODE[sel]],
                                       dtype=np.float64)
        out[f"{name}/seeds"] = np.array(seeds, dtype=np.int64)
        for seed in seeds:
            params = AcoParams(m=m, k=k, alpha=alpha, beta=beta, rho=rho, selection=Selection(sel),
                               gamma_schedule=GammaSchedule(1.5, 1.0, period), seed=seed)
            tau = PheromoneState.initial(n, params.q0_tau)
            prob = antbatch.compute_probability_matrix(tau, inst, params)
            for it in range(iters):
                key = f"{name}/s{seed}/it{it}"
                out[f"{key}/p"] = prob.p
                out[f"{key}/gamma"] = np.array(
                    [antbatch.gamma_at(it, params.gamma_schedule) if sel == "adair" else 1.0])
                out[f"{key}/starts"] = antbatch.rng.start_cities(seed, it, m, n)
                batch = antbatch.construct_tours(prob, inst, params, it)
                elites = antbatch.select_elite(batch, k)
                delta = antbatch.accumulate_increments(elites, n)
                tau = antbatch.apply_update(tau, delta, rho)
                prob = antbatch.compute_probability_matrix(tau, inst, params)
                order = np.argsort(batch.costs, kind="stable")[:k]
                out[f"{key}/tours"] = batch.tours
                out[f"{key}/costs"] = batch.costs
                out[f"{key}/order"] = order
                out[f"{key}/delta"] = delta
                out[f"{key}/tau"] = tau.tau
    # known-answer cases from the reference's own tests
    out["kat/gamma"] = np.array([antbatch.gamma_at(t, GammaSchedule()) for t in (0, 250, 500, 999, 1000)])
    from antbatch.selection import rw_spin
    spins = [(np.array([1.0, 0.0, 3.0]), u) for u in (0.2, 0.25, 0.9, 0.0, 1.0)] + \
            [(np.array([0.3, 0.7, 0.0]), 1.0 - 1e-17), (np.array([0.0, 1.0, 0.0]), 0.999999)]
    out["kat/rw_weights"] = np.array([np.pad(w, (0, 3 - len(w))) for w, _ in spins])
    out["kat/rw_u"] = np.array([u for _, u in spins])
    out["kat/rw_pick"] = np.array([rw_spin(w, u) for w, u in spins])
    out["kat/increment_0_1_2_cost4"] = antbatch.increment_matrix(np.array([0, 1, 2]), 4.0, 3)
    path = os.path.join(HERE, "reference_pipeline.npz")
    np.savez_compressed(path, **out)
    print(f"wrote {path} ({os.path.getsize(path)} bytes, {len(out)} arrays)")


if __name__ == "__main__":
    main()
