"""Solution quality at C2 over 10 seeds: the engine's device stream against
the reference's own streams (BASELINE.json north_star: "best-tour quality
over full runs must agree statistically across 10 seeds"; the reference's
quality gate is tests/test_acceptance.py:387-411).

The reference side is Solver(stream="replay"): it replays antbatch's numpy
streams on the device and reproduces antbatch's run_experiment bit for bit
(tests/test_gpu_parity.py::test_solver_replay_reproduces_reference_runs), so
it IS the reference algorithm's trajectory, at GPU speed.

    python scripts/quality_c2.py [--iters 100] [--seeds 10] [--out file.json]
"""
import argparse
import json
import os
import sys
import time

import numpy as np
from scipy import stats

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2404_04895_b200 as taco  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=1000)
ap.add_argument("--m", type=int, default=1024)
ap.add_argument("--sel", default="adair")
ap.add_argument("--iters", type=int, default=100)
ap.add_argument("--seeds", type=int, default=10)
ap.add_argument("--out", default=None)
args = ap.parse_args()

coords = np.random.default_rng(0).uniform(0.0, 2000.0, (args.n, 2))
inst = taco.euclidean_instance(coords)
rows = []
for seed in range(args.seeds):
    params = taco.AcoParams(m=args.m, k=max(1, args.m // 10), selection=args.sel, seed=seed,
                            gamma_schedule=taco.GammaSchedule(1.5, 1.0, args.iters))
    t0 = time.perf_counter()
    dev_best = taco.Solver(inst, params).run(args.iters)[1]
    t1 = time.perf_counter()
    ref_best = taco.Solver(inst, params, stream="replay").run(args.iters)[1]
    t2 = time.perf_counter()
    rows.append({"seed": seed, "device_stream": dev_best, "reference_stream": ref_best,
                 "device_s": t1 - t0, "replay_s": t2 - t1})
    print(json.dumps(rows[-1]), flush=True)
a = np.array([r["device_stream"] for r in rows])
b = np.array([r["reference_stream"] for r in rows])
welch = stats.ttest_ind(a, b, equal_var=False)
mwu = stats.mannwhitneyu(a, b, alternative="two-sided")
summary = {"config": f"n={args.n} m={args.m} k={max(1, args.m // 10)} {args.sel}, gamma 1.5->1.0 period "
                     f"{args.iters}, {args.iters} iterations, {args.seeds} seeds, U(0,2000)^2 seed 0",
           "device_mean": float(a.mean()), "device_std": float(a.std(ddof=1)),
           "reference_mean": float(b.mean()), "reference_std": float(b.std(ddof=1)),
           "mean_rel_diff": float((a.mean() - b.mean()) / b.mean()),
           "welch_t": float(welch.statistic), "welch_p": float(welch.pvalue),
           "mannwhitney_u": float(mwu.statistic), "mannwhitney_p": float(mwu.pvalue), "runs": rows}
print(json.dumps({k: v for k, v in summary.items() if k != "runs"}))
if args.out:
    with open(args.out, "w") as f:
        json.dump(summary, f, indent=1)
