"""Scan-depth distribution of the pruned sorted-table scan on a Solver's
late-iteration tables (sizing a head-only selection table).

    python scripts/scan_depth.py --n 2392 --m 4096 --iters 20 50 100
Prints, per iteration count, the mean 32-entry windows per ant-step (C oracle
restatement of the kernel's stop rule, cross-checked against the kernel's own
window probe) and the share of steps reading more than T entries.
"""
import argparse
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2404_04895_b200 as taco  # noqa: E402
from paper_2404_04895_b200 import _device, _lib  # noqa: E402
from oracle import fastpath_c  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=2392)
ap.add_argument("--m", type=int, default=4096)
ap.add_argument("--sel", default="adair")
ap.add_argument("--ants", type=int, default=64)
ap.add_argument("--iters", type=int, nargs="+", default=[20])
args = ap.parse_args()

coords = np.random.default_rng(0).uniform(0.0, 2000.0, (args.n, 2))
params = taco.AcoParams(m=args.m, k=max(1, args.m // 10), selection=args.sel, seed=0,
                        gamma_schedule=taco.GammaSchedule(1.5, 1.0, max(args.iters) + 3))
s = taco.Solver(taco.device_euclidean_instance(coords), params, graph=False)
done = 0
for target in sorted(args.iters):
    s.run(target - done)
    done = target
    n, t = args.n, s.tables
    scan = torch.zeros(1, dtype=torch.int64, device=s.dev)
    tours = torch.zeros((args.m, n), dtype=torch.int32, device=s.dev)
    st = _device.new_status(s.dev)
    _device.construct(n, args.m, 0, _lib.CONSTRUCT_SORTED, t, 0, s.iteration, tours, st, scan)
    kernel_windows = int(scan.item()) / (args.m * (n - 1))
    ants = np.unique(np.linspace(0, args.m - 1, args.ants).astype(np.int64))
    hist = fastpath_c.scan_profile(t.sw.cpu().numpy(), t.si.cpu().numpy(), n, 0, s.iteration, ants)
    w = np.arange(1, hist.size + 1)
    total = hist.sum()
    over = {T: float(hist[w * 32 > T].sum() / total) for T in (32, 64, 128, 256, 512, 1024, 2048)}
    cum = np.cumsum(hist) / total
    pct = {p: int(w[np.searchsorted(cum, p / 100.0)]) for p in (50, 90, 99, 99.9)}
    print(json.dumps({"n": n, "m": args.m, "iteration": s.iteration, "kernel_windows_per_step": kernel_windows,
                      "oracle_windows_per_step": float((hist * w).sum() / total),
                      "steps_profiled": int(total), "windows_percentiles": pct,
                      "share_of_steps_reading_more_than_T_entries": over,
                      "windows_beyond_T_share": {T: float((hist * np.maximum(w - T // 32, 0)).sum() /
                                                          (hist * w).sum()) for T in (128, 256, 512, 1024)}}))
