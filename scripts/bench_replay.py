"""Time the reference-stream replay Solver (bit-exact antbatch runs on the GPU).

    python scripts/bench_replay.py --n 2392 --m 4096 --iters 2
"""
import argparse
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2404_04895_b200 as taco  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=2392)
ap.add_argument("--m", type=int, default=4096)
ap.add_argument("--iters", type=int, default=2)
ap.add_argument("--selection", default="adair")
args = ap.parse_args()
inst = taco.euclidean_instance(np.random.default_rng(0).uniform(0.0, 2000.0, (args.n, 2)))
params = taco.AcoParams(m=args.m, k=max(1, args.m // 10), selection=args.selection, seed=0,
                        gamma_schedule=taco.GammaSchedule(1.5, 1.0, args.iters + 1))
s = taco.Solver(inst, params, stream="replay")
s.step()  # warm-up iteration (excluded, like bench.py:228 of the reference)
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(args.iters):
    s.step()
torch.cuda.synchronize()
dt = (time.perf_counter() - t0) / args.iters
print(json.dumps({"mode": "replay (bit-exact reference streams)", "n": args.n, "m": args.m,
                  "s_per_iteration": dt, "iterations_per_s": 1.0 / dt, "best": s.best()[1]}))
