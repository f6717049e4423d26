"""Time the construction kernel alone on realistic tables (tuning helper).

Runs a Solver at the given size for a few iterations (so the pheromone and
the sorted tables look like a real run), then times taco_construct with CUDA
events.  Knobs are read by libtaco from the environment (TACO_SORTED_COST, TACO_SORTED_VIS,
TACO_SORTED_WARPS), so variants are compared in separate processes:

    python scripts/bench_construct.py --n 2392 --m 4096 --iters 5
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

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=2392)
ap.add_argument("--m", type=int, default=4096)
ap.add_argument("--iters", type=int, default=5)
ap.add_argument("--reps", type=int, default=5)
ap.add_argument("--variant", default="sorted", help="sorted | dense | rw")
ap.add_argument("--no-costs", action="store_true", help="tours only (no tour lengths)")
args = ap.parse_args()

inst = taco.euclidean_instance(np.random.default_rng(0).uniform(0, 2000, (args.n, 2)))
rw = args.variant == "rw"
params = taco.AcoParams(m=args.m, k=max(1, args.m // 10), selection="rw" if rw else "adair", seed=0)
s = taco.Solver(inst, params, construct="sorted" if rw else args.variant)
for _ in range(args.iters):
    s.step_async()
s.check()
torch.cuda.synchronize()
dev = s.dev
tours = torch.zeros((args.m, args.n), dtype=torch.int32, device=dev)
costs = None if args.no_costs else torch.zeros(args.m, dtype=torch.float64, device=dev)
st = _device.new_status(dev)
scan = torch.zeros(1, dtype=torch.int64, device=dev)
variant = _lib.CONSTRUCT_SORTED if args.variant == "sorted" else _lib.CONSTRUCT_DENSE
times = []
for r in range(args.reps + 1):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    if rw:
        _device.construct_rw(args.n, args.m, 0, s.p, 0, s.iteration, tours, st, dist=s.di.dist,
                             costs_out=costs, exact_count=scan if r == 0 else None)
    else:
        _device.construct(args.n, args.m, 0, variant, s.tables, 0, s.iteration, tours, st,
                          scan if r == 0 else None, dist=s.di.dist, costs_out=costs)
    b.record()
    torch.cuda.synchronize()
    if r:
        times.append(a.elapsed_time(b))
assert _device.read_status(st)[0] == 0
print(json.dumps({"n": args.n, "m": args.m, "variant": args.variant,
                  "cost": os.environ.get("TACO_SORTED_COST"), "vis": os.environ.get("TACO_SORTED_VIS"), "warps": os.environ.get("TACO_SORTED_WARPS"),
                  "ms": float(np.median(times)), ("exact_recount_steps" if rw else "windows_per_ant_step"):
                      int(scan.item()) if rw else int(scan.item()) / (args.m * (args.n - 1)),
                  "tour_checksum": int(tours.sum().item())}))
