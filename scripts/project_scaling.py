"""Projected multi-GPU scaling from one-GPU measurements.

Only single-GPU boxes are available, so the R-rank iteration is assembled
from its measured parts on one B200:
  construct(m/R)   the construction launch of one rank's m/R ants (its global
                   offset does not matter: the stream is keyed by ant id),
                   timed on the Solver's real late-iteration tables
  rest             elite rank over all m lengths + best tracking + edge map
                   (every rank runs them on the gathered lengths / elite tours)
  update           the replicated row update + row sort (every rank, all rows)
  exchange(R)      the collectives of the costs-first exchange (solver.py):
                   all-gather of the m f64 lengths, SUM all-reduce of the k x n
                   int32 elite tours (+1 stop word), MAX all-reduce of the
                   status key — modelled as 3 x ALPHA + bytes / BW with the
                   NCCL-over-NVSwitch constants below (assumptions, stated)
The per-step latency floor (construction at one ant per SM) bounds the
strong-scaling speed-up whatever the exchange costs.

    python scripts/project_scaling.py --n 2392 --m 4096 [--sel adair]
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

ALPHA_US = 12.0       # assumed NCCL small-message collective latency, 8 x B200 over NVSwitch
ALLGATHER_GBPS = 600.0  # assumed all-gather bus bandwidth per GPU
ALLREDUCE_GBPS = 400.0  # assumed all-reduce (NVLS) algorithm bandwidth

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=2392)
ap.add_argument("--m", type=int, default=4096)
ap.add_argument("--sel", default="adair")
ap.add_argument("--iters", type=int, default=20)
ap.add_argument("--out", default=None)
args = ap.parse_args()

n, m, k = args.n, args.m, max(1, args.m // 10)
coords = np.random.default_rng(0).uniform(0.0, 2000.0, (n, 2))
params = taco.AcoParams(m=m, k=k, selection=args.sel, seed=0, gamma_schedule=taco.GammaSchedule(1.5, 1.0, 50))
s = taco.Solver(taco.device_euclidean_instance(coords), params, graph=False)
s.run(args.iters)
torch.cuda.synchronize()


def timed(fn, reps=5):
    out = []
    for _ in range(reps + 1):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        out.append(a.elapsed_time(b))
    return float(np.median(out[1:]))


# whole iterations, and the construction / update parts of them
timers = {"construct": [], "update": []}
t_iter = timed(lambda: s.step_async(timers=timers))
t_con_full = float(np.median([a.elapsed_time(b) for a, b in timers["construct"]]))
t_upd = float(np.median([a.elapsed_time(b) for a, b in timers["update"]]))
t_rest = max(0.0, t_iter - t_con_full - t_upd)

tours = torch.zeros((m, n), dtype=torch.int32, device=s.dev)
costs = torch.zeros(m, dtype=torch.float64, device=s.dev)
st = _device.new_status(s.dev)
sms = torch.cuda.get_device_properties(s.dev).multi_processor_count


def construct(count):
    return timed(lambda: _device.construct(n, count, 0, s._variant, s.tables, 0, s.iteration, tours, st,
                                           dist=s.di.dist, costs_out=costs))


rows = []
for R in (1, 2, 4, 8):
    t_con = construct(m // R)
    ag_bytes = 8 * m
    ar_bytes = 4 * (k * n + 1)
    t_x = 0.0 if R == 1 else (3 * ALPHA_US * 1e-3 + ag_bytes * (R - 1) / R / (ALLGATHER_GBPS * 1e6)
                              + ar_bytes * 2 * (R - 1) / R / (ALLREDUCE_GBPS * 1e6))
    t = t_con + t_rest + t_upd + t_x
    rows.append({"R": R, "ants_per_rank": m // R, "construct_ms": t_con, "rest_ms": t_rest, "update_ms": t_upd,
                 "exchange_ms_model": t_x, "iteration_ms": t, "it_per_s": 1000.0 / t})
base = rows[0]["it_per_s"]
for r in rows:
    r["speedup"] = r["it_per_s"] / base
    r["efficiency"] = r["speedup"] / r["R"]
floor = construct(min(m, sms))
out = {"n": n, "m": m, "k": k, "selection": args.sel, "iteration_ms_measured_1gpu": t_iter,
       "construct_floor_ms_one_ant_per_sm": floor,
       "speedup_ceiling": t_iter / (floor + t_rest + t_upd),
       "assumptions": {"alpha_us": ALPHA_US, "allgather_GBps": ALLGATHER_GBPS, "allreduce_GBps": ALLREDUCE_GBPS},
       "projection": rows}
print(json.dumps(out))
if args.out:
    with open(args.out, "w") as f:
        json.dump(out, f, indent=1)
