"""Phase timing of the end-to-end path (instance -> Solver -> K x step())."""
import sys
import os
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2404_04895_b200 as taco  # noqa: E402
from paper_2404_04895_b200 import _device  # noqa: E402

n, m = int(sys.argv[1]), int(sys.argv[2])
coords = np.random.default_rng(0).uniform(0.0, 2000.0, (n, 2))
inst = taco.euclidean_instance(coords)
params = taco.AcoParams(m=m, k=max(1, m // 10), selection="adair", seed=0)


def phases(kind):
    torch.cuda.synchronize()
    t = [time.perf_counter()]
    di = taco.device_euclidean_instance(coords) if kind == "dev" else inst
    torch.cuda.synchronize(); t.append(time.perf_counter())
    s = taco.Solver(di, params)
    torch.cuda.synchronize(); t.append(time.perf_counter())
    s.step()
    t.append(time.perf_counter())
    s.step()
    t.append(time.perf_counter())
    for _ in range(18):
        s.step()
    t.append(time.perf_counter())
    _device._INSTANCES.clear()
    return [round((b - a) * 1e3, 3) for a, b in zip(t, t[1:])]


for rep in range(3):
    for kind in ("dev", "host"):
        print(kind, rep, "inst, solver, step1(eager), step2(capture), 18 steps [ms]:", phases(kind))
