"""One Solver iteration at a large n (beyond the sorted table and the fused
row kernel): dense construction + split update."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2404_04895_b200 as taco  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 30000
m = int(sys.argv[2]) if len(sys.argv) > 2 else 256
coords = np.random.default_rng(0).uniform(0, 2000, (n, 2))
t0 = time.perf_counter()
inst = taco.device_euclidean_instance(coords)
s = taco.Solver(inst, taco.AcoParams(m=m, k=max(1, m // 10), selection="ir", seed=0))
torch.cuda.synchronize()
t1 = time.perf_counter()
tour, length = s.step()
t2 = time.perf_counter()
assert sorted(tour.tolist()) == list(range(n))
print({"n": n, "m": m, "construct": s.construct, "split_update": s._split_update, "setup_s": round(t1 - t0, 2),
       "iteration_s": round(t2 - t1, 3), "best": length, "mem_GB": round(torch.cuda.max_memory_allocated() / 1e9, 1)})
