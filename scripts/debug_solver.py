"""Debug helper: run Solver iterations with a sync after every launch."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
import paper_2404_04895_b200 as taco
from paper_2404_04895_b200 import _device, solver as S

for n, m in [(48, 32), (129, 16), (300, 64), (1000, 128), (2392, 256), (2392, 4096)]:
    inst = taco.euclidean_instance(np.random.default_rng(0).uniform(0, 2000, (n, 2)))
    params = taco.AcoParams(m=m, k=max(1, m // 10), selection="adair", seed=0)
    print("n", n, "m", m, flush=True)
    s = taco.Solver(inst, params)
    torch.cuda.synchronize(); print(" init ok", flush=True)
    for it in range(2):
        s.step(); torch.cuda.synchronize(); print(" step ok", it, s.best()[1], flush=True)
