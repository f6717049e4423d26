"""Exercise every libtaco kernel once at small sizes (crash / status smoke; also
the input for compute-sanitizer where a pool allows it):

    python scripts/kernel_smoke.py
    compute-sanitizer --tool memcheck python scripts/kernel_smoke.py

"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2404_04895_b200 as taco  # noqa: E402
from paper_2404_04895_b200 import _device, _lib  # noqa: E402

g = np.random.default_rng(0)
n, m = 37, 21
coords = g.uniform(0, 1000, (n, 2))
inst = taco.device_euclidean_instance(coords)
host_inst = taco.euclidean_instance(coords)
for sel in ("adair", "ir", "rw"):
    params = taco.AcoParams(m=m, k=3, selection=sel, seed=1, gamma_schedule=taco.GammaSchedule(1.5, 1.0, 4))
    for construct in ("sorted", "dense"):
        s = taco.Solver(inst, params, construct=construct, graph=False)
        s.run(2)
    taco.Solver(inst, params, graph=True).run(3)
params = taco.AcoParams(m=m, k=3, selection="adair", seed=1)
taco.Solver(host_inst, params, stream="replay").run(1)
prob = taco.compute_probability_matrix(taco.PheromoneState.initial(n, 1.0), host_inst, params)
for stream in ("numpy", "replay"):
    taco.construct_tours(prob, host_inst, params, 0, stream=stream)
rw = taco.AcoParams(m=m, k=3, selection="rw", seed=1)
taco.construct_tours(prob, host_inst, rw, 0, stream="numpy")
# lane-group kernels: force them through the env knob in-process
dev = _device.device()
t = _device.SelectionTables(n, dev, dense=True, sorted_=True)
_device.selection_table_from_p(_device.upload(prob.p, dev), 1 / 1.3, t)
tours = torch.zeros((m, n), dtype=torch.int32, device=dev)
costs = torch.zeros(m, dtype=torch.float64, device=dev)
for knob in ("g4e4", "g8e2", "g16e2", "warp"):
    os.environ["TACO_SORTED_KERNEL"] = knob
    _device.construct(n, m, 0, _lib.CONSTRUCT_SORTED, t, 5, 1, tours, _device.new_status(dev), dist=inst.dist,
                      costs_out=costs)
os.environ.pop("TACO_SORTED_KERNEL")
batch = taco.TourBatch(tours=tours.cpu().numpy().astype(np.int64), costs=costs.cpu().numpy())
elites = taco.select_elite(batch, 4)
delta = taco.accumulate_increments(elites, n)
taco.apply_update(taco.PheromoneState.initial(n, 1.0), delta, 0.1)
taco.batch_costs(batch.tours, host_inst)
taco.scaled_log_weights(prob.p, 1.3)
big = taco.AcoParams(m=17000, k=5, selection="ir", seed=3)  # CUB elite sort path (m > 16384)
taco.Solver(inst, big, graph=False).run(1)
# gamma < 1: stalled tours rebuilt in-kernel (MODE 1, lane groups, dense) and
# by k_rebuild_stalled (MODE 2, > 32 ants per SM)
pts = g.uniform(0.0, 10.0, (n, 2))
pts[n // 2:] += 1e4
far = taco.device_euclidean_instance(pts)
for mm, knob in ((m, None), (m, "g8e2"), (5000, "warp")):
    if knob:
        os.environ["TACO_SORTED_KERNEL"] = knob
    greedy = taco.AcoParams(m=mm, k=3, selection="adair", seed=2, gamma_schedule=taco.GammaSchedule(1.0, 0.1, 4))
    for construct in ("sorted", "dense"):
        taco.Solver(far, greedy, construct=construct, graph=False).run(3)
    os.environ.pop("TACO_SORTED_KERNEL", None)
# argmax_select_block drop-in
logw = np.log(g.uniform(0.0, 1.0, (n, n)))
taco.argmax_select_block(logw, g.integers(0, n, m), g.standard_exponential((m, n)), g.uniform(size=(m, n)) < 0.3,
                         np.empty((m, n)))
torch.cuda.synchronize()
print("kernel smoke: ok")
