"""Solver-mode update paths on the same inputs: the fused row kernel
(taco_row_update) and the split kernels (taco_update_split) — timing (CUDA
events, median) and bit-equality of tau', the row sums, W and the sorted
table.  (Round 2 also measured a two-pass streaming update here — a warp per
(row, pairwise leaf) tile, then a warp per row: bit-exact but 0.52 vs 0.19 ms
at C3 and 9.3 vs 2.25 ms at C4, see profiles/README.md.)

    python scripts/update_paths.py --n 2392 --k 409 [--same 4] [--gamma 1.3]
"""
import argparse
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2404_04895_b200 import _device  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=2392)
ap.add_argument("--k", type=int, default=409)
ap.add_argument("--same", type=int, default=1)
ap.add_argument("--gamma", type=float, default=1.3)
ap.add_argument("--reps", type=int, default=7)
args = ap.parse_args()
n, k = args.n, args.k
dev = _device.device()
g = np.random.default_rng(n)
tau0 = torch.from_numpy(g.uniform(1e-6, 2.0, (n, n))).to(dev)
eta = torch.from_numpy(g.uniform(1e-4, 1.0, (n, n)) ** 2).to(dev)
base = [g.permutation(n) for _ in range(max(1, k // args.same))]
tours = np.stack([base[r % len(base)] for r in range(k)])
nbr = np.zeros((n, k, 2), dtype=np.int32)
for r, t in enumerate(tours):
    nbr[t, r, 0], nbr[t, r, 1] = np.roll(t, 1), np.roll(t, -1)
nbr_t = torch.from_numpy(nbr).to(dev)
inc = torch.from_numpy(1.0 / g.uniform(1e5, 1e6, k)).to(dev)
delta_ws, unnorm_ws = torch.empty_like(tau0), torch.empty_like(tau0)
out = {}
for path in ("fused", "split"):
    tau = tau0.clone()
    t = _device.SelectionTables(n, dev, dense=True, sorted_=True)
    rs = torch.zeros(n, dtype=torch.float64, device=dev)
    st = _device.new_status(dev)
    common = dict(tau_in=tau, tau_out=tau, eta_b=eta, nbr=nbr_t, inc=inc, k=k, do_evap=True, keep=0.9, alpha=1.0,
                  inv_gamma=1.0 / args.gamma, rowsum_out=rs, w_out=t.w, ldw=t.ldw, sw_out=t.sw, si_out=t.si,
                  status=st)
    times = []
    for r in range(args.reps + 1):
        tau.copy_(tau0)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        if path == "fused":
            _device.row_update(n, want_p=True, **common)
        else:
            _device.update_split(n, delta_ws=delta_ws, unnorm_ws=unnorm_ws, **common)
        b.record()
        torch.cuda.synchronize()
        if r:
            times.append(a.elapsed_time(b))
    assert _device.read_status(st)[0] == 0
    out[path] = [x.cpu().numpy() for x in (tau, rs, t.w, t.sw, t.si)]
    print(f"{path:6s} {np.median(times):.3f} ms (min {min(times):.3f})", flush=True)
for path in ("split",):
    print(path, "== fused:", [bool(np.array_equal(x, y)) for x, y in zip(out["fused"], out[path])])
