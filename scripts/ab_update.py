"""A/B of the row update (taco_row_update + the row sort, Solver mode) between
libtaco builds in one process: same inputs, CUDA-event timing, and the
outputs compared bit for bit.

    python scripts/ab_update.py <libA.so> <libB.so> [--n 10000 --k 819]
"""
import argparse
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2404_04895_b200 import _lib  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("libs", nargs="+")
ap.add_argument("--n", type=int, default=10000)
ap.add_argument("--k", type=int, default=819)
ap.add_argument("--gamma", type=float, default=1.0)
ap.add_argument("--reps", type=int, default=7)
ap.add_argument("--same", type=int, default=1, help="distinct elite tours (k // same copies each: converged colony)")
args = ap.parse_args()
n, k = args.n, args.k
dev = torch.device("cuda")
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
ldw = -(-n // 32) * 32
sig = _lib.SIGNATURES["taco_row_update"]
results = {}
for path in args.libs:
    lib = ctypes.CDLL(path)
    fn = lib.taco_row_update
    fn.restype, fn.argtypes = sig
    tau = tau0.clone()
    w = torch.zeros((n, ldw), dtype=torch.float32, device=dev)
    sw = torch.zeros_like(w)
    si = torch.zeros((n, ldw), dtype=torch.int16, device=dev)
    rs = torch.zeros(n, dtype=torch.float64, device=dev)
    st = torch.zeros(4, dtype=torch.int32, device=dev)
    st[1] = 2**31 - 1
    times = []
    for r in range(args.reps + 1):
        tau.copy_(tau0)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        code = fn(n, tau.data_ptr(), tau.data_ptr(), eta.data_ptr(), nbr_t.data_ptr(), inc.data_ptr(), k, None, None,
                  1, 0.9, 1, 1.0, 1.0 / args.gamma, None, rs.data_ptr(), w.data_ptr(), ldw, sw.data_ptr(),
                  si.data_ptr(), st.data_ptr(), None, torch.cuda.current_stream().cuda_stream)
        b.record()
        torch.cuda.synchronize()
        assert code == 0, code
        if r:
            times.append(a.elapsed_time(b))
    results[path] = [x.cpu().numpy() for x in (tau, rs, si)]
    print(f"{path}: {np.median(times):.3f} ms (min {min(times):.3f})", flush=True)
if len(results) < 2:
    sys.exit(0)
a, b = list(results.values())[:2]
print("tau, rowsum, sorted indices identical:", [bool(np.array_equal(x, y)) for x, y in zip(a, b)])
