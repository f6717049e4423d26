"""Time k_row_update phases at C3 size: no deposit / k elites (random or
identical tours) / P-only, to locate its bottleneck."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2404_04895_b200 as taco  # noqa: E402
from paper_2404_04895_b200 import _device  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 2392
dev = _device.device()
g = np.random.default_rng(0)
tau = torch.from_numpy(g.uniform(0.1, 1.0, (n, n))).to(dev)
eta = torch.from_numpy(g.uniform(0.1, 1.0, (n, n))).to(dev)
tables = _device.SelectionTables(n, dev, dense=True, sorted_=True)
rowsum = torch.zeros(n, dtype=torch.float64, device=dev)
st = _device.new_status(dev)


def timeit(fn, reps=10):
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps * 1e3


def nbr_for(k, same):
    tours = np.stack([g.permutation(n) for _ in range(1 if same else k)])
    if same:
        tours = np.repeat(tours, k, axis=0)
    nbr = np.zeros((n, k, 2), dtype=np.int32)
    for r, t in enumerate(tours):
        prev, nxt = np.roll(t, 1), np.roll(t, -1)
        nbr[t, r, 0] = prev
        nbr[t, r, 1] = nxt
    return torch.from_numpy(nbr).to(dev)


for label, k, same in (("no deposit", 0, False), ("k=1", 1, False), ("k=409 random", 409, False),
                       ("k=409 identical", 409, True)):
    nb = nbr_for(k, same) if k else None
    inc = torch.full((max(k, 1),), 1e-5, dtype=torch.float64, device=dev)
    tout = tau.clone()

    def run():
        _device.row_update(n, tau_in=tout, tau_out=tout, eta_b=eta, nbr=nb, inc=inc if k else None, k=k,
                           do_evap=True, keep=0.9, want_p=True, alpha=1.0, inv_gamma=1 / 1.3, rowsum_out=rowsum,
                           w_out=tables.w, ldw=tables.ldw, sw_out=None, si_out=None, status=st)
    print(f"{label:18s} row_update (no sort) {timeit(run):8.1f} us")

tout = tau.clone()
print("evaporation only (tau r/w):", round(timeit(lambda: _device.row_update(
    n, tau_in=tout, tau_out=tout, do_evap=True, keep=0.9)), 1), "us")
print("P + W, gamma = 1 (no pow):", round(timeit(lambda: _device.row_update(
    n, tau_in=tout, eta_b=eta, want_p=True, alpha=1.0, inv_gamma=1.0, rowsum_out=rowsum, w_out=tables.w,
    ldw=tables.ldw, status=st)), 1), "us")
print("P + W, gamma = 1.3 (pow):", round(timeit(lambda: _device.row_update(
    n, tau_in=tout, eta_b=eta, want_p=True, alpha=1.0, inv_gamma=1 / 1.3, rowsum_out=rowsum, w_out=tables.w,
    ldw=tables.ldw, status=st)), 1), "us")
print("P + W + sort, gamma = 1.3:", round(timeit(lambda: _device.row_update(
    n, tau_in=tout, eta_b=eta, want_p=True, alpha=1.0, inv_gamma=1 / 1.3, rowsum_out=rowsum, w_out=tables.w,
    ldw=tables.ldw, sw_out=tables.sw, si_out=tables.si, status=st)), 1), "us")

dout = torch.empty_like(tau)
for label, k, same in (("k=409 random", 409, False), ("k=409 identical", 409, True), ("k=40 identical", 40, True)):
    nb = nbr_for(k, same)
    inc = torch.full((k,), 1e-5, dtype=torch.float64, device=dev)
    print(f"deposit only (delta_out) {label}:", round(timeit(lambda: _device.row_update(
        n, nbr=nb, inc=inc, k=k, delta_out=dout)), 1), "us")

# split path (taco_update_split): deposit / evaporation+unnorm / normalize kernels
dws, uws = torch.empty_like(tau), torch.empty_like(tau)
for label, k, same in (("no deposit", 0, False), ("k=409 random", 409, False), ("k=409 identical", 409, True)):
    nb = nbr_for(k, same) if k else None
    inc = torch.full((max(k, 1),), 1e-5, dtype=torch.float64, device=dev)
    tout = tau.clone()
    print(f"split {label:16s} (no sort)", round(timeit(lambda: _device.update_split(
        n, tau_in=tout, tau_out=tout, eta_b=eta, nbr=nb, inc=inc if k else None, k=k, do_evap=True, keep=0.9,
        alpha=1.0, inv_gamma=1 / 1.3, delta_ws=dws, unnorm_ws=uws, rowsum_out=rowsum, w_out=tables.w,
        ldw=tables.ldw, status=st)), 1), "us")
