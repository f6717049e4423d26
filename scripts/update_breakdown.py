"""Row-update time on a Solver's real late-iteration state: the full update
(deposit + evaporation + P/W + sort) against the same without the deposit and
without the sort, to size the deposit's share.  (Round 2
also measured a per-row pre-fold of the deposit into a shared-memory hash of
the row's distinct columns, k_deposit_lists: bit-identical but slower — C4
3.12 vs 2.79 ms, n = 5000 0.66 vs 0.58 — the hash, sized for the worst case
of 2k distinct columns, leaves 4 warps per SM.)

    python scripts/update_breakdown.py --n 2392 --m 4096 --iters 20
"""
import argparse
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2404_04895_b200 as taco  # noqa: E402
from paper_2404_04895_b200 import _device  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=2392)
ap.add_argument("--m", type=int, default=4096)
ap.add_argument("--sel", default="adair")
ap.add_argument("--iters", type=int, default=20)
args = ap.parse_args()
coords = np.random.default_rng(0).uniform(0.0, 2000.0, (args.n, 2))
params = taco.AcoParams(m=args.m, k=max(1, args.m // 10), selection=args.sel, seed=0,
                        gamma_schedule=taco.GammaSchedule(1.5, 1.0, 50))
s = taco.Solver(taco.device_euclidean_instance(coords), params, graph=False)
s.run(args.iters)
torch.cuda.synchronize()
n, t = s.n, s.tables
tau0 = s.tau.clone()
gamma = taco.colony.construction_gamma(params, s.iteration)


def run(deposit: bool, sort: bool, reps=7):
    out = []
    for r in range(reps + 1):
        tau = tau0.clone()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        _device.row_update(n, tau_in=tau, tau_out=tau, eta_b=s.eta_b, nbr=s.nbr if deposit else None,
                           inc=s.inc if deposit else None, k=params.k if deposit else 0, do_evap=True, keep=s.keep,
                           want_p=True, alpha=float(params.alpha), inv_gamma=1.0 / gamma, rowsum_out=s.rowsum,
                           w_out=t.w, ldw=t.ldw, sw_out=t.sw if sort else None, si_out=t.si if sort else None,
                           status=s.status)
        b.record()
        torch.cuda.synchronize()
        if r:
            out.append(a.elapsed_time(b))
    return float(np.median(out))


full, nodep, nosort = run(True, True), run(False, True), run(True, False)
# elite-edge statistics of this state: distinct deposit columns per row
nbr = s.nbr.cpu().numpy()
distinct = np.array([len(np.unique(nbr[i].ravel())) for i in range(0, n, max(1, n // 200))])
print({"n": n, "m": args.m, "k": params.k, "iteration": s.iteration, "full_ms": full, "no_deposit_ms": nodep,
       "no_sort_ms": nosort, "deposit_ms": full - nodep, "sort_ms": full - nosort,
       "distinct_deposit_columns_per_row": {"median": float(np.median(distinct)), "max": int(distinct.max())}})
