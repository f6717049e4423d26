"""Row-update launch timing by row count (taco_row_update_rows, rows [0, R)):
separates the per-launch fixed cost (R = 148: one row per CTA) from the
per-row cost.  A sleep kernel ahead of each timed launch hides the host's
launch latency.  Random elites (the warp-fold deposit) or none.

    python scripts/row_range_probe.py <n> <k>
"""
import ctypes, os, sys
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2404_04895_b200 import _lib
n, k = int(sys.argv[1]), int(sys.argv[2])
dev = torch.device("cuda")
g = np.random.default_rng(n)
tau0 = torch.from_numpy(g.uniform(1e-6, 2.0, (n, n))).to(dev)
eta = torch.from_numpy(g.uniform(1e-4, 1.0, (n, n)) ** 2).to(dev)
base = [g.permutation(n) for _ in range(k)]
nbr = np.zeros((n, k, 2), dtype=np.int32)
for r, t in enumerate(base):
    nbr[t, r, 0], nbr[t, r, 1] = np.roll(t, 1), np.roll(t, -1)
nbr_t = torch.from_numpy(nbr).to(dev)
inc = torch.from_numpy(1.0 / g.uniform(1e5, 1e6, k)).to(dev)
ldw = -(-n // 32) * 32
lib = _lib.load()
fn = lib.taco_row_update_rows
tau = tau0.clone()
w = torch.zeros((n, ldw), dtype=torch.float32, device=dev)
rs = torch.zeros(n, dtype=torch.float64, device=dev)
st = torch.zeros(4, dtype=torch.int32, device=dev); st[1] = 2**31 - 1
for gamma in (1.0, 1.5):
  for nb in (0, 1):
    for R in (148, 296, 592, 1184, 2392):
        times = []
        for r in range(6):
            tau.copy_(tau0)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda._sleep(400000)  # covers the host's launch latency
            a.record()
            code = fn(0, R, n, tau.data_ptr(), tau.data_ptr(), eta.data_ptr(), nbr_t.data_ptr() if nb else None, inc.data_ptr(), k if nb else 0, None, None,
                      1, 0.9, 1, 1.0, 1.0 / gamma, None, rs.data_ptr(), w.data_ptr(), ldw, None, None, st.data_ptr(), None,
                      torch.cuda.current_stream().cuda_stream)
            b.record(); torch.cuda.synchronize(); assert code == 0, code
            if r: times.append(a.elapsed_time(b))
        print(f"gamma={gamma} deposit={nb} rows={R}: {np.median(times)*1000:.1f} us", flush=True)
