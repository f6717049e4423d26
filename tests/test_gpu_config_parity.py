"""GPU parity at the BASELINE configs (BASELINE.json configs 2-5), on the
Solver's own late-iteration state.

For each config the Solver (device-built instance, the bench's parameters)
runs ITERS iterations; then, on its selection table for the next iteration:

* every production instantiation of the construction kernels — warp-per-ant
  MODE 1 / 2 / 3 x byte / bit-map visited set, the fused-length MODE 0, the
  lane-group kernels g4e2 / g4e4 / g8e2 / g8e4 / g16e2, and the dense
  full-row kernel — is forced (the TACO_SORTED_* knobs) and its tours of a
  spread sample of global ant ids must equal the C oracle's full-scan
  product rule (oracle/c/fastpath.c) bit for bit: the sorted stream
  (uniforms keyed by sorted position) for the sorted-table kernels, the dense
  stream (keyed by city) for the dense kernel.  Ants are independent and
  keyed by their global id, so restating a sample is exact.
* the Solver's own next iteration (production kernel choice) must give the
  same sampled tours, their lengths bit-exact (numpy's pairwise order over
  the device dist), and tau' / P / the selection table rows equal to the
  reference restatement (evaporate, rank-ordered deposit, transition) on a
  sample of rows: the fused 256-thread row kernel (n <= 7000), the
  512-thread one (C4) and the split update (C5 m = 65536, k = 6553).
* at C2 / C3 (AdaIR, gamma != 1) and C4 (IR) the selection-level agreement with the
  reference's f64 log-domain rule is COUNTED on the same uniforms and on
  refined 53-bit uniforms (oracle fastpath_c.count_mismatches) and written to
  $TACO_PARITY_REPORT (profiles/r02_selection_mismatches.json).
"""

import json
import os

import numpy as np
import pytest
import torch

import paper_2404_04895_b200 as taco
from paper_2404_04895_b200 import _device, _lib
from oracle import fastpath, fastpath_c, reference_port as ref

pytestmark = pytest.mark.gpu

ITERS = 20
CONFIGS = {
    # name: (n, m, selection, sampled ants)
    "c2": (1000, 1024, "adair", 64),
    "c2_m8192": (1000, 8192, "adair", 64),  # > 32 ants/SM with the byte visited set (warp MODE 2 + VIS8)
    "c3": (2392, 4096, "adair", 64),
    "c3_m4400": (2392, 4400, "adair", 32),  # 29.7 ants/SM: one 32-warp CTA per SM (warp MODE 3)
    "c4": (10000, 8192, "ir", 24),
    "c5_256": (5000, 256, "ir", 32),  # 1.7 ants/SM: the latency MODE 4 at n = 5000
    "c5_65536": (5000, 65536, "ir", 48),
}
# label -> (variant, env overrides)
KERNELS = {
    "auto": ("sorted", {}),
    "warp_vis8": ("sorted", {"TACO_SORTED_KERNEL": "warp"}),
    "warp_bits": ("sorted", {"TACO_SORTED_KERNEL": "warp", "TACO_SORTED_VIS": "bits"}),
    "warp_fused_len": ("sorted", {"TACO_SORTED_KERNEL": "warp", "TACO_SORTED_COST": "fused"}),
    # one CTA per SM: the issue-bound MODE 1 and the latency MODE 4 (<= 24 ants per SM by default)
    "warp_mode1": ("sorted", {"TACO_SORTED_KERNEL": "warp", "TACO_SORTED_MODE": "1"}),
    "warp_mode4": ("sorted", {"TACO_SORTED_KERNEL": "warp", "TACO_SORTED_MODE": "4"}),
    "g4e2": ("sorted", {"TACO_SORTED_KERNEL": "g4e2"}),
    "g4e4": ("sorted", {"TACO_SORTED_KERNEL": "g4e4"}),
    "g8e2": ("sorted", {"TACO_SORTED_KERNEL": "g8e2"}),
    "g8e4": ("sorted", {"TACO_SORTED_KERNEL": "g8e4"}),
    "g16e2": ("sorted", {"TACO_SORTED_KERNEL": "g16e2"}),
    "dense": ("dense", {}),
}
_ENV_KEYS = ("TACO_SORTED_KERNEL", "TACO_SORTED_VIS", "TACO_SORTED_COST", "TACO_SORTED_WARPS", "TACO_SORTED_MODE")


def _sample(m: int, count: int) -> np.ndarray:
    spread = np.linspace(0, m - 1, count - 8).astype(np.int64)
    extra = np.random.default_rng(m).integers(0, m, 8)
    return np.unique(np.concatenate([spread, extra, [0, m - 1]]))


def _with_env(env: dict, fn):
    old = {k: os.environ.get(k) for k in _ENV_KEYS}
    try:
        for k in _ENV_KEYS:
            os.environ.pop(k, None)
        os.environ.update(env)
        return fn()
    finally:
        for k, v in old.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v


def _pairwise_lengths(dist_dev: torch.Tensor, tours: np.ndarray) -> np.ndarray:
    """model.batch_costs (model.py:292-295) of host tours over the device dist:
    the gathered edges, then numpy's pairwise row sum."""
    t = torch.from_numpy(tours).to(dist_dev.device)
    edges = dist_dev[t, torch.roll(t, -1, dims=1)].cpu().numpy()
    return edges.sum(axis=1)


def _deposit_rows(elite_tours: np.ndarray, elite_costs: np.ndarray, rows: np.ndarray, n: int) -> np.ndarray:
    """Rows of accumulate_increments (pheromone.py:52-68): per elite in rank
    order, 1.0/cost onto (i, prev_i) and (i, next_i) — each cell at most once
    per elite, so the row-restricted sums are the reference's bit for bit."""
    d = np.zeros((rows.size, n))
    for t, c in zip(elite_tours, elite_costs):
        inc = 1.0 / float(c)
        pos = np.empty(n, dtype=np.int64)
        pos[t] = np.arange(n)
        s = pos[rows]
        d[np.arange(rows.size), t[(s - 1) % n]] += inc
        d[np.arange(rows.size), t[(s + 1) % n]] += inc
    return d


def _report(record: dict) -> None:
    path = os.environ.get("TACO_PARITY_REPORT")
    if path:
        with open(path, "a") as f:
            f.write(json.dumps(record) + "\n")


@pytest.fixture(scope="module")
def solvers():
    return {}


def _solver(solvers, name):
    if name not in solvers:
        n, m, sel, _ = CONFIGS[name]
        coords = np.random.default_rng(0).uniform(0.0, 2000.0, (n, 2))  # the bench instance
        params = taco.AcoParams(m=m, k=max(1, m // 10), selection=sel, seed=0,
                                gamma_schedule=taco.GammaSchedule(1.5, 1.0, 50))
        s = taco.Solver(taco.device_euclidean_instance(coords), params, graph=False)
        s.run(ITERS)
        solvers.clear()  # one config's state on the device at a time
        solvers[name] = s
    return solvers[name]


@pytest.mark.parametrize("name", list(CONFIGS))
def test_construction_kernels_match_oracle_at_config(solvers, name):
    n, m, sel, count = CONFIGS[name]
    s = _solver(solvers, name)
    it, seed = s.iteration, s.params.seed
    ants = _sample(m, count)
    w = s.tables.w[:, :n].cpu().numpy()
    wants = {"sorted": fastpath_c.build_tours_sorted(s.tables.sw.cpu().numpy(), s.tables.si.cpu().numpy(), seed,
                                                     it, ants, n=n)}
    assert fastpath_c.build_tours.last_fallbacks == 0
    if name != "c5_65536":
        wants["dense"] = fastpath_c.build_tours(w, seed, it, ants)
        assert fastpath_c.build_tours.last_fallbacks == 0
    dev = s.dev
    tours = torch.zeros((m, n), dtype=torch.int32, device=dev)
    costs = torch.zeros(m, dtype=torch.float64, device=dev)
    checked = []
    for label, (variant, env) in KERNELS.items():
        if variant == "dense" and name == "c5_65536":
            continue  # 6.5 TB of full-row streaming; dense is covered at the other configs
        code = _lib.CONSTRUCT_SORTED if variant == "sorted" else _lib.CONSTRUCT_DENSE
        status = _device.new_status(dev)
        tours.zero_()

        def run():
            _device.construct(n, m, 0, code, s.tables, seed, it, tours, status, dist=s.di.dist, costs_out=costs,
                              fallback=(s.tau, 1.0, s.eta_b), inv_gamma=1.0 / taco.colony.construction_gamma(s.params, it))
            torch.cuda.synchronize()

        try:
            _with_env(env, run)
        except _lib.TacoError as e:  # a forced layout that does not fit this config (shared memory)
            assert "unsupported" in str(e).lower(), (label, e)
            continue
        assert _device.read_status(status)[0] == 0, label
        want = wants[variant]
        got = tours[torch.from_numpy(ants).to(dev)].cpu().numpy()
        assert np.array_equal(got, want), f"{name}/{label}: tours differ from the oracle"
        assert np.array_equal(costs[torch.from_numpy(ants).to(dev)].cpu().numpy(),
                              _pairwise_lengths(s.di.dist, want)), f"{name}/{label}: lengths"
        checked.append(label)
    assert "auto" in checked and "dense" in checked or name == "c5_65536"
    _report({"test": "construction", "config": name, "n": n, "m": m, "iteration": it,
             "sampled_ants": int(ants.size), "kernels_bit_exact": checked})


@pytest.mark.parametrize("name", list(CONFIGS))
def test_solver_iteration_matches_reference_at_config(solvers, name):
    """The Solver's next iteration: production construction (sampled ants),
    lengths, elite order, tau' / P / W rows against the reference restatement."""
    n, m, sel, count = CONFIGS[name]
    s = _solver(solvers, name)
    it, seed, p = s.iteration, s.params.seed, s.params
    ants = _sample(m, count)
    want = fastpath_c.build_tours_sorted(s.tables.sw.cpu().numpy(), s.tables.si.cpu().numpy(), seed, it, ants, n=n)
    g = np.random.default_rng(it)
    rows = np.unique(np.concatenate([g.integers(0, n, 40), [0, n - 1]]))
    rows_t = torch.from_numpy(rows).to(s.dev)
    tau_rows = s.tau[rows_t].cpu().numpy()
    s.step()
    tours_all = s.tours_all
    got = tours_all[torch.from_numpy(ants).to(s.dev)].cpu().numpy()
    assert np.array_equal(got, want)
    costs = s.costs_all.cpu().numpy()
    assert np.array_equal(costs[ants], _pairwise_lengths(s.di.dist, want))
    order = ref.elite_ranks(costs, p.k)
    assert np.array_equal(s.order.cpu().numpy()[:p.k], order)
    elite_tours = tours_all[torch.from_numpy(order).to(s.dev)].cpu().numpy().astype(np.int64)
    delta = _deposit_rows(elite_tours, costs[order], rows, n)
    tau_new = ref.evaporate(tau_rows, delta, p.rho)
    assert np.array_equal(s.tau[rows_t].cpu().numpy(), tau_new)
    # P rows (colony.py:51-69) and the next selection table
    eta = s.di.eta[rows_t].cpu().numpy()
    unnorm = tau_new * (eta * eta)
    unnorm[np.arange(rows.size), rows] = 0.0
    p_rows = unnorm / np.array([r.sum() for r in unnorm])[:, None]
    p_dev = torch.empty_like(s.tau[:n])
    _device.row_update(n, tau_in=s.tau, eta_b=s.eta_b, want_p=True, alpha=float(p.alpha), p_out=p_dev)
    assert np.array_equal(p_dev[rows_t].cpu().numpy(), p_rows)
    del p_dev
    gamma = taco.colony.construction_gamma(p, s.iteration)
    w_new = s.tables.w[rows_t, :n].cpu().numpy()
    w_want = fastpath.selection_table(p_rows, gamma)
    if gamma == 1.0:
        assert np.array_equal(w_new, w_want)
    else:  # numpy's exp2/log2 vs CUDA's: at most one fp32 ulp
        d = np.abs(w_new.view(np.int32).astype(np.int64) - w_want.view(np.int32).astype(np.int64))
        assert d.max() <= 1
    _report({"test": "iteration", "config": name, "n": n, "m": m, "k": p.k, "iteration": it,
             "sampled_ants": int(ants.size), "sampled_rows": int(rows.size),
             "update_path": "split" if s._split_update else ("fused-512" if n > 7000 else "fused-256")})


@pytest.mark.parametrize("name", ["c2", "c3", "c4"])
def test_selection_mismatch_count_against_log_rule(solvers, name):
    """count where the fp32 product rule (the device's choice)
    differs from the reference's f64 log rule on the same uniforms, and from
    the log rule on refined 53-bit uniforms, along the device's own tours of
    a late iteration (C2 / C3 AdaIR with gamma != 1; C4 IR)."""
    n, m, sel, count = CONFIGS[name]
    s = _solver(solvers, name)
    it, seed = s.iteration, s.params.seed
    gamma = taco.colony.construction_gamma(s.params, it)
    assert gamma != 1.0 or CONFIGS[name][2] == "ir"
    ants = _sample(m, 4 * count)
    sw, si = s.tables.sw.cpu().numpy(), s.tables.si.cpu().numpy()
    pmat = s.probability().p
    logw = ref.log_table(pmat, gamma)
    # the production (sorted-stream) choices, checked against the device first
    tours = fastpath_c.build_tours_sorted(sw, si, seed, it, ants, n=n).astype(np.int32)
    dev_tours = torch.zeros((m, n), dtype=torch.int32, device=s.dev)
    _device.construct(n, m, 0, _lib.CONSTRUCT_SORTED, s.tables, seed, it, dev_tours, _device.new_status(s.dev))
    assert np.array_equal(dev_tours[torch.from_numpy(ants).to(s.dev)].cpu().numpy(), tours)
    c = fastpath_c.count_mismatches(sw, logw, seed, it, ants, tours, si=si)
    assert c["selections"] == ants.size * (n - 1)
    assert c["product_rule"] == 0
    rate = c["log_rule_same_u"] / c["selections"]
    _report({"test": "mismatch", "config": name, "n": n, "m": m, "iteration": it, "gamma": gamma,
             "sampled_ants": int(ants.size), **c, "rate_same_u": rate,
             "rate_u53": c["log_rule_u53"] / c["selections"]})
    # the fp32 table rounds W to 24 bits: disagreement with the f64 rule is
    # confined to near-ties (expected ~1e-7 per selection)
    assert rate < 1e-4
