"""GPU parity: the CUDA path through the C ABI against the oracle and the
golden vectors of the reference.

Bars (BASELINE.json north_star): tours / argmax choices bit-exact given the
same P and the same uniform stream; P, tau, deltas bit-exact (alpha, beta in
numpy's exact power set) else <= 1e-12 relative (tolerance well inside the
1e-6 the north star allows); tour lengths bit-exact (pairwise order).
"""

import os

import numpy as np
import pytest
import torch

import paper_2404_04895_b200 as taco
from paper_2404_04895_b200 import _device, _lib
from paper_2404_04895_b200 import rng as trng
from conftest import euclid
from oracle import fastpath, reference_port as ref

pytestmark = pytest.mark.gpu


def _params(golden, name, seed):
    n, m, k, iters, alpha, beta, rho, period, sel = golden[f"{name}/meta"]
    return taco.AcoParams(m=int(m), k=int(k), alpha=alpha, beta=beta, rho=rho,
                          selection=("ir", "adair", "rw")[int(sel)],
                          gamma_schedule=taco.GammaSchedule(1.5, 1.0, int(period)), seed=seed), int(iters)


def _inst(golden, name):
    return taco.TspInstance(n=golden[f"{name}/dist"].shape[0], dist=golden[f"{name}/dist"],
                            eta=golden[f"{name}/eta"])


# ---------------------------------------------------------------------------
# RNG
# ---------------------------------------------------------------------------
def test_device_philox_known_answers():
    dev = _device.device()
    ctr = torch.tensor([[0, 0], [-1, -1], [0x243F6A88, 0x85A308D3 - 2**32]], dtype=torch.int32, device=dev)
    key = torch.tensor([0, -1, 0x13198A2E], dtype=torch.int32, device=dev)
    out = torch.empty((3, 2), dtype=torch.int32, device=dev)
    _lib.check(_lib.load().taco_philox2x32_10(3, ctr.data_ptr(), key.data_ptr(), out.data_ptr(),
                                              _device.stream_handle()), "philox")
    got = out.cpu().numpy().astype(np.uint32)
    assert got.tolist() == [[0xFF1DAE59, 0x6CD10DF2], [0x2C3F628B, 0xAB4FD7AD], [0xDD7CE038, 0xF62A4C12]]


def test_device_uniforms_and_starts_match_restatement():
    g = np.random.default_rng(0)
    step = g.integers(1, 5000, 4096)
    ant = g.integers(0, 70000, 4096)
    city = g.integers(0, 10000, 4096)
    seed = 2**40 + 12345
    u = trng.device_uniforms(seed, 77, step, ant, city)
    assert np.array_equal(u, fastpath.uniforms(seed, 77, step, ant, city))
    assert np.array_equal(trng.device_starts(seed, 3, 2392, 4096, ant_offset=100),
                          fastpath.starts(seed, 3, np.arange(100, 4196), 2392))
    # the counter's extremes (n <= 65535: city, step <= 65534), 32-bit ants,
    # iterations and seeds whose key wraps around 2^32
    step = np.array([1, 65534, 65534, 1, 40000, 2])
    city = np.array([65534, 65534, 0, 1, 65533, 32768])
    ant = np.array([0, 2**32 - 1, 2**31, 7, 123456789, 2**32 - 2])
    for seed_, it in ((0, 0), (2**64 - 1, 2**32 - 1), (5, 2**31 + 3)):
        assert np.array_equal(trng.device_uniforms(seed_, it, step, ant, city),
                              fastpath.uniforms(seed_, it, step, ant, city))
        assert np.array_equal(trng.device_starts(seed_, it, 65535, 64, ant_offset=2**31 - 64),
                              fastpath.starts(seed_, it, np.arange(2**31 - 64, 2**31), 65535))


# ---------------------------------------------------------------------------
# drop-ins against the reference's golden pipeline
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("stream", ["numpy", "replay"])
@pytest.mark.parametrize("name", ["int12_ir", "int12_adair", "euc23_adair", "euc17_ab"])
def test_dropin_pipeline_matches_reference_golden(golden, name, stream):
    inst = _inst(golden, name)
    for seed in golden[f"{name}/seeds"].tolist():
        params, iters = _params(golden, name, seed)
        tau = taco.PheromoneState.initial(inst.n, params.q0_tau)
        prob = taco.compute_probability_matrix(tau, inst, params)
        for it in range(iters):
            key = f"{name}/s{seed}/it{it}"
            if params.alpha in (0.5, 1.0, 2.0) and params.beta in (0.0, 0.5, 1.0, 2.0):
                assert np.array_equal(prob.p, golden[f"{key}/p"])
            else:
                np.testing.assert_allclose(prob.p, golden[f"{key}/p"], rtol=1e-12, atol=0)
            # reference-stream replay: feed the golden P so tours are comparable bitwise
            batch = taco.construct_tours(taco.ProbabilityMatrix(golden[f"{key}/p"]), inst, params, it,
                                         stream=stream)
            assert np.array_equal(batch.tours, golden[f"{key}/tours"])
            assert np.array_equal(batch.costs, golden[f"{key}/costs"])
            elites = taco.select_elite(batch, params.k)
            assert [c for _, c in elites] == golden[f"{key}/costs"][golden[f"{key}/order"]].tolist()
            delta = taco.accumulate_increments(elites, inst.n)
            assert np.array_equal(delta, golden[f"{key}/delta"])
            tau = taco.apply_update(tau, delta, params.rho)
            assert np.array_equal(tau.tau, golden[f"{key}/tau"])
            assert tau.iteration == it + 1
            prob = taco.compute_probability_matrix(tau, inst, params)


@pytest.mark.parametrize("stream", ["numpy", "replay"])
@pytest.mark.parametrize("mech", ["ir", "adair"])
@pytest.mark.parametrize("n,m", [(5, 1), (10, 7), (51, 64)])
def test_reference_stream_tours_bit_exact(mech, n, m, stream):
    inst = euclid(n + m, n)
    for seed in range(3):
        params = taco.AcoParams(m=m, k=1, selection=mech, seed=seed,
                                gamma_schedule=taco.GammaSchedule(1.5, 1.0, 7))
        tau = ref.initial_tau(n, 1.0)
        p = ref.transition(tau, inst.eta, 1.0, 2.0)
        for it in (0, 3):
            got = taco.construct_tours(taco.ProbabilityMatrix(p), inst, params, it, stream=stream)
            want = ref.build_tours(p, m, seed, it, ref.gamma(it, 1.5, 1.0, 7) if mech == "adair" else 1.0)
            assert np.array_equal(got.tours, want)
            assert np.array_equal(got.costs, ref.lengths(want, inst.dist))


@pytest.mark.parametrize("n,m", [(257, 300), (600, 512)])
def test_device_replay_of_reference_stream_at_scale(n, m):
    # 77k / 307k deviates per step decoded on the device from numpy's Philox
    # keys (slow ziggurat paths included): the reference's tours exactly
    inst = euclid(n, n)
    g = np.random.default_rng(n)
    tau = g.uniform(0.05, 3.0, (n, n))
    p = ref.transition((tau + tau.T) / 2, inst.eta, 1.0, 2.0)
    params = taco.AcoParams(m=m, k=1, selection="adair", seed=99,
                            gamma_schedule=taco.GammaSchedule(1.5, 1.0, 10))
    got = taco.construct_tours(taco.ProbabilityMatrix(p), inst, params, 3, stream="replay")
    want = ref.build_tours(p, m, 99, 3, ref.gamma(3, 1.5, 1.0, 10))
    assert np.array_equal(got.tours, want)
    assert np.array_equal(got.costs, ref.lengths(want, inst.dist))


# ---------------------------------------------------------------------------
# fast path: both construction variants against the product-rule restatement
# ---------------------------------------------------------------------------
def _device_tables(p, gamma):
    dev = _device.device()
    n = p.shape[0]
    t = _device.SelectionTables(n, dev, dense=True, sorted_=True)
    _device.selection_table_from_p(_device.upload(p, dev), 1.0 / gamma, t)
    return t


@pytest.mark.parametrize("n,m,gamma", [(3, 4, 1.0), (7, 5, 1.0), (40, 33, 1.0), (97, 64, 1.37),
                                         (300, 40, 1.5), (700, 150, 1.2)])
def test_fast_construction_matches_restatement(n, m, gamma):
    inst = euclid(n, n)
    g = np.random.default_rng(n)
    tau = g.uniform(0.05, 3.0, (n, n))
    tau = (tau + tau.T) / 2
    p = ref.transition(tau, inst.eta, 1.0, 2.0)
    t = _device_tables(p, gamma)
    w = t.w[:, :n].cpu().numpy()
    # the tables hold exactly fp32(P^(1/gamma)), row-sorted descending
    if gamma == 1.0:
        assert np.array_equal(w, fastpath.selection_table(p, 1.0))
    sw, si = t.sw[:, :n].cpu().numpy(), t.si[:, :n].cpu().numpy().astype(np.int64)
    assert (t.sw[:, n:] == 0).all()  # pad columns are never selectable
    assert np.array_equal(np.take_along_axis(w, si, axis=1), sw)
    # rows descend in the W bits above bit 16, ties keep ascending column order
    prefix = (sw.view(np.uint32) >> 16).astype(np.int64)
    assert (np.diff(prefix, axis=1) <= 0).all()
    same = np.diff(prefix, axis=1) == 0
    assert (np.diff(si, axis=1)[same] > 0).all()
    assert (np.sort(si, axis=1) == np.arange(n)).all()
    seed, it = 11, 5
    # two streams: uniforms keyed by sorted position (sorted kernels) or by city (dense)
    wants = {_lib.CONSTRUCT_SORTED: fastpath.build_tours_sorted(sw, si, seed, it, np.arange(m)),
             _lib.CONSTRUCT_DENSE: fastpath.build_tours(w, seed, it, np.arange(m))}
    dist = _device.upload(inst.dist, t.w.device)
    for variant in (_lib.CONSTRUCT_SORTED, _lib.CONSTRUCT_DENSE):
        want = wants[variant]
        tours = torch.zeros((m, n), dtype=torch.int32, device=t.w.device)
        costs = torch.zeros(m, dtype=torch.float64, device=t.w.device)
        status = _device.new_status(t.w.device)
        _device.construct(n, m, 0, variant, t, seed, it, tours, status, dist=dist, costs_out=costs)
        assert _device.read_status(status)[0] == 0
        assert np.array_equal(tours.cpu().numpy(), want), variant
        # lengths accumulated during construction == numpy's pairwise batch_costs
        assert np.array_equal(costs.cpu().numpy(), ref.lengths(want, inst.dist)), variant


def test_fast_rule_agrees_with_reference_log_rule():
    # same device uniforms, reference log-domain rule vs the fast kernel
    n, m = 120, 48
    inst = euclid(5, n)
    p = ref.transition(ref.initial_tau(n, 1.0), inst.eta, 1.0, 2.0)
    params = taco.AcoParams(m=m, k=1, selection="ir", seed=4)
    # the dense (city-keyed) stream; the sorted stream's count is in test_gpu_config_parity
    got = taco.construct_tours(taco.ProbabilityMatrix(p), inst, params, 2, variant="dense").tours
    want = fastpath.log_rule_tours(p, 1.0, 4, 2, np.arange(m))
    mismatches = int((got != want).any(axis=1).sum())
    assert mismatches == 0


def test_dense_and_sorted_match_their_oracles_at_scale():
    from oracle import fastpath_c

    n, m = 1000, 256
    inst = euclid(1, n)
    params = taco.AcoParams(m=m, k=25, selection="adair", seed=3)
    p = taco.compute_probability_matrix(taco.PheromoneState.initial(n, 1.0), inst, params)
    a = taco.construct_tours(p, inst, params, 0, variant="sorted")
    b = taco.construct_tours(p, inst, params, 0, variant="dense")
    t = _device_tables(p.p, taco.gamma_at(0, params.gamma_schedule))
    ants = np.arange(m)
    assert np.array_equal(a.tours, fastpath_c.build_tours_sorted(t.sw.cpu().numpy(), t.si.cpu().numpy(), 3, 0,
                                                                 ants, n=n))
    assert np.array_equal(b.tours, fastpath_c.build_tours(t.w.cpu().numpy(), 3, 0, ants, n=n))
    for x in (a, b):
        assert np.array_equal(np.sort(x.tours, axis=1), np.broadcast_to(np.arange(n), (m, n)))
        assert np.array_equal(x.costs, ref.lengths(x.tours, inst.dist))
    # two streams of the same rule: same tour-length distribution (KS)
    from scipy import stats
    assert stats.ks_2samp(a.costs, b.costs).pvalue > 1e-3


# ---------------------------------------------------------------------------
# individual ops and error behaviour
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("n", [3, 8, 129, 1000, 2392])
def test_batch_costs_bit_exact(n):
    inst = euclid(n, n)
    g = np.random.default_rng(n)
    tours = np.stack([g.permutation(n) for _ in range(17)])
    assert np.array_equal(taco.batch_costs(tours, inst), ref.lengths(tours, inst.dist))


def test_probability_general_exponents_and_underflow():
    inst = euclid(2, 31)
    tau = np.random.default_rng(0).uniform(0.1, 2.0, (31, 31))
    for alpha, beta in ((1.0, 2.0), (0.5, 0.0), (1.3, 2.7), (2.0, 1.0)):
        params = taco.AcoParams(m=4, k=1, alpha=alpha, beta=beta)
        got = taco.compute_probability_matrix(taco.PheromoneState(tau), inst, params).p
        want = ref.transition(tau, inst.eta, alpha, beta)
        if alpha in (0.5, 1.0, 2.0) and beta in (0.0, 0.5, 1.0, 2.0):
            assert np.array_equal(got, want)
        else:
            np.testing.assert_allclose(got, want, rtol=1e-12, atol=0)
    with pytest.raises(taco.NumericalUnderflow):
        taco.compute_probability_matrix(taco.PheromoneState(np.zeros((31, 31))), inst,
                                        taco.AcoParams(m=4, k=1))
    hot = np.full((31, 31), 1e308)
    with pytest.raises(taco.NumericalUnderflow):
        taco.compute_probability_matrix(taco.PheromoneState(hot), inst, taco.AcoParams(m=4, k=1, alpha=4.0))


def test_select_elite_ties_and_bounds():
    b = taco.TourBatch(tours=np.array([[0, 1, 2], [1, 2, 0], [2, 0, 1]]), costs=np.array([4.0, 4.0, 1.0]))
    e = taco.select_elite(b, 2)
    assert np.array_equal(e[0][0], [2, 0, 1]) and np.array_equal(e[1][0], [0, 1, 2])
    with pytest.raises(ValueError):
        taco.select_elite(b, 0)
    g = np.random.default_rng(1)
    for m in (5000, 20000):  # counting-rank kernel and the CUB radix path
        costs = g.integers(0, 50, m).astype(np.float64) + 0.25  # many ties
        order = np.argsort(costs, kind="stable")
        batch = taco.TourBatch(tours=np.zeros((m, 3), dtype=np.int64) + np.arange(3), costs=costs)
        dev = _device.device()
        got = _device.download(_device.elite_order(_device.upload(costs, dev), _device.EliteWorkspace(m, dev)))
        assert np.array_equal(got, order)
        assert [c for _, c in taco.select_elite(batch, 7)] == costs[order[:7]].tolist()


def test_accumulate_matches_reference_with_duplicates():
    g = np.random.default_rng(7)
    for n, k in ((3, 1), (9, 40), (64, 33), (500, 3)):
        base = [g.permutation(n) for _ in range(max(1, k // 3))]
        elites = [(base[g.integers(len(base))], float(g.uniform(1.0, 50.0))) for _ in range(k)]
        want = ref.deposit(np.stack([t for t, _ in elites]), np.array([c for _, c in elites]), n)
        assert np.array_equal(taco.accumulate_increments(elites, n), want)
    with pytest.raises(taco.InvalidPermutation):
        taco.accumulate_increments([(np.array([0, 1, 1]), 3.0)], 3)
    with pytest.raises(ValueError):
        taco.accumulate_increments([], 3)


def test_apply_update_floor_and_formula():
    tau0 = taco.PheromoneState(tau=np.full((3, 3), 2.0) - 2.0 * np.eye(3), iteration=4)
    delta = np.zeros((3, 3))
    delta[0, 1] = delta[1, 0] = 0.5
    out = taco.apply_update(tau0, delta, rho=0.25)
    assert out.iteration == 5 and out.tau[0, 1] == 2.0 * 0.75 + 0.5 and out.tau[0, 2] == 1.5
    assert out.tau[0, 0] == taco.TAU_MIN
    with pytest.raises(ValueError):
        taco.apply_update(tau0, delta, rho=1.0)


# ---------------------------------------------------------------------------
# Solver
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("construct", ["sorted", "dense"])
def test_solver_matches_chained_dropins(construct):
    n, m = 60, 40
    inst = euclid(8, n)
    params = taco.AcoParams(m=m, k=4, selection="adair", seed=6, gamma_schedule=taco.GammaSchedule(1.5, 1.0, 5))
    s = taco.Solver(inst, params, construct=construct)
    tau = taco.PheromoneState.initial(n, 1.0)
    best = np.inf
    for it in range(6):
        prob = taco.compute_probability_matrix(tau, inst, params)
        batch = taco.construct_tours(prob, inst, params, it, variant=construct)
        elites = taco.select_elite(batch, params.k)
        tau = taco.apply_update(tau, taco.accumulate_increments(elites, n), params.rho)
        tour, length = s.step()
        got = s.last_batch()
        assert np.array_equal(got.tours, batch.tours)
        assert np.array_equal(got.costs, batch.costs)
        assert np.array_equal(s.pheromone().tau, tau.tau)
        best = min(best, batch.costs.min())
        assert length == best
        assert taco.tour_cost(tour, inst) == length


def test_solver_shard_offsets_are_invisible():
    # two "ranks" emulated by construction offsets on one GPU: same rows
    n, m = 80, 24
    inst = euclid(9, n)
    params = taco.AcoParams(m=m, k=3, selection="ir", seed=1)
    p = taco.compute_probability_matrix(taco.PheromoneState.initial(n, 1.0), inst, params)
    t = _device_tables(p.p, 1.0)
    dev = t.w.device
    whole = torch.zeros((m, n), dtype=torch.int32, device=dev)
    st = _device.new_status(dev)
    _device.construct(n, m, 0, _lib.CONSTRUCT_SORTED, t, 1, 0, whole, st)
    a = torch.zeros((10, n), dtype=torch.int32, device=dev)
    b = torch.zeros((14, n), dtype=torch.int32, device=dev)
    _device.construct(n, 10, 0, _lib.CONSTRUCT_SORTED, t, 1, 0, a, st)
    _device.construct(n, 14, 10, _lib.CONSTRUCT_SORTED, t, 1, 0, b, st)
    assert torch.equal(torch.cat([a, b]), whole)


def test_solver_quality_matches_reference_statistically():
    # best-tour quality over 10 seeds: engine vs the reference algorithm
    n, m, iters = 30, 30, 40
    coords = np.random.default_rng(123).uniform(0, 1000, (n, 2))
    inst = taco.euclidean_instance(coords)
    dist, eta = ref.instance_arrays(coords)
    ours, theirs = [], []
    for seed in range(10):
        params = taco.AcoParams(m=m, k=3, selection="adair", seed=seed,
                                gamma_schedule=taco.GammaSchedule(1.5, 1.0, iters))
        ours.append(taco.Solver(inst, params).run(iters)[1])
        cfg = ref.Config(m=m, k=3, selection="adair", period=iters, seed=seed)
        theirs.append(ref.run(dist, eta, cfg, iters)[-1])
    ours, theirs = np.array(ours), np.array(theirs)
    # mean best lengths within 3%, and neither side systematically better by > 3 sigma
    assert abs(ours.mean() - theirs.mean()) / theirs.mean() < 0.03
    se = np.sqrt(ours.var(ddof=1) / 10 + theirs.var(ddof=1) / 10)
    assert abs(ours.mean() - theirs.mean()) <= 3 * se + 1e-9 * theirs.mean()


@pytest.mark.parametrize("name", ["int12_ir", "int12_adair", "euc23_adair"])
def test_solver_replay_reproduces_reference_runs(golden, name):
    # full runs on the reference's own streams: every iteration's tours, lengths
    # and pheromone equal antbatch's run (golden vectors) bit for bit
    inst = _inst(golden, name)
    for seed in golden[f"{name}/seeds"].tolist():
        params, iters = _params(golden, name, seed)
        s = taco.Solver(inst, params, stream="replay")
        for it in range(iters):
            key = f"{name}/s{seed}/it{it}"
            tour, length = s.step()
            b = s.last_batch()
            assert np.array_equal(b.tours, golden[f"{key}/tours"])
            assert np.array_equal(b.costs, golden[f"{key}/costs"])
            assert np.array_equal(s.pheromone().tau, golden[f"{key}/tau"])
            assert length == min(golden[f"{name}/s{seed}/it{i}/costs"].min() for i in range(it + 1))


def _golden_instances():
    return np.load(os.path.join(os.path.dirname(__file__), "golden", "reference_instances.npz"))


@pytest.mark.parametrize("kind", ["EXACT", "EUC_2D", "CEIL_2D", "ATT"])
def test_device_instance_matches_reference_builders(kind):
    """f4: dist/eta built on the device == the reference builders' (golden), bitwise."""
    z = _golden_instances()
    dev = taco.device_euclidean_instance(z["conv/coords"], kind)
    assert np.array_equal(dev.dist.cpu().numpy(), z[f"conv/{kind}/dist"])
    assert np.array_equal(dev.eta.cpu().numpy(), z[f"conv/{kind}/eta"])


def test_device_instance_degenerate_and_lenient():
    z = _golden_instances()
    for kind in ("EUC_2D", "EXACT"):
        with pytest.raises(taco.DegenerateInstance) as e:
            taco.device_euclidean_instance(z["degen/coords"], kind)
        assert str(e.value) == str(z[f"degen/{kind}/message"])
        dev = taco.device_euclidean_instance(z["degen/coords"], kind, lenient=True)
        assert np.array_equal(dev.dist.cpu().numpy(), z[f"degen/{kind}/dist"])
        assert np.array_equal(dev.eta.cpu().numpy(), z[f"degen/{kind}/eta"])
    with pytest.raises(taco.UnsupportedEdgeWeightType):
        taco.device_euclidean_instance(z["degen/coords"], "EXPLICIT")


def test_device_instance_large_and_synthetic():
    from paper_2404_04895_b200.harness import ExperimentConfig, SyntheticSpec, load_instance

    z = _golden_instances()
    for key in [k for k in z.files if k.startswith("syn_") and k.endswith("/spec")]:
        tag = key[: -len("/spec")]
        n, seed = (int(v) for v in z[key])
        kind = "clustered" if "clustered" in tag else "uniform"
        cfg = ExperimentConfig(params=taco.AcoParams(m=4, k=1), synthetic=SyntheticSpec(n=n, seed=seed, kind=kind))
        inst = load_instance(cfg)
        assert inst.name == f"rnd{n}"
        assert np.array_equal(inst.dist.cpu().numpy(), z[f"{tag}/dist"])
        assert np.array_equal(inst.eta.cpu().numpy(), z[f"{tag}/eta"])
    g = np.random.default_rng(3)
    coords = g.uniform(0.0, 2000.0, (3001, 2))  # multi-block rows, n not a multiple of 256
    host = taco.euclidean_instance(coords)
    dev = taco.device_euclidean_instance(coords)
    assert np.array_equal(dev.dist.cpu().numpy(), host.dist)
    assert np.array_equal(dev.eta.cpu().numpy(), host.eta)
    # a Solver on the device instance runs exactly like one on the host instance
    coords = g.uniform(0.0, 2000.0, (90, 2))
    params = taco.AcoParams(m=20, k=2, selection="ir", seed=2)
    a = taco.Solver(taco.device_euclidean_instance(coords), params).run(5)
    b = taco.Solver(taco.euclidean_instance(coords), params).run(5)
    assert a[1] == b[1] and np.array_equal(a[0], b[0])


def test_device_build_instance_from_raw_tsplib_record():
    from types import SimpleNamespace

    z = _golden_instances()
    coords = z["conv/coords"]
    raw = SimpleNamespace(name="x37", dimension=len(coords), edge_weight_type="ATT",
                          node_coords=tuple((i + 1, float(x), float(y)) for i, (x, y) in enumerate(coords)))
    inst = taco.device_build_instance(raw, best_known=123.0)
    assert inst.name == "x37" and inst.best_known == 123.0
    assert np.array_equal(inst.dist.cpu().numpy(), z["conv/ATT/dist"])


@pytest.mark.parametrize("selection", ["adair", "ir", "rw"])
def test_graph_replay_equals_eager_solver(selection):
    """CUDA-graph replay (device iteration state) == eager launches, bit for bit,
    including run()'s multi-iteration graphs and the remainder."""
    n, m = 45, 20
    inst = euclid(12, n)
    params = taco.AcoParams(m=m, k=3, selection=selection, seed=5, gamma_schedule=taco.GammaSchedule(1.5, 1.0, 6))
    g = taco.Solver(inst, params, graph=True, graph_warmup=1)
    e = taco.Solver(inst, params, graph=False)
    for _ in range(3):  # step(): eager warm-up, then 1-iteration graph replays
        assert g.step()[1] == e.step()[1]
        assert np.array_equal(g.last_batch().tours, e.last_batch().tours)
    bg, be = g.run(19), e.run(19)  # 2 x 8-iteration graph + 3 single replays
    assert bg[1] == be[1] and np.array_equal(bg[0], be[0])
    assert g.iteration == e.iteration == 22
    assert np.array_equal(g.pheromone().tau, e.pheromone().tau)
    assert np.array_equal(g.last_batch().costs, e.last_batch().costs)
    assert int(g.best_iter.item()) == int(e.best_iter.item())
    # default warm-up: GRAPH_WARMUP eager iterations, then captured batches
    d = taco.Solver(inst, params)
    assert d.graph
    bd = d.run(22 + 2 * taco.Solver.GRAPH_WARMUP)
    be = e.run(2 * taco.Solver.GRAPH_WARMUP)
    assert bd[1] == be[1] and np.array_equal(d.pheromone().tau, e.pheromone().tau)
    assert len(d._graphs) > 0


@pytest.mark.parametrize("selection", ["adair", "rw"])
def test_checkpoint_resume_is_bit_identical(tmp_path, selection):
    inst = euclid(40, 64)
    params = taco.AcoParams(m=24, k=3, selection=selection, seed=8, gamma_schedule=taco.GammaSchedule(1.5, 1.0, 7))
    full = taco.Solver(inst, params)
    full.run(9)
    first = taco.Solver(inst, params)
    first.run(4)
    first.save(str(tmp_path / "ck.npz"))
    second = taco.Solver(inst, params)
    second.load(str(tmp_path / "ck.npz"))
    assert second.iteration == 4
    tour, length = second.run(5)
    assert second.iteration == full.iteration == 9
    assert np.array_equal(second.pheromone().tau, full.pheromone().tau)
    assert length == full.best()[1] and np.array_equal(tour, full.best()[0])
    assert np.array_equal(second.last_batch().tours, full.last_batch().tours)
    with pytest.raises(ValueError):
        taco.Solver(euclid(40, 65), params).restore(first.checkpoint())


@pytest.mark.parametrize("n,k,gamma,same", [(37, 5, 1.3, False), (300, 40, 1.0, True), (2392, 409, 1.17, False),
                                            (1001, 102, 1.4, True)])
def test_split_update_equals_fused_row_kernel(n, k, gamma, same):
    """taco_update_split (Solver path) == taco_row_update (fused) bit for bit:
    tau', row sums, P, W and the sorted table, with duplicate-heavy deposits."""
    dev = _device.device()
    g = np.random.default_rng(n)
    tau0 = torch.from_numpy(g.uniform(1e-13, 2.0, (n, n))).to(dev)
    eta = torch.from_numpy(g.uniform(0.01, 1.0, (n, n))).to(dev)
    tours = np.stack([g.permutation(n) for _ in range(1 if same else k)])
    tours = np.repeat(tours, k, axis=0) if same else tours
    nbr = np.zeros((n, k, 2), dtype=np.int32)
    for r, t in enumerate(tours):
        nbr[t, r, 0], nbr[t, r, 1] = np.roll(t, 1), np.roll(t, -1)
    nbr_t = torch.from_numpy(nbr).to(dev)
    inc = torch.from_numpy(1.0 / g.uniform(1e3, 1e4, k)).to(dev)
    outs = []
    for split in (False, True):
        tau = tau0.clone()
        t = _device.SelectionTables(n, dev, dense=True, sorted_=True)
        p = torch.zeros((n, n), dtype=torch.float64, device=dev)
        rs = torch.zeros(n, dtype=torch.float64, device=dev)
        st = _device.new_status(dev)
        common = dict(tau_in=tau, tau_out=tau, eta_b=eta, nbr=nbr_t, inc=inc, k=k, do_evap=True, keep=0.9,
                      alpha=1.0, inv_gamma=1.0 / gamma, p_out=p, rowsum_out=rs, w_out=t.w, ldw=t.ldw,
                      sw_out=t.sw, si_out=t.si, status=st)
        if split:
            _device.update_split(n, delta_ws=torch.empty_like(tau), unnorm_ws=torch.empty_like(tau), **common)
        else:
            _device.row_update(n, want_p=True, **common)
        torch.cuda.synchronize()
        assert _device.read_status(st)[0] == 0
        outs.append([x.cpu().numpy() for x in (tau, rs, p, t.w, t.sw, t.si)])
    for a, b in zip(*outs):
        assert np.array_equal(a, b)


@pytest.mark.parametrize("n,cuts", [(300, (0, 1, 150, 299, 300)), (1000, (0, 333, 666, 1000))])
def test_row_range_update_pieces_equal_whole(n, cuts):
    """taco_row_update_rows over a row partition (the multi-GPU row-partitioned
    update) == taco_row_update over all rows, and rows outside the range are
    untouched."""
    dev = _device.device()
    g = np.random.default_rng(n + 1)
    tau0 = torch.from_numpy(g.uniform(1e-3, 2.0, (n, n))).to(dev)
    eta = torch.from_numpy(g.uniform(0.01, 1.0, (n, n))).to(dev)
    k = 7
    tours = np.stack([g.permutation(n) for _ in range(k)])
    nbr = np.zeros((n, k, 2), dtype=np.int32)
    for r, t in enumerate(tours):
        nbr[t, r, 0], nbr[t, r, 1] = np.roll(t, 1), np.roll(t, -1)
    nbr_t = torch.from_numpy(nbr).to(dev)
    inc = torch.from_numpy(1.0 / g.uniform(1e3, 1e4, k)).to(dev)
    outs = []
    for pieces in (False, True):
        tau = tau0.clone()
        t = _device.SelectionTables(n, dev, dense=True, sorted_=True)
        p = torch.zeros((n, n), dtype=torch.float64, device=dev)
        rs = torch.zeros(n, dtype=torch.float64, device=dev)
        st = _device.new_status(dev)
        common = dict(tau_in=tau, tau_out=tau, eta_b=eta, nbr=nbr_t, inc=inc, k=k, do_evap=True, keep=0.9,
                      alpha=1.0, inv_gamma=1.0 / 1.5, p_out=p, rowsum_out=rs, w_out=t.w, ldw=t.ldw,
                      sw_out=t.sw, si_out=t.si, status=st)
        if pieces:
            _device.row_update_rows(cuts[1], cuts[2], n, want_p=True, **common)
            torch.cuda.synchronize()
            assert torch.equal(tau[:cuts[1]], tau0[:cuts[1]]) and torch.equal(tau[cuts[2]:], tau0[cuts[2]:])
            assert not p[:cuts[1]].any() and not p[cuts[2]:].any()
            for a, b in zip(cuts[2:-1], cuts[3:]):
                _device.row_update_rows(a, b, n, want_p=True, **common)
            _device.row_update_rows(cuts[0], cuts[1], n, want_p=True, **common)
        else:
            _device.row_update(n, want_p=True, **common)
        torch.cuda.synchronize()
        assert _device.read_status(st)[0] == 0
        outs.append([x.cpu().numpy() for x in (tau, rs, p, t.w, t.sw, t.si)])
    for a, b in zip(*outs):
        assert np.array_equal(a, b)
    with pytest.raises(ValueError):
        _device.row_update_rows(5, 4, n, want_p=True, **common)


@pytest.mark.parametrize("selection", ["adair", "rw"])
def test_solver_split_update_path_is_bit_identical(monkeypatch, selection):
    """Rows too long for the fused kernel's shared memory take the split
    update; forced here at small n, the runs are identical."""
    inst = euclid(77, 90)
    params = taco.AcoParams(m=30, k=4, selection=selection, seed=3, gamma_schedule=taco.GammaSchedule(1.5, 1.0, 5))
    fused = taco.Solver(inst, params)
    fused.run(6)
    monkeypatch.setattr(taco.Solver, "FUSED_MAX_N", 10)
    split = taco.Solver(inst, params)
    assert split._split_update
    split.run(6)
    assert np.array_equal(split.pheromone().tau, fused.pheromone().tau)
    assert split.best()[1] == fused.best()[1]
    assert np.array_equal(split.last_batch().tours, fused.last_batch().tours)


def test_iterate_yields_what_step_returns():
    """Solver.iterate (pipelined: iteration t+1 queued before t is read)
    yields exactly the per-iteration results of blocking step() calls, in
    graph and eager mode."""
    inst = euclid(91, 60)
    for graph, warm in ((True, 0), (True, None), (False, None)):
        params = taco.AcoParams(m=32, k=3, selection="adair", seed=5, gamma_schedule=taco.GammaSchedule(1.5, 1.0, 7))
        a = taco.Solver(inst, params, graph=graph, graph_warmup=warm)
        want = [a.step() for _ in range(7)]
        b = taco.Solver(inst, params, graph=graph, graph_warmup=warm)
        got = list(b.iterate(7))
        assert [g[0] for g in got] == list(range(7))
        for (tw, lw), (_, tg, lg) in zip(want, got):
            assert np.array_equal(tw, tg) and lw == lg
        assert np.array_equal(a.pheromone().tau, b.pheromone().tau)


def test_row_update_plan_built_in_kernel_equals_prebuilt_image():
    """The row update copies the pairwise plan from a per-n image built at the
    first eager launch (k_plan_image); a launch captured into a CUDA graph
    before any image exists for that n builds the plan in the kernel
    instead.  Both give the same tau / row sums / P / selection table bits.
    n = 1237 is used by no other test, so the capture runs first."""
    dev = _device.device()
    n, k = 1237, 9
    g = np.random.default_rng(n)
    tau0 = torch.from_numpy(g.uniform(1e-6, 2.0, (n, n))).to(dev)
    eta = torch.from_numpy(g.uniform(0.01, 1.0, (n, n))).to(dev)
    tours = np.stack([g.permutation(n) for _ in range(k)])
    nbr = np.zeros((n, k, 2), dtype=np.int32)
    for r, t in enumerate(tours):
        nbr[t, r, 0], nbr[t, r, 1] = np.roll(t, 1), np.roll(t, -1)
    nbr_t = torch.from_numpy(nbr).to(dev)
    inc = torch.from_numpy(1.0 / g.uniform(1e3, 1e4, k)).to(dev)
    outs = []
    for captured in (True, False):
        tau = tau0.clone()
        t = _device.SelectionTables(n, dev, dense=True, sorted_=True)
        p = torch.zeros((n, n), dtype=torch.float64, device=dev)
        rs = torch.zeros(n, dtype=torch.float64, device=dev)
        st = _device.new_status(dev)
        common = dict(tau_in=tau, tau_out=tau, eta_b=eta, nbr=nbr_t, inc=inc, k=k, do_evap=True, keep=0.9,
                      want_p=True, alpha=1.0, inv_gamma=1.0 / 1.5, p_out=p, rowsum_out=rs, w_out=t.w,
                      ldw=t.ldw, sw_out=t.sw, si_out=t.si, status=st)
        torch.cuda.synchronize()
        if captured:
            side = torch.cuda.Stream(device=dev)
            graph = torch.cuda.CUDAGraph()
            with torch.cuda.stream(side):
                graph.capture_begin(capture_error_mode="thread_local")
                try:
                    _device.row_update(n, **common)
                finally:
                    graph.capture_end()
            graph.replay()
        else:
            _device.row_update(n, **common)
        torch.cuda.synchronize()
        assert _device.read_status(st)[0] == 0
        outs.append([x.cpu().numpy() for x in (tau, rs, p, t.w, t.sw, t.si)])
    for a, b in zip(*outs):
        assert np.array_equal(a, b)


@pytest.mark.parametrize("n", [97, 1000, 1024, 1025, 2392, 2400, 2401, 2560, 2561, 5000, 5120, 5121, 10000, 10240])
def test_row_sort_order_at_every_cta_shape(n):
    """The sorted table is row i of W in descending order of the W bits above
    bit 16, stable in the column (the order the pruned scan and the sorted
    stream's positions are defined on), for every row-sort CTA shape and at
    both ends of each one's n range (k_row_sort: 96x11 up to 1024, 96x25 up
    to 2400, 128x20 up to 2560, 192x27 up to 5120, 384x27 up to 10240)."""
    dev = _device.device()
    g = np.random.default_rng(n)
    rows = np.unique(np.concatenate([[0, n - 1], g.integers(0, n, 6)]))
    p = g.uniform(0.0, 1.0, (n, n)) ** 8  # wide exponent range: many equal 16-bit prefixes
    p[g.uniform(size=(n, n)) < 0.05] = 0.0
    np.fill_diagonal(p, 0.0)
    p /= p.sum(axis=1, keepdims=True)
    t = _device.SelectionTables(n, dev, dense=True, sorted_=True)
    _device.selection_table_from_p(_device.upload(p, dev), 1.0, t)
    torch.cuda.synchronize()
    w = t.w.cpu().numpy()[rows, :n]
    key = (w.view(np.uint32) >> 16).astype(np.int64)
    want_si = np.argsort(-key, axis=1, kind="stable")
    assert np.array_equal(t.si.cpu().numpy()[rows, :n].astype(np.int64), want_si)
    assert np.array_equal(t.sw.cpu().numpy()[rows, :n], np.take_along_axis(w, want_si, axis=1))
