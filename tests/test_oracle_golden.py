"""CPU: pin the oracle restatements before trusting them.

* oracle.reference_port reproduces the golden vectors produced by running the
  reference package itself (tests/golden/make_golden.py) bit for bit.
* oracle.fastpath's Philox2x32-10 reproduces the Random123 known-answer
  vectors, and its pairwise-sum restatement equals numpy's ndarray.sum.
"""

import os

import numpy as np
import pytest

from conftest import golden_cases
from oracle import fastpath, reference_port as ref


def _case(golden, name):
    n, m, k, iters, alpha, beta, rho, period, sel = golden[f"{name}/meta"]
    cfg = ref.Config(m=int(m), k=int(k), alpha=alpha, beta=beta, rho=rho,
                     selection=("ir", "adair", "rw")[int(sel)], period=int(period))
    return int(n), int(iters), cfg, golden[f"{name}/dist"], golden[f"{name}/eta"]


def test_golden_has_cases(golden):
    assert len(golden_cases(golden)) >= 6


@pytest.mark.parametrize("name", ["int12_ir", "int12_adair", "euc23_adair", "euc17_ab", "int12_rw", "euc29_rw"])
def test_reference_port_reproduces_reference_pipeline(golden, name):
    n, iters, cfg, dist, eta = _case(golden, name)
    for seed in golden[f"{name}/seeds"].tolist():
        cfg.seed = seed
        tau = ref.initial_tau(n, cfg.q0_tau)
        p = ref.transition(tau, eta, cfg.alpha, cfg.beta)
        for it in range(iters):
            key = f"{name}/s{seed}/it{it}"
            assert np.array_equal(p, golden[f"{key}/p"])
            assert cfg.gamma(it) == golden[f"{key}/gamma"][0]
            assert np.array_equal(ref.start_block(seed, it, cfg.m, n), golden[f"{key}/starts"])
            out = ref.iterate(tau, p, dist, eta, cfg, it)
            assert np.array_equal(out["tours"], golden[f"{key}/tours"])
            assert np.array_equal(out["costs"], golden[f"{key}/costs"])
            assert np.array_equal(out["order"], golden[f"{key}/order"])
            assert np.array_equal(out["delta"], golden[f"{key}/delta"])
            assert np.array_equal(out["tau"], golden[f"{key}/tau"])
            tau, p = out["tau"], out["p"]


def test_gamma_known_answers(golden):
    got = [ref.gamma(t) for t in (0, 250, 500, 999, 1000)]
    assert got == golden["kat/gamma"].tolist()
    assert got[0] == 1.5 and got[-1] == 1.5
    assert abs(got[1] - 1.4268) < 5e-5  # reference tests/test_selection.py:28-41


def test_spin_known_answers(golden):
    # reference tests/test_selection.py:76-93 and the u = 0 / u = 1 edges
    for w, u, want in zip(golden["kat/rw_weights"], golden["kat/rw_u"], golden["kat/rw_pick"]):
        got = ref.spin_round(w[None, :], np.array([0]), np.ones((1, 3)), np.array([u]))[0]
        assert got == want


def test_device_rw_restatement_is_the_reference_rule():
    """fastpath.rw_tours applies the reference's spin rule (spin_round) to the
    device thresholds: with thresholds swapped in, it is the same function."""
    g = np.random.default_rng(8)
    n, m = 15, 6
    p = g.uniform(0.0, 1.0, (n, n))
    np.fill_diagonal(p, 0.0)
    p /= p.sum(axis=1, keepdims=True)
    tours = fastpath.rw_tours(p, 5, 3, np.arange(m))
    for t in tours:
        assert sorted(t.tolist()) == list(range(n))
    # step-by-step replay with spin_round
    cur = fastpath.starts(5, 3, np.arange(m), n)
    unvisited = np.ones((m, n))
    unvisited[np.arange(m), cur] = 0.0
    for step in range(1, n):
        u = fastpath.rw_uniform(5, 3, np.full(m, step), np.arange(m))
        nxt = ref.spin_round(p, cur, unvisited, u)
        assert np.array_equal(nxt, tours[:, step])
        unvisited[np.arange(m), nxt] = 0.0
        cur = nxt


def test_deposit_hand_case(golden):
    # reference tests/test_pheromone.py:59-67: tour [0,1,2] of cost 4
    d = ref.deposit(np.array([[0, 1, 2]]), np.array([4.0]), 3)
    assert np.array_equal(d, golden["kat/increment_0_1_2_cost4"])
    assert np.array_equal(d, 0.25 * (1 - np.eye(3)))


def test_update_hand_case():
    # reference tests/test_pheromone.py:110-124
    tau = np.full((3, 3), 2.0) - 2.0 * np.eye(3)
    delta = np.zeros((3, 3))
    delta[0, 1] = delta[1, 0] = 0.5
    out = ref.evaporate(tau, delta, 0.25)
    assert out[0, 1] == 2.0 * 0.75 + 0.5 and out[0, 2] == 1.5
    assert out[0, 0] == ref.TAU_MIN


def test_probability_known_answer():
    # SPEC.md:183 example: tau = 1, alpha = beta = 1, dist row 0 = [0, 1, 2]
    dist = np.array([[0.0, 1.0, 2.0], [1.0, 0.0, 1.0], [2.0, 1.0, 0.0]])
    eta = np.where(dist > 0, 1.0 / np.where(dist > 0, dist, 1.0), 0.0)
    p = ref.transition(np.ones((3, 3)), eta, 1.0, 1.0)
    assert np.allclose(p[0], [0.0, 2 / 3, 1 / 3], rtol=0, atol=1e-15)


# ---------------------------------------------------------------------------
# fast-path restatement
# ---------------------------------------------------------------------------
KAT = [  # Random123 philox2x32-10 known-answer vectors (kat_vectors)
    ((0, 0), 0, (0xFF1DAE59, 0x6CD10DF2)),
    ((0xFFFFFFFF, 0xFFFFFFFF), 0xFFFFFFFF, (0x2C3F628B, 0xAB4FD7AD)),
    ((0x243F6A88, 0x85A308D3), 0x13198A2E, (0xDD7CE038, 0xF62A4C12)),
]


@pytest.mark.parametrize("ctr,key,want", KAT)
def test_philox_known_answers(ctr, key, want):
    got = fastpath.philox2x32_10(np.array([ctr], dtype=np.uint64), key)[0]
    assert tuple(int(v) for v in got) == want


def test_stream_keys_and_counters():
    # H(seed) is a fixed function (MurmurHash3 fmix64, xor-folded); the
    # iteration offsets it, so the iterations of one run never share a key
    assert fastpath.seed_hash32(0) == 0
    h = fastpath.seed_hash32(12345)
    assert fastpath.stream_key(12345, 7) == (h + 7) & 0xFFFFFFFF
    assert len({fastpath.stream_key(3, it) for it in range(5000)}) == 5000
    assert len({fastpath.seed_hash32(s) for s in range(100_000)}) == 100_000  # fmix64 is a bijection
    # the start counter (ant, 0) and RW counters (ant, 0xffff | step << 16)
    # never collide with a selection counter (ant, (j >> 1) | step << 16),
    # step >= 1, j >> 1 <= 0x7fff
    sel_low = np.arange(0, 65535) >> 1
    assert sel_low.max() < fastpath.RW_LOW
    u = fastpath.uniforms(9, 2, np.array([1, 1, 2]), np.array([0, 0, 0]), np.array([4, 5, 4]))
    w = fastpath.philox2x32_10(np.array([[0, 2 | 1 << 16], [0, 2 | 2 << 16]], dtype=np.uint64),
                               fastpath.stream_key(9, 2))
    assert np.array_equal(u, fastpath.bits_to_uniform(np.array([w[0, 0], w[0, 1], w[1, 0]])))
    # sorted stream: position p at steps 2t - 1 and 2t shares counter
    # (ant, p | t << 16), words 0 and 1; t >= 1, so never the start counter
    # (ant, 0), and p <= 65534 never reaches RW_LOW
    u = fastpath.position_uniforms(9, 2, np.array([1, 2, 3, 4]), np.array([7, 7, 7, 7]), np.array([5, 5, 5, 5]))
    w = fastpath.philox2x32_10(np.array([[7, 5 | 1 << 16], [7, 5 | 2 << 16]], dtype=np.uint64),
                               fastpath.stream_key(9, 2))
    assert np.array_equal(u, fastpath.bits_to_uniform(np.array([w[0, 0], w[0, 1], w[1, 0], w[1, 1]])))


def test_uniform_conversion_is_exact_and_open():
    x = np.array([0, 1 << 9, 0xFFFFFFFF, 0x80000000], dtype=np.uint32)
    u = fastpath.bits_to_uniform(x)
    assert u.dtype == np.float32
    k = (x >> 9).astype(np.float64)
    assert np.array_equal(u.astype(np.float64), (k + 0.5) * 2.0 ** -23)
    assert 0.0 < u.min() and u.max() < 1.0


def test_pairwise_restatement_matches_numpy():
    g = np.random.default_rng(3)
    for n in list(range(1, 140)) + [255, 256, 257, 1000, 2392]:
        a = g.uniform(0, 1, n) * 10.0 ** g.uniform(-6, 6, n)
        assert fastpath.pairwise_sum(a) == a.sum()
        rows = g.uniform(0, 1, (3, n))
        s = rows.sum(axis=1)
        for i in range(3):
            assert fastpath.pairwise_sum(rows[i]) == s[i]


def test_fastpath_tours_are_permutations_and_shard_invariant():
    g = np.random.default_rng(0)
    n = 29
    dist, eta = ref.instance_arrays(g.uniform(0, 100, (n, 2)))
    p = ref.transition(ref.initial_tau(n, 1.0), eta, 1.0, 2.0)
    w = fastpath.selection_table(p, 1.0)
    whole = fastpath.build_tours(w, 9, 4, np.arange(12))
    assert np.array_equal(np.sort(whole, axis=1), np.broadcast_to(np.arange(n), whole.shape))
    parts = np.concatenate([fastpath.build_tours(w, 9, 4, np.arange(0, 5)),
                            fastpath.build_tours(w, 9, 4, np.arange(5, 12))])
    assert np.array_equal(whole, parts)


def test_product_rule_agrees_with_log_rule_on_shared_uniforms():
    # same uniforms, product form vs the reference's log form: count mismatches
    g = np.random.default_rng(1)
    n = 40
    dist, eta = ref.instance_arrays(g.uniform(0, 1000, (n, 2)))
    p = ref.transition(ref.initial_tau(n, 1.0), eta, 1.0, 2.0)
    w = fastpath.selection_table(p, 1.0)
    a = fastpath.build_tours(w, 2, 0, np.arange(32))
    b = fastpath.log_rule_tours(p, 1.0, 2, 0, np.arange(32))
    assert (a != b).sum() == 0


# ---------------------------------------------------------------------------
# instance builders, pinned on tests/golden/reference_instances.npz
# ---------------------------------------------------------------------------
def _instances():
    return np.load(os.path.join(os.path.dirname(__file__), "golden", "reference_instances.npz"))


@pytest.mark.parametrize("kind", ["EXACT", "EUC_2D", "CEIL_2D", "ATT"])
def test_oracle_coord_instance_matches_reference(kind):
    z = _instances()
    dist, eta = ref.coord_instance(z["conv/coords"], kind)
    assert np.array_equal(dist, z[f"conv/{kind}/dist"])
    assert np.array_equal(eta, z[f"conv/{kind}/eta"])


def test_oracle_degenerate_instance_matches_reference():
    z = _instances()
    for kind in ("EUC_2D", "EXACT"):
        with pytest.raises(ref.Degenerate) as e:
            ref.coord_instance(z["degen/coords"], kind)
        assert str(e.value) == str(z[f"degen/{kind}/message"])
        dist, eta = ref.coord_instance(z["degen/coords"], kind, lenient=True)
        assert np.array_equal(dist, z[f"degen/{kind}/dist"]) and np.array_equal(eta, z[f"degen/{kind}/eta"])


def test_synthetic_coords_match_reference():
    from paper_2404_04895_b200.harness import SyntheticSpec, synthetic_coords

    z = _instances()
    for kind in ("clustered", "uniform"):
        key = [k for k in z.files if k.startswith(f"syn_{kind}") and k.endswith("/spec")][0]
        tag = key[: -len("/spec")]
        n, seed = (int(v) for v in z[key])
        coords = synthetic_coords(SyntheticSpec(n=n, seed=seed, kind=kind))
        assert np.array_equal(coords, z[f"{tag}/coords"])
        dist, eta = ref.coord_instance(coords, "EUC_2D")
        assert np.array_equal(dist, z[f"{tag}/dist"]) and np.array_equal(eta, z[f"{tag}/eta"])


def test_c_oracle_equals_numpy_restatement():
    """oracle/c/fastpath.c (the parity oracle at the BASELINE sizes) == the
    numpy restatement, including the f64 fallback and the all -inf rule."""
    from oracle import fastpath_c

    g = np.random.default_rng(4)
    for n in (3, 7, 130, 301):
        w = g.uniform(0.0, 1.0, (n, n)).astype(np.float32)
        np.fill_diagonal(w, 0.0)
        w[g.uniform(size=(n, n)) < 0.1] = 0.0
        ldw = -(-n // 32) * 32
        padded = np.zeros((n, ldw), dtype=np.float32)
        padded[:, :n] = w
        src = g.uniform(0.0, 1.0, (n, n))
        ants = np.concatenate([np.arange(9), [2**31 + 5, 2**32 - 1]])
        for fb in (None, (src, 1.0, None), (src, 2.0, src)):
            try:
                want = fastpath.build_tours(w, 77, 3, ants, fallback=fb, inv_gamma=0.25)
            except AssertionError:  # an ant left with only zero weights and city 0 visited
                with pytest.raises(AssertionError):
                    fastpath_c.build_tours(padded, 77, 3, ants, n=n, fallback=fb, inv_gamma=0.25)
                continue
            assert np.array_equal(fastpath_c.build_tours(padded, 77, 3, ants, n=n, fallback=fb, inv_gamma=0.25), want)
    # the sorted stream: uniforms keyed by the entry's position in the sorted row
    for n in (5, 40, 201):
        w = g.uniform(0.0, 1.0, (n, n)).astype(np.float32)
        np.fill_diagonal(w, 0.0)
        w[g.uniform(size=(n, n)) < 0.1] = 0.0
        key = (w.view(np.uint32) >> 16).astype(np.int64)
        si = np.argsort(-key, axis=1, kind="stable").astype(np.uint16)  # the kernels' row order
        sw = np.take_along_axis(w, si.astype(np.int64), axis=1)
        src = g.uniform(0.0, 1.0, (n, n))
        for fb in (None, (src, 1.0, None)):
            try:
                want = fastpath.build_tours_sorted(sw, si, 5, 2, np.arange(9), fallback=fb, inv_gamma=0.5)
            except AssertionError:
                with pytest.raises(AssertionError):
                    fastpath_c.build_tours_sorted(sw, si, 5, 2, np.arange(9), fallback=fb, inv_gamma=0.5)
                continue
            assert np.array_equal(fastpath_c.build_tours_sorted(sw, si, 5, 2, np.arange(9), fallback=fb,
                                                                inv_gamma=0.5), want)
    # Philox and the key schedule
    ctr = np.array([[0, 0], [0xFFFFFFFF, 0xFFFFFFFF], [0x243F6A88, 0x85A308D3]], dtype=np.uint64)
    key = np.array([0, 0xFFFFFFFF, 0x13198A2E], dtype=np.uint64)
    assert np.array_equal(fastpath_c.philox2x32_10(ctr, key), fastpath.philox2x32_10(ctr, key))
    for seed in (0, 1, 2**40 + 3, 2**64 - 1):
        assert fastpath_c.seed_hash32(seed) == fastpath.seed_hash32(seed)


def test_c_oracle_all_zero_rows_follow_numpy_argmax():
    """No W > 0 and no fallback source: city 0 while unvisited (numpy's argmax
    of an all -inf row), else the reference's assertion (colony.py:149)."""
    from oracle import fastpath_c

    n = 20
    w = np.zeros((n, n), dtype=np.float32)
    side = np.arange(n) >= 10
    w[side[:, None] == side[None, :]] = 1.0
    np.fill_diagonal(w, 0.0)
    st = fastpath.starts(5, 0, np.arange(64), n)
    far = np.arange(64)[side[st]]
    near = np.arange(64)[~side[st]]
    t = fastpath_c.build_tours(w, 5, 0, far)
    assert (t[:, 10] == 0).all() and np.array_equal(t, fastpath.build_tours(w, 5, 0, far))
    with pytest.raises(AssertionError):
        fastpath_c.build_tours(w, 5, 0, near[:1])
    with pytest.raises(AssertionError):
        fastpath.build_tours(w, 5, 0, near[:1])


def test_mismatch_counter_agrees_with_the_rules():
    from oracle import fastpath_c

    n = 150
    g = np.random.default_rng(8)
    p = g.uniform(0.0, 1.0, (n, n))
    np.fill_diagonal(p, 0.0)
    p /= p.sum(axis=1, keepdims=True)
    gamma = 1.37
    w = fastpath.selection_table(p, gamma)
    ants = np.arange(40)
    tours = fastpath_c.build_tours(w, 3, 2, ants).astype(np.int32)
    c = fastpath_c.count_mismatches(w, ref.log_table(p, gamma), 3, 2, ants, tours)
    assert c["selections"] == 40 * (n - 1) and c["product_rule"] == 0
    # the log rule's own tours: counted against themselves, the log rule never disagrees
    logt = fastpath.log_rule_tours(p, gamma, 3, 2, ants).astype(np.int32)
    c2 = fastpath_c.count_mismatches(w, ref.log_table(p, gamma), 3, 2, ants, logt)
    assert c2["log_rule_same_u"] == 0
    assert c["log_rule_same_u"] <= 2 and c["log_rule_u53"] <= 40
