"""Drop-in replacements of the reference's colony functions (colony.py) and
tour lengths (model.py:285-295), executed on the B200 through libtaco.

Signatures, return types and error behaviour follow the reference:
``compute_probability_matrix(tau, inst, params) -> ProbabilityMatrix``
(colony.py:51-69), ``construct_tours(p, inst, params, iteration,
chunk_size=None, probe=None) -> TourBatch`` (colony.py:87-154),
``init_starts`` (colony.py:72-78), ``batch_costs`` / ``tour_cost``.
"""

from __future__ import annotations

import numpy as np
import torch

from . import _device, _lib
from . import rng as _rng
from .model import ProbabilityMatrix, Selection, TourBatch, check_permutations
from .selection import gamma_at


class NumericalUnderflow(ValueError):
    """A transition-matrix row normalizer vanished or became non-finite
    (colony.py:32-33)."""


def _underflow_from_sums(sums: np.ndarray) -> NumericalUnderflow:
    # same row choice as the reference's message (colony.py:64-68)
    bad = int(np.argmin(np.where(np.isfinite(sums), sums, -np.inf)))
    return NumericalUnderflow(
        f"row {bad} normalizer is {float(sums[bad])!r}; "
        "pheromone or heuristic values out of representable range")


def _selection(params) -> Selection:
    return Selection(getattr(params, "selection", Selection.ADAIR))


def construction_gamma(params, iteration: int) -> float:
    """gamma for one iteration: the cosine schedule for AdaIR, 1.0 for IR
    (colony.py:103)."""
    if _selection(params) is Selection.ADAIR:
        return gamma_at(iteration, params.gamma_schedule)
    return 1.0


def compute_probability_matrix(tau, inst, params) -> ProbabilityMatrix:
    """P = RowNorm(tau^alpha * eta^beta) with a zero diagonal (colony.py:51-69).

    Bit-exact with the reference for alpha, beta in {0.5, 1, 2} (numpy's
    scalar-power fast paths; beta also 0); other exponents go through pow and
    agree to ~1 ulp.  Raises NumericalUnderflow when a row normalizer is zero
    or non-finite.
    """
    n = int(inst.n)
    di = _device.device_instance(inst)
    dev = di.dev
    tau_t = _device.upload(np.asarray(tau.tau, dtype=np.float64), dev)
    p_t = torch.empty_like(tau_t)
    sums = torch.empty(n, dtype=torch.float64, device=dev)
    status = _device.new_status(dev)
    if n > 27000:  # beyond the fused row kernel's shared-memory row: the split kernels
        _device.update_split(n, tau_in=tau_t, tau_out=None, eta_b=di.eta_beta(params.beta), nbr=None, inc=None,
                             k=0, do_evap=False, keep=1.0, alpha=float(params.alpha), inv_gamma=1.0,
                             delta_ws=None, unnorm_ws=torch.empty_like(tau_t), p_out=p_t, rowsum_out=sums,
                             status=status)
    else:
        _device.row_update(n, tau_in=tau_t, eta_b=di.eta_beta(params.beta), want_p=True,
                           alpha=float(params.alpha), p_out=p_t, rowsum_out=sums, status=status)
    code, _ = _device.read_status(status)
    if code == _lib.TACO_UNDERFLOW:
        raise _underflow_from_sums(_device.download(sums))
    return ProbabilityMatrix(p=_device.download(p_t))


def init_starts(m: int, n: int, rng_stream: np.random.Generator) -> np.ndarray:
    """Uniform start city per ant from a host generator (colony.py:72-78);
    kept for API compatibility — the device stream draws starts on chip."""
    if m < 1:
        raise ValueError(f"m must be >= 1, got {m}")
    if n < 3:
        raise ValueError(f"n must be >= 3, got {n}")
    return rng_stream.integers(0, n, size=m, dtype=np.int64)


def construct_tours(p, inst, params, iteration: int, chunk_size: int | None = None,
                    probe=None, *, stream: str = "device", variant: str = "sorted") -> TourBatch:
    """Build m complete tours in n-1 lockstep selection rounds (colony.py:87-154).

    stream="device" (default): keyed on-chip Philox2x32-10 uniforms and the
    product-form rule argmax(W * u) — the fast path.
    stream="replay": the reference's own stream, regenerated on the device —
    the per-step Philox4x64 keys of SeedSequence(seed, spawn_key=(0, it, step))
    come from the host, and the (m, n) Exp(1) blocks are decoded from them on
    the device with numpy's ziggurat (k_numpy_stream.cu); tours equal the
    reference's bit for bit at GPU speed.
    stream="numpy": the same, with the deviate blocks produced by numpy on the
    host and uploaded step by step (slow; the replay's cross-check).
    In both reference-stream modes the start cities and the log-weight table
    are numpy's own (rng.py:65-68, selection.py:62-75).
    ``chunk_size`` is accepted and has no effect (chunking is bit-invisible in
    the reference too, colony.py:119-124); ``probe`` is not supported.
    variant: "sorted" (pruned scan of the row-sorted table) or "dense" (full
    row streaming); both return identical tours.
    Roulette wheel (selection="rw", colony.py:127-141) spins on P itself:
    stream="device" draws one threshold per (step, ant) on chip; "numpy" and
    "replay" use the reference's thresholds exp(-E[:, 0]) (rng.py:52-62) —
    generated by numpy, or decoded on the device with numpy taking the exp —
    and return its tours bit for bit.
    """
    if probe is not None:
        raise NotImplementedError("construction probes are not supported by the device engine")
    if chunk_size is not None and chunk_size < 1:
        raise ValueError(f"chunk_size must be >= 1, got {chunk_size}")
    n, m = int(inst.n), int(params.m)
    gamma = construction_gamma(params, iteration)
    di = _device.device_instance(inst)
    dev = di.dev
    p_host = np.asarray(p.p, dtype=np.float64)
    if _selection(params) is Selection.RW:
        tours_t, costs_t = _construct_roulette(p_host, n, m, params.seed, iteration, dev, di.dist, stream)
    elif stream in ("numpy", "replay"):
        tours_t = _construct_reference_stream(p_host, n, m, params.seed, iteration, gamma, dev,
                                              replay=(stream == "replay"))
        costs_t = _device.tour_cost(tours_t, di.dist)
    elif stream == "device":
        tours_t, costs_t = _construct_device_stream(p_host, n, m, params.seed, iteration, gamma, dev,
                                                    variant, di.dist)
    else:
        raise ValueError(f"stream must be 'device', 'replay' or 'numpy', got {stream!r}")
    return TourBatch(tours=_device.download(tours_t).astype(np.int64, copy=False),
                     costs=_device.download(costs_t))


def _construct_device_stream(p_host, n, m, seed, iteration, gamma, dev, variant, dist):
    if variant == "sorted" and n > _lib.load().taco_max_sorted_n():
        variant = "dense"
    if variant not in ("sorted", "dense"):
        raise ValueError(f"variant must be 'sorted' or 'dense', got {variant!r}")
    p_t = _device.upload(p_host, dev)
    tables = _device.SelectionTables(n, dev, dense=(variant == "dense"), sorted_=(variant == "sorted"))
    _device.selection_table_from_p(p_t, 1.0 / gamma, tables)
    tours = torch.zeros((m, n), dtype=torch.int32, device=dev)
    costs = torch.empty(m, dtype=torch.float64, device=dev)
    status = _device.new_status(dev)
    code = _lib.CONSTRUCT_SORTED if variant == "sorted" else _lib.CONSTRUCT_DENSE
    # f64 fallback source when no W > 0 candidate is left: P itself
    _device.construct(n, m, 0, code, tables, seed, iteration, tours, status, dist=dist, costs_out=costs,
                      fallback=(p_t, 1.0, None), inv_gamma=1.0 / gamma)
    _raise_construct_status(status)
    return tours, costs


def _construct_roulette(p_host, n, m, seed, iteration, dev, dist, stream):
    p_t = _device.upload(p_host, dev)
    status = _device.new_status(dev)
    if stream == "device":
        tours = torch.zeros((m, n), dtype=torch.int32, device=dev)
        costs = torch.empty(m, dtype=torch.float64, device=dev)
        _device.construct_rw(n, m, 0, p_t, seed, iteration, tours, status, dist=dist, costs_out=costs)
        _raise_construct_status(status)
        return tours, costs
    if stream not in ("numpy", "replay"):
        raise ValueError(f"stream must be 'device', 'replay' or 'numpy', got {stream!r}")
    starts = _rng.start_cities(seed, iteration, m, n)
    current = _device.upload(starts, dev)
    visited = torch.zeros((m, n), dtype=torch.uint8, device=dev)
    visited[torch.arange(m, device=dev), current] = 1
    tours = torch.zeros((m, n), dtype=torch.int64, device=dev)
    tours[:, 0] = current
    lib, hs = _lib.load(), _device.stream_handle()
    replay = rw_replay_thresholds(seed, iteration, m, n, dev) if stream == "replay" else None
    for step in range(1, n):
        u = replay(step) if replay else _rng.step_uniforms(seed, iteration, step, m, n)
        u_t = _device.upload(u, dev)
        _lib.check(lib.taco_rw_parity(n, m, step, p_t.data_ptr(), u_t.data_ptr(), current.data_ptr(),
                                      visited.data_ptr(), tours.data_ptr(), status.data_ptr(), None, 0, hs),
                   "taco_rw_parity")
    if replay:
        replay.check()
    _raise_construct_status(status)
    return tours, _device.tour_cost(tours, dist)


class rw_replay_thresholds:
    """The reference's roulette thresholds u = exp(-E[:, 0]) of each step
    (rng.step_uniforms rng.py:52-62): column 0 of the step's Exp(1) block is
    decoded on the device from numpy's Philox key (taco_replay_first_column),
    and the exponential is taken by numpy itself, so u is the reference's bit
    for bit (one m-element round trip per step instead of the (m, n) block)."""

    def __init__(self, seed: int, iteration: int, m: int, n: int, dev):
        self.m, self.n, self.dev = m, n, dev
        self.keys = _rng.step_keys(seed, iteration, n)
        lib = _lib.load()
        self.ws_bytes = int(lib.taco_replay_workspace_bytes(m, n))
        self.ws = torch.empty(self.ws_bytes, dtype=torch.uint8, device=dev)
        self.flags = torch.zeros(2, dtype=torch.int32, device=dev)
        self.e0 = torch.empty(m, dtype=torch.float64, device=dev)

    def __call__(self, step: int) -> np.ndarray:
        k0, k1 = (int(v) for v in self.keys[step - 1])
        _lib.check(_lib.load().taco_replay_first_column(self.n, self.m, k0, k1, self.ws.data_ptr(), self.ws_bytes,
                                                        self.e0.data_ptr(), self.flags.data_ptr(),
                                                        _device.stream_handle()), "taco_replay_first_column")
        return np.exp(-_device.download(self.e0))  # numpy's exp, as rng.py:62

    def check(self) -> None:
        ambiguous, overflow = (int(v) for v in self.flags.cpu().tolist())
        if ambiguous or overflow:
            raise ReplayUnreliable(f"replay flags: {ambiguous} close wedge tests, overflow={overflow}")


def _raise_construct_status(status: torch.Tensor) -> None:
    code, _ = _device.read_status(status)
    if code == _lib.TACO_NO_CANDIDATE:
        raise AssertionError("selector chose a visited city")


class ReplayUnreliable(RuntimeError):
    """A replayed ziggurat comparison was too close to call with CUDA's exp
    (or the replay window overflowed); use stream="numpy" for that call."""


def _construct_reference_stream(p_host, n, m, seed, iteration, gamma, dev, replay: bool) -> torch.Tensor:
    # log-weight table with the reference's numpy arithmetic (selection.py:72-74)
    logw = np.full(p_host.shape, -np.inf)
    np.log(p_host, out=logw, where=p_host > 0)
    np.divide(logw, gamma, out=logw)
    logw_t = _device.upload(logw, dev)
    starts = _rng.start_cities(seed, iteration, m, n)
    current = _device.upload(starts, dev)
    visited = torch.zeros((m, n), dtype=torch.uint8, device=dev)
    visited[torch.arange(m, device=dev), current] = 1
    tours = torch.zeros((m, n), dtype=torch.int64, device=dev)
    tours[:, 0] = current
    status = _device.new_status(dev)
    lib = _lib.load()
    stream = _device.stream_handle()
    if replay:
        keys = _rng.step_keys(seed, iteration, n)
        ws_bytes = int(lib.taco_replay_workspace_bytes(m, n))
        ws = torch.empty(ws_bytes, dtype=torch.uint8, device=dev)
        flags = torch.zeros(2, dtype=torch.int32, device=dev)
        for step in range(1, n):
            k0, k1 = (int(v) for v in keys[step - 1])
            _lib.check(lib.taco_select_replay(n, m, step, k0, k1, logw_t.data_ptr(), current.data_ptr(),
                                              visited.data_ptr(), tours.data_ptr(), ws.data_ptr(), ws_bytes,
                                              flags.data_ptr(), status.data_ptr(), stream), "taco_select_replay")
        ambiguous, overflow = (int(v) for v in flags.cpu().tolist())
        if ambiguous or overflow:
            raise ReplayUnreliable(f"replay flags: {ambiguous} close wedge tests, overflow={overflow}")
    else:
        for step in range(1, n):
            e_t = _device.upload(_rng.step_exponentials(seed, iteration, step, m, n), dev)
            _lib.check(lib.taco_select_parity(n, m, step, logw_t.data_ptr(), e_t.data_ptr(), current.data_ptr(),
                                              visited.data_ptr(), tours.data_ptr(), status.data_ptr(), stream),
                       "taco_select_parity")
    _raise_construct_status(status)
    return tours


def batch_costs(tours, inst) -> np.ndarray:
    """Closed-tour lengths of an (m, n) tour array in numpy's pairwise
    summation order (model.py:292-295); bit-exact with the reference."""
    t = np.ascontiguousarray(np.asarray(tours, dtype=np.int64))
    if t.ndim != 2 or t.shape[1] != inst.n:
        raise ValueError(f"tours must have shape (m, {inst.n}), got {t.shape}")
    if t.size and (t.min() < 0 or t.max() >= inst.n):
        raise IndexError("tour entries out of range")
    di = _device.device_instance(inst)
    return _device.download(_device.tour_cost(_device.upload(t, di.dev), di.dist))


def tour_cost(tour, inst) -> float:
    """Length of one closed tour (model.py:285-289)."""
    t = np.asarray(tour, dtype=np.int64)
    check_permutations(t, inst.n)
    return float(batch_costs(t[None, :], inst)[0])
