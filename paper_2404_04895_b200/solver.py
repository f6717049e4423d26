"""Device-resident TensorACO solver: ``Solver(instance, params).step()`` /
``.run()``.

The reference has no solver object; its iteration is the loop body of
``run_experiment`` (bench.py:199-206):
    construct_tours -> select_elite -> accumulate_increments -> apply_update
    -> compute_probability_matrix
The Solver runs exactly that sequence per ``step()`` with all state resident in
HBM and six kernel launches per iteration:

    1. taco_construct        tours (m x n int32) from the row-sorted fp32
                             selection table; the kernel's epilogue sums each
                             tour's length in numpy's pairwise order
       [multi-GPU: all-gather of the m lengths over NCCL]
    2. taco_elite_order      stable rank of the lengths
    3. taco_track_best       best-so-far tour / length on device
    4. taco_elite_neighbors  (prev, next) of every city in the k elite tours
       [multi-GPU: taco_shard_elites + SUM all-reduce of the k elite tours]
    5. taco_row_update       deposit + evaporation + P + W(gamma of it+1), then
    6. (k_row_sort)          the row-sorted table the next construction scans
       [multi-GPU, row-partitioned: this rank's rows only, then an in-place
        all-gather of the selection table and of the status words]

The host synchronizes only when a result is read (``step()`` returns the best
tour and length; ``iterate()`` reads every iteration's result while the next
one runs; ``run()`` reads once at the end).

On one GPU the iteration is captured once as a CUDA graph and replayed
(``graph=True``, the default there): the iteration number and the next 1/gamma
live in a device ``taco_iter_state`` that the kernels read and a final
``taco_iter_advance`` launch moves on, so the captured launches replay
unchanged.  ``run()`` replays a graph of several iterations at a time.
"""

from __future__ import annotations

import math
import struct

import numpy as np
import torch
import torch.distributed as tdist

from . import _device, _lib
from .colony import NumericalUnderflow, construction_gamma
from .distributed import (AntShard, gather_colony, gather_costs, gather_rows, row_partition, shard_ants,
                          share_elites, share_status)
from .model import AcoParams, PheromoneState, ProbabilityMatrix, Selection, TourBatch, instance_from_distances


def _as_instance(instance):
    if hasattr(instance, "dist") and hasattr(instance, "eta") and hasattr(instance, "n"):
        return instance
    return instance_from_distances(np.asarray(instance, dtype=np.float64))


def _as_params(params, n: int, overrides: dict):
    if params is None:
        return AcoParams.for_instance(n, **overrides)
    if overrides:
        raise TypeError("pass either an AcoParams object or keyword parameters, not both")
    return params


class _Timer:
    """CUDA-event pairs around selected launches (no-op without a dict)."""

    def __init__(self, timers: dict | None):
        self.timers = timers
        self._open = {}

    def start(self, name: str) -> None:
        if self.timers is not None and name in self.timers:
            e = torch.cuda.Event(enable_timing=True)
            e.record()
            self._open[name] = e

    def stop(self, name: str) -> None:
        if name in self._open:
            e = torch.cuda.Event(enable_timing=True)
            e.record()
            self.timers[name].append((self._open.pop(name), e))


class Solver:
    """TensorACO on one B200, or sharded over the ranks of a process group.

    instance: a TspInstance (this package's or the reference's), an (n, n)
    distance matrix, or a device instance (``device_euclidean_instance``).  params: an AcoParams, or keyword overrides of
    ``AcoParams.for_instance`` (alpha, beta, rho, n_ants / m, k, selection,
    seed, gamma_schedule, q0_tau, max_iters).
    construct: "auto" (default: "dense" for n < DENSE_MAX_N, else "sorted"),
    "sorted" (pruned scan of the row-sorted table) or "dense" (full-row stream).
    stream: "device" (default, the on-chip Philox2x32 stream) or "replay":
    every iteration replays the reference's own numpy streams on the device
    (colony.construct_tours(stream="replay")) with the reference's log-domain
    rule, so a run reproduces antbatch's run_experiment bit for bit (tours,
    pheromone, best lengths) — the parity mode, one GPU only.
    group: torch.distributed group to shard ants over (default: the world
    group when initialized with more than one rank).
    update: "replicated" (default: every rank updates all rows of its own
    replica, no n^2 collective) or "partitioned" (each rank updates its n/R
    rows of tau / P / the selection table and the table rows are
    all-gathered: 6n^2 B per iteration).
    graph: replay a captured CUDA graph per iteration (default: on for a
    single-GPU device-stream colony; the sharded and replay modes always run
    eagerly).  Measured per iteration, eager -> graph: C1 0.192 -> 0.183 ms,
    C2 -1.9%, C3 1.588 -> 1.578 ms, C4 15.53 -> 15.50 ms.
    graph_warmup: eager iterations before the first capture (default
    GRAPH_WARMUP = 32: a short run does not pay a capture it cannot
    amortize; 0 captures at the second iteration).
    """

    GRAPH_BATCH = 8  # iterations per graph replay in run()
    GRAPH_WARMUP = 32  # eager iterations before the first capture
    FUSED_MAX_N = 27000  # the fused row kernel stages a row of n doubles in shared memory
    # construct="auto": the full-row kernel below this n (no row sort; n = 51,
    # m = 64: 0.040 vs 0.044 ms per iteration; even at n = 100; sorted from 200)
    DENSE_MAX_N = 96

    def __init__(self, instance, params=None, *, construct: str = "auto", stream: str = "device",
                 group=None, graph: bool | None = None, update: str | None = None,
                 graph_warmup: int | None = None, **overrides):
        if isinstance(instance, _device.DeviceInstance):  # built on the device (from_coords)
            self.inst, device_inst = None, instance
        else:
            self.inst, device_inst = _as_instance(instance), None
        self.n = n = int(device_inst.n if device_inst is not None else self.inst.n)
        self.params = p = _as_params(params, n, overrides)
        self.rw = Selection(p.selection) is Selection.RW  # roulette wheel spins on P itself
        if construct not in ("auto", "sorted", "dense"):
            raise ValueError(f"construct must be 'auto', 'sorted' or 'dense', got {construct!r}")
        if construct == "auto":  # tiny rows: the full-row kernel needs no sorted table
            construct = "dense" if n < self.DENSE_MAX_N else "sorted"
        lib = _lib.load()
        if construct == "sorted" and n > lib.taco_max_sorted_n():
            construct = "dense"
        self.construct = construct
        self._variant = _lib.CONSTRUCT_SORTED if construct == "sorted" else _lib.CONSTRUCT_DENSE
        if stream not in ("device", "replay"):
            raise ValueError(f"stream must be 'device' or 'replay', got {stream!r}")
        self.stream = stream

        self.group = group
        if group is None and tdist.is_available() and tdist.is_initialized() and tdist.get_world_size() > 1:
            self.group = tdist.group.WORLD
        world = tdist.get_world_size(self.group) if self.group is not None else 1
        rank = tdist.get_rank(self.group) if self.group is not None else 0
        self.shard: AntShard = shard_ants(p.m, rank, world)
        if stream == "replay" and world > 1:
            raise ValueError("the reference-stream replay runs on one GPU")

        if update is None:
            # replicated (north_star: every rank applies the identical deposit,
            # no n^2 collective); "partitioned" trades an n^2 all-gather of
            # the selection table for 1/R of the update
            update = "replicated"
        if update not in ("replicated", "partitioned"):
            raise ValueError(f"update must be 'replicated' or 'partitioned', got {update!r}")
        # (rows past the fused row kernel's shared memory take the replicated
        # split update)
        self.partitioned = update == "partitioned" and world > 1 and n <= self.FUSED_MAX_N
        if self.partitioned and Selection(p.selection) is Selection.ADAIR and p.gamma_schedule.gamma_min < 1.0:
            # steps left without a W > 0 city are decided from the row's
            # tau^alpha eta^beta (include/taco.h), which a row-partitioned rank
            # holds only for its own rows
            raise ValueError("update='partitioned' needs gamma >= 1 (gamma_min < 1 can leave steps to the f64 "
                             "fallback, which reads every row of tau); use update='replicated'")
        # row partition: this rank updates rows [begin, end); the row buffers
        # carry world * chunk rows so the table all-gather has equal chunks
        self._part = row_partition(n, rank, world) if self.partitioned else row_partition(n, 0, 1)
        rows = self._part.rows if self.partitioned else n

        self.di = device_inst if device_inst is not None else _device.device_instance(self.inst)
        dev = self.dev = self.di.dev
        m, k = p.m, p.k
        self.eta_b = self.di.eta_beta(p.beta)
        self.tau = torch.zeros((rows, n), dtype=torch.float64, device=dev)
        self.tau[:n].fill_(float(p.q0_tau))
        self.tau[:n].fill_diagonal_(0.0)
        replay = stream == "replay"
        table = not (replay or self.rw)
        self.tables = _device.SelectionTables(n, dev, dense=(construct == "dense" and table),
                                              sorted_=(construct == "sorted" and table), rows=rows)
        if self.rw:  # P (f64) is the spin input; steps that needed the exact recount
            self.p = torch.empty((rows, n), dtype=torch.float64, device=dev)
            self.rw_exact_steps = torch.zeros(1, dtype=torch.int64, device=dev)
        if replay:  # reference-stream state: P, the numpy log table, lockstep buffers
            self.p = torch.empty((n, n), dtype=torch.float64, device=dev)
            self.logw = torch.empty((n, n), dtype=torch.float64, device=dev)
            self.tours64 = torch.zeros((m, n), dtype=torch.int64, device=dev)
            self.visited = torch.zeros((m, n), dtype=torch.uint8, device=dev)
            self.current = torch.zeros(m, dtype=torch.int64, device=dev)
            self.replay_ws_bytes = int(lib.taco_replay_workspace_bytes(m, n))
            self.replay_ws = torch.empty(self.replay_ws_bytes, dtype=torch.uint8, device=dev)
            self.replay_flags = torch.zeros(2, dtype=torch.int32, device=dev)
        sh = self.shard
        # zero-initialized so a failed construction never leaves out-of-range cities
        self.tours_local = torch.zeros((sh.per_rank, n), dtype=torch.int32, device=dev)
        self.costs_local = torch.zeros(sh.per_rank, dtype=torch.float64, device=dev)
        if world > 1:
            # costs-first exchange: all m lengths, then only the k elite tours
            self.costs_all = torch.zeros(m, dtype=torch.float64, device=dev)
            uneven = m % world != 0
            self._pad_costs = torch.zeros(world * sh.per_rank, dtype=torch.float64, device=dev) if uneven else None
            # the k elite tours plus one word: every rank's construction stop
            # flag (status[3]) rides the same SUM all-reduce, so a failure on
            # one rank skips the same iteration's update on every rank
            self._elite_buf = torch.zeros(k * n + 1, dtype=torch.int32, device=dev)
            self.elite_tours = self._elite_buf[:k * n].view(k, n)
            self._stop_flag = self._elite_buf[k * n:]
            self.elite_costs = torch.zeros(k, dtype=torch.float64, device=dev)
            self._ident_k = torch.arange(k, dtype=torch.int32, device=dev)
            self._all_tours_iteration = -1  # last_batch() gathers all tours on demand
            self.tours_all = None
        else:
            self.tours_all, self.costs_all = self.tours_local, self.costs_local
        self.order = torch.zeros(m, dtype=torch.int32, device=dev)
        self.elite_ws = _device.EliteWorkspace(m, dev)
        self.nbr = torch.zeros((n, k, 2), dtype=torch.int32, device=dev)  # city-major edge map
        self.inc = torch.zeros(k, dtype=torch.float64, device=dev)
        # status (4 x i32) | best length (f64) | best iteration (i32, pad) | best tour (n x i32):
        # one device block, so step() reads everything back in a single copy
        self._io = torch.zeros(32 + 4 * n, dtype=torch.uint8, device=dev)
        self._io_host = torch.empty_like(self._io, device="cpu").pin_memory()
        self.best_cost = self._io[16:24].view(torch.float64)
        self.best_cost.fill_(math.inf)
        self.best_iter = self._io[24:28].view(torch.int32)
        self.best_iter.fill_(-1)
        self.best_tour = self._io[32:].view(torch.int32)
        self.rowsum = torch.zeros(n, dtype=torch.float64, device=dev)
        # rows longer than the fused kernel's shared-memory row use the split
        # update, with its delta / tau^alpha eta^beta workspaces
        # the split kernels also win for large elite sets at n >= 4000: their
        # deposit spreads a row's 2k additions over warp-per-row blocks
        # (n = 5000: k = 6553 1.52 vs 2.42 ms, k = 3276 1.11 vs 1.43, k = 1638
        # 0.90 vs 0.94; n = 2392, k = 1638 and n = 10000, k = 819 stay fused)
        self._split_update = n > self.FUSED_MAX_N or (n >= 4000 and p.k >= 1500 and not self.partitioned)
        self._delta_ws = torch.empty((n, n), dtype=torch.float64, device=dev) if self._split_update else None
        self._unnorm_ws = torch.empty((n, n), dtype=torch.float64, device=dev) if self._split_update else None
        self.status = self._io[0:16].view(torch.int32)
        self.status[1] = 2**31 - 1  # _device.new_status layout: smallest offending index
        self.iteration = 0
        self.keep = 1.0 - p.rho  # pheromone.py:81 evaluates (1.0 - rho) in float64
        # device iteration state (taco_iter_state) + 1/gamma per t mod period
        period = int(p.gamma_schedule.period) if Selection(p.selection) is Selection.ADAIR else 1
        self._period = period
        self._inv_gamma = torch.tensor([1.0 / construction_gamma(p, t) for t in range(period)],
                                       dtype=torch.float64, device=dev)
        self.state = torch.zeros(32, dtype=torch.uint8, device=dev)  # taco_iter_state
        self._write_state(0)
        # default: graphs on one GPU (small colonies: 9.5k -> 16.7k it/s; the
        # launch gaps still cost 0.6% at C3); GRAPH_WARMUP keeps the capture,
        # ~2-10 ms, out of runs too short to amortize it
        if graph is None:
            use_graph = world == 1 and stream == "device"
        else:
            use_graph = bool(graph)
        if use_graph and (world > 1 or stream != "device"):
            raise ValueError("CUDA-graph replay covers the single-GPU device-stream solver")
        self.graph = use_graph
        self._graphs: dict[int, torch.cuda.CUDAGraph] = {}
        self._eager_left = self.GRAPH_WARMUP if graph_warmup is None else int(graph_warmup)
        # P / W for iteration 0 from the initial pheromone (bench.py:191-192);
        # the reference raises NumericalUnderflow right there
        self._rebuild_tables(evaporate=False, gamma_next=construction_gamma(p, 0))
        self.check()

    # ------------------------------------------------------------------
    def _rebuild_tables(self, evaporate: bool, gamma_next: float, state=None) -> None:
        """End-of-iteration update: deposit + evaporation + P / W.  The fused
        row kernel (taco_row_update) is faster while a row fits in shared
        memory; longer rows use the split streaming kernels (taco_update_split,
        bit-identical, any n)."""
        t = self.tables
        p_mode = self.stream == "replay" or self.rw  # P itself is the next iteration's input
        common = dict(
            tau_in=self.tau, tau_out=self.tau if evaporate else None, eta_b=self.eta_b,
            nbr=self.nbr if evaporate else None, inc=self.inc if evaporate else None,
            k=self.params.k if evaporate else 0, do_evap=evaporate, keep=self.keep,
            alpha=float(self.params.alpha), inv_gamma=1.0 / gamma_next, p_out=self.p if p_mode else None,
            rowsum_out=self.rowsum, w_out=None if p_mode else t.w, ldw=t.ldw,
            sw_out=None if p_mode else t.sw, si_out=None if p_mode else t.si, status=self.status, state=state)
        if self.partitioned:  # my rows, then every rank's rows of the construction input
            _device.row_update_rows(self._part.begin, self._part.end, self.n, want_p=True, **common)
            if p_mode:
                self._gather_rows(self.p)
            elif t.sw is not None:
                self._gather_rows(t.sw)
                self._gather_rows(t.si)
            else:
                self._gather_rows(t.w)
        elif self._split_update:
            _device.update_split(self.n, delta_ws=self._delta_ws, unnorm_ws=self._unnorm_ws, **common)
        else:
            _device.row_update(self.n, want_p=True, **common)
        if self.shard.world > 1:
            self._share_status()

    def _gather_rows(self, buf: torch.Tensor) -> None:
        gather_rows(buf, self._part, self.group)

    def _share_status(self) -> None:
        """Fail-stop across ranks: a failure seen by one rank's ants or rows
        stops every rank's next construction, and every rank raises it at the
        same step (device-side, no host sync)."""
        share_status(self.status, self.group)

    def _write_state(self, it: int) -> None:
        """Device state for iteration `it`: (it, 1/gamma(it + 1), 1/gamma(it))."""
        inv = 1.0 / construction_gamma(self.params, it + 1)
        cur = 1.0 / construction_gamma(self.params, it)
        host = torch.frombuffer(bytearray(struct.pack("<IIddd", it & 0xFFFFFFFF, 0, inv, cur, 0.0)),
                                dtype=torch.uint8)
        self.state.copy_(host)

    def step_async(self, timers: dict | None = None, scan_count: torch.Tensor | None = None) -> None:
        """Enqueue one full iteration on the current stream (no host sync).

        timers: optional {"construct": [...], "update": [...]} lists that get
        a (start, end) CUDA-event pair around those launches (bench.py).
        scan_count: optional device u64 that accumulates the table windows
        the sorted construction kernel read.  Either forces the eager path.
        """
        if self.graph and timers is None and scan_count is None:
            self._replay(1)
        else:
            self._enqueue(timers, scan_count)

    def _replay(self, iters: int) -> None:
        g = self._graphs.get(iters)
        if g is None:
            if self._eager_left > 0:
                # the first GRAPH_WARMUP iterations run eagerly (same launches,
                # same device state): one-time host work (kernel attributes,
                # device queries) stays outside any capture, and a short run
                # does not pay a capture (~2 ms) it cannot amortize
                for _ in range(iters):
                    self._enqueue(None, None)
                self._eager_left -= iters
                return
            g = self._capture(iters)
        g.replay()
        self.iteration += iters

    def _capture(self, iters: int) -> torch.cuda.CUDAGraph:
        # the device state already holds self.iteration (every iteration of a
        # graph-mode solver advances it on the stream); capture does not run
        # capture_begin/end directly: torch.cuda.graph() would also synchronize,
        # empty the device and pinned-host caches (and optionally gc.collect()),
        # which costs milliseconds per capture; the iteration allocates nothing
        side = torch.cuda.Stream(device=self.dev)
        side.wait_stream(torch.cuda.current_stream(self.dev))
        g = torch.cuda.CUDAGraph()
        it0 = self.iteration
        with torch.cuda.stream(side):
            g.capture_begin(capture_error_mode="thread_local")
            try:
                for _ in range(iters):
                    self._enqueue(None, None)
            finally:
                g.capture_end()
        self.iteration = it0  # _enqueue counted the captured (not yet run) iterations
        torch.cuda.current_stream(self.dev).wait_stream(side)
        self._graphs[iters] = g
        return g

    def _enqueue(self, timers: dict | None, scan_count: torch.Tensor | None) -> None:
        """Launch one iteration (eagerly, or into a graph being captured)."""
        with _device.pinned_stream():
            self._enqueue_launches(timers, scan_count)

    def _enqueue_launches(self, timers: dict | None, scan_count: torch.Tensor | None) -> None:
        p, sh, it = self.params, self.shard, self.iteration
        st = self.state if self.graph else None
        lib = _lib.load()
        ev = _Timer(timers)
        ev.start("construct")
        if self.stream == "replay":
            self._construct_replay(it)
        elif self.rw:
            _device.construct_rw(self.n, sh.count, sh.offset, self.p, p.seed, it, self.tours_local, self.status,
                                 dist=self.di.dist, costs_out=self.costs_local, exact_count=self.rw_exact_steps,
                                 state=st)
        else:
            # f64 fallback source (no W > 0 candidate left): the row's
            # tau^alpha eta^beta, current on every rank unless row-partitioned
            fb = None if self.partitioned else (self.tau, float(p.alpha), self.eta_b)
            _device.construct(self.n, sh.count, sh.offset, self._variant, self.tables, p.seed, it,
                              self.tours_local, self.status, scan_count, dist=self.di.dist,
                              costs_out=self.costs_local, state=st, fallback=fb,
                              inv_gamma=1.0 / construction_gamma(p, it))
        ev.stop("construct")
        if sh.world > 1:
            gather_costs(self.costs_local, sh, self.costs_all, self.group, self._pad_costs)
        _device.elite_order(self.costs_all, self.elite_ws, self.order)
        if sh.world > 1:
            _lib.check(lib.taco_shard_elites(self.n, p.k, self.order.data_ptr(), sh.offset, sh.count,
                                             self.tours_local.data_ptr(), self.costs_all.data_ptr(),
                                             self.elite_tours.data_ptr(), self.elite_costs.data_ptr(),
                                             _device.stream_handle()), "taco_shard_elites")
            self._stop_flag.copy_(self.status[3:4])
            share_elites(self._elite_buf, self.group)
            torch.maximum(self.status[3:4], self._stop_flag, out=self.status[3:4])
            tours, costs, order = self.elite_tours, self.elite_costs, self._ident_k
        else:
            tours, costs, order = self.tours_all, self.costs_all, self.order
        _lib.check(lib.taco_track_best(self.n, tours.data_ptr(), costs.data_ptr(), order.data_ptr(),
                                       self.best_cost.data_ptr(), self.best_tour.data_ptr(),
                                       self.best_iter.data_ptr(), it & 0xFFFFFFFF, self.status.data_ptr(), _lib.ptr(st),
                                       _device.stream_handle()), "taco_track_best")
        _device.elite_neighbors(tours, order, costs, p.k, self.nbr, self.inc)
        ev.start("update")
        self._rebuild_tables(evaporate=True, gamma_next=construction_gamma(p, it + 1), state=st)
        ev.stop("update")
        if st is not None:
            _lib.check(lib.taco_iter_advance(st.data_ptr(), self._inv_gamma.data_ptr(), self._period,
                                             _device.stream_handle()), "taco_iter_advance")
        self.iteration = it + 1

    def _construct_replay(self, it: int) -> None:
        """Lockstep construction on the reference's streams (colony.py:101-152):
        numpy's start cities and log table (host), the step deviates replayed
        on the device from numpy's Philox keys."""
        from . import rng as _rng
        from .colony import ReplayUnreliable

        n, p, lib = self.n, self.params, _lib.load()
        self.check()  # the host drives this mode step by step: raise where the reference would
        starts = torch.from_numpy(_rng.start_cities(p.seed, it, p.m, n)).to(self.dev)
        self.current.copy_(starts)
        self.visited.zero_()
        self.visited[torch.arange(p.m, device=self.dev), starts] = 1
        self.tours64[:, 0] = starts
        stream = _device.stream_handle()
        if self.rw:  # roulette wheel on the reference's thresholds (colony.py:127-134)
            from .colony import rw_replay_thresholds

            thresholds = rw_replay_thresholds(p.seed, it, p.m, n, self.dev)
            for step in range(1, n):
                u_t = _device.upload(thresholds(step), self.dev)
                _lib.check(lib.taco_rw_parity(n, p.m, step, self.p.data_ptr(), u_t.data_ptr(),
                                              self.current.data_ptr(), self.visited.data_ptr(),
                                              self.tours64.data_ptr(), self.status.data_ptr(), None, 0, stream),
                           "taco_rw_parity")
            self.tours_local.copy_(self.tours64)
            _device.tour_cost(self.tours64, self.di.dist, self.costs_local)
            thresholds.check()
            return
        gamma = construction_gamma(p, it)
        ph = _device.download(self.p)
        logw = np.full(ph.shape, -np.inf)
        np.log(ph, out=logw, where=ph > 0)  # selection.py:72-74, numpy's own log
        np.divide(logw, gamma, out=logw)
        self.logw.copy_(torch.from_numpy(logw))
        keys = _rng.step_keys(p.seed, it, n)
        for step in range(1, n):
            k0, k1 = (int(v) for v in keys[step - 1])
            _lib.check(lib.taco_select_replay(n, p.m, step, k0, k1, self.logw.data_ptr(), self.current.data_ptr(),
                                              self.visited.data_ptr(), self.tours64.data_ptr(),
                                              self.replay_ws.data_ptr(), self.replay_ws_bytes,
                                              self.replay_flags.data_ptr(), self.status.data_ptr(), stream),
                       "taco_select_replay")
        self.tours_local.copy_(self.tours64)
        _device.tour_cost(self.tours64, self.di.dist, self.costs_local)
        ambiguous, overflow = (int(v) for v in self.replay_flags.cpu().tolist())
        if ambiguous or overflow:
            raise ReplayUnreliable(f"replay flags: {ambiguous} close wedge tests, overflow={overflow}")

    def check(self) -> None:
        """Raise the reference's exception for any failure recorded so far
        (with a row-partitioned update, the underflow report is a collective;
        every rank raises it at the same step)."""
        code, _ = _device.read_status(self.status)  # identical on every rank (_share_status)
        self._raise_status(code)

    def _raise_status(self, code: int) -> None:
        if code == _lib.TACO_UNDERFLOW:
            from .colony import _underflow_from_sums
            sums = self.rowsum
            if self.partitioned:  # each rank wrote its own rows of the sums (the rest stay 0)
                sums = sums.clone()
                tdist.all_reduce(sums, op=tdist.ReduceOp.SUM, group=self.group)
            raise _underflow_from_sums(_device.download(sums))
        if code == _lib.TACO_NO_CANDIDATE:
            raise AssertionError("selector chose a visited city")
        if code != 0:
            raise RuntimeError(f"device status {code}")

    def best(self) -> tuple[np.ndarray, float]:
        """(best tour so far as int64 array, its length)."""
        tour = _device.download(self.best_tour).astype(np.int64)
        return tour, float(self.best_cost.item())

    def step(self) -> tuple[np.ndarray, float]:
        """Run one iteration; return the best tour so far and its length
        (one device-to-host copy: status, best length and best tour)."""
        self.step_async()
        return self._read_back()

    def iterate(self, iters: int):
        """Run ``iters`` iterations, yielding ``(iteration, best_tour,
        best_length)`` after each one — the same values ``step()`` returns.

        Pipelined: iteration t+1 is already queued on the device when the
        result of iteration t is read (an async D2H copy into a pinned double
        buffer, waited on by event), so the device never idles on the host.
        The reference's per-iteration records (bench.py:199-207) come out of
        this loop at device speed."""
        bufs = [torch.empty_like(self._io_host).pin_memory() for _ in range(2)]
        events = [torch.cuda.Event(), torch.cuda.Event()]
        pending = None
        for t in range(int(iters)):
            self.step_async()
            b = t & 1
            bufs[b].copy_(self._io, non_blocking=True)
            events[b].record()
            if pending is not None:
                yield self._decode_io(*pending)
            pending = (bufs[b], events[b], self.iteration - 1)
        if pending is not None:
            yield self._decode_io(*pending)

    def _decode_io(self, buf: torch.Tensor, event, iteration: int):
        event.synchronize()
        raw = buf.numpy()
        self._raise_status(int(raw[0:4].view(np.int32)[0]))
        return (iteration, raw[32:].view(np.int32).astype(np.int64), float(raw[16:24].view(np.float64)[0]))

    def _read_back(self) -> tuple[np.ndarray, float]:
        self._io_host.copy_(self._io)  # synchronizes the stream
        raw = self._io_host.numpy()
        self._raise_status(int(raw[0:4].view(np.int32)[0]))
        return (raw[32:].view(np.int32).astype(np.int64),
                float(raw[16:24].view(np.float64)[0]))

    def run(self, max_iters: int | None = None) -> tuple[np.ndarray, float]:
        """Run ``max_iters`` iterations (default params.max_iters) and return
        the best tour and length."""
        iters = self.params.max_iters if max_iters is None else int(max_iters)
        if self.graph:
            batch = self.GRAPH_BATCH
            for _ in range(iters // batch):
                self._replay(batch)
            for _ in range(iters % batch):
                self._replay(1)
        else:
            for _ in range(iters):
                self.step_async()
        return self._read_back()

    # ---- checkpoint / resume ----------------------------------------------
    def checkpoint(self) -> dict:
        """Host copy of the whole iteration state: tau, the iteration counter
        and the best-so-far tour.  The streams are keyed by (seed, iteration),
        so ``restore`` continues bit-identically (the reference's
        state is (tau, iteration), model.py:218-232)."""
        self.check()
        tour, length = self.best()
        if self.partitioned:
            self._gather_rows(self.tau)
        return {"tau": _device.download(self.tau[:self.n]).copy(), "iteration": int(self.iteration),
                "best_tour": tour, "best_length": length, "best_iteration": int(self.best_iter.item()),
                "n": int(self.n), "seed": int(self.params.seed)}

    def restore(self, ckpt: dict) -> None:
        """Load a ``checkpoint()`` of a Solver on the same instance and params."""
        if int(ckpt["n"]) != self.n or int(ckpt["seed"]) != int(self.params.seed):
            raise ValueError("checkpoint is for a different instance size or seed")
        tau = np.asarray(ckpt["tau"], dtype=np.float64)
        if tau.shape != (self.n, self.n):
            raise ValueError(f"tau must have shape ({self.n}, {self.n})")
        it = int(ckpt["iteration"])
        self.status.copy_(_device.new_status(self.dev))  # a restored solver starts healthy
        self.tau[:self.n].copy_(torch.from_numpy(np.ascontiguousarray(tau)))
        self.best_tour.copy_(torch.from_numpy(np.asarray(ckpt["best_tour"], dtype=np.int32)))
        self.best_cost.fill_(float(ckpt["best_length"]))
        self.best_iter.fill_(int(ckpt["best_iteration"]))
        self.iteration = it
        self._write_state(it)
        # P / W of iteration `it` from the restored tau (what the end of
        # iteration it-1 built)
        self._rebuild_tables(evaporate=False, gamma_next=construction_gamma(self.params, it))

    def save(self, path: str) -> None:
        """``checkpoint()`` to an .npz file."""
        np.savez(path, **{k: np.asarray(v) for k, v in self.checkpoint().items()})

    def load(self, path: str) -> None:
        """``restore()`` from a ``save()`` file."""
        with np.load(path) as z:
            self.restore({k: z[k] for k in z.files})

    # ---- state inspection (host copies) ---------------------------------
    def pheromone(self) -> PheromoneState:
        """tau (a collective when row-partitioned: the rows are all-gathered)."""
        if self.partitioned:
            self._gather_rows(self.tau)
        return PheromoneState(tau=_device.download(self.tau[:self.n]), iteration=self.iteration)

    def probability(self) -> ProbabilityMatrix:
        if self.partitioned:
            self._gather_rows(self.tau)
        p = torch.empty_like(self.tau[:self.n])
        _device.row_update(self.n, tau_in=self.tau, eta_b=self.eta_b, want_p=True,
                           alpha=float(self.params.alpha), p_out=p)
        return ProbabilityMatrix(p=_device.download(p))

    def last_batch(self) -> TourBatch:
        """Tours and lengths of the most recent iteration (all ranks' ants;
        sharded runs all-gather the tours here, on demand — a collective every
        rank must call)."""
        if self.shard.world > 1 and self._all_tours_iteration != self.iteration:
            sh, m, n = self.shard, self.params.m, self.n
            if self.tours_all is None:
                self.tours_all = torch.zeros((m, n), dtype=torch.int32, device=self.dev)
            pad_t = torch.zeros((sh.world * sh.per_rank, n), dtype=torch.int32, device=self.dev) \
                if m % sh.world else None
            scratch = torch.zeros_like(self.costs_all)
            pad_c = torch.zeros_like(self._pad_costs) if self._pad_costs is not None else None
            gather_colony(self.tours_local, self.costs_local, sh, self.tours_all, scratch, self.group, pad_t, pad_c)
            self._all_tours_iteration = self.iteration
        return TourBatch(tours=_device.download(self.tours_all).astype(np.int64),
                         costs=_device.download(self.costs_all))

    def elite_order(self) -> np.ndarray:
        return _device.download(self.order)


__all__ = ["Solver", "NumericalUnderflow"]
