"""TensorACO-B200 benchmark (driver contract: one JSON line on rank 0).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--config c3] [--construct auto|sorted|dense]

A "step" is one full ACO iteration of the hot path (bench.py:199-206 of the
reference): construct m tours -> lengths -> stable elite sort -> index-mapped
deposit + evaporation -> P and the selection table for the next iteration.
The default workload is BASELINE.json's metric config: synthetic uniform
Euclidean n=2392 cities, m=4096 ants (k=409), AdaIR, on 1 GPU.  Under
torchrun the ants are sharded over the ranks (weak in the colony sense: the
whole colony is fixed and split).

--impl reference times the reference's own CPU implementation on the host
cores: the UNMODIFIED antbatch package installed in baseline/_ref (git-ignored,
it travels with the repo) through its own functions — run_experiment as-is
for C1, and for the larger configs one sampled-and-extrapolated iteration per
step (n-1 x the mean of sampled lockstep rounds + P, logw,
lengths and update), one independent colony per core (the reference is
single-threaded numpy).  Without baseline/_ref it falls back to
oracle/reference_port, the numpy restatement pinned to the reference's golden
vectors.
"""

from __future__ import annotations

import argparse
import gc
import json
import math
import os
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

CONFIGS = {
    # name: (n, m, selection)  — BASELINE.json configs
    "c1": (51, 64, "ir"),
    "c2": (1000, 1024, "adair"),
    "c3": (2392, 4096, "adair"),
    "c3ir": (2392, 4096, "ir"),
    "c3rw": (2392, 4096, "rw"),  # roulette-wheel ablation
    "c4": (10000, 8192, "ir"),
    "c5_256": (5000, 256, "ir"),
    "c5_4096": (5000, 4096, "ir"),
    "c5_65536": (5000, 65536, "ir"),
}
METRIC = "ACO iterations/sec at n=2392, m=4096 (city-selections/sec = m*(n-1)*it/s)"


def _metric(n: int, m: int) -> str:
    """BASELINE.json's metric at C3 (the default config); the same metric
    named with the config's own n and m elsewhere."""
    return METRIC if (n, m) == (2392, 4096) else (
        f"ACO iterations/sec at n={n}, m={m} (city-selections/sec = m*(n-1)*it/s)")
PEAKS_PATH = os.path.join(ROOT, "MEASURED_PEAKS.json")
HBM_FALLBACK = 6650.0  # GB/s, /opt/skills/guides/B200_PROFILING.md fallback


def _peaks() -> tuple[float, str]:
    try:
        with open(PEAKS_PATH) as f:
            return float(json.load(f)["hbm_gbs"]), "measured"
    except (OSError, KeyError, ValueError):
        return HBM_FALLBACK, "fallback"


def _capture(kernel: str, config: str) -> dict | None:
    """The committed ncu --set full summary of `kernel` captured on this config
    (profiles/traffic.json, written by scripts/summarize_profiles.py): DRAM
    bytes and warp instructions per launch, L2 hit rate, issue activity."""
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as f:
            return json.load(f).get(f"{kernel}@{config}")
    except (OSError, ValueError):
        return None


def _traffic(kernel: str, config: str):
    rec = _capture(kernel, config)
    return (rec["dram_bytes_per_launch"], rec["capture"]) if rec else (None, None)


def _config_dict(config: str, n: int, m: int, k: int, selection: str, period: int, world: int) -> dict:
    """The workload description, identical in both arms."""
    return {"workload": f"{config}: n={n} cities, m={m} ants, k={k}, {selection}, alpha=1 beta=2 rho=0.1, "
                        f"gamma 1.5->1.0 period {period}",
            "n": n, "m": m, "k": k, "selection": selection, "gamma_period": period,
            "instance": "U(0,2000)^2 Euclidean cities (seed 0), unrounded distances",
            "parallelism": f"ants sharded over {world} rank(s)"}


class _null:
    def __enter__(self):
        return self

    def __exit__(self, *exc):
        return False


class ClockSampler:
    """SM clock and clock-event (throttle) reasons sampled through NVML every
    ~2 ms, kept only inside the marked timed regions (``window()``), so short
    timed regions still get tens of samples and host-side gaps (instance
    setup, CPU baseline) do not dilute the median."""

    REASONS = (("hw_slowdown", 0x8), ("hw_thermal_slowdown", 0x40), ("sw_thermal_slowdown", 0x20),
               ("sw_power_cap", 0x4), ("hw_power_brake_slowdown", 0x80))

    def __init__(self, local_rank: int, period_s: float = 0.002):
        self.period = period_s
        self.samples: list[tuple[float, int]] = []
        self.max_mhz = None
        self._in_window = threading.Event()
        self._stop = threading.Event()
        self._thread = None
        self._nvml = None
        self._handle = None
        self._local = local_rank

    def _open(self):
        import pynvml
        import torch

        pynvml.nvmlInit()
        self._nvml = pynvml
        try:
            props = torch.cuda.get_device_properties(self._local)
            bus = f"{props.pci_domain_id:08x}:{props.pci_bus_id:02x}:{props.pci_device_id:02x}.0"
            self._handle = pynvml.nvmlDeviceGetHandleByPciBusId(bus)
        except Exception:  # noqa: BLE001 - fall back to the NVML index
            self._handle = pynvml.nvmlDeviceGetHandleByIndex(self._local)
        self.max_mhz = float(pynvml.nvmlDeviceGetMaxClockInfo(self._handle, pynvml.NVML_CLOCK_SM))

    def _poll(self):
        nv, h = self._nvml, self._handle
        get_reasons = getattr(nv, "nvmlDeviceGetCurrentClocksEventReasons",
                              getattr(nv, "nvmlDeviceGetCurrentClocksThrottleReasons", None))
        while not self._stop.is_set():
            if self._in_window.wait(timeout=0.05):
                try:
                    self.samples.append((float(nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)),
                                         int(get_reasons(h)) if get_reasons else 0))
                except Exception:  # noqa: BLE001
                    pass
                time.sleep(self.period)

    def __enter__(self):
        try:
            self._open()
            self._thread = threading.Thread(target=self._poll, daemon=True)
            self._thread.start()
        except Exception:  # noqa: BLE001 - no NVML: the line says "unavailable"
            self._nvml = None
        return self

    def __exit__(self, *exc):
        self._stop.set()
        self._in_window.set()
        if self._thread is not None:
            self._thread.join(timeout=2)

    class _Window:
        def __init__(self, ev):
            self.ev = ev

        def __enter__(self):
            self.ev.set()

        def __exit__(self, *exc):
            self.ev.clear()

    def window(self):
        """Context manager marking a timed region (enter before the first
        launch, exit after the closing synchronize)."""
        return self._Window(self._in_window)

    def summary(self) -> dict:
        if self._nvml is None or not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["unavailable"], "samples": 0}
        sm = [c for c, _ in self.samples]
        reasons = sorted({name for _, bits in self.samples for name, bit in self.REASONS if bits & bit})
        return {"sm_mhz": float(np.median(sm)), "sm_min_mhz": min(sm), "sm_max_mhz": self.max_mhz,
                "reasons": reasons, "samples": len(sm), "source": "NVML, 2 ms, timed regions only"}


# ---------------------------------------------------------------------------
# distributed plumbing
# ---------------------------------------------------------------------------
def _dist_init(gpus: int):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch
        import torch.distributed as dist

        # TACO_BENCH_SMOKE=1: every rank on cuda:0 over gloo (host-side
        # collectives, no kernel waits on another rank's): a functional check
        # of the N > 1 path on a one-GPU box, not a measurement
        if os.environ.get("TACO_BENCH_SMOKE") == "1":
            local = 0
            torch.cuda.set_device(0)
            dist.init_process_group("gloo")
        else:
            torch.cuda.set_device(local)
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    return rank, world, local


def _max_over_ranks(x: float, world: int) -> float:
    if world == 1:
        return x
    import torch
    import torch.distributed as dist

    t = torch.tensor([x], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def _barrier(world: int) -> None:
    if world > 1:
        import torch.distributed as dist

        dist.barrier()


# ---------------------------------------------------------------------------
# our arm
# ---------------------------------------------------------------------------
def run_ours(args) -> dict | None:
    import torch

    rank, world, local = _dist_init(args.gpus)
    import paper_2404_04895_b200 as taco
    from paper_2404_04895_b200 import _device, _lib

    n, m, selection = CONFIGS[args.config]
    if args.weak:  # population scaling: the colony grows with the GPUs (m per GPU fixed)
        m *= int(os.environ.get("WORLD_SIZE", "1"))
    if args.construct == "auto":  # the Solver's own choice (full-row kernel for tiny rows)
        args.construct = "dense" if n < taco.Solver.DENSE_MAX_N else "sorted"
    k = max(1, m // 10)
    period = args.warmup + args.steps
    # NVML clock sampler (rank 0): samples only inside the timed regions
    sampler = ClockSampler(local) if rank == 0 else None
    if sampler:
        sampler.__enter__()
    coords = np.random.default_rng(0).uniform(0.0, 2000.0, (n, 2))
    inst = taco.euclidean_instance(coords)
    params = taco.AcoParams(m=m, k=k, selection=selection, seed=0,
                            gamma_schedule=taco.GammaSchedule(1.5, 1.0, period))
    dev = _device.device()

    # ---- e2e: solve from host buffers through the public API ---------------
    # headline e2e: host coordinates (pinned) -> device_euclidean_instance
    # (16n B H2D, dist/eta built on the device) -> Solver -> K iterations of
    # Solver.iterate(), each iteration's status + best length + best tour read
    # back in one D2H copy (pipelined: the next iteration is queued first).
    # e2e_host_instance: the same from a host TspInstance (dist + eta H2D);
    # e2e_step: the device instance with K blocking step() calls instead.
    coords_pinned = torch.from_numpy(coords).pin_memory()

    def e2e_run(make_instance, steps, blocking=False):
        solver_ = taco.Solver(make_instance(), params, construct=args.construct)
        out = None
        if blocking:
            for _ in range(steps):
                out = solver_.step()
        else:
            for _it, tour_, len_ in solver_.iterate(steps):
                out = (tour_, len_)
        return out

    def dev_inst():
        return taco.device_euclidean_instance(coords_pinned.numpy())

    e2e_run(dev_inst, args.warmup)
    e2e_run(lambda: inst, args.warmup)
    _device._INSTANCES.clear()
    torch.cuda.synchronize()
    # each e2e figure is the median of three complete runs (instance, Solver,
    # K steps): millisecond-scale host timings pick up scheduler / GC noise
    e2e_times = {"device_instance": [], "host_instance": [], "step": []}
    for _rep in range(3):
        for name, make, blocking in (("device_instance", dev_inst, False), ("host_instance", lambda: inst, False),
                                     ("step", dev_inst, True)):
            gc.collect()
            _barrier(world)
            with sampler.window() if sampler else _null():
                t0 = time.perf_counter()
                best_tour, best_len = e2e_run(make, args.steps, blocking)
                torch.cuda.synchronize()
                e2e_times[name].append(_max_over_ranks(time.perf_counter() - t0, world))
            _device._INSTANCES.clear()
    e2e_times = {k: float(np.median(v)) for k, v in e2e_times.items()}

    # ---- device-timed value ------------------------------------------------
    # steady state of a long run: graph replays (where the Solver uses them)
    # from the first timed iteration on
    solver = taco.Solver(inst, params, construct=args.construct, graph_warmup=0)
    for _ in range(args.warmup):
        solver.step_async()
    solver.check()
    torch.cuda.synchronize()
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    _barrier(world)
    torch.cuda.synchronize()
    # timed: K iterations through the Solver's own path (one CUDA-graph replay
    # per iteration on a single GPU; eager launches when sharded)
    with sampler.window() if sampler else _null():
        start.record()
        for _ in range(args.steps):
            solver.step_async()
        end.record()
        torch.cuda.synchronize()
    if sampler:
        sampler.__exit__()
    solver.check()
    _barrier(world)
    elapsed_ms = _max_over_ranks(start.elapsed_time(end), world)
    ms_per_step = elapsed_ms / args.steps

    # ---- per-kernel breakdown: eager iterations with events around the
    # construction and the row update, plus the sorted kernel's window probe
    timers = {"construct": [], "update": []}
    scan = torch.zeros(1, dtype=torch.int64, device=dev)
    bd_steps = min(args.steps, 10)
    for _ in range(bd_steps):
        solver.step_async(timers=timers, scan_count=scan if args.construct == "sorted" else None)
    torch.cuda.synchronize()
    solver.check()
    t_construct = float(np.mean([a.elapsed_time(b) for a, b in timers["construct"]]))
    t_update = float(np.mean([a.elapsed_time(b) for a, b in timers["update"]]))
    windows = int(scan.item()) / bd_steps

    # ---- L2-flushed variant: 256 MB scrub before every iteration ----------
    scrub = torch.empty(256 * 2**20, dtype=torch.uint8, device=dev)
    flushed = []
    for _ in range(min(args.steps, 10)):
        scrub.fill_(1)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        solver.step_async()
        b.record()
        torch.cuda.synchronize()
        flushed.append(a.elapsed_time(b))
    flushed_ms = _max_over_ranks(float(np.mean(flushed)), world)

    # ---- the north-star full-row streaming kernel on the same state -------
    dense_ms = None
    rw = selection == "rw"
    if args.construct == "sorted" and n <= 20480 and not rw:
        pmat = torch.from_numpy(solver.probability().p).to(dev)
        dt = _device.SelectionTables(n, dev, dense=True, sorted_=False)
        g = taco.colony.construction_gamma(params, solver.iteration)
        _device.selection_table_from_p(pmat, 1.0 / g, dt)
        tours = torch.zeros((solver.shard.count, n), dtype=torch.int32, device=dev)
        st = _device.new_status(dev)
        reps = []
        for r in range(3):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            _device.construct(n, solver.shard.count, solver.shard.offset, _lib.CONSTRUCT_DENSE, dt, 0,
                              solver.iteration, tours, st)
            b.record()
            torch.cuda.synchronize()
            reps.append(a.elapsed_time(b))
        dense_ms = float(np.median(reps))
        del dt, tours

    if rank != 0:
        return None

    it_per_s = 1000.0 / ms_per_step
    peak, peak_kind = _peaks()
    sharded = solver.shard.world > 1
    launches_per_iter = 5 + (0 if rw else 1) + (1 if solver.graph else 0) + (1 if sharded else 0)
    sms_ = torch.cuda.get_device_properties(dev).multi_processor_count
    # > 32 ants per SM on the warp kernel (MODE 2): + the k_rebuild_stalled follow-up
    mode2 = (not rw and args.construct == "sorted" and 32 * sms_ < solver.shard.count <= 64 * sms_)
    launches_per_iter += 1 if mode2 else 0
    launches_per_iter += 2 if solver._split_update else 0  # deposit + evaporation + normalization
    m_local = solver.shard.count
    # roofline.achieved = ALGORITHMIC bytes per launch / launch time, with the
    # per-unit figure of SURVEY §8(d): each ant streams its current row of the
    # selection table every step, m (n-1) n x 4 B (fp32 W) for IR / AdaIR, and
    # m (n-1) (8n + 2048) B for RW (f64 P row + the crossing tile).  The sorted
    # kernel moves far fewer bytes than that (pruned scan: table_bytes_read);
    # `traffic` is ncu's measured DRAM bytes per launch of the same kernel.
    alg_full = m_local * (n - 1) * n * 4
    alg_sorted = windows * 32 * 6 + m_local * n * 4  # sorted-table windows read + tours written
    dom_ms = t_construct
    kernel = "k_construct_rw" if rw else f"k_construct_{args.construct}"
    alg = m_local * (n - 1) * (n * 8 + 2048) if rw else alg_full
    cap = _capture(kernel, args.config)
    traffic = cap["dram_bytes_per_launch"] if cap else None
    clocks = sampler.summary() if sampler else {}
    sm_mhz = clocks.get("sm_mhz") or clocks.get("sm_max_mhz") or 1965.0
    sms = torch.cuda.get_device_properties(dev).multi_processor_count
    inst = cap.get("warp_instructions_per_launch") if cap else None
    if rw or args.construct == "sorted":
        # The pruned scan reads ~2% of the full-row bytes (table_bytes_read,
        # counted live) and the roulette kernel's f64 rows are L2-resident, so
        # HBM does not bound either: instruction issue and the n-1 dependent
        # steps do.  roofline = issue: ncu's warp instructions per launch (the
        # committed capture of this config) / the event-timed launch, against
        # 4 issue slots per SM per cycle at the sampled clock.
        if rw:
            hbm_side = {"alg_bytes_per_launch": alg, "dram_bytes_per_launch_ncu": traffic,
                        "l2_hit_rate_ncu": cap.get("l2_hit_rate") if cap else None,
                        "alg_bytes_def": "SURVEY 8(d): f64 P row per ant-step, m*(n-1)*(8n+2048) B"}
            bytes_live = traffic / (dom_ms * 1e-3) / 1e9 if traffic else None
        else:
            hbm_side = {"table_bytes_read_per_launch": alg_sorted, "GBps": alg_sorted / (dom_ms * 1e-3) / 1e9,
                        "frac_of_hbm_peak": alg_sorted / (dom_ms * 1e-3) / 1e9 / peak,
                        "dram_bytes_per_launch_ncu": traffic,
                        "l2_hit_rate_ncu": cap.get("l2_hit_rate") if cap else None,
                        "alg_bytes_full_row": alg_full,
                        "alg_bytes_def": "SURVEY 8(d) full-row figure m*(n-1)*n*4 B is reported under "
                                         "roofline_dense, the kernel that streams it"}
            bytes_live = hbm_side["GBps"]
        if inst:
            issue_peak = sms * 4 * sm_mhz * 1e6
            roof = {"kernel": kernel, "bound": "issue", "achieved": inst / (dom_ms * 1e-3), "peak": issue_peak,
                    "unit": "warp-instructions/s", "frac": inst / (dom_ms * 1e-3) / issue_peak,
                    "warp_instructions_per_launch": inst,
                    "peak_def": f"{sms} SMs x 4 issue slots x {sm_mhz:.0f} MHz (sampled SM clock)",
                    "traffic": traffic, "traffic_source": cap["capture"], "hbm": hbm_side}
        else:  # no capture of this config: the bytes it really moves, against HBM
            roof = {"kernel": kernel, "bound": "hbm", "achieved": bytes_live, "peak": peak, "unit": "GB/s",
                    "frac": bytes_live / peak if bytes_live else None, "traffic": traffic, "hbm": hbm_side,
                    "note": "no ncu capture of this config: the bytes it reads (live probe) against HBM"}
        roof.update({"ms_per_launch": dom_ms, "share_of_step": dom_ms / ms_per_step, "peak_kind": peak_kind})
    else:
        roof = {"kernel": kernel, "bound": "hbm", "achieved": alg / (dom_ms * 1e-3) / 1e9, "peak": peak,
                "unit": "GB/s", "peak_kind": peak_kind, "traffic": traffic,
                "traffic_source": cap["capture"] if cap else None,
                "ms_per_launch": dom_ms, "share_of_step": dom_ms / ms_per_step, "alg_bytes_per_launch": alg,
                "alg_bytes_def": "SURVEY 8(d): full-row stream of the fp32 table, m*(n-1)*n*4 B"}
        roof["frac"] = roof["achieved"] / peak
    line = {
        "metric": _metric(n, m), "value": it_per_s, "unit": "iterations/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step,
        "higher_is_better": True, "scaling": "weak" if args.weak else "strong", "vs_baseline": None, "dtype": "f64+f32",
        "data": "synthetic: U(0,2000)^2 Euclidean cities (seed 0), unrounded distances",
        "config": _config_dict(args.config, n, m, k, selection, period, world),
        "construct": "rw" if rw else args.construct,
        "l2": ("back-to-back iterations; per-iteration state (tau, eta^b, dist, tables, tours) > 126 MB L2; "
               "value_l2_flushed scrubs 256 MB before each iteration"),
        "selections_per_s": m * (n - 1) * it_per_s,
        "value_l2_flushed": 1000.0 / flushed_ms,
        "kernel_ms": {"construct": t_construct, "update_p": t_update,
                      "construct_dense_full_row": dense_ms},
        "roofline": roof,
        "e2e": {"value": args.steps / e2e_times["device_instance"], "unit": "iterations/s",
                "h2d_bytes_per_step": (n * 2 * 8) / args.steps,
                "d2h_bytes_per_step": 32 + n * 4,
                "what": ("pinned host coords -> device_euclidean_instance -> Solver -> K iterations of "
                         "Solver.iterate(), each iteration's status + best length + best tour read back in one "
                         "D2H copy (the next iteration queued before the read); median of 3 complete runs")},
        "e2e_host_instance": {"value": args.steps / e2e_times["host_instance"], "unit": "iterations/s",
                              "h2d_bytes_per_step": (2 * n * n * 8) / args.steps,
                              "d2h_bytes_per_step": 32 + n * 4,
                              "what": "host TspInstance (dist + eta H2D) -> Solver -> Solver.iterate(K)"},
        "e2e_step": {"value": args.steps / e2e_times["step"], "unit": "iterations/s",
                     "h2d_bytes_per_step": (n * 2 * 8) / args.steps, "d2h_bytes_per_step": 32 + n * 4,
                     "what": "as e2e, with K blocking Solver.step() calls (host waits for every iteration)"},
        "gpu_launches": args.steps * launches_per_iter,
        "gpu_launches_note": (f"{launches_per_iter} libtaco kernels per iteration: k_construct_"
                              f"{'rw' if rw else args.construct} (or the lane-group variant)"
                              f"{' + k_rebuild_stalled' if mode2 else ''}, k_elite_rank, "
                              "k_track_best, k_elite_neighbors, "
                              f"{'k_deposit_rows, k_evap_unnorm, k_row_normalize' if solver._split_update else 'k_row_update'}"
                              f"{'' if rw else ', k_row_sort'}{', k_iter_advance' if solver.graph else ''}"
                              f"{', k_shard_elites (+ NCCL collectives)' if sharded else ''}"
                              f"{' (+ CUB radix-sort kernels: m > 16384)' if m > 16384 else ''}; "
                              f"{'replayed as one CUDA graph per iteration' if solver.graph else 'eager launches'}"),
        "best_length": best_len,
    }
    if dense_ms is not None:
        line["roofline_dense"] = {"kernel": "k_construct_dense", "bound": "hbm",
                                  "achieved": alg_full / (dense_ms * 1e-3) / 1e9, "peak": peak,
                                  "unit": "GB/s", "frac": alg_full / (dense_ms * 1e-3) / 1e9 / peak,
                                  "ms_per_launch": dense_ms, "traffic": _traffic("k_construct_dense", args.config)[0],
                                  "alg_bytes_def": "full-row stream m*(n-1)*n*4 B (SURVEY 8d)"}
    if sampler:
        line["clocks"] = clocks
    if world == 1 and not args.no_cpu_baseline:
        from oracle import cpu_baseline

        ref_ok = cpu_baseline.reference_available()
        sampler_fn = cpu_baseline.sample_iteration_reference if ref_ok else cpu_baseline.sample_iteration
        s = sampler_fn(n, m, k, selection, seed=0, steps=args.cpu_steps, period=period)
        line["cpu_baseline"] = {
            "value": 1.0 / s["t_iter"], "unit": "iterations/s", "cores": 1,
            "kind": "reference" if ref_ok else "port",
            "sample": (f"{'antbatch (unmodified, baseline/_ref)' if ref_ok else 'oracle/reference_port'}, 1 thread: "
                       f"{s['steps_sampled']} construction steps "
                       f"(mean {s['t_step'] * 1e3:.1f} ms) x (n-1) + P {s['t_p'] * 1e3:.0f} ms + logw "
                       f"{s['t_logw'] * 1e3:.0f} ms + lengths {s['t_costs'] * 1e3:.0f} ms + update "
                       f"{s['t_update'] * 1e3:.0f} ms; extrapolated"),
            "t_iter_s": s["t_iter"]}
    return line


# ---------------------------------------------------------------------------
# reference arm
# ---------------------------------------------------------------------------
def run_reference(args) -> dict | None:
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if rank != 0:
        return None
    from oracle import cpu_baseline

    n, m, selection = CONFIGS[args.config]
    if args.weak:
        m *= world
    k = max(1, m // 10)
    period = args.warmup + args.steps  # the same gamma schedule as our arm
    host = len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else (os.cpu_count() or 1)
    cores = max(1, min(host, args.ref_procs) if args.ref_procs > 0 else host)
    ref_ok = cpu_baseline.reference_available()
    # C1 is small enough for the reference's own run_experiment, whole; the
    # larger configs take hours per iteration on one core: sampled + extrapolated
    as_is = ref_ok and n * m <= 51 * 64
    kind = "as-is" if as_is else ("reference" if ref_ok else "port")
    per_job = args.steps + 1 if as_is else args.cpu_steps  # iterations (as-is) or sampled rounds
    # warm-up round (untimed), then K rounds; a round = one iteration on each
    # of `cores` independent single-threaded colonies at once
    if args.warmup:
        cpu_baseline.parallel_samples(n, m, k, selection, cores, cores, steps=2, period=period, kind=kind)
    t0 = time.perf_counter()
    rounds = 1 if as_is else args.steps
    times = cpu_baseline.parallel_samples(n, m, k, selection, rounds * cores, cores, steps=per_job, period=period,
                                          kind=kind)
    wall = time.perf_counter() - t0
    per_colony = 1.0 / float(np.mean(times))
    value = per_colony * cores
    what = ("antbatch (the unmodified reference, baseline/_ref)" if ref_ok else
            "oracle/reference_port (numpy restatement of antbatch, pinned to its golden vectors)")
    how = (f"run_experiment as-is, {per_job} iterations per colony (its own clock; the warm-up iteration "
           f"excluded, bench.py:228)" if as_is else
           f"each step = one iteration extrapolated from {args.cpu_steps} sampled lockstep rounds "
           f"(SURVEY 8(d))")
    return {
        "metric": _metric(n, m), "value": value, "unit": "iterations/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": 1000.0 / value, "higher_is_better": True, "scaling": "weak" if args.weak else "strong",
        "vs_baseline": None, "dtype": "f64", "impl": "reference",
        "timing": "measured" if as_is else "extrapolated",
        "data": "synthetic: U(0,2000)^2 Euclidean cities (seed 0), unrounded distances",
        "config": _config_dict(args.config, n, m, k, selection, period, world),
        "cpu_baseline": {"value": value, "unit": "iterations/s", "cores": cores,
                         "kind": "reference" if ref_ok else "port",
                         "sample": (f"{what}: {how}; {cores} independent single-threaded colonies in parallel; "
                                    f"per-colony {per_colony:.3g} it/s"),
                         "wall_s": wall},
        "e2e": {"value": value, "unit": "iterations/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }


def main() -> None:
    ap = argparse.ArgumentParser(description=__doc__, formatter_class=argparse.RawDescriptionHelpFormatter)
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=("ours", "reference"), default="ours")
    ap.add_argument("--config", choices=sorted(CONFIGS), default="c3")
    ap.add_argument("--construct", choices=("auto", "sorted", "dense"), default="auto")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-steps", type=int, default=6)
    ap.add_argument("--ref-procs", type=int, default=0, help="reference arm processes (0: all host cores)")
    ap.add_argument("--weak", action="store_true",
                    help="weak (population) scaling: the config's m ants per GPU, m x N in total; default strong "
                         "(the config's colony split over the GPUs)")
    args = ap.parse_args()
    if args.warmup < 0 or args.steps < 1:
        ap.error("need --steps >= 1 and --warmup >= 0")
    line = run_reference(args) if args.impl == "reference" else run_ours(args)
    if line is not None:
        print(json.dumps(line), flush=True)
    if int(os.environ.get("WORLD_SIZE", "1")) > 1 and args.impl == "ours":
        import torch.distributed as dist

        dist.destroy_process_group()


if __name__ == "__main__":
    main()
