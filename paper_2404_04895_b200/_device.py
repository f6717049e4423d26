"""Device-side plumbing: torch owns memory and streams, libtaco does the math.

Every helper here takes/returns CUDA torch tensors and launches on torch's
current stream.  There is deliberately no CPU path: without a CUDA device or
without libtaco.so the calls raise.
"""

from __future__ import annotations

import threading
import warnings
import weakref

import numpy as np
import torch

from . import _lib
from ._lib import check, ptr

INT32_MAX = 2**31 - 1


class NoCudaDevice(RuntimeError):
    """The engine needs an sm_100a CUDA device; there is no CPU fallback."""


def device() -> torch.device:
    if not torch.cuda.is_available():
        raise NoCudaDevice("TensorACO-B200 needs a CUDA (sm_100a) device; no CPU fallback exists")
    _lib.load()
    return torch.device("cuda", torch.cuda.current_device())


_PINNED_STREAM = threading.local()


def stream_handle() -> int:
    """The current CUDA stream as a raw handle (a Solver pins it for the
    launches of one iteration: torch's current_stream() lookup costs
    microseconds per call, several per iteration)."""
    h = getattr(_PINNED_STREAM, "handle", None)
    return h if h is not None else torch.cuda.current_stream().cuda_stream


class pinned_stream:
    """Context: stream_handle() returns the stream current at entry."""

    def __enter__(self):
        self._prev = getattr(_PINNED_STREAM, "handle", None)
        _PINNED_STREAM.handle = torch.cuda.current_stream().cuda_stream
        return self

    def __exit__(self, *exc):
        _PINNED_STREAM.handle = self._prev
        return False


def new_status(dev) -> torch.Tensor:
    return torch.tensor([0, INT32_MAX, 0, 0], dtype=torch.int32, device=dev)


def read_status(status: torch.Tensor) -> tuple[int, int]:
    code, idx, _, _ = (int(v) for v in status.cpu().tolist())
    return code, idx


def upload(a: np.ndarray, dev, dtype=None) -> torch.Tensor:
    """Host array -> new device tensor.  The reference's value objects are
    read-only numpy arrays; they are only read here (copied to the device), so
    torch's non-writable-array warning does not apply."""
    with warnings.catch_warnings():
        warnings.filterwarnings("ignore", message="The given NumPy array is not writable")
        t = torch.from_numpy(np.ascontiguousarray(a))
    if dtype is not None:
        t = t.to(dtype)
    return t.to(dev, non_blocking=False)


def download(t: torch.Tensor) -> np.ndarray:
    return t.detach().cpu().numpy()


def pad_ld(n: int) -> int:
    """Leading dimension of the dense fp32 table: rows start 128-byte aligned."""
    return (n + 31) // 32 * 32


# ---------------------------------------------------------------------------
# per-instance device cache (dist, eta, eta^beta), keyed by object identity
# ---------------------------------------------------------------------------
class UnsupportedEdgeWeightType(ValueError):
    """Edge-weight convention outside EXACT / EUC_2D / CEIL_2D / ATT
    (tsplib.py:45-46, raised by tsplib.distance tsplib.py:215)."""


class DeviceInstance:
    """dist / eta (and eta^beta per beta) resident on the device."""

    def __init__(self, inst, dev):
        self.n = int(inst.n)
        self.dev = dev
        self.best_known = getattr(inst, "best_known", None)
        self.name = getattr(inst, "name", "")
        self.dist = upload(np.asarray(inst.dist, dtype=np.float64), dev)
        self.eta = upload(np.asarray(inst.eta, dtype=np.float64), dev)
        self._eta_b: dict[float, torch.Tensor] = {}

    @classmethod
    def from_coords(cls, coords, edge_weight_type: str = "EXACT", lenient: bool = False,
                    best_known: float | None = None, name: str = "") -> "DeviceInstance":
        """Instance built on the device from (n, 2) coordinates, bit-exact with
        the host builders: ``"EXACT"`` = euclidean_instance (model.py:124-134),
        ``"EUC_2D"`` / ``"CEIL_2D"`` / ``"ATT"`` = build_instance's TSPLIB
        conventions (model.py:98-119, tsplib.py:198-215).  Only the 16n bytes of
        coordinates cross PCIe; the host never holds the n^2 matrices."""
        from .model import DegenerateInstance

        kind = _lib.EDGE_WEIGHT_TYPES.get(str(edge_weight_type))
        if kind is None:
            raise UnsupportedEdgeWeightType(f"edge weight type {edge_weight_type!r} not supported")
        xy = np.ascontiguousarray(np.asarray(coords, dtype=np.float64))
        if xy.ndim != 2 or xy.shape[1] != 2:
            raise ValueError(f"coords must have shape (n, 2), got {xy.shape}")
        n = xy.shape[0]
        if n < 3:
            raise DegenerateInstance(f"need at least 3 cities, got {n}")
        if n > 65535:
            raise ValueError(f"n = {n} exceeds the engine's 65535-city limit")
        dev = device()
        obj = cls.__new__(cls)
        obj.n, obj.dev, obj._eta_b = n, dev, {}
        obj.best_known, obj.name = best_known, name
        obj.dist = torch.empty((n, n), dtype=torch.float64, device=dev)
        obj.eta = torch.empty((n, n), dtype=torch.float64, device=dev)
        status = new_status(dev)
        check(_lib.load().taco_coord_instance(n, ptr(upload(xy, dev)), kind, ptr(obj.dist), ptr(obj.eta),
                                              int(bool(lenient)), ptr(status), stream_handle()),
              "taco_coord_instance")
        code, row = read_status(status)
        if code == _lib.TACO_DEGENERATE:
            # the first row-major zero off the diagonal lies in the smallest such row
            d = download(obj.dist[row])
            d[row] = 1.0
            col = int(np.flatnonzero(d == 0.0)[0])
            raise DegenerateInstance(f"cities {row} and {col} are at distance 0 (duplicate coordinates)")
        return obj

    def eta_beta(self, beta: float) -> torch.Tensor:
        beta = float(beta)
        t = self._eta_b.get(beta)
        if t is None:
            t = torch.empty_like(self.eta)
            check(_lib.load().taco_eta_power(t.numel(), ptr(self.eta), beta, ptr(t), stream_handle()),
                  "taco_eta_power")
            self._eta_b[beta] = t
        return t


def device_build_instance(raw, best_known: float | None = None, lenient: bool = False) -> DeviceInstance:
    """build_instance (model.py:98-119) on the device from a parsed TSPLIB file:
    any object with ``dimension``, ``node_coords`` ((id, x, y) triples),
    ``edge_weight_type`` and ``name`` (the reference's RawTspFile).  The
    reference's bundled best-known table is not consulted (TSPLIB data is out
    of scope): pass ``best_known``."""
    coords = np.array([(float(x), float(y)) for _, x, y in raw.node_coords], dtype=np.float64).reshape(-1, 2)
    if coords.shape[0] != int(raw.dimension):
        raise ValueError(f"DIMENSION {raw.dimension} but {coords.shape[0]} coordinates")
    return DeviceInstance.from_coords(coords, raw.edge_weight_type, lenient=lenient, best_known=best_known,
                                      name=getattr(raw, "name", ""))


_INSTANCES: "weakref.WeakKeyDictionary" = weakref.WeakKeyDictionary()


def device_instance(inst) -> DeviceInstance:
    dev = device()
    try:
        cached = _INSTANCES.get(inst)
    except TypeError:  # unhashable / not weak-referenceable: no caching
        return DeviceInstance(inst, dev)
    if cached is None or cached.dev != dev:
        cached = DeviceInstance(inst, dev)
        _INSTANCES[inst] = cached
    return cached


# ---------------------------------------------------------------------------
# thin typed wrappers over the C ABI
# ---------------------------------------------------------------------------
def row_update(n, *, tau_in=None, tau_out=None, eta_b=None, nbr=None, inc=None, k=0,
               delta_in=None, delta_out=None, do_evap=False, keep=1.0, want_p=False,
               alpha=1.0, inv_gamma=1.0, p_out=None, rowsum_out=None, w_out=None, ldw=0,
               sw_out=None, si_out=None, status=None, state=None) -> None:
    code = _lib.load().taco_row_update(
        n, ptr(tau_in), ptr(tau_out), ptr(eta_b), ptr(nbr), ptr(inc), int(k), ptr(delta_in),
        ptr(delta_out), int(bool(do_evap)), float(keep), int(bool(want_p)), float(alpha),
        float(inv_gamma), ptr(p_out), ptr(rowsum_out), ptr(w_out), int(ldw), ptr(sw_out),
        ptr(si_out), ptr(status), ptr(state), stream_handle())
    check(code, "taco_row_update")


def row_update_rows(row_begin, row_end, n, *, tau_in=None, tau_out=None, eta_b=None, nbr=None, inc=None, k=0,
                    delta_in=None, delta_out=None, do_evap=False, keep=1.0, want_p=False, alpha=1.0,
                    inv_gamma=1.0, p_out=None, rowsum_out=None, w_out=None, ldw=0, sw_out=None, si_out=None,
                    status=None, state=None) -> None:
    """row_update on rows [row_begin, row_end) only (taco_row_update_rows)."""
    code = _lib.load().taco_row_update_rows(
        int(row_begin), int(row_end), n, ptr(tau_in), ptr(tau_out), ptr(eta_b), ptr(nbr), ptr(inc), int(k),
        ptr(delta_in), ptr(delta_out), int(bool(do_evap)), float(keep), int(bool(want_p)), float(alpha),
        float(inv_gamma), ptr(p_out), ptr(rowsum_out), ptr(w_out), int(ldw), ptr(sw_out), ptr(si_out), ptr(status),
        ptr(state), stream_handle())
    check(code, "taco_row_update_rows")


def update_split(n, *, tau_in, tau_out, eta_b, nbr, inc, k, do_evap, keep, alpha, inv_gamma, delta_ws,
                 unnorm_ws, p_out=None, rowsum_out=None, w_out=None, ldw=0, sw_out=None, si_out=None,
                 status=None, state=None) -> None:
    """Solver-mode update as three streaming kernels (taco_update_split)."""
    code = _lib.load().taco_update_split(
        n, ptr(tau_in), ptr(tau_out), ptr(eta_b), ptr(nbr), ptr(inc), int(k), int(bool(do_evap)), float(keep),
        float(alpha), float(inv_gamma), ptr(delta_ws), ptr(unnorm_ws), ptr(p_out), ptr(rowsum_out), ptr(w_out),
        int(ldw), ptr(sw_out), ptr(si_out), ptr(status), ptr(state), stream_handle())
    check(code, "taco_update_split")


class SelectionTables:
    """fp32 selection table W = P^(1/gamma): dense and/or row-sorted (values
    sw + column indices si), all with row pitch ldw (multiple of 32).  The
    sorted rows' pad columns stay W = 0 (zero-initialized, never selectable)."""

    def __init__(self, n: int, dev, dense: bool, sorted_: bool, rows: int | None = None):
        self.n = n
        self.ldw = pad_ld(n)
        rows = n if rows is None else rows  # > n: padding rows for equal all-gather chunks
        # the sorted table is built from the dense one, so sorted implies dense
        self.w = torch.empty((rows, self.ldw), dtype=torch.float32, device=dev) if dense or sorted_ else None
        self.sw = torch.zeros((rows, self.ldw), dtype=torch.float32, device=dev) if sorted_ else None
        self.si = torch.zeros((rows, self.ldw), dtype=torch.uint16, device=dev) if sorted_ else None


def selection_table_from_p(p: torch.Tensor, inv_gamma: float, tables: SelectionTables) -> None:
    code = _lib.load().taco_selection_table(
        tables.n, ptr(p), float(inv_gamma), ptr(tables.w), tables.ldw, ptr(tables.sw), ptr(tables.si),
        stream_handle())
    check(code, "taco_selection_table")


def construct(n: int, m_local: int, ant_offset: int, variant: int, tables: SelectionTables,
              seed: int, iteration: int, tours_out: torch.Tensor, status: torch.Tensor,
              scan_count: torch.Tensor | None = None, dist: torch.Tensor | None = None,
              costs_out: torch.Tensor | None = None, state: torch.Tensor | None = None,
              fallback: tuple | None = None, inv_gamma: float = 1.0) -> None:
    """Build tours (and, with dist + costs_out, their lengths) on the device.

    fallback: (A, alpha, B or None) device f64 (n, n) tensors, the source of
    the f64 decision when no W > 0 candidate is left (include/taco.h); None:
    only the all -inf rule (city 0 when unvisited)."""
    fb_a, fb_alpha, fb_b = fallback if fallback is not None else (None, 1.0, None)
    code = _lib.load().taco_construct(
        n, m_local, ant_offset, variant, ptr(tables.w), tables.ldw, ptr(tables.sw), ptr(tables.si),
        int(seed), int(iteration) & 0xFFFFFFFF, ptr(dist), ptr(tours_out), ptr(costs_out), ptr(status),
        ptr(scan_count), ptr(fb_a), float(fb_alpha), ptr(fb_b), float(inv_gamma), ptr(state), stream_handle())
    check(code, "taco_construct")


def construct_rw(n: int, m_local: int, ant_offset: int, p: torch.Tensor, seed: int, iteration: int,
                 tours_out: torch.Tensor, status: torch.Tensor, dist: torch.Tensor | None = None,
                 costs_out: torch.Tensor | None = None, exact_count: torch.Tensor | None = None,
                 force_exact: bool = False, state: torch.Tensor | None = None) -> None:
    """Roulette-wheel tours from the f64 probability matrix (device stream)."""
    code = _lib.load().taco_construct_rw(
        n, m_local, ant_offset, ptr(p), int(seed), int(iteration) & 0xFFFFFFFF, ptr(dist), ptr(tours_out),
        ptr(costs_out), ptr(status), ptr(exact_count), int(bool(force_exact)), ptr(state), stream_handle())
    check(code, "taco_construct_rw")


def tour_cost(tours: torch.Tensor, dist: torch.Tensor, out: torch.Tensor | None = None) -> torch.Tensor:
    m, n = tours.shape
    if out is None:
        out = torch.empty(m, dtype=torch.float64, device=tours.device)
    is64 = 1 if tours.dtype == torch.int64 else 0
    if not is64 and tours.dtype != torch.int32:
        raise TypeError(f"tours must be int32 or int64, got {tours.dtype}")
    check(_lib.load().taco_tour_cost(n, m, ptr(tours), is64, ptr(dist), ptr(out), stream_handle()),
          "taco_tour_cost")
    return out


class EliteWorkspace:
    def __init__(self, m: int, dev):
        self.m = m
        self.nbytes = int(_lib.load().taco_elite_workspace_bytes(m))
        self.buf = torch.empty(max(self.nbytes, 1), dtype=torch.uint8, device=dev)


def elite_order(costs: torch.Tensor, ws: EliteWorkspace, out: torch.Tensor | None = None) -> torch.Tensor:
    m = costs.numel()
    if out is None:
        out = torch.empty(m, dtype=torch.int32, device=costs.device)
    check(_lib.load().taco_elite_order(m, ptr(costs), ptr(out), ptr(ws.buf), ws.nbytes, stream_handle()),
          "taco_elite_order")
    return out


def elite_neighbors(tours: torch.Tensor, order: torch.Tensor, costs: torch.Tensor, k: int,
                    nbr: torch.Tensor, inc: torch.Tensor) -> None:
    n = tours.shape[1]
    is64 = 1 if tours.dtype == torch.int64 else 0
    check(_lib.load().taco_elite_neighbors(n, k, ptr(tours), is64, ptr(order), ptr(costs), ptr(nbr),
                                           ptr(inc), stream_handle()), "taco_elite_neighbors")
