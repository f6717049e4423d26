"""ctypes binding of libtaco.so (the C ABI declared in include/taco.h).

The library is built in-tree by ``python -m paper_2404_04895_b200.build`` (or
``__graft_entry__.build()``) into ``paper_2404_04895_b200/lib/libtaco.so``.
There is no CPU fallback: if the library is missing every device entry point
raises ``TacoLibraryMissing``.
"""

from __future__ import annotations

import ctypes
import os

LIB_PATH = os.environ.get("TACO_LIB_PATH") or os.path.join(os.path.dirname(os.path.abspath(__file__)), "lib",
                                                           "libtaco.so")

TACO_OK = 0
TACO_UNDERFLOW = 1
TACO_NO_CANDIDATE = 2
TACO_DEGENERATE = 3
EDGE_WEIGHT_TYPES = {"EXACT": 0, "EUC_2D": 1, "CEIL_2D": 2, "ATT": 3}
TACO_ERR_ARG = -1
TACO_ERR_CUDA = -2
TACO_ERR_UNSUPPORTED = -3

CONSTRUCT_SORTED = 0
CONSTRUCT_DENSE = 1

_c_int = ctypes.c_int
_c_i64 = ctypes.c_int64
_c_u32 = ctypes.c_uint32
_c_u64 = ctypes.c_uint64
_c_f64 = ctypes.c_double
_c_size = ctypes.c_size_t
_p = ctypes.c_void_p

# name -> (restype, argtypes); mirrors include/taco.h one for one
SIGNATURES = {
    "taco_abi_version": (_c_int, []),
    "taco_status_string": (ctypes.c_char_p, [_c_int]),
    "taco_last_cuda_error": (ctypes.c_char_p, []),
    "taco_max_sorted_n": (_c_int, []),
    "taco_row_update": (_c_int, [
        _c_int, _p, _p, _p, _p, _p, _c_int, _p, _p, _c_int, _c_f64, _c_int, _c_f64, _c_f64,
        _p, _p, _p, _c_int, _p, _p, _p, _p, _p]),
    "taco_row_update_rows": (_c_int, [
        _c_int, _c_int, _c_int, _p, _p, _p, _p, _p, _c_int, _p, _p, _c_int, _c_f64, _c_int, _c_f64, _c_f64,
        _p, _p, _p, _c_int, _p, _p, _p, _p, _p]),
    "taco_update_split": (_c_int, [_c_int, _p, _p, _p, _p, _p, _c_int, _c_int, _c_f64, _c_f64, _c_f64, _p, _p,
                                   _p, _p, _p, _c_int, _p, _p, _p, _p, _p]),
    "taco_selection_table": (_c_int, [_c_int, _p, _c_f64, _p, _c_int, _p, _p, _p]),
    "taco_eta_power": (_c_int, [_c_i64, _p, _c_f64, _p, _p]),
    "taco_construct": (_c_int, [
        _c_int, _c_int, _c_int, _c_int, _p, _c_int, _p, _p, _c_u64, _c_u32, _p, _p, _p, _p, _p,
        _p, _c_f64, _p, _c_f64, _p, _p]),
    "taco_starts": (_c_int, [_c_int, _c_int, _c_int, _c_u64, _c_u32, _p, _p]),
    "taco_uniforms": (_c_int, [_c_int, _p, _p, _p, _c_u64, _c_u32, _p, _p]),
    "taco_philox2x32_10": (_c_int, [_c_int, _p, _p, _p, _p]),
    "taco_select_parity": (_c_int, [_c_int, _c_int, _c_int, _p, _p, _p, _p, _p, _p, _p]),
    "taco_argmax_select_block": (_c_int, [_c_int, _c_int, _p, _p, _p, _p, _p, _p, _p]),
    "taco_replay_workspace_bytes": (_c_size, [_c_int, _c_int]),
    "taco_select_replay": (_c_int, [_c_int, _c_int, _c_int, _c_u64, _c_u64, _p, _p, _p, _p, _p, _c_size, _p, _p,
                                    _p]),
    "taco_replay_first_column": (_c_int, [_c_int, _c_int, _c_u64, _c_u64, _p, _c_size, _p, _p, _p]),
    "taco_construct_rw": (_c_int, [_c_int, _c_int, _c_int, _p, _c_u64, _c_u32, _p, _p, _p, _p, _p, _c_int, _p,
                                   _p]),
    "taco_rw_parity": (_c_int, [_c_int, _c_int, _c_int, _p, _p, _p, _p, _p, _p, _p, _c_int, _p]),
    "taco_rw_uniforms": (_c_int, [_c_int, _p, _p, _c_u64, _c_u32, _p, _p]),
    "taco_coord_instance": (_c_int, [_c_int, _p, _c_int, _p, _p, _c_int, _p, _p]),
    "taco_log_weights": (_c_int, [_c_i64, _p, _c_f64, _p, _p]),
    "taco_tour_cost": (_c_int, [_c_int, _c_int, _p, _c_int, _p, _p, _p]),
    "taco_elite_workspace_bytes": (_c_size, [_c_int]),
    "taco_elite_order": (_c_int, [_c_int, _p, _p, _p, _c_size, _p]),
    "taco_elite_neighbors": (_c_int, [_c_int, _c_int, _p, _c_int, _p, _p, _p, _p, _p]),
    "taco_track_best": (_c_int, [_c_int, _p, _p, _p, _p, _p, _p, _c_u32, _p, _p, _p]),
    "taco_iter_advance": (_c_int, [_p, _p, _c_int, _p]),
    "taco_shard_elites": (_c_int, [_c_int, _c_int, _p, _c_int, _c_int, _p, _p, _p, _p, _p]),
}

ABI_VERSION = 4


class TacoLibraryMissing(ImportError):
    """libtaco.so is not built (run __graft_entry__.build())."""


class TacoError(RuntimeError):
    """A libtaco call returned an argument, CUDA or size error."""


_LIB = None


def load(path: str = LIB_PATH) -> ctypes.CDLL:
    """Load (once) and type the library; raises TacoLibraryMissing if absent."""
    global _LIB
    if _LIB is not None:
        return _LIB
    if not os.path.exists(path):
        raise TacoLibraryMissing(
            f"{path} not found: build it with `python -c 'import __graft_entry__ as g; g.build()'`")
    lib = ctypes.CDLL(path)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    if lib.taco_abi_version() != ABI_VERSION:
        raise TacoLibraryMissing(f"libtaco ABI {lib.taco_abi_version()} != {ABI_VERSION}; rebuild")
    _LIB = lib
    return lib


def check(code: int, what: str) -> None:
    """Raise on a synchronous (launch-time) error code."""
    if code == TACO_OK:
        return
    msg = load().taco_status_string(code).decode()
    if code == TACO_ERR_ARG:
        raise ValueError(f"{what}: {msg}")
    if code == TACO_ERR_CUDA:
        msg += f" ({load().taco_last_cuda_error().decode()})"
    raise TacoError(f"{what}: {msg} (code {code})")


def ptr(t) -> int | None:
    """Device pointer of a torch tensor (None passes NULL)."""
    return None if t is None else t.data_ptr()
