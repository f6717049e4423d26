"""ORACLE (test infrastructure only): ctypes front end of oracle/c/fastpath.c,
the C restatement of the engine's device stream and product-form selection
rule used for parity at the BASELINE sizes (n up to 10000),
where the numpy restatement (oracle/fastpath.py) would take hours.

The library is compiled by ``build()`` (gcc, -O2 -fopenmp -ffp-contract=off,
no fast-math: every float operation is one IEEE round-to-nearest, as on the
device) into oracle/lib/ and is pinned against oracle/fastpath.py in
tests/test_oracle_golden.py.  Only tests/, __graft_entry__.smoke() and bench.py
load it; the product never does.
"""

from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(HERE, "c", "fastpath.c")
LIB = os.path.join(HERE, "lib", "libfastpath_oracle.so")
CFLAGS = ["-O2", "-fopenmp", "-ffp-contract=off", "-fno-fast-math", "-fPIC", "-shared", "-std=c11"]

_lib = None
_logu = None


def build(force: bool = False) -> str:
    """Compile oracle/c/fastpath.c (skipped when up to date)."""
    if not force and os.path.exists(LIB) and os.path.getmtime(LIB) >= os.path.getmtime(SRC):
        return LIB
    os.makedirs(os.path.dirname(LIB), exist_ok=True)
    tmp = LIB + ".tmp"
    subprocess.run(["gcc", *CFLAGS, "-o", tmp, SRC, "-lm"], check=True)
    os.replace(tmp, LIB)
    return LIB


def _load():
    global _lib
    if _lib is None:
        lib = ctypes.CDLL(build())
        P = ctypes.c_void_p
        lib.fpo_build_tours.argtypes = [P, ctypes.c_int, ctypes.c_int, ctypes.c_uint64, ctypes.c_uint32, P,
                                        ctypes.c_int, P, ctypes.c_double, P, ctypes.c_double, P, P, P]
        lib.fpo_build_tours.restype = ctypes.c_int
        lib.fpo_build_tours_sorted.argtypes = [P, P, ctypes.c_int, ctypes.c_int, ctypes.c_uint64, ctypes.c_uint32,
                                               P, ctypes.c_int, P, ctypes.c_double, P, ctypes.c_double, P, P, P]
        lib.fpo_build_tours_sorted.restype = ctypes.c_int
        lib.fpo_count_mismatches.argtypes = [P, P, ctypes.c_int, ctypes.c_int, P, P, ctypes.c_uint64,
                                             ctypes.c_uint32, P, ctypes.c_int, P, P]
        lib.fpo_count_mismatches.restype = None
        lib.fpo_scan_profile.argtypes = [P, P, ctypes.c_int, ctypes.c_int, ctypes.c_uint64, ctypes.c_uint32, P,
                                         ctypes.c_int, P, ctypes.c_int]
        lib.fpo_scan_profile.restype = None
        lib.fpo_seed_hash32.argtypes = [ctypes.c_uint64]
        lib.fpo_seed_hash32.restype = ctypes.c_uint32
        lib.fpo_philox.argtypes = [ctypes.c_int, P, P, P]
        lib.fpo_philox.restype = None
        _lib = lib
    return _lib


def _ptr(a):
    return None if a is None else a.ctypes.data


def _table(w: np.ndarray) -> tuple[np.ndarray, int]:
    w = np.ascontiguousarray(w, dtype=np.float32)
    return w, w.shape[1]


def _fallback(fallback):
    if fallback is None:
        return None, 1.0, None
    fb_b = None if fallback[2] is None else np.ascontiguousarray(fallback[2], dtype=np.float64)
    return np.ascontiguousarray(fallback[0], dtype=np.float64), float(fallback[1]), fb_b


def build_tours_sorted(sw: np.ndarray, si: np.ndarray, seed: int, iteration: int, ants, n: int | None = None,
                       fallback: tuple | None = None, inv_gamma: float = 1.0) -> np.ndarray:
    """Full-scan product-rule tours of the SORTED stream (the kernels that scan
    the row-sorted table): uniforms keyed by the entry's position in the row.
    sw / si: (n, ld) sorted values and their cities.  Otherwise as build_tours."""
    sw, ld = _table(sw)
    si = np.ascontiguousarray(si, dtype=np.uint16)
    assert si.shape == sw.shape
    n = sw.shape[0] if n is None else int(n)
    ants = np.ascontiguousarray(np.asarray(ants, dtype=np.int64))
    out = np.zeros((ants.size, n), dtype=np.int32)
    fb_a, alpha, fb_b = _fallback(fallback)
    fbs = np.zeros(1, dtype=np.int64)
    fail = np.zeros(1, dtype=np.int32)
    rc = _load().fpo_build_tours_sorted(_ptr(sw), _ptr(si), n, ld, int(seed) & 0xFFFFFFFFFFFFFFFF,
                                        int(iteration) & 0xFFFFFFFF, _ptr(ants), ants.size, _ptr(fb_a), alpha,
                                        _ptr(fb_b), float(inv_gamma), _ptr(out), _ptr(fbs), _ptr(fail))
    if rc == 2:
        raise AssertionError("selector chose a visited city")
    build_tours.last_fallbacks = int(fbs[0])
    return out.astype(np.int64)


def build_tours(w: np.ndarray, seed: int, iteration: int, ants, n: int | None = None,
                fallback: tuple | None = None, inv_gamma: float = 1.0) -> np.ndarray:
    """Full-scan product-rule tours of the DENSE stream (uniforms keyed by
    city; int64, one row per entry of `ants`).

    w: (n, ldw) fp32 selection table (ldw >= n; pad columns ignored).
    fallback: (A, alpha, B or None), the f64 source the kernel falls back to
    when no W > 0 candidate is left (v = A^alpha * B); None: no source (the
    all -inf rule only).  Raises AssertionError like the reference (colony.py:149).
    Both builders set build_tours.last_fallbacks.
    """
    w, ldw = _table(w)
    n = w.shape[0] if n is None else int(n)
    ants = np.ascontiguousarray(np.asarray(ants, dtype=np.int64))
    out = np.zeros((ants.size, n), dtype=np.int32)
    fb_a = fb_b = None
    alpha = 1.0
    if fallback is not None:
        fb_a = np.ascontiguousarray(fallback[0], dtype=np.float64)
        alpha = float(fallback[1])
        fb_b = None if fallback[2] is None else np.ascontiguousarray(fallback[2], dtype=np.float64)
    fbs = np.zeros(1, dtype=np.int64)
    fail = np.zeros(1, dtype=np.int32)
    rc = _load().fpo_build_tours(_ptr(w), n, ldw, int(seed) & 0xFFFFFFFFFFFFFFFF, int(iteration) & 0xFFFFFFFF,
                                 _ptr(ants), ants.size, _ptr(fb_a), alpha, _ptr(fb_b), float(inv_gamma),
                                 _ptr(out), _ptr(fbs), _ptr(fail))
    if rc == 2:
        raise AssertionError("selector chose a visited city")
    build_tours.last_fallbacks = int(fbs[0])
    return out.astype(np.int64)


build_tours.last_fallbacks = 0


def logu_table() -> np.ndarray:
    """numpy's log of every device uniform value (k + 1/2) 2^-23, k < 2^23."""
    global _logu
    if _logu is None:
        k = np.arange(1 << 23, dtype=np.float64)
        _logu = np.log((k + 0.5) * 2.0**-23)
    return _logu


def count_mismatches(w: np.ndarray, logw: np.ndarray, seed: int, iteration: int, ants, tours,
                     si: np.ndarray | None = None) -> dict:
    """Selection-level agreement of recorded tours (the device's) with the
    product rule, the reference's log rule on the same uniforms and the log
    rule on refined 53-bit uniforms (see fastpath.c fpo_count_mismatches).
    w: the dense table, or with `si` the row-sorted table (sorted stream)."""
    w, ldw = _table(w)
    n = w.shape[0]
    if si is not None:
        si = np.ascontiguousarray(si, dtype=np.uint16)
        assert si.shape == w.shape
    logw = np.ascontiguousarray(logw, dtype=np.float64)
    assert logw.shape == (n, n)
    ants = np.ascontiguousarray(np.asarray(ants, dtype=np.int64))
    tours = np.ascontiguousarray(tours, dtype=np.int32)
    assert tours.shape == (ants.size, n)
    out = np.zeros(5, dtype=np.int64)
    _load().fpo_count_mismatches(_ptr(w), _ptr(si), n, ldw, _ptr(logw), _ptr(logu_table()),
                                 int(seed) & 0xFFFFFFFFFFFFFFFF,
                                 int(iteration) & 0xFFFFFFFF, _ptr(ants), ants.size, _ptr(tours), _ptr(out))
    return {"selections": int(out[0]), "product_rule": int(out[1]), "log_rule_same_u": int(out[2]),
            "log_rule_u53": int(out[3]), "u53_below_uniform_floor": int(out[4])}


def seed_hash32(seed: int) -> int:
    return int(_load().fpo_seed_hash32(int(seed) & 0xFFFFFFFFFFFFFFFF))


def philox2x32_10(ctr: np.ndarray, key) -> np.ndarray:
    ctr = np.ascontiguousarray(np.asarray(ctr, dtype=np.uint32).reshape(-1, 2))
    key = np.ascontiguousarray(np.broadcast_to(np.asarray(key, dtype=np.uint32), (ctr.shape[0],)))
    out = np.zeros_like(ctr)
    _load().fpo_philox(ctr.shape[0], _ptr(ctr), _ptr(key), _ptr(out))
    return out


def scan_profile(sw: np.ndarray, si: np.ndarray, n: int, seed: int, iteration: int, ants,
                 bins: int = 4096) -> np.ndarray:
    """Histogram of 32-entry windows read per step by the pruned sorted scan
    (index w: w + 1 windows; last bin: that many or more)."""
    sw = np.ascontiguousarray(sw, dtype=np.float32)
    si = np.ascontiguousarray(si, dtype=np.uint16)
    ants = np.ascontiguousarray(np.asarray(ants, dtype=np.int64))
    hist = np.zeros(bins, dtype=np.int64)
    _load().fpo_scan_profile(_ptr(sw), _ptr(si), int(n), sw.shape[1], int(seed) & 0xFFFFFFFFFFFFFFFF,
                             int(iteration) & 0xFFFFFFFF, _ptr(ants), ants.size, _ptr(hist), bins)
    return hist
