"""Selection helpers of the drop-in (reference: selection.py).

IR picks argmax(r * p) and AdaIR argmax(r**gamma * p) over the unvisited
cities; the reference evaluates the equivalent log form argmax(log p / gamma -
E) with E = -log r (selection.py:1-32).  The engine evaluates the product form
argmax(W * u) with the fp32 table W = p**(1/gamma); both forms
choose the same city given the same uniforms (tests/test_gpu_parity.py counts
mismatches against the log form).  As in the reference, larger gamma makes
selection MORE exploratory (selection.py:27-32).
"""

from __future__ import annotations

import math

import numpy as np
import torch

from . import _device, _lib
from .model import GammaSchedule


class AllZeroWeights(ValueError):
    """No positive entry to select from (selection.py:44-45)."""


def gamma_at(iteration: int, schedule: GammaSchedule) -> float:
    """Cosine-annealed exponent at a 0-based iteration (selection.py:48-59):
    gamma_min + (gamma_max - gamma_min)/2 * (1 + cos(pi * (t mod T) / T))."""
    if iteration < 0:
        raise ValueError(f"iteration must be non-negative, got {iteration}")
    t = iteration % schedule.period
    lo, hi = schedule.gamma_min, schedule.gamma_max
    return lo + 0.5 * (hi - lo) * (1.0 + math.cos(math.pi * t / schedule.period))


def scaled_log_weights(p, gamma: float) -> np.ndarray:
    """log(p) / gamma with -inf where p == 0, computed on the device
    (selection.py:62-75).  CUDA's log is within 1 ulp of numpy's."""
    if not gamma > 0:
        raise ValueError(f"gamma must be > 0, got {gamma}")
    arr = np.ascontiguousarray(np.asarray(p, dtype=np.float64))
    dev = _device.device()
    src = _device.upload(arr, dev)
    out = torch.empty_like(src)
    _lib.check(_lib.load().taco_log_weights(src.numel(), src.data_ptr(), float(gamma), out.data_ptr(),
                                            _device.stream_handle()), "taco_log_weights")
    return _device.download(out).reshape(arr.shape)


def argmax_select_block(logw, current, e_block, visited, scores) -> np.ndarray:
    """Lockstep perturbed argmax of all m ants at one step (selection.py:
    143-155), on the device: scores = logw[current] - e_block, visited cities
    at -inf, row argmax (first of ties; an all -inf row gives 0).  ``scores``
    (caller-owned (m, n) f64 scratch, as in the reference) receives the masked
    scores; returns the (m,) int64 choices.  Bit-exact with the reference: one
    IEEE subtraction per element and exact comparisons."""
    logw = np.ascontiguousarray(np.asarray(logw, dtype=np.float64))
    current = np.ascontiguousarray(np.asarray(current, dtype=np.int64))
    e_block = np.ascontiguousarray(np.asarray(e_block, dtype=np.float64))
    visited = np.ascontiguousarray(np.asarray(visited, dtype=bool))
    m, n = e_block.shape
    if logw.ndim != 2 or logw.shape[1] != n or current.shape != (m,) or visited.shape != (m, n):
        raise ValueError("shapes: logw (r, n), current (m,), e_block (m, n), visited (m, n)")
    if m and (current.min() < 0 or current.max() >= logw.shape[0]):
        raise IndexError("current city out of range")
    dev = _device.device()
    lw, cur, e, vis = (_device.upload(a, dev) for a in (logw, current, e_block, visited.view(np.uint8)))
    sc = torch.empty((m, n), dtype=torch.float64, device=dev)
    nxt = torch.empty(m, dtype=torch.int64, device=dev)
    _lib.check(_lib.load().taco_argmax_select_block(n, m, lw.data_ptr(), cur.data_ptr(), e.data_ptr(),
                                                    vis.data_ptr(), sc.data_ptr(), nxt.data_ptr(),
                                                    _device.stream_handle()), "taco_argmax_select_block")
    if scores is not None:
        scores[...] = _device.download(sc)
    return _device.download(nxt)
