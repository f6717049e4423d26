"""Random streams of the engine.

Two streams exist:

* ``"device"`` (default, the hot path) — counter-based Philox4x32-10 evaluated
  on chip inside the construction kernel.  Every uniform is addressed by
  (seed, iteration, step, global ant, city), so results do not depend on how
  ants are scheduled or sharded across GPUs (the property the reference gets
  from keyed numpy streams, rng.py:1-20).  Nothing is materialized in HBM.

* ``"numpy"`` — the reference's own keyed numpy streams (rng.py:26-68:
  ``Philox(SeedSequence(seed, spawn_key=(domain, *key)))``), generated on the
  host and uploaded step by step.  This is the bit-exact parity mode of
  ``construct_tours(..., stream="numpy")``; it is slow by construction (the
  reference's deviate generation is half of its CPU time) and exists to prove
  that the device argmax reproduces the reference's tours exactly.
"""

from __future__ import annotations

import numpy as np

DOMAIN_CONSTRUCT = 0  # rng.py:26 spawn-key domains of the reference
DOMAIN_START = 1
DOMAIN_MC = 2


def stream(seed: int, domain: int, *key: int) -> np.random.Generator:
    """The reference's keyed generator (rng.py:33-39)."""
    ss = np.random.SeedSequence(entropy=seed, spawn_key=(domain, *key))
    return np.random.Generator(np.random.Philox(ss))


def step_exponentials(seed: int, iteration: int, step: int, m: int, n: int) -> np.ndarray:
    """(m, n) Exp(1) block of one construction step (rng.py:42-49)."""
    return stream(seed, DOMAIN_CONSTRUCT, iteration, step).standard_exponential((m, n))


def step_keys(seed: int, iteration: int, n: int) -> np.ndarray:
    """Philox4x64 keys of the construction steps 1..n-1 of one iteration: the
    state SeedSequence(seed, spawn_key=(0, it, step)) hands to numpy's Philox
    (rng.py:33-39).  Shape (n-1, 2) uint64; the device replays the streams."""
    return np.stack([np.random.SeedSequence(entropy=seed, spawn_key=(DOMAIN_CONSTRUCT, iteration, step))
                     .generate_state(2, np.uint64) for step in range(1, n)])


def start_cities(seed: int, iteration: int, m: int, n: int) -> np.ndarray:
    """Reference start city per ant (rng.py:65-68)."""
    return stream(seed, DOMAIN_START, iteration).integers(0, n, size=m, dtype=np.int64)


def device_starts(seed: int, iteration: int, n: int, m: int, ant_offset: int = 0) -> np.ndarray:
    """Start cities of the device stream for ants [ant_offset, ant_offset + m)."""
    import torch

    from . import _device, _lib

    dev = _device.device()
    out = torch.empty(m, dtype=torch.int32, device=dev)
    _lib.check(_lib.load().taco_starts(n, m, ant_offset, int(seed), int(iteration) & 0xFFFFFFFF,
                                       out.data_ptr(), _device.stream_handle()), "taco_starts")
    return out.cpu().numpy().astype(np.int64)


def device_uniforms(seed: int, iteration: int, step, ant, city) -> np.ndarray:
    """Device-stream uniforms u(seed, iteration, step, ant, city) (fp32)."""
    import torch

    from . import _device, _lib

    dev = _device.device()
    s = torch.as_tensor(np.asarray(step, dtype=np.uint32).astype(np.int32).ravel(), device=dev)
    a = torch.as_tensor(np.asarray(ant, dtype=np.uint32).astype(np.int32).ravel(), device=dev)
    c = torch.as_tensor(np.asarray(city, dtype=np.uint32).astype(np.int32).ravel(), device=dev)
    out = torch.empty(s.numel(), dtype=torch.float32, device=dev)
    _lib.check(_lib.load().taco_uniforms(s.numel(), s.data_ptr(), a.data_ptr(), c.data_ptr(), int(seed),
                                         int(iteration) & 0xFFFFFFFF, out.data_ptr(),
                                         _device.stream_handle()), "taco_uniforms")
    return out.cpu().numpy()
