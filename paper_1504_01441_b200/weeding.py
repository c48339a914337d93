"""Drop-in for `hdrflow.weeding` (weeding.py:30-145) on the GPU.

All iterations run concurrently (one thread draws+fits each hypothesis, one
block tests it against every match); each iteration keeps its own
Philox4x64-10 stream keyed by SeedSequence(seed, spawn_key=(it,)), so the
result is the reference's for any worker count (weeding.py:8-11).
"""

from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass

import numpy as np
import torch

from . import _native
from .engine import device_of, engine_for_rows, ptr, to_dev

DEFAULT_ITERATIONS = 256
DEFAULT_COARSE_ITERATIONS = 64
MAX_RESAMPLE = 10


def default_delta(n_matches: int) -> int:
    """weeding.py:30-32."""
    return max(12, math.ceil(0.15 * n_matches))


@dataclass
class WeedParams:
    """weeding.py:35-53."""
    iterations: int = DEFAULT_ITERATIONS
    delta: int | None = None
    eps: float = 2.0 * 2.0 / 640.0
    seed: int = 0

    def __post_init__(self):
        if self.iterations < 1:
            raise ValueError("iterations must be >= 1")
        if self.delta is not None and self.delta < 4:
            raise ValueError("delta must be >= 4")
        if self.eps <= 0:
            raise ValueError("eps must be positive")


@dataclass
class WeedResult:
    kept: np.ndarray
    witness: np.ndarray


def weed(matches, image_size, params: WeedParams) -> WeedResult:
    """weeding.py:100-111 (K7)."""
    dev = device_of(matches)
    m = to_dev(matches, torch.float64, dev).reshape(-1, 5)
    n = m.shape[0]
    if n < 4:
        raise ValueError("need at least 4 matches to weed")
    width, height = image_size
    kept = torch.empty((n,), dtype=torch.int64, device=m.device)
    witness = torch.zeros((n,), dtype=torch.int64, device=m.device)
    nk = ctypes.c_int32(0)
    e = engine_for_rows(n, dev)  # the weed workspace scales with the tile count
    delta = -1 if params.delta is None else int(params.delta)
    _native.check(_native.lib().hdr_weed(e.handle, ptr(m), n, width, height, params.iterations,
                                         float(params.eps), int(params.seed), delta, ptr(kept),
                                         ctypes.byref(nk), ptr(witness)), "weed")
    return WeedResult(kept[:nk.value].cpu().numpy(), witness.cpu().numpy())


def weed_parallel(matches, image_size, params: WeedParams, workers: int) -> WeedResult:
    """weeding.py:114-145 — same argument checks; the GPU run is already parallel."""
    if workers < 1:
        raise ValueError("workers must be >= 1")
    if params.iterations % workers != 0:
        raise ValueError("iterations must be divisible by the worker count")
    if len(matches) < 4:
        raise ValueError("need at least 4 matches to weed")
    return weed(matches, image_size, params)
