"""Drop-in for `hdrflow.metering` (metering.py:1-57): the reference choice on
the file path -- the darkest exposure; ties go to the
lower mean luminance, computed on the GPU (`hdr_mean_luminance`, f64
accumulation of the f32 luminance) -- and the exposure-offset plan
(`select_offset` from the GPU's dark-pixel count, `hdr_dark_count`)."""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _native
from .engine import engine, ptr, to_dev


def mean_luminance(img) -> float:
    """np.mean(luminance(img)) of metering.py:46-48 (grey images: their mean)."""
    t = to_dev(img, torch.float32)
    h, w = t.shape[:2]
    res = torch.zeros((1,), dtype=torch.float64, device=t.device)
    e = engine(w, h, t.device.index)
    _native.check(_native.lib().hdr_mean_luminance(e.handle, ptr(t), 1 if t.dim() == 2 else 3,
                                                   h * w, ptr(res)), "mean_luminance")
    return float(res.item())


def choose_reference(images, exposures) -> int:
    """Index of the darkest exposure; ties resolve to the lowest mean luminance."""
    if not images or len(images) != len(exposures):
        raise ValueError("need one exposure per image")
    exposures = [float(e) for e in exposures]
    shortest = min(exposures)
    candidates = [i for i, e in enumerate(exposures) if e == shortest]
    if len(candidates) == 1:
        return candidates[0]
    return min(candidates, key=lambda i: (mean_luminance(images[i]), i))


DARK_LEVEL = 0.05                  # metering.py:11
OFFSET_CUTOFFS = (0.02, 0.10)      # metering.py:12


@dataclass
class ExposurePlan:
    """metering.py:15-18."""
    offset_stops: int
    reference_index: int


def dark_fraction(img, dark_level: float = DARK_LEVEL) -> float:
    """np.mean(luminance(img) < dark_level) (metering.py:28-29); grey images
    are compared directly, like the reference."""
    t = to_dev(img, torch.float32)
    h, w = t.shape[:2]
    res = torch.zeros((1,), dtype=torch.int64, device=t.device)
    e = engine(w, h, t.device.index)
    _native.check(_native.lib().hdr_dark_count(e.handle, ptr(t), 1 if t.dim() == 2 else 3, h * w,
                                               float(np.float32(dark_level)), ptr(res)), "dark_count")
    return int(res.item()) / float(h * w)


def select_offset(img, dark_level: float = DARK_LEVEL,
                  cutoffs: tuple = OFFSET_CUTOFFS) -> int:
    """Second-exposure offset (2, 3 or 4 stops) from the underexposed
    fraction (metering.py:21-34)."""
    q = dark_fraction(img, dark_level)
    if q < cutoffs[0]:
        return 2
    if q < cutoffs[1]:
        return 3
    return 4


def plan_stack(images, exposures) -> ExposurePlan:
    """metering.py:54-57."""
    ref = choose_reference(images, exposures)
    return ExposurePlan(offset_stops=select_offset(images[ref]), reference_index=ref)
