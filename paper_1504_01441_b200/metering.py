"""Drop-in for `hdrflow.metering.choose_reference` (metering.py:37-51), the
one metering decision on the file path: the darkest
exposure is the reference; ties go to the lower mean luminance, computed on
the GPU (`hdr_mean_luminance`, f64 accumulation of the f32 luminance)."""

from __future__ import annotations

import torch

from . import _native
from .engine import engine, ptr, to_dev


def mean_luminance(img) -> float:
    """np.mean(luminance(img)) of metering.py:46-48 (grey images: their mean)."""
    t = to_dev(img, torch.float32)
    if t.dim() == 2:
        t = t.unsqueeze(-1).expand(*t.shape, 3).contiguous()
    h, w = t.shape[:2]
    res = torch.zeros((1,), dtype=torch.float64, device=t.device)
    e = engine(w, h, t.device.index)
    _native.check(_native.lib().hdr_mean_luminance(e.handle, ptr(t), h * w, ptr(res)),
                  "mean_luminance")
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
