"""Drop-in for `hdrflow.fusion` (fusion.py:28-157) on the GPU: SSIM (K13),
quality and fusion weights (K14), Laplacian-pyramid fusion (K15)."""

from __future__ import annotations

import numpy as np
import torch

from . import _native
from .engine import device_of, engine, is_torch, out, ptr, to_dev

SSIM_WINDOW = 11
SSIM_SIGMA = 1.5
SSIM_C1 = 0.01 ** 2
SSIM_C2 = 0.03 ** 2
WELL_EXPOSED_SIGMA = 0.2
WEIGHT_FLOOR = 1e-12


def ssim_map(a, b, window: int = SSIM_WINDOW, sigma: float = SSIM_SIGMA):
    """fusion.py:34-64 — float64 result (computed in f64, stored f32)."""
    if a.shape != b.shape or a.ndim != 2:
        raise ValueError("ssim_map expects two single-channel images of equal size")
    if window % 2 != 1:
        raise ValueError("window must be odd")
    as_torch = is_torch(a, b)
    dev = device_of(a, b)
    ta, tb = to_dev(a, torch.float32, dev), to_dev(b, torch.float32, dev)
    h, w = ta.shape
    res = torch.empty((h, w), dtype=torch.float32, device=ta.device)
    e = engine(1, 1, dev)
    _native.check(_native.lib().hdr_ssim_map(e.handle, ptr(ta), ptr(tb), w, h, window,
                                             float(sigma), ptr(res)), "ssim_map")
    return out(res.double(), as_torch)


def quality_weights(img):
    """fusion.py:67-77 — contrast x saturation x well-exposedness + 1e-12."""
    if img.ndim != 3 or img.shape[2] != 3:
        raise ValueError("quality_weights expects an (h, w, 3) image")
    as_torch = is_torch(img)
    t = to_dev(img, torch.float32, device_of(img))
    h, w = t.shape[:2]
    res = torch.empty((h, w), dtype=torch.float32, device=t.device)
    e = engine(1, 1, t.device.index)
    _native.check(_native.lib().hdr_quality_weights(e.handle, ptr(t), w, h, ptr(res)),
                  "quality_weights")
    return out(res.double(), as_torch)


def fusion_weights(ref, warped, ssim, valid):
    """fusion.py:117-128 — normalised (w_ref, w_src) per pixel (f32 on the
    device, widened to float64 like the reference's result)."""
    as_torch = is_torch(ref, warped, ssim, valid)
    dev = device_of(ref, warped, ssim, valid)
    r, wp = to_dev(ref, torch.float32, dev), to_dev(warped, torch.float32, dev)
    s = to_dev(ssim, torch.float32, dev)
    v = to_dev(np.asarray(valid) != 0 if not isinstance(valid, torch.Tensor) else valid != 0,
               torch.uint8, dev)
    h, w = r.shape[:2]
    wr = torch.empty((h, w), dtype=torch.float32, device=r.device)
    ws = torch.empty((h, w), dtype=torch.float32, device=r.device)
    e = engine(1, 1, dev)
    _native.check(_native.lib().hdr_fusion_weights(e.handle, ptr(r), ptr(wp), ptr(s), ptr(v), w, h,
                                                   ptr(wr), ptr(ws)), "fusion_weights")
    return out(wr.double(), as_torch), out(ws.double(), as_torch)


def default_fusion_levels(height: int, width: int) -> int:
    """fusion.py:131-132."""
    return max(1, int(np.floor(np.log2(min(height, width)))) - 1)


def fuse(ref, warped, ssim, valid, levels: int | None = None):
    """fusion.py:135-157 — float32 composite clipped to [0, 1]."""
    if ref.shape != warped.shape:
        raise ValueError("reference and warped source dimensions differ")
    if ssim.shape != ref.shape[:2] or valid.shape != ref.shape[:2]:
        raise ValueError("ssim/valid dimensions differ from the images")
    as_torch = is_torch(ref, warped, ssim, valid)
    dev = device_of(ref, warped, ssim, valid)
    r, wp = to_dev(ref, torch.float32, dev), to_dev(warped, torch.float32, dev)
    s = to_dev(ssim, torch.float32, dev)
    v = to_dev(np.asarray(valid) != 0 if not isinstance(valid, torch.Tensor) else valid != 0,
               torch.uint8, dev)
    h, w = r.shape[:2]
    res = torch.empty((h, w, 3), dtype=torch.float32, device=r.device)
    e = engine(w, h, dev)
    _native.check(_native.lib().hdr_fuse(e.handle, ptr(r), ptr(wp), ptr(s), ptr(v), w, h,
                                         0 if levels is None else int(levels), ptr(res)), "fuse")
    return out(res, as_torch)
