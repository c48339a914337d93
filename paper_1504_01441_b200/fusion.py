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


def _as_hwc(t: torch.Tensor) -> torch.Tensor:
    return t.unsqueeze(-1) if t.dim() == 2 else t


def _pyr_down(t: torch.Tensor) -> torch.Tensor:
    """fusion.py:85-86 on a float64 CUDA tensor (h, w[, c])."""
    x = _as_hwc(t).contiguous()
    h, w, c = x.shape
    res = torch.empty(((h + 1) // 2, (w + 1) // 2, c), dtype=torch.float64, device=x.device)
    e = engine(1, 1, x.device.index)
    _native.check(_native.lib().hdr_pyr_down(e.handle, ptr(x), w, h, c, ptr(res)), "pyr_down")
    return res if t.dim() == 3 else res[..., 0]


def _pyr_up(t: torch.Tensor, shape, base: torch.Tensor | None = None, sign: int = 0) -> torch.Tensor:
    """fusion.py:89-93: zero-insert into `shape`, 2x-gain blur; with `base`,
    base - up (sign < 0) or base + up (sign > 0) in the same kernel."""
    x = _as_hwc(t).contiguous()
    ch_, cw, c = x.shape
    h, w = int(shape[0]), int(shape[1])
    res = torch.empty((h, w, c), dtype=torch.float64, device=x.device)
    b = None if base is None else _as_hwc(base).contiguous()
    e = engine(1, 1, x.device.index)
    _native.check(_native.lib().hdr_pyr_up(e.handle, ptr(x), cw, ch_, c, w, h, ptr(b), int(sign),
                                           ptr(res)), "pyr_up")
    return res if t.dim() == 3 else res[..., 0]


def gaussian_pyramid(img, levels: int) -> list:
    """fusion.py:96-100 — float64 levels, 5-tap reflect blur + [::2, ::2]."""
    as_torch = is_torch(img)
    g = [to_dev(img, torch.float64, device_of(img))]
    while len(g) < levels and min(g[-1].shape[:2]) >= 2:
        g.append(_pyr_down(g[-1]))
    return [out(x, as_torch) for x in g]


def laplacian_pyramid(img, levels: int) -> list:
    """fusion.py:103-107."""
    as_torch = is_torch(img)
    g = gaussian_pyramid(to_dev(img, torch.float64, device_of(img)), levels)
    laps = [_pyr_up(g[i + 1], g[i].shape, g[i], -1) for i in range(len(g) - 1)] + [g[-1]]
    return [out(x, as_torch) for x in laps]


def collapse_pyramid(laps) -> object:
    """fusion.py:110-114."""
    as_torch = is_torch(*laps)
    dev = device_of(*laps)
    ts = [to_dev(x, torch.float64, dev) for x in laps]
    res = ts[-1]
    for lap in ts[-2::-1]:
        res = _pyr_up(res, lap.shape, lap, +1)
    return out(res, as_torch)


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
