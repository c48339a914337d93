"""Drop-in for `hdrflow.image` (image.py:18-136): GPU luminance, histogram
matching, box pyramid and summed-area table; coordinate helpers are the
reference's closed forms."""

from __future__ import annotations

import ctypes

import numpy as np
import torch

from . import _native
from .engine import device_of, engine, is_torch, out, ptr, to_dev

REC601 = (0.299, 0.587, 0.114)
PYRAMID_MAX_LEVELS = 5
PYRAMID_MIN_DIM = 100
HISTOGRAM_BINS = 256


def image_size(img):
    """(width, height) of an image array (image.py:18-20)."""
    return img.shape[1], img.shape[0]


def luminance(img):
    """image.py:23-29 — bit-exact Rec.601 luminance (kernel K1)."""
    if img.ndim != 3 or img.shape[2] != 3:
        raise ValueError("luminance expects an (h, w, 3) image")
    as_torch = is_torch(img)
    t = to_dev(img, torch.float32, device_of(img))
    h, w = t.shape[:2]
    res = torch.empty((h, w), dtype=torch.float32, device=t.device)
    e = engine(max(w, 1), max(h, 1), t.device.index)
    _native.check(_native.lib().hdr_luminance(e.handle, ptr(t), h * w, ptr(res)), "luminance")
    return out(res, as_torch)


def match_histogram(src, ref):
    """image.py:109-122 — per-channel 256-bin CDF matching (kernels K1+K2)."""
    if src.ndim != ref.ndim or (src.ndim == 3 and src.shape[2] != ref.shape[2]):
        raise ValueError("source and reference must have the same channel count")
    as_torch = is_torch(src, ref)
    dev = device_of(src, ref)
    s = to_dev(src, torch.float32, dev)
    r = to_dev(ref, torch.float32, dev)
    res = torch.empty_like(s)
    ch = s.shape[2] if s.dim() == 3 else 1
    n_s, n_r = s.numel() // ch, r.numel() // ch
    e = engine(1, 1, dev)
    for c in range(ch):
        off = c * 4
        _native.check(_native.lib().hdr_match_histogram(
            e.handle, ptr(s).value + off, n_s, ptr(r).value + off, n_r, ch, ptr(res).value + off),
            "match_histogram")
    return out(res, as_torch)


def quantize_256(img):
    """image.py:91-93 (host helper, not on the GPU path)."""
    return np.clip(np.floor(np.asarray(img) * 255.0 + 0.5), 0, 255).astype(np.uint8)


def integral(img):
    """image.py:32-44 — f64 SAT in numpy's sequential order (kernel K4)."""
    if img.ndim != 2:
        raise ValueError("integral expects a single-channel image")
    as_torch = is_torch(img)
    t = to_dev(img, torch.float32, device_of(img))
    h, w = t.shape
    table = torch.empty((h + 1, w + 1), dtype=torch.float64, device=t.device)
    e = engine(w, h, t.device.index)
    _native.check(_native.lib().hdr_integral(e.handle, ptr(t), w, h, ptr(table)), "integral")
    return out(table, as_torch)


def rect_sum(table, x0, y0, x1, y1):
    """image.py:47-58 (host helper over an already computed table)."""
    t = table.cpu().numpy() if isinstance(table, torch.Tensor) else table
    h1, w1 = t.shape
    x0, y0, x1, y1 = (np.asarray(v) for v in (x0, y0, x1, y1))
    if (np.any(x0 < 0) or np.any(y0 < 0) or np.any(x0 > x1) or np.any(y0 > y1)
            or np.any(x1 >= w1) or np.any(y1 >= h1)):
        raise ValueError("rectangle bounds out of range")
    return t[y1, x1] - t[y0, x1] - t[y1, x0] + t[y0, x0]


def downsample(img):
    """image.py:61-68 — one 2x2 box level (kernel K3)."""
    h, w = img.shape[:2]
    if h < 2 or w < 2:
        raise ValueError("image too small to downsample")
    if img.ndim != 2:
        raise ValueError("downsample on the GPU path expects a single-channel image")
    lv = build_pyramid(img, max_levels=2, min_dim=0)
    return lv[1]


def build_pyramid(img, max_levels: int = PYRAMID_MAX_LEVELS, min_dim: int = PYRAMID_MIN_DIM):
    """image.py:71-88 — all levels from one device-resident chain (kernel K3)."""
    h, w = img.shape[:2]
    if min(h, w) < min_dim:
        raise ValueError(f"input below {min_dim} pixels in one dimension")
    if img.ndim != 2:
        raise ValueError("the GPU pyramid expects a single-channel image")
    as_torch = is_torch(img)
    t = to_dev(img, torch.float32, device_of(img))
    dims = [(h, w)]
    while len(dims) < max_levels:
        ph, pw = dims[-1]
        if min(ph // 2, pw // 2) < max(min_dim, 1):
            break
        dims.append((ph // 2, pw // 2))
    levels = [t] + [torch.empty(d, dtype=torch.float32, device=t.device) for d in dims[1:]]
    arr = (ctypes.c_void_p * len(levels))(None, *[l.data_ptr() for l in levels[1:]])
    nlev = ctypes.c_int32(0)
    e = engine(w, h, t.device.index)
    _native.check(_native.lib().hdr_build_pyramid(e.handle, ptr(t), w, h, max_levels, min_dim,
                                                  arr, ctypes.byref(nlev)), "build_pyramid")
    assert nlev.value == len(levels)
    return [img if i == 0 and not as_torch else out(l, as_torch) for i, l in enumerate(levels)]


def to_normalized(x, y, width: int, height: int):
    """image.py:125-129."""
    w = float(width)
    return (2.0 * np.asarray(x, dtype=np.float64) - width) / w, \
           (2.0 * np.asarray(y, dtype=np.float64) - height) / w


def from_normalized(xn, yn, width: int, height: int):
    """image.py:132-136."""
    w = float(width)
    return (np.asarray(xn, dtype=np.float64) * w + width) / 2.0, \
           (np.asarray(yn, dtype=np.float64) * w + height) / 2.0
