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
    """image.py:91-93 — floor(x * 255 + 0.5) clipped to uint8 on the GPU
    (float32 samples in float32 arithmetic, anything else in float64)."""
    as_torch = is_torch(img)
    dev = device_of(img)
    f32 = img.dtype in (np.float32, torch.float32)
    t = to_dev(img, torch.float32 if f32 else torch.float64, dev)
    res = torch.empty(t.shape, dtype=torch.uint8, device=t.device)
    e = engine(1, 1, dev)
    _native.check(_native.lib().hdr_quantize_256(e.handle, ptr(t), 0 if f32 else 1, t.numel(),
                                                 ptr(res)), "quantize_256")
    return out(res, as_torch)


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


_INDEX_ERROR = ("only integers, slices (`:`), ellipsis (`...`), numpy.newaxis (`None`) and "
                "integer or boolean arrays are valid indices")


def rect_sum(table, x0, y0, x1, y1):
    """image.py:47-58 — batched rectangle sums on the GPU (scalars or
    broadcastable integer arrays; an out-of-range rectangle raises
    ValueError as the reference does)."""
    as_torch = is_torch(table, x0, y0, x1, y1)
    dev = device_of(table, x0, y0, x1, y1)
    t = to_dev(table, torch.float64, dev)
    h1, w1 = t.shape
    if is_torch(x0, y0, x1, y1):
        b = torch.broadcast_tensors(*(to_dev(v, torch.int64, dev) if isinstance(v, torch.Tensor)
                                      else torch.as_tensor(v, device=f"cuda:{dev}")
                                      for v in (x0, y0, x1, y1)))
        if any(v.dtype.is_floating_point or v.dtype.is_complex for v in b):
            raise IndexError(_INDEX_ERROR)
        shape = tuple(b[0].shape)
        q = torch.stack([v.reshape(-1).to(torch.int64) for v in b]).contiguous()
    else:
        b = np.broadcast_arrays(*(np.asarray(v) for v in (x0, y0, x1, y1)))
        if any(not (np.issubdtype(v.dtype, np.integer) or v.dtype == np.bool_) for v in b):
            raise IndexError(_INDEX_ERROR)
        shape = b[0].shape
        q = to_dev(np.stack([v.reshape(-1).astype(np.int64) for v in b]), torch.int64, dev)
    n = q.shape[1]
    res = torch.empty(n, dtype=torch.float64, device=t.device)
    e = engine(1, 1, dev)
    _native.check(_native.lib().hdr_rect_sum(e.handle, ptr(t), w1, h1, ptr(q), n, ptr(res)),
                  "rect_sum")
    res = res.reshape(shape)
    if as_torch:
        return res
    r = res.cpu().numpy()
    return r[()] if shape == () else r


def downsample(img):
    """image.py:61-68 — one 2x2 box level, any channel count (kernel K3 /
    hdr_downsample); float32 result."""
    h, w = img.shape[:2]
    if h < 2 or w < 2:
        raise ValueError("image too small to downsample")
    as_torch = is_torch(img)
    dev = device_of(img)
    f32 = img.dtype in (np.float32, torch.float32)
    t = to_dev(img, torch.float32 if f32 else torch.float64, dev)
    ch = 1 if t.dim() == 2 else int(t.shape[2])
    res = torch.empty((h // 2, w // 2) + tuple(t.shape[2:]), dtype=torch.float32, device=t.device)
    e = engine(1, 1, dev)
    _native.check(_native.lib().hdr_downsample(e.handle, ptr(t), 0 if f32 else 1, w, h, ch, ptr(res)),
                  "downsample")
    return out(res, as_torch)


def build_pyramid(img, max_levels: int = PYRAMID_MAX_LEVELS, min_dim: int = PYRAMID_MIN_DIM):
    """image.py:71-88 — all levels from one device-resident chain (kernel K3)."""
    h, w = img.shape[:2]
    if min(h, w) < min_dim:
        raise ValueError(f"input below {min_dim} pixels in one dimension")
    if img.ndim != 2 or img.dtype not in (np.float32, torch.float32):
        # multi-channel or non-float32 levels: one hdr_downsample per level
        levels = [img]
        while len(levels) < max_levels:
            ph, pw = levels[-1].shape[:2]
            if min(ph // 2, pw // 2) < min_dim:
                break
            levels.append(downsample(levels[-1]))
        return levels
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
