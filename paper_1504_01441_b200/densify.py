"""Drop-in for `hdrflow.densify` (densify.py:30-174) on the GPU: sparse
splat (K9), domain-transform filter (K10), ratio + fallback finalise (K11)
and the bilinear backward warp (K12)."""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _native
from .engine import device_of, engine, is_torch, out, ptr, to_dev

DEFAULT_SIGMA_S = 400.0
DEFAULT_SIGMA_R = 0.2
DEFAULT_PASSES = 3
NORMALIZATION_FLOOR = 1e-4


@dataclass
class SparseMaps:
    """densify.py:30-35 (planes may be numpy arrays or CUDA tensors)."""
    pu: np.ndarray
    pv: np.ndarray
    n: np.ndarray


def build_sparse_maps(matches, width: int, height: int) -> SparseMaps:
    """densify.py:38-56 — collisions keep the lowest (score, index)."""
    as_torch = is_torch(matches)
    dev = device_of(matches)
    m = to_dev(np.asarray(matches, dtype=np.float64).reshape(-1, 5)
               if not isinstance(matches, torch.Tensor) else matches.reshape(-1, 5),
               torch.float64, dev)
    planes = torch.empty((3, height, width), dtype=torch.float64, device=m.device)
    e = engine(width, height, dev)
    _native.check(_native.lib().hdr_sparse_maps(e.handle, ptr(m), m.shape[0], width, height,
                                                ptr(planes[0]), ptr(planes[1]), ptr(planes[2])),
                  "build_sparse_maps")
    return SparseMaps(out(planes[0], as_torch), out(planes[1], as_torch), out(planes[2], as_torch))


def dt_filter(guide, data, sigma_s: float = DEFAULT_SIGMA_S, sigma_r: float = DEFAULT_SIGMA_R,
              passes: int = DEFAULT_PASSES):
    """densify.py:78-113 — data (h, w) or (h, w, k), float64 result.

    A single-channel float32 guide takes the pair pipeline's kernels (row
    sweeps in shared memory, cluster column sweeps); any other guide (several
    channels, float64 values) takes hdr_dt_filter_general, which sums the
    channel distances as densify.py:59-66 does."""
    if sigma_s <= 0 or sigma_r <= 0:
        raise ValueError("sigma_s and sigma_r must be positive")
    if passes < 1:
        raise ValueError("passes must be >= 1")
    if guide.shape[:2] != data.shape[:2]:
        raise ValueError("guide and data dimensions differ")
    as_torch = is_torch(guide, data)
    dev = device_of(guide, data)
    d = to_dev(data, torch.float64, dev)
    squeeze = d.dim() == 2
    if squeeze:
        d = d[:, :, None]
    h, w, k = d.shape
    planes = d.permute(2, 0, 1).contiguous()
    gch = 1 if guide.ndim == 2 else int(guide.shape[2])
    fast = gch == 1 and guide.dtype in (np.float32, torch.float32)
    e = engine(w, h, dev)
    lib = _native.lib()
    if fast:
        g = to_dev(guide, torch.float32, dev).reshape(h, w)
        rc = lib.hdr_dt_filter(e.handle, ptr(g), ptr(planes), k, w, h, float(sigma_s),
                               float(sigma_r), int(passes))
    else:
        g = to_dev(guide, torch.float64, dev).reshape(h, w, gch)
        rc = lib.hdr_dt_filter_general(e.handle, ptr(g), gch, ptr(planes), k, w, h,
                                       float(sigma_s), float(sigma_r), int(passes))
    _native.check(rc, "dt_filter")
    res = planes.permute(1, 2, 0)
    res = res[:, :, 0] if squeeze else res.contiguous()
    return out(res.contiguous(), as_torch)


def densify_flow(guide, maps: SparseMaps, fallback=None, sigma_s: float = DEFAULT_SIGMA_S,
                 sigma_r: float = DEFAULT_SIGMA_R, passes: int = DEFAULT_PASSES,
                 floor: float = NORMALIZATION_FLOOR):
    """densify.py:116-142 — ratio of filtered planes, H-flow below the floor."""
    h, w = maps.n.shape
    if guide.shape[:2] != (h, w):
        raise ValueError("guide and sparse maps dimensions differ")
    as_torch = is_torch(guide, maps.n)
    dev = device_of(guide, maps.n)
    g = to_dev(guide, torch.float32, dev)
    planes = torch.stack([to_dev(maps.pu, torch.float64, dev), to_dev(maps.pv, torch.float64, dev),
                          to_dev(maps.n, torch.float64, dev)]).contiguous()
    e = engine(w, h, dev)
    lib = _native.lib()
    _native.check(lib.hdr_dt_filter(e.handle, ptr(g), ptr(planes), 3, w, h, float(sigma_s),
                                    float(sigma_r), int(passes)), "dt_filter")
    fb = None if fallback is None else to_dev(fallback, torch.float64, dev)
    flow = torch.empty((h, w, 2), dtype=torch.float32, device=g.device)
    _native.check(lib.hdr_densify_finalize(e.handle, ptr(planes), w, h, ptr(fb), float(floor),
                                           ptr(flow)), "densify_flow")
    return out(flow, as_torch)


def warp_image(src, flow):
    """densify.py:145-174 — bilinear backward warp (f64 coordinates)."""
    h, w = src.shape[:2]
    if flow.shape[:2] != (h, w) or flow.shape[2] != 2:
        raise ValueError("flow must be (h, w, 2) matching the source")
    as_torch = is_torch(src, flow)
    dev = device_of(src, flow)
    s = to_dev(src, torch.float32, dev)
    f = to_dev(flow, torch.float32, dev)
    ch = 1 if s.dim() == 2 else int(s.shape[2])
    warped = torch.empty_like(s)
    valid = torch.empty((h, w), dtype=torch.uint8, device=s.device)
    e = engine(1, 1, dev)
    _native.check(_native.lib().hdr_warp_image(e.handle, ptr(s), ch, w, h, ptr(f), ptr(warped),
                                               ptr(valid)), "warp_image")
    return out(warped, as_torch), out(valid.bool(), as_torch)
