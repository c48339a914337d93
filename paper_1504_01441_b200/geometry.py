"""Drop-in for `hdrflow.geometry` (geometry.py:22-135) on the GPU.

`fit_homography` runs the block-wide DLT of K8 (pivoted Householder for
four points, Gram + Jacobi for least squares) with the reference's
DegenerateFit rules; `inlier_mask` and `homography_pixel_flow` are K7's
transfer test and the fallback flow of K11.
"""

from __future__ import annotations

import numpy as np
import torch

from . import _native
from .engine import device_of, engine, is_torch, out, ptr, to_dev
from .errors import DegenerateFit

MIN_DET = 1e-12

__all__ = ["DegenerateFit", "fit_homography", "apply_homography", "inlier_mask",
           "symmetric_transfer_error", "homography_pixel_flow", "MIN_DET"]


def fit_homography(ref_pts, src_pts):
    """geometry.py:35-77."""
    as_torch = is_torch(ref_pts, src_pts)
    dev = device_of(ref_pts, src_pts)
    r = to_dev(ref_pts, torch.float64, dev).reshape(-1, 2)
    s = to_dev(src_pts, torch.float64, dev).reshape(-1, 2)
    n = r.shape[0]
    if n < 4 or s.shape[0] != n:
        raise ValueError("need at least 4 point pairs")
    hm = torch.empty((3, 3), dtype=torch.float64, device=r.device)
    e = engine(1, 1, dev)
    _native.check(_native.lib().hdr_fit_homography(e.handle, ptr(r), ptr(s), n, ptr(hm)),
                  "fit_homography")
    return out(hm, as_torch)


def apply_homography(h, pts):
    """geometry.py:80-93 (host helper; not on the pair path)."""
    h = h.cpu().numpy() if isinstance(h, torch.Tensor) else np.asarray(h)
    pts = np.asarray(pts, dtype=np.float64)
    x, y = pts[..., 0], pts[..., 1]
    denom = h[2, 0] * x + h[2, 1] * y + h[2, 2]
    if np.any(np.abs(denom) < 1e-12):
        raise ValueError("point maps to infinity")
    res = np.empty_like(pts)
    res[..., 0] = (h[0, 0] * x + h[0, 1] * y + h[0, 2]) / denom
    res[..., 1] = (h[1, 0] * x + h[1, 1] * y + h[1, 2]) / denom
    return res


def inlier_mask(h, ref_pts, src_pts, eps: float):
    """geometry.py:118-121 — hypot(fwd, bwd) < eps on the GPU."""
    as_torch = is_torch(h, ref_pts, src_pts)
    dev = device_of(h, ref_pts, src_pts)
    hm = to_dev(h, torch.float64, dev)
    r = to_dev(ref_pts, torch.float64, dev).reshape(-1, 2)
    s = to_dev(src_pts, torch.float64, dev).reshape(-1, 2)
    n = r.shape[0]
    mask = torch.zeros((max(n, 1),), dtype=torch.uint8, device=r.device)
    e = engine(1, 1, dev)
    _native.check(_native.lib().hdr_inlier_mask(e.handle, ptr(hm), ptr(r), ptr(s), n, float(eps),
                                                ptr(mask)), "inlier_mask")
    return out(mask[:n].bool(), as_torch)


def symmetric_transfer_error(h, ref_pts, src_pts):
    """geometry.py:107-115 (host helper used by diagnostics only)."""
    h = h.cpu().numpy() if isinstance(h, torch.Tensor) else np.asarray(h, dtype=np.float64)
    ref_pts = np.asarray(ref_pts, dtype=np.float64).reshape(-1, 2)
    src_pts = np.asarray(src_pts, dtype=np.float64).reshape(-1, 2)

    def dist(hh, p, t):
        d = hh[2, 0] * p[:, 0] + hh[2, 1] * p[:, 1] + hh[2, 2]
        res = np.full(len(p), np.inf)
        ok = np.abs(d) >= 1e-12
        mx = (hh[0, 0] * p[:, 0] + hh[0, 1] * p[:, 1] + hh[0, 2])[ok] / d[ok]
        my = (hh[1, 0] * p[:, 0] + hh[1, 1] * p[:, 1] + hh[1, 2])[ok] / d[ok]
        res[ok] = np.hypot(mx - t[ok, 0], my - t[ok, 1])
        return res

    return np.hypot(dist(h, ref_pts, src_pts), dist(np.linalg.inv(h), src_pts, ref_pts))


def homography_pixel_flow(h, width: int, height: int):
    """geometry.py:124-135 — dense (h, w, 2) float32 flow."""
    as_torch = is_torch(h)
    dev = device_of(h)
    hm = to_dev(h, torch.float64, dev)
    flow = torch.empty((height, width, 2), dtype=torch.float32, device=hm.device)
    e = engine(1, 1, dev)
    _native.check(_native.lib().hdr_homography_flow(e.handle, ptr(hm), width, height, ptr(flow)),
                  "homography_pixel_flow")
    return out(flow, as_torch)
