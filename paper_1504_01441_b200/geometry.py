"""Drop-in for `hdrflow.geometry` (geometry.py:22-135) on the GPU.

`fit_homography` runs the block-wide DLT of K8 (pivoted Householder for
four points, Gram + Jacobi for least squares) with the reference's
DegenerateFit rules; `inlier_mask`, `symmetric_transfer_error` and
`homography_pixel_flow` are K7's transfer test and the fallback flow of K11;
`apply_homography` maps points on the device.
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
    """geometry.py:80-93 — projective map of (..., 2) points on the GPU;
    ValueError if any point lands at infinity."""
    as_torch = is_torch(h, pts)
    dev = device_of(h, pts)
    hm = to_dev(h, torch.float64, dev)
    p = to_dev(pts, torch.float64, dev)
    shape = tuple(p.shape)
    p2 = p.reshape(-1, 2)
    res = torch.empty_like(p2)
    e = engine(1, 1, dev)
    _native.check(_native.lib().hdr_apply_homography(e.handle, ptr(hm), ptr(p2), p2.shape[0], ptr(res)),
                  "apply_homography")
    return out(res.reshape(shape), as_torch)


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
    """geometry.py:107-115 — per-pair hypot(fwd, bwd) on the GPU, h_inv by
    LU with partial pivoting as np.linalg.inv (LinAlgError if singular)."""
    as_torch = is_torch(h, ref_pts, src_pts)
    dev = device_of(h, ref_pts, src_pts)
    hm = to_dev(h, torch.float64, dev)
    r = to_dev(ref_pts, torch.float64, dev).reshape(-1, 2)
    s = to_dev(src_pts, torch.float64, dev).reshape(-1, 2)
    if r.shape[0] != s.shape[0]:
        raise ValueError("ref_pts and src_pts hold different numbers of points")
    res = torch.empty(r.shape[0], dtype=torch.float64, device=r.device)
    e = engine(1, 1, dev)
    _native.check(_native.lib().hdr_symmetric_transfer_error(e.handle, ptr(hm), ptr(r), ptr(s),
                                                             r.shape[0], ptr(res)),
                  "symmetric_transfer_error")
    return out(res, as_torch)


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
