"""Drop-in for `hdrflow.matcher` (matcher.py:64-263) on the GPU.

`detect_corners`, `ssd_match` (batched), `_match_level` and
`fit_matches_homography` each call one C-ABI twin. `pyramidal_match` over
caller-supplied pyramids drives those twins level by level from the host;
the fused, host-sync-free chain is `pipeline.match_stack` /
`pipeline.register_and_fuse`.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _native
from .engine import device_of, engine, engine_for_rows, is_torch, out, ptr, to_dev
from .errors import DegenerateFit
from .weeding import (DEFAULT_COARSE_ITERATIONS, DEFAULT_ITERATIONS, WeedParams,
                      weed_parallel)

DEFAULT_TILE = 64
DEFAULT_THRESHOLD = 4.0 / 255.0
DEFAULT_QUADRANT_HALF = 8
DEFAULT_RADIUS = 10
DEFAULT_PATCH = 21
DEFAULT_EPS_PX = 2.0


def level_seed(seed: int, level: int) -> int:
    """matcher.py:146-149 (SeedSequence in libhdrb200's host code)."""
    return int(_native.lib().hdr_level_seed(int(seed), int(level)))


@dataclass
class MatcherParams:
    """matcher.py:152-170."""
    tile: int = DEFAULT_TILE
    threshold: float = DEFAULT_THRESHOLD
    quadrant_half: int = DEFAULT_QUADRANT_HALF
    radius: int = DEFAULT_RADIUS
    patch: int = DEFAULT_PATCH
    iterations: int = DEFAULT_ITERATIONS
    coarse_iterations: int = DEFAULT_COARSE_ITERATIONS
    delta: int | None = None
    eps_px: float = DEFAULT_EPS_PX
    seed: int = 0
    workers: int = 1

    def weed_params(self, level: int, width: int) -> WeedParams:
        iterations = self.iterations if level == 0 else self.coarse_iterations
        return WeedParams(iterations=iterations, delta=self.delta,
                          eps=2.0 * self.eps_px / width, seed=level_seed(self.seed, level))


@dataclass
class MatchResult:
    """matcher.py:173-178."""
    matches: np.ndarray
    raw_matches: np.ndarray
    homography: np.ndarray | None
    level_counts: list = field(default_factory=list)


def cornerness(table, x: int, y: int, half: int = DEFAULT_QUADRANT_HALF):
    """matcher.py:51-61 — (cornerness, min contiguous-quadrant contrast) at
    (x, y) of an integral image (image.integral's table)."""
    h1, w1 = table.shape
    if not (half <= x <= w1 - 1 - half and half <= y <= h1 - 1 - half):
        raise ValueError("quadrant neighborhood out of bounds")
    t = to_dev(table, torch.float64, device_of(table))
    xy = torch.tensor([[int(x), int(y)]], dtype=torch.int32).to(t.device)
    res = torch.empty((1, 2), dtype=torch.float64, device=t.device)
    e = engine(w1 - 1, h1 - 1, t.device.index)
    _native.check(_native.lib().hdr_cornerness(e.handle, ptr(t), w1 - 1, h1 - 1, ptr(xy), 1, half,
                                               ptr(res)), "cornerness")
    r = res.cpu().numpy()[0]
    return float(r[0]), float(r[1])


def detect_corners(lum, tile: int = DEFAULT_TILE, threshold: float = DEFAULT_THRESHOLD,
                   half: int = DEFAULT_QUADRANT_HALF):
    """matcher.py:64-105 — (n, 3) rows (x, y, score), tile order (K4 + K5)."""
    if tile < 16:
        raise ValueError("tile must be >= 16")
    as_torch = is_torch(lum)
    t = to_dev(lum, torch.float32, device_of(lum))
    h, w = t.shape
    nt = -(-w // tile) * -(-h // tile)
    corners = torch.empty((max(nt, 1), 3), dtype=torch.float64, device=t.device)
    count = ctypes.c_int32(0)
    e = engine(w, h, t.device.index)
    _native.check(_native.lib().hdr_detect_corners(e.handle, ptr(t), w, h, tile, float(threshold),
                                                   half, ptr(corners), ctypes.byref(count)),
                  "detect_corners")
    return out(corners[:count.value].clone(), as_torch)


def ssd_match_batch(ref, src, pts, radius: int = DEFAULT_RADIUS, patch: int = DEFAULT_PATCH):
    """Batched matcher.ssd_match: pts (n, 4) = (x_ref, y_ref, x_init, y_init).

    Returns (out (n, 3) float64, found (n) bool)."""
    dev = device_of(ref, src)
    r = to_dev(ref, torch.float32, dev)
    s = to_dev(src, torch.float32, dev)
    if r.shape != s.shape:
        raise ValueError("reference and source must have the same shape")
    p = to_dev(np.asarray(pts, dtype=np.int32).reshape(-1, 4), torch.int32, dev)
    n = p.shape[0]
    h, w = r.shape
    res = torch.zeros((max(n, 1), 3), dtype=torch.float64, device=r.device)
    found = torch.zeros((max(n, 1),), dtype=torch.uint8, device=r.device)
    e = engine(w, h, dev)
    _native.check(_native.lib().hdr_ssd_match(e.handle, ptr(r), ptr(s), w, h, ptr(p), n, radius,
                                              patch, ptr(res), ptr(found)), "ssd_match")
    f = found[:n].cpu().numpy()
    if np.any(f == 2):
        raise ValueError("reference patch out of bounds")
    return res[:n].cpu().numpy(), f.astype(bool)


def ssd_match(ref, src, p_ref, p_init, radius: int = DEFAULT_RADIUS, patch: int = DEFAULT_PATCH):
    """matcher.py:108-143 — (x_src, y_src, score) or None."""
    res, found = ssd_match_batch(ref, src, [[int(p_ref[0]), int(p_ref[1]), int(p_init[0]),
                                             int(p_init[1])]], radius, patch)
    if not found[0]:
        return None
    return int(res[0, 0]), int(res[0, 1]), float(res[0, 2])


def _native_params(params: MatcherParams) -> _native.HdrParams:
    from .pipeline import PipelineParams
    return PipelineParams(tile=params.tile, threshold=params.threshold,
                          quadrant_half=params.quadrant_half, radius=params.radius,
                          patch=params.patch, iterations=params.iterations,
                          coarse_iterations=params.coarse_iterations, delta=params.delta,
                          eps_px=params.eps_px, seed=params.seed,
                          workers=params.workers).to_native()


def _match_level(lum_ref, lum_src, h_pred, params: MatcherParams):
    """matcher.py:181-210 — detect, predict through h_pred, SSD (K4-K6)."""
    as_torch = is_torch(lum_ref, lum_src)
    dev = device_of(lum_ref, lum_src)
    r = to_dev(lum_ref, torch.float32, dev)
    s = to_dev(lum_src, torch.float32, dev)
    hp = to_dev(np.asarray(h_pred, dtype=np.float64) if not isinstance(h_pred, torch.Tensor)
                else h_pred, torch.float64, dev)
    h, w = r.shape
    nt = -(-w // params.tile) * -(-h // params.tile)
    raw = torch.empty((max(nt, 1), 5), dtype=torch.float64, device=r.device)
    count = ctypes.c_int32(0)
    e = engine(w, h, dev)
    p = _native_params(params)
    _native.check(_native.lib().hdr_match_level(e.handle, ctypes.byref(p), ptr(r), ptr(s), w, h,
                                                ptr(hp), ptr(raw), ctypes.byref(count)),
                  "match_level")
    return out(raw[:count.value].clone(), as_torch)


match_level = _match_level


def fit_matches_homography(matches, width: int, height: int):
    """matcher.py:213-218 — least-squares H in normalized coordinates (K8)."""
    as_torch = is_torch(matches)
    dev = device_of(matches)
    m = to_dev(matches, torch.float64, dev).reshape(-1, 5)
    n = m.shape[0]
    if n < 4:
        raise ValueError("need at least 4 point pairs")
    hm = torch.empty((3, 3), dtype=torch.float64, device=m.device)
    e = engine_for_rows(n, dev)
    _native.check(_native.lib().hdr_fit_matches_homography(e.handle, ptr(m), n, width, height,
                                                           ptr(hm)), "fit_matches_homography")
    return out(hm, as_torch)


def pyramidal_match(ref_pyr, src_pyr, params: MatcherParams | None = None) -> MatchResult:
    """matcher.py:221-263 over caller pyramids, one GPU twin per stage."""
    params = params or MatcherParams()
    if len(ref_pyr) != len(src_pyr):
        raise ValueError("pyramids must have equal level counts")
    for a, b in zip(ref_pyr, src_pyr):
        if a.shape != b.shape:
            raise ValueError("pyramid levels must have matching dimensions")
    h_pred = np.eye(3)
    homography = None
    counts = [(0, 0)] * len(ref_pyr)
    raw = weeded = np.zeros((0, 5), dtype=np.float64)
    for level in range(len(ref_pyr) - 1, -1, -1):
        lr, ls = ref_pyr[level], src_pyr[level]
        h, w = lr.shape
        raw = _match_level(lr, ls, h_pred, params)
        if isinstance(raw, torch.Tensor):
            raw = raw.cpu().numpy()
        if len(raw) >= 4:
            res = weed_parallel(raw, (w, h), params.weed_params(level, w), params.workers)
            weeded = raw[res.kept]
        else:
            weeded = np.zeros((0, 5), dtype=np.float64)
        counts[level] = (len(raw), len(weeded))
        if len(weeded) >= 4:
            try:
                h_pred = fit_matches_homography(weeded, w, h)
                if level == 0:
                    homography = h_pred
            except DegenerateFit:
                pass
    return MatchResult(matches=weeded, raw_matches=raw, homography=homography,
                       level_counts=counts)
