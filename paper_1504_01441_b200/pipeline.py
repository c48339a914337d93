"""Drop-in for `hdrflow.pipeline` (pipeline.py:35-198): the same entry points,
dataclasses, defaults and exceptions, executed by libhdrb200.so on the GPU.

`register_and_fuse` enqueues the whole pair as one device-resident chain
(no host round trip between the five pyramid levels) and synchronises once
to read the registration verdict. Inputs may be numpy arrays (results come
back as numpy, like the reference) or CUDA tensors (results stay on the
device as tensors).
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _native
from .engine import device_of, engine, is_torch, out, ptr, to_dev
from .errors import ConfigError, RegistrationError

PYRAMID_MAX_LEVELS = 5


@dataclass
class PipelineParams:
    """Mirror of PipelineParams (pipeline.py:35-57); same defaults."""
    tile: int = 64
    threshold: float = 4.0 / 255.0
    quadrant_half: int = 8
    radius: int = 10
    patch: int = 21
    max_levels: int = PYRAMID_MAX_LEVELS
    iterations: int = 256
    coarse_iterations: int = 64
    delta: int | None = None
    eps_px: float = 2.0
    sigma_s: float = 400.0
    sigma_r: float = 0.2
    passes: int = 3
    ssim_window: int = 11
    ssim_sigma: float = 1.5
    normalization_floor: float = 1e-4
    seed: int = 0
    workers: int = 1

    def validate(self):
        """pipeline.py:59-87 — ConfigError with the reference's messages."""
        checks = [
            (self.tile >= 16, "tile must be >= 16"),
            (self.threshold > 0, "threshold must be positive"),
            (self.quadrant_half >= 2, "quadrant_half must be >= 2"),
            (self.radius >= 1, "radius must be >= 1"),
            (self.patch >= 3 and self.patch % 2 == 1, "patch must be odd and >= 3"),
            (1 <= self.max_levels <= PYRAMID_MAX_LEVELS,
             f"max_levels must be in [1, {PYRAMID_MAX_LEVELS}]"),
            (self.iterations >= 1, "iterations must be >= 1"),
            (self.coarse_iterations >= 1, "coarse_iterations must be >= 1"),
            (self.delta is None or self.delta >= 4, "delta must be >= 4"),
            (self.eps_px > 0, "eps_px must be positive"),
            (self.sigma_s > 0, "sigma_s must be positive"),
            (self.sigma_r > 0, "sigma_r must be positive"),
            (self.passes >= 1, "passes must be >= 1"),
            (self.ssim_window >= 3 and self.ssim_window % 2 == 1,
             "ssim_window must be odd and >= 3"),
            (self.ssim_sigma > 0, "ssim_sigma must be positive"),
            (self.normalization_floor > 0, "normalization_floor must be positive"),
            (self.workers >= 1, "workers must be >= 1"),
            (self.workers >= 1 and self.iterations % self.workers == 0,
             "iterations must be divisible by workers"),
            (self.workers >= 1 and self.coarse_iterations % self.workers == 0,
             "coarse_iterations must be divisible by workers"),
        ]
        for ok, message in checks:
            if not ok:
                raise ConfigError(message)

    def matcher_params(self):
        from .matcher import MatcherParams
        return MatcherParams(tile=self.tile, threshold=self.threshold,
                             quadrant_half=self.quadrant_half, radius=self.radius,
                             patch=self.patch, iterations=self.iterations,
                             coarse_iterations=self.coarse_iterations, delta=self.delta,
                             eps_px=self.eps_px, seed=self.seed, workers=self.workers)

    def to_native(self) -> _native.HdrParams:
        p = _native.HdrParams()
        for name, _ in _native.HdrParams._fields_:
            if name == "_pad":
                continue
            val = getattr(self, name)
            if name == "delta":
                val = -1 if val is None else int(val)
            if name == "seed":
                if int(val) < 0 or int(val) >= 2 ** 64:
                    raise ValueError("seed must be in [0, 2**64)")
            setattr(p, name, val)
        return p


@dataclass
class RegistrationOutput:
    """Mirror of RegistrationOutput (pipeline.py:99-109): same fields/dtypes."""
    composite: np.ndarray
    flow: np.ndarray
    warped: np.ndarray
    valid: np.ndarray
    ssim: np.ndarray
    matches: np.ndarray
    raw_matches: np.ndarray
    homography: np.ndarray | None
    level_counts: list = field(default_factory=list)


def as_rgb(img):
    """pipeline.py:112-115 (numpy or tensor)."""
    if isinstance(img, torch.Tensor):
        return img.unsqueeze(-1).expand(*img.shape, 3).contiguous() if img.dim() == 2 else img
    return np.repeat(img[:, :, None], 3, axis=2) if img.ndim == 2 else img


class PairBuffers:
    """Caller-owned device outputs of one pair (hdr_outputs)."""

    def __init__(self, width: int, height: int, device: int, tile: int = 16):
        kw = dict(device=f"cuda:{device}")
        n = _native.lib().hdr_max_matches(width, height, tile)
        self.width, self.height, self.max_matches = width, height, n
        self.composite = torch.empty((height, width, 3), dtype=torch.float32, **kw)
        self.flow = torch.empty((height, width, 2), dtype=torch.float32, **kw)
        self.warped = torch.empty((height, width, 3), dtype=torch.float32, **kw)
        self.valid = torch.empty((height, width), dtype=torch.uint8, **kw)
        self.ssim = torch.empty((height, width), dtype=torch.float32, **kw)
        self.matches = torch.empty((n, 5), dtype=torch.float64, **kw)
        self.raw_matches = torch.empty((n, 5), dtype=torch.float64, **kw)
        self.homography = torch.empty((3, 3), dtype=torch.float64, **kw)
        self.info = torch.zeros((_native.INFO_WORDS,), dtype=torch.int32, **kw)
        self.native = _native.HdrOutputs(*(t.data_ptr() for t in (
            self.composite, self.flow, self.warped, self.valid, self.ssim, self.matches,
            self.raw_matches, self.homography, self.info)))


def enqueue_pair(ref: torch.Tensor, src: torch.Tensor, params: PipelineParams,
                 bufs: PairBuffers, graph: bool = False, stream=None):
    """Asynchronously run the whole pair on the current (or given) stream."""
    h, w = ref.shape[:2]
    e = engine(w, h, ref.device.index)
    e.bind_stream(stream)
    fn = (_native.lib().hdr_register_and_fuse_graph if graph
          else _native.lib().hdr_register_and_fuse)
    p = params.to_native()
    _native.check(fn(e.handle, ctypes.byref(p), w, h, ptr(ref), ptr(src),
                     ctypes.byref(bufs.native)), "register_and_fuse")
    return e


def _level_counts(info: np.ndarray):
    levels = int(info[2])
    return [(int(info[3 + 2 * l]), int(info[4 + 2 * l])) for l in range(levels)]


def register_and_fuse(ref, src, params: PipelineParams | None = None) -> RegistrationOutput:
    """Full in-memory pipeline for a (reference, source) pair (pipeline.py:174-198)."""
    params = params or PipelineParams()
    params.validate()
    as_torch = is_torch(ref, src)
    dev = device_of(ref, src)
    ref_t = as_rgb(to_dev(ref, torch.float32, dev))
    src_t = as_rgb(to_dev(src, torch.float32, dev))
    if ref_t.shape != src_t.shape:
        raise ConfigError("reference and source dimensions differ")
    if ref_t.dim() != 3 or ref_t.shape[2] != 3:
        raise ValueError("luminance expects an (h, w, 3) image")
    h, w = ref_t.shape[:2]
    if min(h, w) < 100:
        raise ValueError("input below 100 pixels in one dimension")
    bufs = PairBuffers(w, h, dev)
    enqueue_pair(ref_t, src_t, params, bufs)
    info = bufs.info.cpu().numpy()  # the one host sync of the pair
    m, n = int(info[16]), int(info[17])
    if info[0] == _native.HDR_ERR_REGISTRATION:
        raise RegistrationError(f"only {m} reliable matches at full resolution")
    hom = bufs.homography if info[1] else None
    return RegistrationOutput(
        composite=out(bufs.composite, as_torch),
        flow=out(bufs.flow, as_torch),
        warped=out(bufs.warped, as_torch),
        valid=out(bufs.valid.bool(), as_torch),
        ssim=out(bufs.ssim.double(), as_torch),
        matches=out(bufs.matches[:m].clone(), as_torch),
        raw_matches=out(bufs.raw_matches[:n].clone(), as_torch),
        homography=None if hom is None else out(hom.clone(), as_torch),
        level_counts=_level_counts(info))


def match_stack(ref, src, params: PipelineParams):
    """pipeline.py:122-130 — equalise, pyramids, coarse-to-fine matching."""
    from .matcher import MatchResult
    as_torch = is_torch(ref, src)
    dev = device_of(ref, src)
    ref_t = as_rgb(to_dev(ref, torch.float32, dev))
    src_t = as_rgb(to_dev(src, torch.float32, dev))
    h, w = ref_t.shape[:2]
    if min(h, w) < 100:
        raise ValueError("input below 100 pixels in one dimension")
    bufs = PairBuffers(w, h, dev)
    e = engine(w, h, dev)
    p = params.to_native()
    _native.check(_native.lib().hdr_match_stack(
        e.handle, ctypes.byref(p), w, h, ptr(ref_t), ptr(src_t), ptr(bufs.matches),
        ptr(bufs.raw_matches), ptr(bufs.homography), ptr(bufs.info)), "match_stack")
    info = bufs.info.cpu().numpy()
    m, n = int(info[16]), int(info[17])
    return MatchResult(matches=out(bufs.matches[:m].clone(), as_torch),
                       raw_matches=out(bufs.raw_matches[:n].clone(), as_torch),
                       homography=out(bufs.homography.clone(), as_torch) if info[1] else None,
                       level_counts=_level_counts(info))


def equalize_source(lum_ref, lum_src):
    """pipeline.py:118-119."""
    from .image import match_histogram
    return match_histogram(lum_src, lum_ref)


def weed_finest(raw_matches, size, params: PipelineParams):
    """pipeline.py:133-140."""
    from .weeding import weed_parallel
    if len(raw_matches) < 4:
        return np.zeros((0, 5), dtype=np.float64)
    wp = params.matcher_params().weed_params(0, size[0])
    result = weed_parallel(raw_matches, size, wp, params.workers)
    return raw_matches[result.kept]


def fit_fallback(matches, width: int, height: int):
    """pipeline.py:143-150 (with the matcher's least-squares fit)."""
    from .errors import DegenerateFit
    from .matcher import fit_matches_homography
    if len(matches) < 4:
        return None
    try:
        return fit_matches_homography(matches, width, height)
    except DegenerateFit:
        return None


def make_flow(matches, lum_ref, params: PipelineParams):
    """pipeline.py:153-162."""
    from . import densify
    h, w = lum_ref.shape[:2]
    maps = densify.build_sparse_maps(matches, w, h)
    fallback = fit_fallback(matches, w, h)
    return densify.densify_flow(lum_ref, maps, fallback, sigma_s=params.sigma_s,
                                sigma_r=params.sigma_r, passes=params.passes,
                                floor=params.normalization_floor)


def make_ssim(lum_ref, warped, params: PipelineParams):
    """pipeline.py:165-171 — SSIM of lum_ref vs equalised luminance(warped)."""
    as_torch = is_torch(lum_ref, warped)
    dev = device_of(lum_ref, warped)
    a = to_dev(lum_ref, torch.float32, dev)
    wrp = as_rgb(to_dev(warped, torch.float32, dev))
    h, w = a.shape
    res = torch.empty((h, w), dtype=torch.float32, device=a.device)
    e = engine(w, h, dev)
    _native.check(_native.lib().hdr_make_ssim(e.handle, ptr(a), ptr(wrp), w, h,
                                              params.ssim_window, params.ssim_sigma, ptr(res)),
                  "make_ssim")
    return out(res.double(), as_torch)
