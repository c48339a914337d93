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
from .engine import device_of, engine, is_torch, out, ptr, to_dev, to_host
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
    return _collect(bufs, as_torch)


def _collect(bufs: PairBuffers, as_torch: bool, composite: bool = True) -> RegistrationOutput:
    """RegistrationOutput from a finished pair's buffers (one host sync to
    read the verdict; RegistrationError as pipeline.py:185-187)."""
    info = bufs.info.cpu().numpy()
    m, n = int(info[16]), int(info[17])
    if info[0] == _native.HDR_ERR_REGISTRATION:
        raise RegistrationError(f"only {m} reliable matches at full resolution")
    hom = bufs.homography if info[1] else None
    fields = {"composite": bufs.composite if composite else None, "flow": bufs.flow,
              "warped": bufs.warped, "valid": bufs.valid.bool(), "ssim": bufs.ssim.double(),
              "matches": bufs.matches[:m].clone(), "raw_matches": bufs.raw_matches[:n].clone(),
              "homography": None if hom is None else hom.clone()}
    if not as_torch:  # every D2H issued before the one synchronisation
        live = [k for k, v in fields.items() if v is not None]
        fields.update(zip(live, to_host(*(fields[k] for k in live))))
    return RegistrationOutput(level_counts=_level_counts(info), **fields)


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


# ---------------------------------------------------------------- file path
@dataclass
class PipelineConfig:
    """Mirror of PipelineConfig (pipeline.py:201-210)."""
    inputs: list = field(default_factory=list)
    exposures: list | None = None
    exposure_file: str | None = None
    output: str = "composite.png"
    dump_all: bool = False
    out_dir: str | None = None
    params: PipelineParams = field(default_factory=PipelineParams)


def _resolve_exposures(config: PipelineConfig):
    """pipeline.py:213-228."""
    from .fileio import load_exposures
    inputs = list(config.inputs)
    if config.exposure_file:
        entries = load_exposures(config.exposure_file)
        if inputs:
            table = dict(entries)
            try:
                return inputs, [table[p] for p in inputs]
            except KeyError as exc:
                raise ConfigError(f"no exposure for input {exc}") from exc
        return [p for p, _ in entries], [e for _, e in entries]
    if config.exposures is not None:
        if len(config.exposures) != len(inputs):
            raise ConfigError("need one exposure per input image")
        return inputs, list(config.exposures)
    return inputs, [1.0] * len(inputs)


def harmonize_raw(raws):
    """Bring raw PNG samples to one layout so both frames share one decode:
    grey -> RGB repeat (pipeline.as_rgb) and 8 -> 16 bit by x257, which is
    exact (v*257/65535 and v/255 are the same real number, so the f64
    quotients of fileio.load_png are identical)."""
    arrs = [a for a, _ in raws]
    bits = max(b for _, b in raws)
    out = []
    for a, b in zip(arrs, (b for _, b in raws)):
        if b != bits:
            a = a.astype(np.uint16) * np.uint16(257)
        out.append(a)
    if any(a.ndim == 3 for a in out):
        out = [np.repeat(a[:, :, None], 3, axis=2) if a.ndim == 2 else a for a in out]
    return [np.ascontiguousarray(a) for a in out], bits


def run_raw(ref_raw, src_raw, bits: int, params: PipelineParams, bufs: PairBuffers,
            composite_u8: torch.Tensor | None = None, graph: bool = False, stream=None):
    """Enqueue a pair from raw device samples (hdr_register_and_fuse_raw):
    decode both frames, register and fuse, and optionally quantise the
    composite for save_png -- asynchronous, no host sync."""
    h, w = ref_raw.shape[:2]
    channels = 1 if ref_raw.dim() == 2 else ref_raw.shape[2]
    e = engine(w, h, ref_raw.device.index)
    e.bind_stream(stream)
    p = params.to_native()
    _native.check(_native.lib().hdr_register_and_fuse_raw(
        e.handle, ctypes.byref(p), w, h, ptr(ref_raw), ptr(src_raw), channels, bits,
        1 if graph else 0, ctypes.byref(bufs.native), ptr(composite_u8)), "register_and_fuse_raw")
    return e


def run_hdr(config: PipelineConfig) -> RegistrationOutput:
    """pipeline.run_hdr (pipeline.py:267-282): load a pair of PNGs, pick the
    reference, register and fuse, write the 8-bit composite (and the debug
    dumps when asked). Only raw samples cross PCIe; scaling, the metering
    statistic, the pair and the 8-bit quantisation run on the GPU."""
    from . import fileio, metering
    config.params.validate()
    inputs, exposures = _resolve_exposures(config)
    if len(inputs) != 2:
        raise ConfigError("exactly 2 input images are required")
    raws, bits = harmonize_raw([fileio.read_png_raw(p) for p in inputs])
    dev = torch.cuda.current_device()
    raw_dev = [fileio.raw_to_device(a, bits, dev) for a in raws]
    images = _LazyFrames(raw_dev, bits)
    k = metering.choose_reference(images, exposures)
    ref_raw, src_raw = raw_dev[k], raw_dev[1 - k]
    if ref_raw.shape != src_raw.shape:
        raise ConfigError("reference and source dimensions differ")
    h, w = ref_raw.shape[:2]
    if min(h, w) < 100:
        raise ValueError("input below 100 pixels in one dimension")
    bufs = PairBuffers(w, h, dev)
    comp8 = torch.empty((h, w, 3), dtype=torch.uint8, device=f"cuda:{dev}")
    run_raw(ref_raw, src_raw, bits, config.params, bufs, comp8)
    result = _collect(bufs, False)
    fileio.write_png_u8(config.output, comp8.cpu().numpy())
    if config.dump_all:
        import os
        directory = config.out_dir or os.path.dirname(os.path.abspath(config.output))
        dump_intermediates(result, images.lum(k), images[k], directory)
    return result


def flow_to_pfm(flow) -> np.ndarray:
    """pipeline.py:253-258: (h, w, 2) flow -> 3-channel PFM data (zero third plane)."""
    f = flow.cpu().numpy() if isinstance(flow, torch.Tensor) else np.asarray(flow)
    h, w = f.shape[:2]
    data = np.zeros((h, w, 3), dtype=np.float32)
    data[:, :, :2] = f
    return data


def pfm_to_flow(data: np.ndarray) -> np.ndarray:
    """pipeline.py:261-264."""
    from .fileio import FileFormatError
    if data.ndim != 3 or data.shape[2] != 3:
        raise FileFormatError("flow PFM must have 3 channels")
    return np.ascontiguousarray(data[:, :, :2])


def dump_intermediates(result: RegistrationOutput, lum_ref, ref, directory: str) -> None:
    """pipeline.py:231-250: the stage dumps (match CSVs, flow / warped /
    valid / SSIM / weight maps as PFM, debug renders as PNG). The fusion
    weights are recomputed on the GPU (hdr_fusion_weights)."""
    import os
    from . import fileio, fusion, viz
    os.makedirs(directory, exist_ok=True)
    j = lambda name: os.path.join(directory, name)  # noqa: E731
    valid = np.asarray(result.valid)
    fileio.save_matches_csv(j("matches_raw.csv"), result.raw_matches)
    fileio.save_matches_csv(j("matches.csv"), result.matches)
    fileio.save_png(j("matches.png"), viz.overlay_matches(lum_ref, result.matches))
    fileio.save_pfm(j("flow.pfm"), flow_to_pfm(result.flow))
    fileio.save_png(j("flow.png"), viz.flow_to_color(result.flow))
    fileio.save_pfm(j("warped.pfm"), result.warped)
    fileio.save_png(j("warped.png"), result.warped)
    fileio.save_pfm(j("valid.pfm"), valid.astype(np.float32))
    fileio.save_pfm(j("ssim.pfm"), np.asarray(result.ssim).astype(np.float32))
    fileio.save_png(j("ssim.png"), viz.heatmap(result.ssim, -1.0, 1.0))
    w_ref, w_src = fusion.fusion_weights(ref, result.warped, result.ssim, valid.astype(np.float32))
    w_ref, w_src = viz._np(w_ref), viz._np(w_src)
    fileio.save_pfm(j("weight_ref.pfm"), w_ref.astype(np.float32))
    fileio.save_pfm(j("weight_src.pfm"), w_src.astype(np.float32))
    fileio.save_png(j("weight_ref.png"), viz.heatmap(w_ref, 0.0, 1.0))
    fileio.save_png(j("weight_src.png"), viz.heatmap(w_src, 0.0, 1.0))


class _LazyFrames:
    """Decoded frames for metering / dumps, materialised on first use."""

    def __init__(self, raw_dev, bits):
        self.raw, self.bits, self.cache = raw_dev, bits, {}

    def __len__(self):
        return len(self.raw)

    def __getitem__(self, i):
        if i not in self.cache:
            from .fileio import decode_rgb
            self.cache[i] = decode_rgb(self.raw[i], self.bits)
        return self.cache[i]

    def lum(self, i):
        from .image import luminance
        return luminance(self[i])


# ---------------------------------------------------------------- n-frame stacks
@dataclass
class StackOutput:
    """register_and_fuse_stack's result: the k-way composite, the index of
    the frame used as reference, and one RegistrationOutput per source frame
    (frame order, reference skipped; their `composite` is None)."""
    composite: np.ndarray
    reference_index: int
    registrations: list = field(default_factory=list)


def register_and_fuse_stack(frames, exposures=None, params: PipelineParams | None = None,
                            reference_index: int | None = None) -> StackOutput:
    """n-frame stack (n = 2..4): the reference is
    metering.choose_reference's pick (darkest exposure; ties -> lower mean
    luminance) unless given, every other frame is registered to it like
    register_and_fuse, and all frames are blended with the reference's
    fusion generalised to n weights. One device pass, one host sync."""
    from . import metering
    params = params or PipelineParams()
    params.validate()
    n = len(frames)
    if not 2 <= n <= 4:
        raise ValueError("stacks take 2..4 frames")
    as_torch = is_torch(*frames)
    dev = device_of(*frames)
    ts = [as_rgb(to_dev(x, torch.float32, dev)) for x in frames]
    if any(t.shape != ts[0].shape for t in ts):
        raise ConfigError("reference and source dimensions differ")
    if ts[0].dim() != 3 or ts[0].shape[2] != 3:
        raise ValueError("luminance expects an (h, w, 3) image")
    h, w = ts[0].shape[:2]
    if min(h, w) < 100:
        raise ValueError("input below 100 pixels in one dimension")
    exposures = [1.0] * n if exposures is None else list(exposures)
    k = metering.choose_reference(ts, exposures) if reference_index is None else int(reference_index)
    order = [k] + [f for f in range(n) if f != k]
    bufs = [PairBuffers(w, h, dev) for _ in range(n - 1)]
    comp = torch.empty((h, w, 3), dtype=torch.float32, device=f"cuda:{dev}")
    e = engine(w, h, dev)
    p = params.to_native()
    fr = (ctypes.c_void_p * n)(*[ts[f].data_ptr() for f in order])
    outs = (ctypes.c_void_p * (n - 1))(*[ctypes.addressof(b.native) for b in bufs])
    _native.check(_native.lib().hdr_register_and_fuse_stack(e.handle, ctypes.byref(p), n, w, h, fr,
                                                            outs, ptr(comp)), "register_and_fuse_stack")
    regs = []
    for b in bufs:
        # raises RegistrationError like the pairwise reference call would
        regs.append(_collect(b, as_torch, composite=False))
    return StackOutput(composite=out(comp, as_torch), reference_index=k, registrations=regs)


def fuse_stack(frames, ssims, valids, levels: int | None = None):
    """The k-way blend alone (hdr_fuse_stack): frames[0] = reference,
    frames[f] = warped source f with ssims[f-1] / valids[f-1]."""
    n = len(frames)
    if not 2 <= n <= 4 or len(ssims) != n - 1 or len(valids) != n - 1:
        raise ValueError("fuse_stack takes 2..4 frames and n-1 ssim/valid maps")
    as_torch = is_torch(*frames, *ssims, *valids)
    dev = device_of(*frames, *ssims, *valids)
    ts = [to_dev(x, torch.float32, dev) for x in frames]
    ss = [to_dev(x, torch.float32, dev) for x in ssims]
    vs = [to_dev(np.asarray(v) != 0 if not isinstance(v, torch.Tensor) else v != 0, torch.uint8, dev)
          for v in valids]
    h, w = ts[0].shape[:2]
    res = torch.empty((h, w, 3), dtype=torch.float32, device=ts[0].device)
    e = engine(w, h, dev)
    arr = lambda xs: (ctypes.c_void_p * max(len(xs), 1))(*[x.data_ptr() for x in xs])  # noqa: E731
    _native.check(_native.lib().hdr_fuse_stack(e.handle, n, arr(ts), arr(ss), arr(vs), w, h,
                                               0 if levels is None else int(levels), ptr(res)),
                  "fuse_stack")
    return out(res, as_torch)
