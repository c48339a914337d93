"""One pair split across GPUs by row bands.

`register_and_fuse_banded` returns what `pipeline.register_and_fuse`
(pipeline.py:174-198) returns, computed by the ranks of a torch.distributed
group (one process per GPU, NCCL over NVLink; any backend works, gloo stages
through the host):

* registration (match_stack: luminance, histogram matching, pyramids,
  corners, SSD, weeding, fits -- a chain of small dependent kernels) runs
  on every rank; it is deterministic, so every rank holds the same matches
  and homography without a collective;
* the domain-transform filter (densify.py:78-113) is split by row bands of
  whole column chunks: each rank sweeps its rows and aggregates its column
  chunks; the chunk aggregates (chunk-major, so a band's are one block) are
  all-gathered, and each rank links them and re-runs its own chunks -- the carries of the column
  recursion crossing the bands (densify.py:69-75). The last pass writes the
  band's f32 flow (densify_flow, densify.py:134-142);
* the flow is all-gathered (every rank needs the rows above and below its
  band for the SSIM window), each rank warps its band plus a 5-row halo
  (densify.py:145-174) and histograms its own rows of the warped luminance;
  the 256-bin histograms are all-reduced for make_ssim's histogram match
  (image.py:96-106), and each rank computes the SSIM of its band
  (fusion.py:34-64);
* warped, validity and SSIM are all-gathered and the merge
  (fusion.py:135-157) runs on every rank (its coarse pyramid levels are
  global and latency-bound; splitting level 0 would cost an all-reduce of the
  8-channel level-1 pyramid, ~40 MB at 5MP, about the level-0 work saved).

Bands are equal runs of whole hdr_band_rows_multiple()-row blocks (the last
may be short). Every step is the
single-GPU pair's own kernel on the same data (the column sweep takes the
chunk agg/link/apply form), so the result equals
`register_and_fuse` run with the options dt_cluster_columns = 0 and
dt_sparse_first = 0 bit for bit, and the reference within the usual bars
(tests/test_gpu_banded.py).
"""

from __future__ import annotations

import ctypes

import torch
import torch.distributed as dist

from . import _native
from .engine import device_of, engine, is_torch, out, ptr, to_dev
from .errors import RegistrationError
from .pipeline import PairBuffers, PipelineParams, RegistrationOutput, _level_counts, as_rgb

SSIM_HALO = 5  # rows of the 11-tap SSIM window beyond a band (window // 2)


def band_size(h: int, world: int, multiple: int | None = None) -> int:
    """Rows of every band but possibly the last (a whole number of
    `multiple`-row blocks): equal bands let the band outputs move by
    all-gather."""
    m = multiple or int(_native.lib().hdr_band_rows_multiple())
    nb = (h + m - 1) // m
    return (nb + world - 1) // world * m


def band_rows(h: int, world: int, rank: int, multiple: int | None = None) -> tuple[int, int]:
    """Rows [y0, y1) of `rank`'s band (the last band may be short or empty)."""
    b = band_size(h, world, multiple)
    return min(h, rank * b), min(h, (rank + 1) * b)


def _group_info(group):
    if not dist.is_initialized():
        return 0, 1, None
    return dist.get_rank(group), dist.get_world_size(group), dist.get_backend(group)


def _allreduce_sum(t: torch.Tensor, group, backend) -> None:
    if backend is None:
        return
    if backend == "nccl" or not t.is_cuda:
        dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)
        return
    h = t.cpu()  # host-staged collective for gloo with device tensors
    dist.all_reduce(h, op=dist.ReduceOp.SUM, group=group)
    t.copy_(h)


def _gather_blocks(t: torch.Tensor, rank: int, n: int, group, backend) -> None:
    """Every rank's block [rank * n, (rank + 1) * n) of the flat t into every
    rank's t (NCCL all-gather in place; other backends sum zero-padded copies
    through the host)."""
    if backend is None:
        return
    if backend == "nccl":
        dist.all_gather_into_tensor(t, t[rank * n:(rank + 1) * n].clone(), group=group)
        return
    t[:rank * n].zero_()
    t[(rank + 1) * n:].zero_()
    _allreduce_sum(t, group, backend)


def _gather_rows(t: torch.Tensor, rank: int, band: int, group, backend) -> None:
    """Every rank's band rows of t (rows padded to world * band) into every
    rank's t: NCCL all-gather in place; other backends sum zero-padded
    copies through the host."""
    if backend is None:
        return
    if backend == "nccl":
        dist.all_gather_into_tensor(t, t[rank * band:(rank + 1) * band].clone(), group=group)
        return
    t[:rank * band].zero_()
    t[(rank + 1) * band:].zero_()
    _allreduce_sum(t, group, backend)


def register_and_fuse_banded(ref, src, params: PipelineParams | None = None, group=None) -> RegistrationOutput:
    """pipeline.register_and_fuse over the ranks of `group` (module docstring);
    every rank gets the full RegistrationOutput."""
    params = params or PipelineParams()
    params.validate()
    lib = _native.lib()
    rank, world, backend = _group_info(group)
    as_torch = is_torch(ref, src)
    dev = device_of(ref, src)
    ref_t = as_rgb(to_dev(ref, torch.float32, dev))
    src_t = as_rgb(to_dev(src, torch.float32, dev))
    if ref_t.shape != src_t.shape:
        from .errors import ConfigError
        raise ConfigError("reference and source dimensions differ")
    h, w = ref_t.shape[:2]
    if min(h, w) < 100:
        raise ValueError("input below 100 pixels in one dimension")
    e = engine(w, h, dev)
    bufs = PairBuffers(w, h, dev)
    p = params.to_native()
    # registration, replicated
    _native.check(lib.hdr_match_stack(e.handle, ctypes.byref(p), w, h, ptr(ref_t), ptr(src_t),
                                      ptr(bufs.matches), ptr(bufs.raw_matches), ptr(bufs.homography),
                                      ptr(bufs.info)), "match_stack")
    info = bufs.info.cpu().numpy()
    m, n = int(info[16]), int(info[17])
    if info[0] == _native.HDR_ERR_REGISTRATION:
        raise RegistrationError(f"only {m} reliable matches at full resolution")
    kw = dict(device=ref_t.device)
    lum_ref = torch.empty((h, w), dtype=torch.float32, **kw)
    _native.check(lib.hdr_luminance(e.handle, ptr(ref_t), h * w, ptr(lum_ref)), "luminance")
    planes = torch.empty((3, h, w), dtype=torch.float64, **kw)
    _native.check(lib.hdr_sparse_maps(e.handle, ptr(bufs.matches), m, w, h, ptr(planes[0]), ptr(planes[1]),
                                      ptr(planes[2])), "build_sparse_maps")
    band = band_size(h, world)
    y0, y1 = band_rows(h, world, rank)
    hp = band * world  # rows of the gathered (padded) outputs
    # densify_flow: rows and column chunks of the band, aggregates gathered
    # chunk aggregates, chunk-major: a band's chunks are one block, padded to
    # `world` equal blocks so they move by all-gather
    per_band = int(lib.hdr_band_agg_doubles(w, band, 3))  # a band is whole chunks
    agg = torch.zeros(max(int(lib.hdr_band_agg_doubles(w, h, 3)), world * per_band), dtype=torch.float64, **kw)
    flow_p = torch.zeros((hp, w, 2), dtype=torch.float32, **kw)
    flow = flow_p[:h]
    has_fb = ctypes.c_void_p(bufs.info.data_ptr() + 4)  # info[1]: the homography exists

    def band_dt(op, i, a=None, fb=None, hf=None, floor=0.0, fl=None):
        _native.check(lib.hdr_band_dt(e.handle, op, ptr(lum_ref), ptr(planes), 3, w, h, y0, y1,
                                      float(params.sigma_s), float(params.sigma_r), int(params.passes), i,
                                      a, fb, hf, floor, fl), "banded dt_filter")

    for i in range(1, params.passes + 1):
        band_dt(0, i)                                    # the band's row sweeps
        band_dt(1, i, ptr(agg))                          # its column-chunk aggregates
        _gather_blocks(agg, rank, per_band, group, backend)  # the carries' inputs from every band
        last = i == params.passes
        band_dt(2, i, ptr(agg), ptr(bufs.homography), has_fb, float(params.normalization_floor),
                ptr(flow) if last else None)             # link + the band's chunks (flow on the last pass)
    _gather_rows(flow_p, rank, band, group, backend)
    # warp_image of the band + halo, histogram of the band's own rows
    warped_p = torch.empty((hp, w, 3), dtype=torch.float32, **kw)
    valid_p = torch.empty((hp, w), dtype=torch.uint8, **kw)
    ssim_p = torch.empty((hp, w), dtype=torch.float32, **kw)
    warped, valid, ssim = warped_p[:h], valid_p[:h], ssim_p[:h]
    qw = torch.empty((h, w), dtype=torch.uint8, **kw)
    hist = torch.zeros(256, dtype=torch.int32, **kw)
    ha, hb = max(0, y0 - SSIM_HALO), min(h, y1 + SSIM_HALO)
    for a, b, hp in ((y0, y1, ptr(hist)), (ha, y0, None), (y1, hb, None)):
        _native.check(lib.hdr_band_warp(e.handle, ptr(flow), w, h, a, b, ptr(src_t), ptr(warped), ptr(valid),
                                        ptr(qw), hp), "band warp")
    _allreduce_sum(hist, group, backend)
    _native.check(lib.hdr_band_ssim(e.handle, ptr(lum_ref), ptr(qw), ptr(hist), w, h, y0, y1,
                                    int(params.ssim_window), float(params.ssim_sigma), ptr(ssim)), "band ssim")
    for t in (warped_p, valid_p, ssim_p):
        _gather_rows(t, rank, band, group, backend)
    # merge, replicated
    _native.check(lib.hdr_fuse(e.handle, ptr(ref_t), ptr(warped), ptr(ssim), ptr(valid), w, h, 0,
                               ptr(bufs.composite)), "fuse")
    hom = bufs.homography if info[1] else None
    return RegistrationOutput(
        composite=out(bufs.composite, as_torch), flow=out(flow, as_torch), warped=out(warped, as_torch),
        valid=out(valid.bool(), as_torch), ssim=out(ssim.double(), as_torch),
        matches=out(bufs.matches[:m].clone(), as_torch), raw_matches=out(bufs.raw_matches[:n].clone(), as_torch),
        homography=None if hom is None else out(hom.clone(), as_torch), level_counts=_level_counts(info))
