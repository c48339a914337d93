"""CPU ORACLE — TEST INFRASTRUCTURE ONLY.

This module is the checker for the GPU path, never part of it: only
`tests/`, `__graft_entry__.smoke()` and `bench.py`'s `cpu_baseline` /
`--impl reference` legs may import it. The product package
(`paper_1504_01441_b200`) must not import anything under `oracle/`.

What it is: a numpy restatement of the reference `hdrflow` register+merge
path (`/root/reference/pkg/src/hdrflow/*.py`), function by function, with
the reference's dtypes and operation order so that, on the same host, it
reproduces the reference bit for bit (numpy ufuncs, `einsum`, `cumsum`,
`np.linalg` (OpenBLAS LAPACK), `np.random.Philox`, `scipy.ndimage`).

Parity pinning: `oracle/gen_golden.py` runs the REAL reference (importable
in the build container only) on seeded synthetic scenes and writes
`tests/golden/*.npz`; `tests/test_oracle_golden.py` checks this oracle
against those fixtures (bit-exact for integer/index outputs and the f32
raster stages, tight tolerances elsewhere). On the GPU box, where the
reference does not exist, the GPU parity tests compare against this oracle.

One deliberate difference from the shipped reference: `pipeline.fit_fallback`
calls `fit_matches_homography`, which `pipeline.py` never imports
(`pipeline.py:148` vs `pipeline.py:18-24`), so the shipped
`register_and_fuse` raises NameError whenever registration succeeds. The
oracle calls the matcher's least-squares fit there, i.e. the behaviour of
the reference with the one-line import shim.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np
from numpy.lib.stride_tricks import sliding_window_view
from scipy import ndimage

# ---------------------------------------------------------------- constants
LUMA = (0.299, 0.587, 0.114)                 # image.py:12
PYR_LEVELS, PYR_MIN = 5, 100                 # image.py:13-14
NBINS = 256                                  # image.py:15
ITERS, COARSE_ITERS, MAX_RESAMPLE = 256, 64, 10   # weeding.py:25-27
RANK_RTOL, MIN_DET = 1e-9, 1e-12             # geometry.py:14-15
SSIM_C1, SSIM_C2 = 0.01 ** 2, 0.03 ** 2      # fusion.py:20-21
EXPOSED_SIGMA, W_FLOOR = 0.2, 1e-12          # fusion.py:22-23
PYR5 = np.array([1.0, 4.0, 6.0, 4.0, 1.0]) / 16.0   # fusion.py:25


class DegenerateFit(ValueError):
    pass


class RegistrationError(RuntimeError):
    pass


class ConfigError(ValueError):
    pass


@dataclass
class Params:
    """Mirror of `PipelineParams` (pipeline.py:35-57)."""
    tile: int = 64
    threshold: float = 4.0 / 255.0
    quadrant_half: int = 8
    radius: int = 10
    patch: int = 21
    max_levels: int = PYR_LEVELS
    iterations: int = ITERS
    coarse_iterations: int = COARSE_ITERS
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


# ------------------------------------------------------------ raster (image.py)
def luminance(rgb):
    """image.py:23-29 — f32, (wr*R + wg*G) + wb*B, each op rounded, clipped."""
    if rgb.ndim != 3 or rgb.shape[2] != 3:
        raise ValueError("luminance expects an (h, w, 3) image")
    y = LUMA[0] * rgb[..., 0] + LUMA[1] * rgb[..., 1] + LUMA[2] * rgb[..., 2]
    return np.clip(y, 0.0, 1.0).astype(np.float32)


def integral(img):
    """image.py:32-44 — f64 SAT, cumsum down columns then along rows."""
    h, w = img.shape
    sat = np.zeros((h + 1, w + 1), dtype=np.float64)
    np.cumsum(img, axis=0, dtype=np.float64, out=sat[1:, 1:])
    np.cumsum(sat[1:, 1:], axis=1, out=sat[1:, 1:])
    return sat


def box_sum(sat, x0, y0, x1, y1):
    """image.py:47-58 (bounds already valid) — ((t11-t01)-t10)+t00."""
    return sat[y1, x1] - sat[y0, x1] - sat[y1, x0] + sat[y0, x0]


def halve(img):
    """image.py:61-68 — 2x2 box mean in f32, odd row/column dropped."""
    h, w = img.shape[:2]
    if h < 2 or w < 2:
        raise ValueError("image too small to downsample")
    v = img[: h - h % 2, : w - w % 2]
    return ((v[0::2, 0::2] + v[0::2, 1::2] + v[1::2, 0::2] + v[1::2, 1::2])
            * np.float32(0.25)).astype(np.float32)


def pyramid(img, max_levels=PYR_LEVELS, min_dim=PYR_MIN):
    """image.py:71-88."""
    if min(img.shape[:2]) < min_dim:
        raise ValueError(f"input below {min_dim} pixels in one dimension")
    out = [img]
    while len(out) < max_levels and min(out[-1].shape[0] // 2, out[-1].shape[1] // 2) >= min_dim:
        out.append(halve(out[-1]))
    return out


def quantize(img):
    """image.py:91-93 — floor(x*255 + .5) in f32, clipped, u8."""
    return np.clip(np.floor(img * 255.0 + 0.5), 0, 255).astype(np.uint8)


def histogram_lut(q_src, q_ref):
    """image.py:96-106, the transfer table only (f32 on the k/255 grid)."""
    cdf_s = np.cumsum(np.bincount(q_src.ravel(), minlength=NBINS)) / q_src.size
    cdf_r = np.cumsum(np.bincount(q_ref.ravel(), minlength=NBINS)) / q_ref.size
    idx = np.searchsorted(cdf_r, cdf_s, side="left")
    return np.minimum(idx, NBINS - 1).astype(np.float32) / np.float32(255.0)


def match_histogram(src, ref):
    """image.py:109-122 for single-channel data."""
    qs = quantize(src)
    return histogram_lut(qs, quantize(ref))[qs]


def to_norm(x, y, w, h):
    """image.py:125-129."""
    return ((2.0 * np.asarray(x, dtype=np.float64) - w) / float(w),
            (2.0 * np.asarray(y, dtype=np.float64) - h) / float(w))


def from_norm(xn, yn, w, h):
    """image.py:132-136."""
    return ((np.asarray(xn, dtype=np.float64) * float(w) + w) / 2.0,
            (np.asarray(yn, dtype=np.float64) * float(w) + h) / 2.0)


# ---------------------------------------------------------- corners (matcher.py)
def _quadrants(sat, xs, ys, half):
    """matcher.py:37-47 — cyclic |tr-tl|,|br-tr|,|bl-br|,|tl-bl|; sum, min."""
    a = float(half * half)
    tl = box_sum(sat, xs - half, ys - half, xs, ys) / a
    tr = box_sum(sat, xs, ys - half, xs + half, ys) / a
    br = box_sum(sat, xs, ys, xs + half, ys + half) / a
    bl = box_sum(sat, xs - half, ys, xs, ys + half) / a
    d = np.stack([np.abs(tr - tl), np.abs(br - tr), np.abs(bl - br), np.abs(tl - bl)])
    return d.sum(axis=0), d.min(axis=0)


def candidate_axis(n, tile):
    """matcher.py:75-81 — per-tile offsets spacing//2, +spacing, ... clipped."""
    step = max(1, tile // 16)
    offs = np.arange(step // 2, tile, step)
    return np.concatenate([t0 + offs[offs < min(tile, n - t0)] for t0 in range(0, n, tile)])


def detect_corners(lum, tile=64, threshold=4.0 / 255.0, half=8):
    """matcher.py:64-105 — best admissible candidate per tile, tile order."""
    if tile < 16:
        raise ValueError("tile must be >= 16")
    h, w = lum.shape
    gx, gy = np.meshgrid(candidate_axis(w, tile), candidate_axis(h, tile))
    gx, gy = gx.ravel(), gy.ravel()
    inside = (gx >= half) & (gx <= w - half) & (gy >= half) & (gy <= h - half)
    gx, gy = gx[inside], gy[inside]
    if gx.size == 0:
        return np.zeros((0, 3))
    score, low = _quadrants(integral(lum), gx, gy, half)
    keep = low > threshold
    gx, gy, score = gx[keep], gy[keep], score[keep]
    if gx.size == 0:
        return np.zeros((0, 3))
    tid = (gy // tile) * (-(-w // tile)) + gx // tile
    order = np.lexsort((np.arange(gx.size), -score, tid))
    ts = tid[order]
    heads = order[np.flatnonzero(np.r_[True, ts[1:] != ts[:-1]])]
    return np.column_stack([gx[heads], gy[heads], score[heads]]).astype(np.float64)


def ssd_search(ref, src, p_ref, p_init, radius=10, patch=21):
    """matcher.py:108-143 — exhaustive f64 SSD; ties: d2, then y, then x."""
    hp = patch // 2
    xr, yr = int(p_ref[0]), int(p_ref[1])
    xi, yi = int(p_init[0]), int(p_init[1])
    hs, ws = src.shape
    if not (hp <= xr <= ref.shape[1] - 1 - hp and hp <= yr <= ref.shape[0] - 1 - hp):
        raise ValueError("reference patch out of bounds")
    x0, x1 = max(xi - radius, hp), min(xi + radius, ws - 1 - hp)
    y0, y1 = max(yi - radius, hp), min(yi + radius, hs - 1 - hp)
    if x0 > x1 or y0 > y1:
        return None
    tpl = ref[yr - hp:yr + hp + 1, xr - hp:xr + hp + 1].astype(np.float64)
    win = sliding_window_view(src[y0 - hp:y1 + hp + 1, x0 - hp:x1 + hp + 1]
                              .astype(np.float64), (patch, patch))
    diff = win - tpl
    ssd = np.einsum("ijkl,ijkl->ij", diff, diff)
    tied = np.flatnonzero(ssd.ravel() == ssd.min())
    ty, tx = np.unravel_index(tied, ssd.shape)
    cx, cy = tx + x0, ty + y0
    best = tied[np.lexsort((cx, cy, (cx - xi) ** 2 + (cy - yi) ** 2))[0]]
    by, bx = np.unravel_index(best, ssd.shape)
    return bx + x0, by + y0, float(ssd[by, bx])


def level_seed(seed, level):
    """matcher.py:146-149."""
    return int(np.random.SeedSequence(entropy=seed, spawn_key=(level,)).generate_state(1)[0])


def match_level(lum_ref, lum_src, h_pred, p: Params, corners=None):
    """matcher.py:181-210 — predict through h_pred, SSD-search each corner."""
    h, w = lum_ref.shape
    hp = p.patch // 2
    if corners is None:
        corners = detect_corners(lum_ref, p.tile, p.threshold, p.quadrant_half)
    rows = []
    for cx, cy, _ in corners:
        x, y = int(cx), int(cy)
        if not (hp <= x <= w - 1 - hp and hp <= y <= h - 1 - hp):
            continue
        xn, yn = to_norm(x, y, w, h)
        den = h_pred[2, 0] * xn + h_pred[2, 1] * yn + h_pred[2, 2]
        if abs(den) < 1e-12:
            continue
        mx = (h_pred[0, 0] * xn + h_pred[0, 1] * yn + h_pred[0, 2]) / den
        my = (h_pred[1, 0] * xn + h_pred[1, 1] * yn + h_pred[1, 2]) / den
        px, py = from_norm(mx, my, w, h)
        if not (np.isfinite(px) and np.isfinite(py)):
            continue
        if abs(px) > 8 * w or abs(py) > 8 * h:
            continue
        hit = ssd_search(lum_ref, lum_src, (x, y), (int(round(px)), int(round(py))),
                         p.radius, p.patch)
        if hit is not None:
            rows.append((float(x), float(y), float(hit[0]), float(hit[1]), hit[2]))
    return np.asarray(rows, dtype=np.float64) if rows else np.zeros((0, 5))


# --------------------------------------------------------- geometry.py
def _hartley(pts):
    """geometry.py:22-32."""
    c = pts.mean(axis=0)
    d = pts - c
    md = np.mean(np.hypot(d[:, 0], d[:, 1]))
    if md < 1e-12:
        raise DegenerateFit("coincident points")
    s = np.sqrt(2.0) / md
    return np.array([[s, 0.0, -s * c[0]], [0.0, s, -s * c[1]], [0.0, 0.0, 1.0]]), d * s


def dlt_matrix(p, q):
    """geometry.py:51-63 — two rows per correspondence, conditioned coords."""
    n = len(p)
    a = np.zeros((2 * n, 9))
    a[0::2, 0], a[0::2, 1], a[0::2, 2] = -p[:, 0], -p[:, 1], -1.0
    a[0::2, 6], a[0::2, 7], a[0::2, 8] = p[:, 0] * q[:, 0], p[:, 1] * q[:, 0], q[:, 0]
    a[1::2, 3], a[1::2, 4], a[1::2, 5] = -p[:, 0], -p[:, 1], -1.0
    a[1::2, 6], a[1::2, 7], a[1::2, 8] = p[:, 0] * q[:, 1], p[:, 1] * q[:, 1], q[:, 1]
    return a


def fit_homography(ref_pts, src_pts):
    """geometry.py:35-77 — Hartley DLT via SVD; DegenerateFit rules A.5."""
    ref_pts = np.asarray(ref_pts, dtype=np.float64).reshape(-1, 2)
    src_pts = np.asarray(src_pts, dtype=np.float64).reshape(-1, 2)
    if len(ref_pts) < 4 or len(src_pts) != len(ref_pts):
        raise ValueError("need at least 4 point pairs")
    t_r, p = _hartley(ref_pts)
    t_s, q = _hartley(src_pts)
    _, sv, vt = np.linalg.svd(dlt_matrix(p, q))
    if sv[-2] <= RANK_RTOL * sv[0]:
        raise DegenerateFit("rank-deficient correspondence set")
    hm = np.linalg.inv(t_s) @ vt[-1].reshape(3, 3) @ t_r
    if abs(hm[2, 2]) < 1e-12:
        raise DegenerateFit("homography maps the origin to infinity")
    hm = hm / hm[2, 2]
    if abs(np.linalg.det(hm)) <= MIN_DET:
        raise DegenerateFit("singular homography")
    return hm


def _transfer(hm, pts, tgt):
    """geometry.py:96-104."""
    x, y = pts[:, 0], pts[:, 1]
    den = hm[2, 0] * x + hm[2, 1] * y + hm[2, 2]
    out = np.full(len(pts), np.inf)
    ok = np.abs(den) >= 1e-12
    mx = (hm[0, 0] * x + hm[0, 1] * y + hm[0, 2])[ok] / den[ok]
    my = (hm[1, 0] * x + hm[1, 1] * y + hm[1, 2])[ok] / den[ok]
    out[ok] = np.hypot(mx - tgt[ok, 0], my - tgt[ok, 1])
    return out


def apply_homography(hm, pts):
    """geometry.py:80-93 — projective map of (..., 2) points."""
    pts = np.asarray(pts, dtype=np.float64)
    x, y = pts[..., 0], pts[..., 1]
    den = hm[2, 0] * x + hm[2, 1] * y + hm[2, 2]
    if np.any(np.abs(den) < 1e-12):
        raise ValueError("point maps to infinity")
    out = np.empty_like(pts)
    out[..., 0] = (hm[0, 0] * x + hm[0, 1] * y + hm[0, 2]) / den
    out[..., 1] = (hm[1, 0] * x + hm[1, 1] * y + hm[1, 2]) / den
    return out


def symmetric_transfer_error(hm, ref_pts, src_pts):
    """geometry.py:107-115 — hypot(fwd, bwd) per pair."""
    ref_pts = np.asarray(ref_pts, dtype=np.float64).reshape(-1, 2)
    src_pts = np.asarray(src_pts, dtype=np.float64).reshape(-1, 2)
    return np.hypot(_transfer(hm, ref_pts, src_pts),
                    _transfer(np.linalg.inv(hm), src_pts, ref_pts))


def inlier_mask(hm, ref_pts, src_pts, eps):
    """geometry.py:107-121 — hypot(fwd, bwd) < eps."""
    ref_pts = np.asarray(ref_pts, dtype=np.float64).reshape(-1, 2)
    src_pts = np.asarray(src_pts, dtype=np.float64).reshape(-1, 2)
    err = np.hypot(_transfer(hm, ref_pts, src_pts),
                   _transfer(np.linalg.inv(hm), src_pts, ref_pts))
    return err < eps


def homography_flow(hm, w, h):
    """geometry.py:124-135 — dense pixel flow of a normalized-coords H, f32."""
    ys, xs = np.mgrid[0:h, 0:w]
    xn, yn = to_norm(xs, ys, w, h)
    den = hm[2, 0] * xn + hm[2, 1] * yn + hm[2, 2]
    bad = np.abs(den) < 1e-12
    safe = np.where(bad, 1.0, den)
    px, py = from_norm((hm[0, 0] * xn + hm[0, 1] * yn + hm[0, 2]) / safe,
                       (hm[1, 0] * xn + hm[1, 1] * yn + hm[1, 2]) / safe, w, h)
    f = np.stack([px - xs, py - ys], axis=-1)
    f[bad] = 0.0
    return f.astype(np.float32)


def fit_matches_homography(m, w, h):
    """matcher.py:213-218."""
    m = np.asarray(m, dtype=np.float64)
    rx, ry = to_norm(m[:, 0], m[:, 1], w, h)
    sx, sy = to_norm(m[:, 2], m[:, 3], w, h)
    return fit_homography(np.column_stack([rx, ry]), np.column_stack([sx, sy]))


# ---------------------------------------------------------- weeding.py
def default_delta(n):
    """weeding.py:30-32."""
    return max(12, math.ceil(0.15 * n))


def weed(matches, w, h, iterations, eps, seed, delta=None):
    """weeding.py:62-111 — union of inlier sets larger than delta.

    Returns (kept sorted indices, witness i64). Each iteration owns
    Generator(Philox(SeedSequence(seed, spawn_key=(it,)))) and resamples at
    most 10 times on DegenerateFit.
    """
    n = len(matches)
    if n < 4:
        raise ValueError("need at least 4 matches to weed")
    m = np.asarray(matches, dtype=np.float64)
    rx, ry = to_norm(m[:, 0], m[:, 1], w, h)
    sx, sy = to_norm(m[:, 2], m[:, 3], w, h)
    rp, sp = np.column_stack([rx, ry]), np.column_stack([sx, sy])
    d = default_delta(n) if delta is None else delta
    keep = np.zeros(n, dtype=bool)
    wit = np.zeros(n, dtype=np.int64)
    for it in range(iterations):
        gen = np.random.Generator(np.random.Philox(
            np.random.SeedSequence(entropy=seed, spawn_key=(it,))))
        hm = None
        for _ in range(MAX_RESAMPLE):
            pick = gen.choice(n, size=4, replace=False)
            try:
                hm = fit_homography(rp[pick], sp[pick])
                break
            except DegenerateFit:
                continue
        if hm is None:
            continue
        inl = inlier_mask(hm, rp, sp, eps)
        cnt = int(inl.sum())
        if cnt > d:
            keep |= inl
            np.maximum(wit, np.where(inl, cnt, 0), out=wit)
    return np.flatnonzero(keep), wit


def level_weed_args(p: Params, level, width):
    """matcher.py:166-170 — (iterations, eps, seed) for one level."""
    iters = p.iterations if level == 0 else p.coarse_iterations
    return iters, 2.0 * p.eps_px / width, level_seed(p.seed, level)


@dataclass
class LevelTrace:
    corners: np.ndarray
    raw: np.ndarray
    kept: np.ndarray
    h_pred_in: np.ndarray
    h_fit: np.ndarray | None


def pyramidal_match(ref_pyr, src_pyr, p: Params, trace=None):
    """matcher.py:221-263 — coarse-to-fine; carries H when a level fails."""
    h_pred = np.eye(3)
    hom = None
    counts = [(0, 0)] * len(ref_pyr)
    raw = weeded = np.zeros((0, 5))
    for lev in range(len(ref_pyr) - 1, -1, -1):
        lr, ls = ref_pyr[lev], src_pyr[lev]
        h, w = lr.shape
        corners = detect_corners(lr, p.tile, p.threshold, p.quadrant_half)
        h_in = h_pred.copy()
        raw = match_level(lr, ls, h_pred, p, corners)
        kept = np.zeros(0, dtype=np.int64)
        if len(raw) >= 4:
            iters, eps, sd = level_weed_args(p, lev, w)
            kept, _ = weed(raw, w, h, iters, eps, sd, p.delta)
        weeded = raw[kept] if len(raw) >= 4 else np.zeros((0, 5))
        counts[lev] = (len(raw), len(weeded))
        fit = None
        if len(weeded) >= 4:
            try:
                fit = fit_matches_homography(weeded, w, h)
                h_pred = fit
                if lev == 0:
                    hom = fit
            except DegenerateFit:
                pass
        if trace is not None:
            trace[lev] = LevelTrace(corners, raw, kept, h_in, fit)
    return weeded, raw, hom, counts


# ---------------------------------------------------------- densify.py
def sparse_maps(matches, w, h):
    """densify.py:38-56 — splat flow + indicator; collisions keep min (score, i)."""
    pu, pv, nn = np.zeros((h, w)), np.zeros((h, w)), np.zeros((h, w))
    best = {}
    m = np.asarray(matches, dtype=np.float64).reshape(-1, 5)
    for i, row in enumerate(m):
        x, y = int(round(row[0])), int(round(row[1]))
        if not (0 <= x < w and 0 <= y < h):
            raise ValueError(f"match reference position ({row[0]}, {row[1]}) out of bounds")
        if (x, y) not in best or (row[4], i) < best[(x, y)]:
            best[(x, y)] = (row[4], i)
    for (x, y), (_, i) in best.items():
        pu[y, x] = m[i, 2] - m[i, 0]
        pv[y, x] = m[i, 3] - m[i, 1]
        nn[y, x] = 1.0
    return pu, pv, nn


def _scan(buf, a):
    """densify.py:69-75 — in-place fwd then bwd one-pole recursion on axis 0."""
    for i in range(1, buf.shape[0]):
        buf[i] += a[i - 1] * (buf[i - 1] - buf[i])
    for i in range(buf.shape[0] - 2, -1, -1):
        buf[i] += a[i] * (buf[i + 1] - buf[i])


def dt_filter(guide, data, sigma_s=400.0, sigma_r=0.2, passes=3):
    """densify.py:78-113 — domain-transform recursive filter, f64."""
    flat = data.ndim == 2
    out = np.asarray(data, dtype=np.float64).copy()
    if flat:
        out = out[:, :, None]
    h, w, _ = out.shape
    g = np.asarray(guide, dtype=np.float64)
    if g.ndim == 2:
        g = g[:, :, None]
    r = sigma_s / sigma_r
    dx = 1.0 + r * np.abs(np.diff(g, axis=1)).sum(axis=2)
    dy = 1.0 + r * np.abs(np.diff(g, axis=0)).sum(axis=2)
    den = np.sqrt(4.0 ** passes - 1.0)
    for i in range(1, passes + 1):
        sig = sigma_s * np.sqrt(3.0) * 2.0 ** (passes - i) / den
        ax = np.exp(-np.sqrt(2.0) / sig * dx)
        ay = np.exp(-np.sqrt(2.0) / sig * dy)
        if w > 1:
            cols = np.ascontiguousarray(out.transpose(1, 0, 2))
            _scan(cols, np.ascontiguousarray(ax.T)[:, :, None])
            out = np.ascontiguousarray(cols.transpose(1, 0, 2))
        if h > 1:
            _scan(out, ay[:, :, None])
    return out[:, :, 0] if flat else out


def densify_flow(guide, maps, fallback, sigma_s=400.0, sigma_r=0.2, passes=3,
                 floor=1e-4, return_smooth=False):
    """densify.py:116-142 — ratio of filtered maps, H-flow below the floor."""
    pu, pv, nn = maps
    h, w = nn.shape
    sm = dt_filter(guide, np.stack([pu, pv, nn], axis=-1), sigma_s, sigma_r, passes)
    wgt = sm[:, :, 2]
    ok = wgt > floor
    if fallback is not None:
        flow = homography_flow(fallback, w, h).astype(np.float64)
    else:
        flow = np.zeros((h, w, 2))
    np.divide(sm[:, :, 0], wgt, out=flow[:, :, 0], where=ok)
    np.divide(sm[:, :, 1], wgt, out=flow[:, :, 1], where=ok)
    flow = flow.astype(np.float32)
    return (flow, sm) if return_smooth else flow


def warp_image(src, flow):
    """densify.py:145-174 — bilinear backward warp in f64, validity mask."""
    h, w = src.shape[:2]
    sx = np.arange(w, dtype=np.float64)[None, :] + flow[:, :, 0].astype(np.float64)
    sy = np.arange(h, dtype=np.float64)[:, None] + flow[:, :, 1].astype(np.float64)
    valid = (sx >= 0) & (sx <= w - 1) & (sy >= 0) & (sy <= h - 1)
    cx, cy = np.clip(sx, 0, w - 1), np.clip(sy, 0, h - 1)
    x0, y0 = np.floor(cx).astype(np.intp), np.floor(cy).astype(np.intp)
    x1, y1 = np.minimum(x0 + 1, w - 1), np.minimum(y0 + 1, h - 1)
    fx, fy = cx - x0, cy - y0
    if src.ndim == 3:
        fx, fy = fx[:, :, None], fy[:, :, None]
    top = src[y0, x0] * (1.0 - fx) + src[y0, x1] * fx
    bot = src[y1, x0] * (1.0 - fx) + src[y1, x1] * fx
    return (top * (1.0 - fy) + bot * fy).astype(np.float32), valid


# ---------------------------------------------------------- fusion.py
def gauss_taps(sigma, radius):
    """fusion.py:28-31."""
    x = np.arange(-radius, radius + 1, dtype=np.float64)
    k = np.exp(-0.5 * (x / sigma) ** 2)
    return k / k.sum()


def ssim_map(a, b, window=11, sigma=1.5):
    """fusion.py:34-64 — five separable reflect blurs, clipped to [-1, 1]."""
    k = gauss_taps(sigma, window // 2)

    def blur(x):
        return ndimage.convolve1d(ndimage.convolve1d(x, k, axis=0, mode="reflect"),
                                  k, axis=1, mode="reflect")

    af, bf = a.astype(np.float64), b.astype(np.float64)
    ma, mb = blur(af), blur(bf)
    va = blur(af * af) - ma * ma
    vb = blur(bf * bf) - mb * mb
    cv = blur(af * bf) - ma * mb
    s = ((2.0 * ma * mb + SSIM_C1) * (2.0 * cv + SSIM_C2)) / \
        ((ma * ma + mb * mb + SSIM_C1) * (va + vb + SSIM_C2))
    return np.clip(s, -1.0, 1.0)


def quality_weights(img):
    """fusion.py:67-77 — |laplace(lum)| * std(rgb) * well-exposedness + 1e-12."""
    f = img.astype(np.float64)
    con = np.abs(ndimage.laplace(luminance(img).astype(np.float64), mode="reflect"))
    sat = f.std(axis=2)
    ex = np.exp(-((f - 0.5) ** 2).sum(axis=2) / (2.0 * EXPOSED_SIGMA ** 2))
    return con * sat * ex + W_FLOOR


def _blur5(x):
    return ndimage.convolve1d(ndimage.convolve1d(x, PYR5, axis=0, mode="reflect"),
                              PYR5, axis=1, mode="reflect")


def pyr_down(x):
    """fusion.py:85-86."""
    return _blur5(x)[::2, ::2]


def pyr_up(x, shape):
    """fusion.py:89-93 — zero-insert then 2x-gain blur."""
    z = np.zeros(shape[:2] + x.shape[2:], dtype=x.dtype)
    z[::2, ::2] = x
    return ndimage.convolve1d(ndimage.convolve1d(z, 2.0 * PYR5, axis=0, mode="reflect"),
                              2.0 * PYR5, axis=1, mode="reflect")


def gaussian_pyramid(x, levels):
    """fusion.py:96-100."""
    g = [np.asarray(x, dtype=np.float64)]
    while len(g) < levels and min(g[-1].shape[:2]) >= 2:
        g.append(pyr_down(g[-1]))
    return g


def laplacian_pyramid(x, levels):
    """fusion.py:103-107."""
    g = gaussian_pyramid(x, levels)
    return [g[i] - pyr_up(g[i + 1], g[i].shape) for i in range(len(g) - 1)] + [g[-1]]


def collapse(laps):
    """fusion.py:110-114."""
    out = laps[-1]
    for lap in laps[-2::-1]:
        out = lap + pyr_up(out, lap.shape)
    return out


def fusion_weights(ref, warped, ssim, valid):
    """fusion.py:117-128."""
    wr = quality_weights(ref)
    ws = quality_weights(warped) * np.clip(ssim, 0.0, 1.0) * np.asarray(valid, dtype=np.float64)
    tot = wr + ws
    return wr / tot, ws / tot


def fusion_levels(h, w):
    """fusion.py:131-132."""
    return max(1, int(np.floor(np.log2(min(h, w)))) - 1)


def fuse(ref, warped, ssim, valid, levels=None):
    """fusion.py:135-157."""
    h, w = ref.shape[:2]
    if levels is None:
        levels = fusion_levels(h, w)
    wr, ws = fusion_weights(ref, warped, ssim, valid)
    lr, ls = laplacian_pyramid(ref, levels), laplacian_pyramid(warped, levels)
    gr, gs = gaussian_pyramid(wr, levels), gaussian_pyramid(ws, levels)
    out = collapse([a[:, :, None] * x + b[:, :, None] * y
                    for a, b, x, y in zip(gr, gs, lr, ls)])
    return np.clip(out, 0.0, 1.0).astype(np.float32)


# ---------------------------------------------------------- pipeline.py
def as_rgb(img):
    """pipeline.py:112-115."""
    return np.repeat(img[:, :, None], 3, axis=2) if img.ndim == 2 else img


def make_ssim(lum_ref, warped, p: Params):
    """pipeline.py:165-171."""
    eq = match_histogram(luminance(as_rgb(warped)), lum_ref)
    return ssim_map(lum_ref, eq, p.ssim_window, p.ssim_sigma)


@dataclass
class OracleOutput:
    composite: np.ndarray
    flow: np.ndarray
    warped: np.ndarray
    valid: np.ndarray
    ssim: np.ndarray
    matches: np.ndarray
    raw_matches: np.ndarray
    homography: np.ndarray | None
    level_counts: list = field(default_factory=list)
    stages: dict = field(default_factory=dict)


def register_and_fuse(ref, src, p: Params | None = None, keep_stages=False):
    """pipeline.py:174-198 (with the fit_matches_homography shim)."""
    p = p or Params()
    ref = as_rgb(np.asarray(ref, dtype=np.float32))
    src = as_rgb(np.asarray(src, dtype=np.float32))
    if ref.shape != src.shape:
        raise ConfigError("reference and source dimensions differ")
    st = {}
    lum_ref = luminance(ref)
    lum_src = luminance(src)
    eq_src = match_histogram(lum_src, lum_ref)
    rp = pyramid(lum_ref, p.max_levels)
    sp = pyramid(eq_src, p.max_levels)
    trace = {}
    weeded, raw, hom, counts = pyramidal_match(rp, sp, p, trace)
    if keep_stages:
        st.update(lum_ref=lum_ref, lum_src=lum_src, eq_src=eq_src, ref_pyr=rp,
                  src_pyr=sp, trace=trace)
    if len(weeded) < 4:
        raise RegistrationError(f"only {len(weeded)} reliable matches at full resolution")
    h, w = lum_ref.shape
    maps = sparse_maps(weeded, w, h)
    fb = None
    if len(weeded) >= 4:
        try:
            fb = fit_matches_homography(weeded, w, h)
        except DegenerateFit:
            fb = None
    flow, smooth = densify_flow(lum_ref, maps, fb, p.sigma_s, p.sigma_r, p.passes,
                                p.normalization_floor, return_smooth=True)
    warped, valid = warp_image(src, flow)
    ssim = make_ssim(lum_ref, warped, p)
    comp = fuse(ref, warped, ssim, valid.astype(np.float32))
    if keep_stages:
        st.update(smooth=smooth, fallback=fb)
    return OracleOutput(comp, flow, warped, valid, ssim, weeded, raw, hom, counts, st)


# ---------------------------------------------------------- file path (fileio.py, metering.py, pipeline.run_hdr)
def load_png(path):
    """fileio.load_png (fileio.py:21-41): float32 in [0, 1], (h, w) or (h, w, 3)."""
    from PIL import Image
    with Image.open(path) as im:
        im.load()
        if im.mode in ("I", "I;16", "I;16B", "I;16L"):
            arr = np.asarray(im.convert("I"), dtype=np.float64) / 65535.0
        elif im.mode in ("L", "RGB"):
            arr = np.asarray(im, dtype=np.float64) / 255.0
        elif im.mode in ("LA", "RGBA", "P", "1"):
            conv = "L" if im.mode in ("LA", "1") else "RGB"
            arr = np.asarray(im.convert(conv), dtype=np.float64) / 255.0
        else:
            raise ValueError(f"unsupported PNG mode {im.mode!r}: {path}")
    return np.clip(arr, 0.0, 1.0).astype(np.float32)


def png_quantize(img):
    """fileio.save_png's sample values (fileio.py:46-47)."""
    return np.clip(np.floor(np.asarray(img, dtype=np.float64) * 255.0 + 0.5), 0, 255).astype(np.uint8)


def choose_reference(images, exposures):
    """metering.choose_reference (metering.py:37-51)."""
    exposures = [float(e) for e in exposures]
    shortest = min(exposures)
    cands = [i for i, e in enumerate(exposures) if e == shortest]
    if len(cands) == 1:
        return cands[0]

    def mean_lum(i):
        img = images[i]
        return float(np.mean(luminance(img) if img.ndim == 3 else img))
    return min(cands, key=lambda i: (mean_lum(i), i))


def run_hdr(inputs, exposures=None, p: Params | None = None):
    """pipeline.run_hdr (pipeline.py:267-282) without the file writes:
    returns (output, 8-bit composite as save_png would write it, ref index)."""
    if len(inputs) != 2:
        raise ConfigError("exactly 2 input images are required")
    exposures = [1.0, 1.0] if exposures is None else exposures
    images = [as_rgb(load_png(x)) for x in inputs]
    k = choose_reference(images, exposures)
    out = register_and_fuse(images[k], images[1 - k], p)
    return out, png_quantize(out.composite), k


# ---------------------------------------------------------- n-frame stacks
# Not reference code: the reference registers and fuses exactly two images
# (pipeline.py:271-272, fusion.py:135-157); the paper prescribes n-1 pairwise
# registrations against the reference. This composes the
# reference's own functions -- the pairwise register_and_fuse stages,
# quality_weights, laplacian/gaussian pyramids and collapse -- into the k-way
# blend (weights normalised over all frames). For n = 2 it is exactly fuse().
def fuse_stack(frames, ssims, valids, levels=None):
    """frames[0] = reference, frames[f] = warped source f (ssims/valids[f-1])."""
    h, w = frames[0].shape[:2]
    if levels is None:
        levels = fusion_levels(h, w)
    ws = [quality_weights(frames[0])]
    for f in range(1, len(frames)):
        ws.append(quality_weights(frames[f]) * np.clip(ssims[f - 1], 0.0, 1.0)
                  * np.asarray(valids[f - 1], dtype=np.float64))
    tot = ws[0]
    for x in ws[1:]:
        tot = tot + x
    ws = [x / tot for x in ws]
    laps = [laplacian_pyramid(x, levels) for x in frames]
    gps = [gaussian_pyramid(x, levels) for x in ws]
    blended = []
    for lev in range(len(laps[0])):
        acc = gps[0][lev][:, :, None] * laps[0][lev]
        for f in range(1, len(frames)):
            acc = acc + gps[f][lev][:, :, None] * laps[f][lev]
        blended.append(acc)
    return np.clip(collapse(blended), 0.0, 1.0).astype(np.float32)


def register_and_fuse_stack(frames, exposures=None, p: Params | None = None):
    """Pick the reference (metering.choose_reference), register every other
    frame to it as register_and_fuse does, blend all frames. Returns
    (composite, reference index, [OracleOutput per source, frame order])."""
    p = p or Params()
    frames = [as_rgb(np.asarray(x, dtype=np.float32)) for x in frames]
    exposures = [1.0] * len(frames) if exposures is None else exposures
    k = choose_reference(frames, exposures)
    ref = frames[k]
    regs, warped, ssims, valids = [], [ref], [], []
    for f, src in enumerate(frames):
        if f == k:
            continue
        r = register_and_fuse(ref, src, p)
        regs.append(r)
        warped.append(r.warped)
        ssims.append(r.ssim)
        valids.append(r.valid.astype(np.float32))
    return fuse_stack(warped, ssims, valids), k, regs


def select_offset(img, dark_level=0.05, cutoffs=(0.02, 0.10)):
    """metering.select_offset (metering.py:21-34)."""
    lum = luminance(img) if img.ndim == 3 else img
    q = float(np.mean(lum < dark_level))
    return 2 if q < cutoffs[0] else 3 if q < cutoffs[1] else 4


def plan_stack(images, exposures):
    """metering.plan_stack (metering.py:54-57): (offset_stops, reference_index)."""
    k = choose_reference(images, exposures)
    return select_offset(images[k]), k
