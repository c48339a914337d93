"""The reference SPEC's invariants (SPEC.md "Invariants & Properties" of the
image, matcher, geometry, weeding, densify and fusion sections), checked on
the GPU path with hypothesis-generated inputs. Property tests complement the
oracle parity tests: they hold for inputs no golden vector covers."""

import numpy as np
import pytest
from hypothesis import HealthCheck, given, settings
from hypothesis import strategies as st

from oracle import hdr_oracle as O
from paper_1504_01441_b200 import densify, fusion, geometry, image, matcher, pipeline, weeding

pytestmark = pytest.mark.gpu
SETTINGS = settings(max_examples=12, deadline=None, derandomize=True,
                    suppress_health_check=[HealthCheck.function_scoped_fixture])


def rng_image(seed, h, w, c=None, scale=1.0):
    r = np.random.default_rng(seed)
    shape = (h, w) if c is None else (h, w, c)
    return (r.random(shape) * scale).astype(np.float32)


@SETTINGS
@given(seed=st.integers(0, 10 ** 6), h=st.integers(1, 90), w=st.integers(1, 90),
       q=st.integers(0, 3))
def test_rect_sum_equals_direct_summation(cuda, seed, h, w, q):
    """SPEC image invariant: rect_sum = direct summation within 1e-9 relative."""
    img = rng_image(seed, h, w)
    t = image.integral(img)
    r = np.random.default_rng(seed + 1)
    for _ in range(4):
        y0, y1 = sorted(r.integers(0, h + 1, 2))
        x0, x1 = sorted(r.integers(0, w + 1, 2))
        direct = float(img[y0:y1, x0:x1].astype(np.float64).sum())
        got = float(image.rect_sum(t, x0, y0, x1, y1))
        assert abs(got - direct) <= 1e-9 * max(1.0, abs(direct))


@SETTINGS
@given(seed=st.integers(0, 10 ** 6), h=st.integers(4, 120), w=st.integers(4, 120))
def test_match_histogram_idempotent_to_one_bin(cuda, seed, h, w):
    src, ref = rng_image(seed, h, w), rng_image(seed + 7, h, w) ** 2
    once = image.match_histogram(src, ref)
    twice = image.match_histogram(once, ref)
    assert np.abs(twice - once).max() <= 1.0 / 255.0 + 1e-7


@SETTINGS
@given(seed=st.integers(0, 10 ** 6), c=st.sampled_from([0.125, 0.25, 0.5]),
       a=st.sampled_from([0.5, 2.0]))
def test_cornerness_shift_and_scale(cuda, seed, c, a):
    """SPEC matcher invariants: C(img + c) = C(img) and C(a img) = a C(img).
    On a 2^-10 lattice the shift and the power-of-two scale are exact in f32,
    so the quadrant differences -- and with them corners and scores -- carry
    over exactly (threshold scaled with a)."""
    img = (np.round(rng_image(seed, 200, 256, scale=0.4) * 1024) / 1024).astype(np.float32)
    base = matcher.detect_corners(img, threshold=4.0 / 255.0)
    shifted = matcher.detect_corners((img + np.float32(c)).astype(np.float32), threshold=4.0 / 255.0)
    np.testing.assert_array_equal(base, shifted)
    scaled = matcher.detect_corners((img * np.float32(a)).astype(np.float32),
                                    threshold=a * 4.0 / 255.0)
    np.testing.assert_array_equal(base[:, :2], scaled[:, :2])
    np.testing.assert_array_equal(scaled[:, 2], a * base[:, 2])


@SETTINGS
@given(seed=st.integers(0, 10 ** 6), n=st.integers(4, 200))
def test_inliers_monotone_in_eps(cuda, seed, n):
    r = np.random.default_rng(seed)
    ref = r.uniform(-1, 1, (n, 2))
    H = np.array([[1.01, 0.02, 0.01], [-0.01, 0.99, -0.02], [0.01, 0.0, 1.0]])
    src = O.apply_homography(H, ref) if hasattr(O, "apply_homography") else None
    if src is None:
        p = np.c_[ref, np.ones(n)] @ H.T
        src = p[:, :2] / p[:, 2:]
    src = src + r.normal(0, 0.01, src.shape)
    masks = [np.asarray(geometry.inlier_mask(H, ref, src, eps)) for eps in (0.005, 0.01, 0.02, 0.05)]
    for a, b in zip(masks, masks[1:]):
        assert not np.any(a & ~b)


@SETTINGS
@given(seed=st.integers(0, 10 ** 6), n=st.integers(8, 300), frac=st.floats(0.3, 1.0))
def test_weed_subset_and_delta_soundness(cuda, seed, n, frac):
    """SPEC weeding invariants: M is a subset of the matches and every kept
    match belongs to an inlier set larger than delta (its witness count)."""
    r = np.random.default_rng(seed)
    xr = r.uniform(20, 620, (n, 2))
    good = r.random(n) < frac
    xs = xr + np.array([3.0, -2.0])
    xs[~good] = r.uniform(20, 620, (int((~good).sum()), 2))
    m = np.c_[xr, xs, r.random(n)]
    p = weeding.WeedParams(iterations=64, seed=seed)
    res = weeding.weed(m, (640, 480), p)
    kept = np.asarray(res.kept)
    assert np.all((kept >= 0) & (kept < n)) and np.all(np.diff(kept) > 0)
    delta = weeding.default_delta(n)
    assert np.all(np.asarray(res.witness)[kept] > delta)
    o = O.weed(m, 640, 480, 64, p.eps, seed)
    assert np.array_equal(kept, o[0])


@SETTINGS
@given(seed=st.integers(0, 10 ** 6), h=st.integers(2, 150), w=st.integers(2, 150),
       v=st.floats(-5, 5))
def test_dt_filter_preserves_constants(cuda, seed, h, w, v):
    guide = rng_image(seed, h, w)
    out = densify.dt_filter(guide, np.full((h, w), v))
    assert np.abs(np.asarray(out) - v).max() <= 1e-5 * max(1.0, abs(v))


@SETTINGS
@given(seed=st.integers(0, 10 ** 6), m=st.integers(0, 30))
def test_densify_flow_finite_and_exact_on_common_flow(cuda, seed, m):
    """SPEC densify invariants: finite everywhere (also with no matches) and
    equal to the common flow at every corner pixel when all corners share one
    flow value."""
    h, w = 96, 128
    r = np.random.default_rng(seed)
    guide = rng_image(seed, h, w)
    xr = np.c_[r.integers(0, w, m), r.integers(0, h, m)].astype(np.float64)
    mt = np.c_[xr, xr + np.array([5.0, 2.0]), r.random(m)] if m else np.zeros((0, 5))
    maps = densify.build_sparse_maps(mt, w, h)
    flow = densify.densify_flow(guide, maps)
    assert np.isfinite(flow).all()
    for x, y in xr.astype(int):
        np.testing.assert_allclose(flow[y, x], [5.0, 2.0], rtol=0, atol=1e-5)


@SETTINGS
@given(seed=st.integers(0, 10 ** 6), h=st.integers(8, 80), w=st.integers(8, 80))
def test_fusion_weights_and_output_range(cuda, seed, h, w):
    """SPEC fusion invariants: normalised weights sum to 1, output in [0, 1],
    monotone trust (lower SSIM never raises the source weight), and fusing
    identical frames returns the frame."""
    ref, warped = rng_image(seed, h, w, 3), rng_image(seed + 1, h, w, 3)
    s_hi = np.random.default_rng(seed).uniform(0, 1, (h, w)).astype(np.float32)
    s_lo = (s_hi * np.float32(0.5)).astype(np.float32)
    valid = np.ones((h, w), bool)
    wr, ws = fusion.fusion_weights(ref, warped, s_hi, valid)
    assert np.abs(wr + ws - 1.0).max() < 1e-6
    _, ws_lo = fusion.fusion_weights(ref, warped, s_lo, valid)
    assert np.all(ws_lo <= ws + 1e-7)
    comp = fusion.fuse(ref, warped, s_hi, valid)
    assert np.isfinite(comp).all() and comp.min() >= 0.0 and comp.max() <= 1.0
    same = pipeline.fuse_stack([ref, ref, ref], [s_hi, s_lo], [valid, valid])
    assert np.abs(same - ref).max() < 1e-4


@settings(max_examples=8, deadline=None, derandomize=True,
          suppress_health_check=[HealthCheck.function_scoped_fixture])
@given(seed=st.integers(0, 10 ** 6), h=st.integers(30, 90), w=st.integers(30, 90),
       radius=st.integers(1, 12), patch=st.sampled_from([3, 5, 9, 21]), quant=st.booleans())
def test_ssd_match_equals_bruteforce(cuda, seed, h, w, radius, patch, quant):
    """SPEC matcher invariant: ssd_match equals the brute-force oracle on
    random configurations (quantised images force exact score ties)."""
    r = np.random.default_rng(seed)
    ref, src = rng_image(seed, h, w), rng_image(seed + 3, h, w)
    if quant:
        ref, src = (np.round(ref * 4) / 4).astype(np.float32), (np.round(src * 4) / 4).astype(np.float32)
    hp = patch // 2
    pts = []
    for _ in range(25):
        xr, yr = r.integers(hp, w - hp), r.integers(hp, h - hp)
        pts.append((xr, yr, r.integers(-5, w + 5), r.integers(-5, h + 5)))
    got, found = matcher.ssd_match_batch(ref, src, pts, radius, patch)
    for (xr, yr, xi, yi), g, f in zip(pts, got, found):
        want = O.ssd_search(ref, src, (xr, yr), (xi, yi), radius, patch)
        assert f == (want is not None)
        if want is not None:
            assert (int(g[0]), int(g[1])) == (want[0], want[1])
            assert abs(g[2] - want[2]) <= 1e-12 * max(1.0, want[2])


@settings(max_examples=10, deadline=None, derandomize=True,
          suppress_health_check=[HealthCheck.function_scoped_fixture])
@given(seed=st.integers(0, 10 ** 6), h=st.integers(1, 70), w=st.integers(1, 70),
       amp=st.floats(0.0, 40.0))
def test_warp_bit_exact_random_flow(cuda, seed, h, w, amp):
    """warp_image (densify.py:145-174) is bit-exact for arbitrary flows,
    including samples far outside the frame (clamped, marked invalid)."""
    src = rng_image(seed, h, w, 3)
    flow = (np.random.default_rng(seed).normal(size=(h, w, 2)) * amp).astype(np.float32)
    got, valid = densify.warp_image(src, flow)
    want, wvalid = O.warp_image(src, flow)
    np.testing.assert_array_equal(got, want)
    np.testing.assert_array_equal(valid, wvalid)


@settings(max_examples=8, deadline=None, derandomize=True,
          suppress_health_check=[HealthCheck.function_scoped_fixture])
@given(seed=st.integers(0, 10 ** 6), h=st.integers(2, 140), w=st.integers(2, 140),
       levels=st.integers(0, 6))
def test_fuse_random_sizes_match_oracle(cuda, seed, h, w, levels):
    """fusion.fuse at odd sizes and explicit level counts (reflect edges at
    every level) within the 1e-3 composite bar."""
    ref, warped = rng_image(seed, h, w, 3), rng_image(seed + 1, h, w, 3)
    ssim = np.random.default_rng(seed).uniform(-0.5, 1, (h, w)).astype(np.float32)
    valid = np.random.default_rng(seed + 2).random((h, w)) > 0.2
    lv = None if levels == 0 else levels
    got = fusion.fuse(ref, warped, ssim, valid, lv)
    want = O.fuse(ref, warped, ssim, valid.astype(np.float32), lv)
    assert np.abs(got - want).max() < 1e-3


@settings(max_examples=10, deadline=None, derandomize=True,
          suppress_health_check=[HealthCheck.function_scoped_fixture])
@given(seed=st.integers(0, 10 ** 6), h=st.integers(100, 900), w=st.integers(100, 900))
def test_pyramid_random_sizes_bit_exact(cuda, seed, h, w):
    """SPEC image invariant: level dims halve exactly (floor) with the
    retention rule; values bit-exact (separately rounded f32)."""
    img = rng_image(seed, h, w)
    got = image.build_pyramid(img)
    want = O.pyramid(img)
    assert len(got) == len(want)
    for a, b in zip(got, want):
        np.testing.assert_array_equal(np.asarray(a), b)


@settings(max_examples=6, deadline=None, derandomize=True,
          suppress_health_check=[HealthCheck.function_scoped_fixture])
@given(seed=st.integers(0, 10 ** 6), w=st.integers(120, 360), h=st.integers(120, 300),
       stops=st.sampled_from([1.0, 2.0, 3.0]), rot=st.sampled_from([0.0, 0.4]))
def test_register_and_fuse_random_scenes(cuda, seed, w, h, stops, rot):
    """End to end on random scene recipes and sizes: the same verdict as the
    oracle (RegistrationError or not), identical level counts and match
    coordinates, composite within 1e-3."""
    from harness import synth
    from paper_1504_01441_b200.errors import RegistrationError
    st_ = synth.synth_stack(synth.working_spec(w, h, stops=stops, rotation_deg=rot), seed)
    try:
        want = O.register_and_fuse(st_.ref, st_.src)
    except O.RegistrationError:
        with pytest.raises(RegistrationError):
            pipeline.register_and_fuse(st_.ref, st_.src)
        return
    got = pipeline.register_and_fuse(st_.ref, st_.src)
    assert got.level_counts == want.level_counts
    np.testing.assert_array_equal(got.matches[:, :4], want.matches[:, :4])
    assert np.abs(got.composite - want.composite).max() < 1e-3


@settings(max_examples=12, deadline=None, derandomize=True,
          suppress_health_check=[HealthCheck.function_scoped_fixture])
@given(seed=st.integers(0, 10 ** 6), h=st.integers(1, 67), w=st.integers(1, 67))
def test_luminance_and_histogram_match_any_size(cuda, seed, h, w):
    """image.luminance / match_histogram bit-exact at every size (pixel
    counts not a multiple of the kernels' 4-pixel vectors included)."""
    rgb, rgb2 = rng_image(seed, h, w, 3), rng_image(seed + 5, h, w, 3) * np.float32(0.7)
    lum = image.luminance(rgb)
    np.testing.assert_array_equal(lum, O.luminance(rgb))
    lum2 = O.luminance(rgb2)
    np.testing.assert_array_equal(image.match_histogram(lum2, lum), O.match_histogram(lum2, lum))


@settings(max_examples=10, deadline=None, derandomize=True,
          suppress_health_check=[HealthCheck.function_scoped_fixture])
@given(seed=st.integers(0, 10 ** 6), h=st.integers(1, 80), w=st.integers(1, 80),
       window=st.sampled_from([3, 7, 11, 15]))
def test_ssim_and_quality_any_size(cuda, seed, h, w, window):
    """fusion.ssim_map (reflect edges, windows larger than the image) within
    1e-4 and quality_weights within 1e-5 relative of the oracle."""
    a, b = rng_image(seed, h, w), rng_image(seed + 9, h, w)
    got = fusion.ssim_map(a, b, window, 1.5)
    want = O.ssim_map(a, b, window, 1.5)
    assert np.abs(np.asarray(got) - want).max() < 1e-4
    img = rng_image(seed + 2, h, w, 3)
    q, oq = np.asarray(fusion.quality_weights(img)), O.quality_weights(img)
    assert np.abs(q - oq).max() <= 1e-5 * oq.max() + 1e-12


@settings(max_examples=12, deadline=None, derandomize=True,
          suppress_health_check=[HealthCheck.function_scoped_fixture])
@given(seed=st.integers(0, 10 ** 6), h=st.integers(1, 70), w=st.integers(1, 70),
       c=st.sampled_from([0, 1, 3]), levels=st.integers(1, 8))
def test_pyramid_functions_bit_exact(cuda, seed, h, w, c, levels):
    """fusion.gaussian_pyramid / laplacian_pyramid / collapse_pyramid match
    the reference's scipy arithmetic bit for bit (f64, symmetric correlate
    order), for grey and colour arrays of any size."""
    x = np.random.default_rng(seed).random((h, w) if c == 0 else (h, w, c))
    for got, want in zip(fusion.gaussian_pyramid(x, levels), O.gaussian_pyramid(x, levels)):
        np.testing.assert_array_equal(got, want)
    laps, olaps = fusion.laplacian_pyramid(x, levels), O.laplacian_pyramid(x, levels)
    assert len(laps) == len(olaps)
    for got, want in zip(laps, olaps):
        np.testing.assert_array_equal(got, want)
    np.testing.assert_array_equal(fusion.collapse_pyramid(olaps), O.collapse(olaps))
