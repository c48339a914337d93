"""GPU parity at BASELINE.json's headline shapes, pinned to the REAL reference.

tests/golden/c2_5mp_s0.npz (configs[1], 2592x1944) and c4_12mp_s0.npz
(configs[3], 4000x3000) were written by oracle/gen_golden.py running hdrflow
itself: per-level corners, raw matches, kept sets, witness counts and
least-squares H, the final matches / H / level_counts, full-array digests of
every dense output and a 1-in-32 lattice sample of each. The device path is
compared with those fixtures directly, then with the oracle at full
resolution (the oracle reproduces every one of those digests bit for bit,
tests/test_oracle_golden.py), which pins every pixel.

Bars (north_star): keypoints / match coordinates / kept sets bit-exact, SSD
scores 1e-12 relative, H 1e-4 relative, flow 1e-4 px, warped and composite
1e-3 max-abs, `valid` identical, SSIM 1e-4 (see check_dense for the one
documented exception: pixels near a quantisation flip of the warped frame's
luminance).
"""

import numpy as np
import pytest

from golden_util import BIG_SCENES, WIDE_SCENES, digest, load, scene_inputs
from oracle import hdr_oracle as O
from paper_1504_01441_b200 import matcher, pipeline, weeding

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

FLOW_TOL = 1e-4
RADIANCE_TOL = 1e-3
SSIM_TOL = 1e-4
H_RTOL = 1e-4


@pytest.fixture(scope="module", params=BIG_SCENES + WIDE_SCENES)
def big(request, cuda):
    fx = load(request.param)
    ref, src = scene_inputs(fx)
    assert [digest(ref), digest(src)] == list(fx["inputs_digest"])
    res = pipeline.register_and_fuse(ref, src)
    return request.param, fx, ref, src, res


def rows_equal(got, want):
    got, want = np.asarray(got), np.asarray(want)
    assert got.shape == want.shape
    np.testing.assert_array_equal(got[:, :4], want[:, :4])
    np.testing.assert_allclose(got[:, 4], want[:, 4], rtol=1e-12, atol=1e-15)


def test_headline_pair_against_reference_fixture(big):
    """The whole pair against what hdrflow.register_and_fuse returned."""
    _, fx, _, _, res = big
    np.testing.assert_array_equal(np.asarray(res.level_counts), fx["level_counts"])
    rows_equal(res.raw_matches, fx["raw_matches"])
    rows_equal(res.matches, fx["matches"])
    hm = fx["homography"]
    assert np.abs(res.homography - hm).max() / np.abs(hm).max() < H_RTOL
    # validity is decided in f64 on the flow: it must be the reference's, pixel for pixel
    assert digest(res.valid) == str(fx["valid_digest"])
    st = int(fx["stride"])
    sub = lambda a: np.asarray(a)[::st, ::st]  # noqa: E731
    assert np.abs(sub(res.flow) - fx["flow_sub"]).max() < FLOW_TOL
    assert np.abs(sub(res.warped) - fx["warped_sub"]).max() < RADIANCE_TOL
    assert np.abs(sub(res.composite) - fx["composite_sub"]).max() < RADIANCE_TOL
    assert np.abs(sub(res.ssim) - fx["ssim_sub"]).max() < SSIM_TOL


def test_headline_level_trace_against_reference_fixture(big):
    """Every pyramid level's corners, raw matches, RANSAC kept set, witness
    counts and least-squares H, each stage run on the GPU from the
    reference's own inputs for that level."""
    _, fx, ref, src, _ = big
    lum_ref = O.luminance(ref)
    rp = O.pyramid(lum_ref)
    sp = O.pyramid(O.match_histogram(O.luminance(src), lum_ref))
    mp = matcher.MatcherParams()
    for lev in range(len(rp) - 1, -1, -1):
        h, w = rp[lev].shape
        corners = matcher.detect_corners(rp[lev], mp.tile, mp.threshold, mp.quadrant_half)
        np.testing.assert_array_equal(corners, fx[f"L{lev}_corners"])
        raw = matcher._match_level(rp[lev], sp[lev], fx[f"L{lev}_hpred"], mp)
        rows_equal(raw, fx[f"L{lev}_raw"])
        raw = fx[f"L{lev}_raw"]
        if len(raw) >= 4:
            r = weeding.weed_parallel(raw, (w, h), mp.weed_params(lev, w), 1)
            np.testing.assert_array_equal(r.kept, fx[f"L{lev}_kept"])
            np.testing.assert_array_equal(r.witness, fx[f"L{lev}_witness"])
        if f"L{lev}_hfit" in fx:
            hf = matcher.fit_matches_homography(raw[fx[f"L{lev}_kept"]], w, h)
            assert np.abs(hf - fx[f"L{lev}_hfit"]).max() / np.abs(fx[f"L{lev}_hfit"]).max() < 1e-9


def quant_flips(warped_a, warped_b):
    """Pixels where quantize_256(luminance(warped)) differs between two warped
    frames (image.py:91-93): the SSIM input there moves by a whole LUT step."""
    qa = O.quantize(O.luminance(np.asarray(warped_a)))
    qb = O.quantize(O.luminance(np.asarray(warped_b)))
    return qa != qb


def check_dense(res, o, window=11):
    """Full-resolution dense outputs against the oracle.

    SSIM is held to 1e-4 everywhere except inside the 11x11 SSIM window of a
    pixel whose quantised warped luminance differs from the reference's.
    Such a flip needs luminance(warped) * 255 within ~1e-7 of a rounding
    boundary (the warped frames agree to ~1e-7), and it changes that
    pixel's equalised value by a full 1/255 LUT step, which the Gaussian
    moments spread over the window (up to ~1e-3 of SSIM). It is a
    property of the reference's 8-bit quantisation, not of the SSIM kernel:
    the kernel alone is held to 1e-4 on identical inputs
    (test_gpu_parity.test_ssim_and_fuse_stages). The number of flips is
    bounded too."""
    assert np.abs(res.flow - o.flow).max() < FLOW_TOL
    np.testing.assert_array_equal(res.valid, o.valid)
    assert np.abs(res.warped - o.warped).max() < RADIANCE_TOL
    flips = quant_flips(res.warped, o.warped)
    assert flips.sum() <= max(4, 1e-5 * flips.size), int(flips.sum())
    near = flips.copy()
    if flips.any():
        from scipy.ndimage import binary_dilation
        near = binary_dilation(flips, np.ones((window, window), bool))
    err = np.abs(np.asarray(res.ssim) - o.ssim)
    assert err[~near].max() < SSIM_TOL
    assert np.abs(res.composite - o.composite).max() < RADIANCE_TOL
    return int(flips.sum()), float(err.max())


def test_headline_pair_full_resolution_against_oracle(big):
    _, fx, ref, src, res = big
    o = O.register_and_fuse(ref, src)
    assert res.level_counts == o.level_counts
    rows_equal(res.matches, o.matches)
    # the oracle reproduces the reference's digests on the build host; on
    # this host it is the full-resolution checker
    check_dense(res, o)
