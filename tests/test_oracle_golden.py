"""Pin the CPU oracle (oracle/hdr_oracle.py) against fixtures produced by the
REAL reference (oracle/gen_golden.py). CPU only."""

import numpy as np
import pytest

from golden_util import BIG_SCENES, WIDE_SCENES, SCENES, digest, load, scene_inputs
from oracle import hdr_oracle as O
from harness import synth


@pytest.fixture(scope="module", params=SCENES + BIG_SCENES + WIDE_SCENES)
def scene(request):
    fx = load(request.param)
    ref, src = scene_inputs(fx)
    return request.param, fx, ref, src


def test_synth_inputs_match_reference(scene):
    _, fx, ref, src = scene
    assert [digest(ref), digest(src)] == list(fx["inputs_digest"])


def test_raster_stages_bit_exact(scene):
    _, fx, ref, src = scene
    lum_ref = O.luminance(ref)
    eq = O.match_histogram(O.luminance(src), lum_ref)
    assert digest(lum_ref) == str(fx["lum_ref_digest"])
    assert digest(eq) == str(fx["eq_src_digest"])
    rp, sp = O.pyramid(lum_ref), O.pyramid(eq)
    assert [digest(a) for a in rp] + [digest(a) for a in sp] == list(fx["pyr_digests"])


def test_level_trace_bit_exact(scene):
    _, fx, ref, src = scene
    lum_ref = O.luminance(ref)
    rp = O.pyramid(lum_ref)
    sp = O.pyramid(O.match_histogram(O.luminance(src), lum_ref))
    p = O.Params()
    for lev in range(len(rp) - 1, -1, -1):
        h, w = rp[lev].shape
        corners = O.detect_corners(rp[lev], p.tile, p.threshold, p.quadrant_half)
        np.testing.assert_array_equal(corners, fx[f"L{lev}_corners"])
        raw = O.match_level(rp[lev], sp[lev], fx[f"L{lev}_hpred"], p, corners)
        np.testing.assert_array_equal(raw, fx[f"L{lev}_raw"])
        if len(raw) >= 4:
            iters, eps, sd = O.level_weed_args(p, lev, w)
            kept, wit = O.weed(raw, w, h, iters, eps, sd, p.delta)
            np.testing.assert_array_equal(kept, fx[f"L{lev}_kept"])
            np.testing.assert_array_equal(wit, fx[f"L{lev}_witness"])
        if f"L{lev}_hfit" in fx:
            hf = O.fit_matches_homography(raw[kept], w, h)
            np.testing.assert_array_equal(hf, fx[f"L{lev}_hfit"])


def test_end_to_end_bit_exact(scene):
    _, fx, ref, src = scene
    o = O.register_and_fuse(ref, src)
    np.testing.assert_array_equal(o.matches, fx["matches"])
    np.testing.assert_array_equal(o.raw_matches, fx["raw_matches"])
    np.testing.assert_array_equal(np.asarray(o.level_counts), fx["level_counts"])
    np.testing.assert_array_equal(o.homography, fx["homography"])
    for k in ("composite", "flow", "warped", "valid", "ssim"):
        assert digest(getattr(o, k)) == str(fx[f"{k}_digest"]), k


def test_default_scene_raises():
    fx = load("default_scene_error")
    st = synth.synth_stack(synth.SceneSpec(), 0)
    assert [digest(st.ref), digest(st.src)] == list(fx["inputs_digest"])
    with pytest.raises(O.RegistrationError) as ei:
        O.register_and_fuse(st.ref, st.src)
    assert str(ei.value) == str(fx["message"])


def test_spec_kats():
    """SPEC.md KATs the reference satisfies."""
    # cornerness on a checkerboard quadrant pattern: C = 4, min = 1
    img = np.zeros((32, 32), dtype=np.float32)
    img[:16, 16:] = 1.0
    img[16:, :16] = 1.0
    c, lo = O._quadrants(O.integral(img), np.array([16]), np.array([16]), 8)
    assert (c[0], lo[0]) == (4.0, 1.0)
    edge = np.zeros((32, 32), dtype=np.float32)
    edge[:, 16:] = 1.0
    c, lo = O._quadrants(O.integral(edge), np.array([16]), np.array([16]), 8)
    assert (c[0], lo[0]) == (2.0, 0.0)
    assert O.detect_corners(np.full((128, 128), 0.5, np.float32)).shape == (0, 3)
    assert [len(O.pyramid(np.zeros((h, w), np.float32))) for w, h in
            [(640, 480), (2592, 1944), (4000, 3000), (100, 100)]] == [3, 5, 5, 1]
    assert O.to_norm(0, 0, 640, 480) == (-1.0, -0.75)
    a = np.random.default_rng(0).random((64, 64)).astype(np.float32)
    assert O.ssd_search(a, a, (30, 30), (30, 30)) == (30, 30, 0.0)
    s = np.full((40, 40), 0.25, np.float32)
    t = np.full((40, 40), 0.75, np.float32)
    assert abs(O.ssim_map(s, t)[20, 20] - 0.600064) < 1e-6
    assert abs(O.ssim_map(a, a) - 1.0).max() < 1e-12
