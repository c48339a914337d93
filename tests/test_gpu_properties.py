"""Size-independent properties of the GPU stages at the BASELINE sizes
(5MP, 12MP), where a full oracle comparison would take minutes per case:
identities the reference's arithmetic guarantees exactly, and linearity of
the domain-transform filter."""

import numpy as np
import pytest

from oracle import hdr_oracle as O
from harness import synth
from paper_1504_01441_b200 import densify, fusion, image

pytestmark = pytest.mark.gpu

SIZES = [(2592, 1944), (4000, 3000)]


@pytest.mark.parametrize("w,h", SIZES)
def test_warp_zero_flow_is_identity(cuda, w, h):
    rng = np.random.default_rng(w)
    src = rng.random((h, w, 3), dtype=np.float32)
    warped, valid = densify.warp_image(src, np.zeros((h, w, 2), np.float32))
    np.testing.assert_array_equal(warped, src)
    assert valid.all()


@pytest.mark.parametrize("w,h", SIZES)
def test_warp_integer_shift(cuda, w, h):
    """An integer flow (u, v) is a pure shift: warped[y, x] = src[y+v, x+u]
    inside, invalid exactly where the sample leaves the frame."""
    rng = np.random.default_rng(h)
    src = rng.random((h, w, 3), dtype=np.float32)
    u, v = -3, 2
    flow = np.empty((h, w, 2), np.float32)
    flow[..., 0], flow[..., 1] = u, v
    warped, valid = densify.warp_image(src, flow)
    np.testing.assert_array_equal(warped[: h - v, -u:], src[v:, : w + u])
    want_valid = np.zeros((h, w), bool)
    want_valid[: h - v, -u:] = True
    np.testing.assert_array_equal(valid, want_valid)


def test_dt_filter_linear_at_5mp(cuda):
    w, h = 2592, 1944
    rng = np.random.default_rng(1)
    guide = synth.synth_stack(synth.working_spec(640, 480), 0).ref[..., 0]
    guide = np.ascontiguousarray(np.tile(guide, (5, 5))[:h, :w])
    a = np.zeros((h, w, 2))
    b = np.zeros((h, w, 2))
    idx = rng.integers(0, h * w, 1300)
    a.reshape(-1, 2)[idx] = rng.normal(size=(1300, 2))
    b.reshape(-1, 2)[rng.permutation(idx)] = rng.normal(size=(1300, 2))
    fa, fb = densify.dt_filter(guide, a), densify.dt_filter(guide, b)
    fab = densify.dt_filter(guide, 2.0 * a - 0.5 * b)
    scale = np.abs(fab).max()
    assert np.abs(fab - (2.0 * fa - 0.5 * fb)).max() <= 1e-12 * scale


@pytest.mark.parametrize("w,h", SIZES)
def test_fuse_identical_frames_reconstructs(cuda, w, h):
    """Fusing a frame with itself (SSIM 1, all valid) gives weights 1/2 + 1/2
    and collapse(laplacian_pyramid(x)) = x up to f32 rounding."""
    rng = np.random.default_rng(3)
    img = rng.random((h, w, 3), dtype=np.float32)
    comp = fusion.fuse(img, img, np.ones((h, w), np.float32), np.ones((h, w), bool))
    assert np.abs(comp - img).max() < 1e-5


def test_histogram_match_self_is_quantisation(cuda):
    """match_histogram(x, x) maps every pixel onto its own 8-bit level (the
    CDF-matching LUT of identical histograms is the identity on bins)."""
    w, h = 2592, 1944
    lum = O.luminance(synth.synth_stack(synth.working_spec(640, 480), 0).ref)
    lum = np.ascontiguousarray(np.tile(lum, (5, 5))[:h, :w])
    got = image.match_histogram(lum, lum)
    want = (O.quantize(lum).astype(np.float32) / np.float32(255.0)).astype(np.float32)
    np.testing.assert_array_equal(got, want)
