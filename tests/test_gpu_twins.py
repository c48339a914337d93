"""Stage twins with the general arguments the reference accepts (and the pair
pipeline never passes), on the GPU, against tests/golden/twins.npz written by
the REAL reference and against the oracle on fresh inputs:

* dt_filter: multi-channel and float64 guides (hdr_dt_filter_general, the
  reference's sequential recursion), more than three planes, and rows wider
  than the shared-memory row kernels (densify.py:59-113);
* warp_image with any channel count (densify.py:145-174);
* rect_sum, quantize_256, downsample / build_pyramid on multi-channel and
  float64 images (image.py:47-93);
* apply_homography, symmetric_transfer_error (geometry.py:80-115) and their
  error cases.

Bars: bit-exact where the reference's arithmetic is reproduced step for step
(warp, raster helpers, geometry); dt_filter 1e-12 relative for the
sequential twin (exp may differ in the last bit) and 1e-9 for the
shared-memory scan kernels (reassociated affine scans, as in
test_gpu_parity.py)."""

import numpy as np
import pytest
import torch

from golden_util import load
from oracle import hdr_oracle as O
from paper_1504_01441_b200 import densify, geometry, image

pytestmark = pytest.mark.gpu
FX = load("twins")


def rel_err(got, want):
    return float(np.abs(np.asarray(got) - want).max() / max(1.0, np.abs(want).max()))


@pytest.mark.parametrize("tag,args,tol", [("g3", (40.0, 0.3, 2), 1e-12), ("g64", (), 1e-12),
                                          ("g9", (25.0, 0.1, 3), 1e-12), ("k5", (60.0, 0.2, 3), 1e-9)])
def test_dt_filter_general_vs_reference(cuda, tag, args, tol):
    got = densify.dt_filter(FX[f"dt_{tag}_guide"], FX[f"dt_{tag}_data"], *args)
    assert got.shape == FX[f"dt_{tag}_out"].shape and got.dtype == np.float64
    assert rel_err(got, FX[f"dt_{tag}_out"]) <= tol


@pytest.mark.parametrize("w,h,k", [(7300, 24, 3), (9001, 9, 1), (8192, 17, 2)])
def test_dt_filter_wide_rows(cuda, w, h, k):
    """Rows wider than dt_rows_kernel's shared memory: the sequential row twin
    inside the fast filter (columns stay on the cluster kernel)."""
    r = np.random.default_rng(w + h)
    g = r.random((h, w)).astype(np.float32)
    d = r.random((h, w, k))
    d[r.random((h, w)) < 0.9] = 0.0  # sparse, like the splat planes
    got = densify.dt_filter(g, d, 400.0, 0.2, 3)
    assert rel_err(got, O.dt_filter(g, d, 400.0, 0.2, 3)) <= 1e-9


def test_dt_filter_torch_multichannel_guide(cuda):
    r = np.random.default_rng(3)
    g = r.random((40, 50, 3)).astype(np.float32)
    d = r.random((40, 50))
    got = densify.dt_filter(torch.from_numpy(g).cuda(), torch.from_numpy(d).cuda(), 30.0, 0.5, 2)
    assert isinstance(got, torch.Tensor) and got.is_cuda
    assert rel_err(got.cpu().numpy(), O.dt_filter(g, d, 30.0, 0.5, 2)) <= 1e-12


@pytest.mark.parametrize("c", [2, 4, 5])
def test_warp_any_channels_vs_reference(cuda, c):
    w, v = densify.warp_image(FX[f"warp{c}_src"], FX[f"warp{c}_flow"])
    np.testing.assert_array_equal(w, FX[f"warp{c}_out"])
    np.testing.assert_array_equal(v, FX[f"warp{c}_valid"])


def test_warp_grey_2d_matches_oracle(cuda):
    r = np.random.default_rng(5)
    src = r.random((33, 47)).astype(np.float32)
    flow = (r.random((33, 47, 2)) * 10 - 5).astype(np.float32)
    w, v = densify.warp_image(src, flow)
    ow, ov = O.warp_image(src, flow)
    np.testing.assert_array_equal(w, ow)
    np.testing.assert_array_equal(v, ov)


def test_rect_sum_vs_reference(cuda):
    t, q = FX["rs_table"], FX["rs_q"]
    np.testing.assert_array_equal(image.rect_sum(t, q[0], q[1], q[2], q[3]), FX["rs_out"])
    s = image.rect_sum(t, 3, 2, 19, 11)
    assert np.ndim(s) == 0 and s == FX["rs_scalar"]
    # broadcasting: one column against many rows
    ys = np.arange(0, 17)
    np.testing.assert_array_equal(image.rect_sum(t, 2, ys, 9, 17), O.box_sum(t, 2, ys, 9, 17))
    # device tensors in, device tensor out
    got = image.rect_sum(torch.from_numpy(t).cuda(), torch.tensor(q[0]).cuda(), torch.tensor(q[1]).cuda(),
                         torch.tensor(q[2]).cuda(), torch.tensor(q[3]).cuda())
    np.testing.assert_array_equal(got.cpu().numpy(), FX["rs_out"])


@pytest.mark.parametrize("bounds", [(-1, 0, 3, 3), (4, 0, 3, 3), (0, 0, 24, 3), (0, 5, 3, 4), (0, 0, 3, 18)])
def test_rect_sum_rejects_out_of_range(cuda, bounds):
    with pytest.raises(ValueError, match="rectangle bounds out of range"):
        image.rect_sum(FX["rs_table"], *bounds)


def test_rect_sum_float_bounds_raise_index_error(cuda):
    with pytest.raises(IndexError):
        image.rect_sum(FX["rs_table"], 0.5, 0, 3, 3)


def test_quantize_vs_reference(cuda):
    np.testing.assert_array_equal(image.quantize_256(FX["q32_in"]), FX["q32_out"])
    np.testing.assert_array_equal(image.quantize_256(FX["q64_in"]), FX["q64_out"])
    img = np.random.default_rng(2).random((19, 23, 3)).astype(np.float32)
    q = image.quantize_256(img)
    assert q.dtype == np.uint8 and q.shape == img.shape
    np.testing.assert_array_equal(q, O.quantize(img))


def test_downsample_multichannel_vs_reference(cuda):
    np.testing.assert_array_equal(image.downsample(FX["ds3_in"]), FX["ds3_out"])
    got = image.downsample(FX["ds64_in"])
    assert got.dtype == np.float32
    np.testing.assert_array_equal(got, FX["ds64_out"])
    with pytest.raises(ValueError, match="too small"):
        image.downsample(np.zeros((1, 5, 3), np.float32))


def test_build_pyramid_rgb_matches_oracle(cuda):
    img = np.random.default_rng(4).random((250, 333, 3)).astype(np.float32)
    got = image.build_pyramid(img, max_levels=4, min_dim=30)
    want = O.pyramid(img, 4, 30)
    assert len(got) == len(want)
    for a, b in zip(got, want):
        np.testing.assert_array_equal(a, b)


def test_apply_homography_vs_reference(cuda):
    got = geometry.apply_homography(FX["h"], FX["h_pts"])
    assert got.shape == FX["h_pts"].shape
    np.testing.assert_array_equal(got, FX["h_out"])
    hm = np.array([[1.0, 0, 0], [0, 1.0, 0], [1.0, 0, -2.0]])
    with pytest.raises(ValueError, match="point maps to infinity"):
        geometry.apply_homography(hm, np.array([[2.0, 5.0], [1.0, 1.0]]))


def test_symmetric_transfer_error_vs_reference(cuda):
    got = geometry.symmetric_transfer_error(FX["h"], FX["ste_ref"], FX["ste_src"])
    np.testing.assert_allclose(got, FX["ste_out"], rtol=1e-13, atol=0)
    # points mapped to infinity give inf, as _transfer_distance does
    hm = np.array([[1.0, 0, 0], [0, 1.0, 0], [0.5, 0, 1.0]])
    rp = np.array([[-2.0, 0.0], [1.0, 1.0]])
    sp = np.array([[0.0, 0.0], [1.0, 1.0]])
    np.testing.assert_allclose(geometry.symmetric_transfer_error(hm, rp, sp),
                               O.symmetric_transfer_error(hm, rp, sp), rtol=1e-13)
    with pytest.raises(np.linalg.LinAlgError):
        geometry.symmetric_transfer_error(np.zeros((3, 3)), rp, sp)
