"""Pin the oracle's general-argument stage functions to tests/golden/twins.npz,
written by the REAL reference (oracle/gen_golden.py --wide): dt_filter with
multi-channel / float64 guides and five planes, warp_image with 2/4/5
channels, batched rect_sum, quantize_256 and downsample on float32/float64,
apply_homography and symmetric_transfer_error. CPU only."""

import numpy as np

from golden_util import load
from oracle import hdr_oracle as O

FX = load("twins")


def test_dt_filter_general_guides_bit_exact():
    for tag, args in (("g3", (40.0, 0.3, 2)), ("g64", ()), ("g9", (25.0, 0.1, 3)), ("k5", (60.0, 0.2, 3))):
        got = O.dt_filter(FX[f"dt_{tag}_guide"], FX[f"dt_{tag}_data"], *args)
        np.testing.assert_array_equal(got, FX[f"dt_{tag}_out"], err_msg=tag)


def test_warp_any_channels_bit_exact():
    for c in (2, 4, 5):
        w, v = O.warp_image(FX[f"warp{c}_src"], FX[f"warp{c}_flow"])
        np.testing.assert_array_equal(w, FX[f"warp{c}_out"])
        np.testing.assert_array_equal(v, FX[f"warp{c}_valid"])


def test_raster_helpers_bit_exact():
    q = FX["rs_q"]
    np.testing.assert_array_equal(O.box_sum(FX["rs_table"], q[0], q[1], q[2], q[3]), FX["rs_out"])
    np.testing.assert_array_equal(O.quantize(FX["q32_in"]), FX["q32_out"])
    np.testing.assert_array_equal(O.quantize(FX["q64_in"]), FX["q64_out"])
    np.testing.assert_array_equal(O.halve(FX["ds3_in"]), FX["ds3_out"])
    np.testing.assert_array_equal(O.halve(FX["ds64_in"]), FX["ds64_out"])


def test_geometry_helpers_bit_exact():
    np.testing.assert_array_equal(O.apply_homography(FX["h"], FX["h_pts"]), FX["h_out"])
    np.testing.assert_array_equal(O.symmetric_transfer_error(FX["h"], FX["ste_ref"], FX["ste_src"]),
                                  FX["ste_out"])
