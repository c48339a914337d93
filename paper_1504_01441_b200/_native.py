"""ctypes binding of libhdrb200.so (include/hdrb200.h).

Loading fails loudly: there is no CPU fallback anywhere in this package. If
the library is missing, build it with `__graft_entry__.build()` (or
`python -m paper_1504_01441_b200.build`).
"""

from __future__ import annotations

import ctypes
import os

from .errors import ConfigError, DegenerateFit, RegistrationError

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libhdrb200.so")

HDR_OK, HDR_ERR_INVALID, HDR_ERR_DEGENERATE = 0, 1, 2
HDR_ERR_REGISTRATION, HDR_ERR_CONFIG, HDR_ERR_CUDA, HDR_ERR_EMPTY = 3, 4, 5, 6
HDR_ERR_SINGULAR = 7
INFO_WORDS = 32
NUM_STAGES = 7
STAGES = ("raster", "corners", "match_chain", "dt_filter", "finalize_warp", "ssim", "fuse")
# kernel-probe families (HDR_KP_* in include/hdrb200.h)
KPROBES = ("dt_rows", "dt_cols", "warp", "ssim", "fuse_weights0", "fuse_collapse0")


class HdrParams(ctypes.Structure):
    _fields_ = [
        ("tile", ctypes.c_int32), ("quadrant_half", ctypes.c_int32),
        ("radius", ctypes.c_int32), ("patch", ctypes.c_int32),
        ("max_levels", ctypes.c_int32), ("iterations", ctypes.c_int32),
        ("coarse_iterations", ctypes.c_int32), ("delta", ctypes.c_int32),
        ("passes", ctypes.c_int32), ("ssim_window", ctypes.c_int32),
        ("workers", ctypes.c_int32), ("_pad", ctypes.c_int32),
        ("threshold", ctypes.c_double), ("eps_px", ctypes.c_double),
        ("sigma_s", ctypes.c_double), ("sigma_r", ctypes.c_double),
        ("ssim_sigma", ctypes.c_double), ("normalization_floor", ctypes.c_double),
        ("seed", ctypes.c_uint64),
    ]


class HdrOutputs(ctypes.Structure):
    _fields_ = [(n, ctypes.c_void_p) for n in
                ("composite", "flow", "warped", "valid", "ssim", "matches",
                 "raw_matches", "homography", "info")]


# (name, restype, argtypes) for every symbol include/hdrb200.h declares
_P, _I, _I64, _D, _U64 = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_double, ctypes.c_uint64
SIGNATURES = {
    "hdr_params_default": (None, [_P]),
    "hdr_params_validate": (_I, [_P, ctypes.c_char_p, ctypes.c_size_t]),
    "hdr_ctx_create": (_I, [_I, _I, _P, ctypes.POINTER(_P)]),
    "hdr_ctx_destroy": (_I, [_P]),
    "hdr_ctx_set_stream": (_I, [_P, _P]),
    "hdr_max_matches": (_I, [_I, _I, _I]),
    "hdr_last_error": (ctypes.c_char_p, []),
    "hdr_set_option": (_I, [ctypes.c_char_p, ctypes.c_int64]),
    "hdr_ctx_sync": (_I, [_P]),
    "hdr_register_and_fuse": (_I, [_P, _P, _I, _I, _P, _P, _P]),
    "hdr_register_and_fuse_graph": (_I, [_P, _P, _I, _I, _P, _P, _P]),
    "hdr_ctx_set_probes": (_I, [_P, _P]),
    "hdr_ctx_graph_kernels": (_I, [_P]),
    "hdr_ctx_set_kernel_probes": (_I, [_P, _I, _P, _I]),
    "hdr_luminance": (_I, [_P, _P, _I64, _P]),
    "hdr_match_histogram": (_I, [_P, _P, _I64, _P, _I64, _I, _P]),
    "hdr_build_pyramid": (_I, [_P, _P, _I, _I, _I, _I, _P, _P]),
    "hdr_integral": (_I, [_P, _P, _I, _I, _P]),
    "hdr_cornerness": (_I, [_P, _P, _I, _I, _P, _I, _I, _P]),
    "hdr_detect_corners": (_I, [_P, _P, _I, _I, _I, _D, _I, _P, _P]),
    "hdr_ssd_match": (_I, [_P, _P, _P, _I, _I, _P, _I, _I, _I, _P, _P]),
    "hdr_match_level": (_I, [_P, _P, _P, _P, _I, _I, _P, _P, _P]),
    "hdr_weed": (_I, [_P, _P, _I, _I, _I, _I, _D, _U64, _I, _P, _P, _P]),
    "hdr_fit_matches_homography": (_I, [_P, _P, _I, _I, _I, _P]),
    "hdr_fit_homography": (_I, [_P, _P, _P, _I, _P]),
    "hdr_inlier_mask": (_I, [_P, _P, _P, _P, _I, _D, _P]),
    "hdr_homography_flow": (_I, [_P, _P, _I, _I, _P]),
    "hdr_match_stack": (_I, [_P, _P, _I, _I, _P, _P, _P, _P, _P, _P]),
    "hdr_sparse_maps": (_I, [_P, _P, _I, _I, _I, _P, _P, _P]),
    "hdr_dt_filter": (_I, [_P, _P, _P, _I, _I, _I, _D, _D, _I]),
    "hdr_dt_filter_general": (_I, [_P, _P, _I, _P, _I, _I, _I, _D, _D, _I]),
    "hdr_rect_sum": (_I, [_P, _P, _I, _I, _P, _I64, _P]),
    "hdr_quantize_256": (_I, [_P, _P, _I, _I64, _P]),
    "hdr_downsample": (_I, [_P, _P, _I, _I, _I, _I, _P]),
    "hdr_apply_homography": (_I, [_P, _P, _P, _I64, _P]),
    "hdr_symmetric_transfer_error": (_I, [_P, _P, _P, _P, _I64, _P]),
    "hdr_densify_finalize": (_I, [_P, _P, _I, _I, _P, _D, _P]),
    "hdr_warp_image": (_I, [_P, _P, _I, _I, _I, _P, _P, _P]),
    "hdr_ssim_map": (_I, [_P, _P, _P, _I, _I, _I, _D, _P]),
    "hdr_make_ssim": (_I, [_P, _P, _P, _I, _I, _I, _D, _P]),
    "hdr_quality_weights": (_I, [_P, _P, _I, _I, _P]),
    "hdr_fuse": (_I, [_P, _P, _P, _P, _P, _I, _I, _I, _P]),
    "hdr_fusion_weights": (_I, [_P, _P, _P, _P, _P, _I, _I, _P, _P]),
    "hdr_pyr_down": (_I, [_P, _P, _I, _I, _I, _P]),
    "hdr_pyr_up": (_I, [_P, _P, _I, _I, _I, _I, _I, _P, _I, _P]),
    "hdr_fuse_stack": (_I, [_P, _I, _P, _P, _P, _I, _I, _I, _P]),
    "hdr_register_and_fuse_stack": (_I, [_P, _P, _I, _I, _I, _P, _P, _P]),
    "hdr_decode_image": (_I, [_P, _P, _I, _I, _I, _I, _P]),
    "hdr_encode_u8": (_I, [_P, _P, _I64, _P]),
    "hdr_mean_luminance": (_I, [_P, _P, _I, _I64, _P]),
    "hdr_dark_count": (_I, [_P, _P, _I, _I64, ctypes.c_float, _P]),
    "hdr_register_and_fuse_raw": (_I, [_P, _P, _I, _I, _P, _P, _I, _I, _I, _P, _P]),
    "hdr_trace_dump": (_I, [ctypes.c_char_p, _I64]),
    "hdr_band_rows_multiple": (_I, []),
    "hdr_band_agg_doubles": (_I64, [_I, _I, _I]),
    "hdr_band_dt": (_I, [_P, _I, _P, _P, _I, _I, _I, _I, _I, _D, _D, _I, _I, _P, _P, _P, _D, _P]),
    "hdr_band_warp": (_I, [_P, _P, _I, _I, _I, _I, _P, _P, _P, _P, _P]),
    "hdr_band_ssim": (_I, [_P, _P, _P, _P, _I, _I, _I, _I, _I, _D, _P]),
    "hdr_level_seed": (ctypes.c_uint32, [_U64, _I]),
    "hdr_iteration_keys": (_I, [_U64, _I, _P]),
    "hdr_choice4_host": (_I, [_P, _I, _I, _P]),
    "hdr_fit_homography_host": (_I, [_P, _P, _I, _P]),
}

_lib = None


def lib():
    """The loaded library; raises RuntimeError when it was never built."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(
                f"{LIB_PATH} is missing: the CUDA path has no CPU fallback. "
                "Build it with __graft_entry__.build().")
        handle = ctypes.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(handle, name)
            fn.restype = res
            fn.argtypes = args
        _lib = handle
    return _lib


def last_error() -> str:
    msg = lib().hdr_last_error()
    return msg.decode() if msg else ""


def check(rc: int, what: str = "") -> None:
    """Map an hdr status code onto the reference's exception types."""
    if rc == HDR_OK:
        return
    msg = last_error() or what
    if rc == HDR_ERR_CONFIG:
        raise ConfigError(msg)
    if rc == HDR_ERR_DEGENERATE:
        raise DegenerateFit(msg)
    if rc == HDR_ERR_REGISTRATION:
        raise RegistrationError(msg)
    if rc == HDR_ERR_INVALID:
        raise ValueError(msg)
    if rc == HDR_ERR_SINGULAR:
        import numpy as np
        raise np.linalg.LinAlgError(msg)
    raise RuntimeError(f"{what}: {msg}" if what else msg)
