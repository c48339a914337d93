"""C-ABI checks that need no GPU: the library loads, exports every symbol the
header declares, and its host-side key schedule / sampler reproduce numpy's
SeedSequence + Philox + Generator.choice (golden vectors from the reference
environment)."""

import ctypes
import os
import re

import numpy as np
import pytest

from golden_util import load
from paper_1504_01441_b200 import _native
from paper_1504_01441_b200.pipeline import PipelineParams

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    text = open(os.path.join(ROOT, "include", "hdrb200.h")).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(hdr_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_header_symbol():
    lib = _native.lib()
    syms = header_symbols()
    assert len(syms) >= 30
    for s in syms:
        assert hasattr(lib, s), s
        assert s in _native.SIGNATURES, f"{s} has no ctypes signature"


def test_level_seeds_match_numpy():
    fx = load("philox_choice")
    for row, seed in zip(fx["level_seeds"], (0, 1, 12345, 2 ** 40 + 3)):
        got = [_native.lib().hdr_level_seed(seed, l) for l in range(5)]
        assert got == [int(v) for v in row]


def test_iteration_keys_and_choice_match_numpy():
    fx = load("philox_choice")
    lib = _native.lib()
    for seed, it, n, key, draws in zip(fx["seed"], fx["it"], fx["n"], fx["key"], fx["draws"]):
        keys = (ctypes.c_uint64 * (2 * (int(it) + 1)))()
        assert lib.hdr_iteration_keys(int(seed), int(it) + 1, keys) == 0
        assert [keys[2 * it], keys[2 * it + 1]] == [int(key[0]), int(key[1])]
        k2 = (ctypes.c_uint64 * 2)(int(key[0]), int(key[1]))
        out = np.zeros((10, 4), dtype=np.int64)
        assert lib.hdr_choice4_host(k2, int(n), 10, out.ctypes.data) == 0
        np.testing.assert_array_equal(out, draws)


def test_choice_small_populations_match_numpy():
    lib = _native.lib()
    for n in (4, 5, 6, 7, 13, 1000):
        for it in range(20):
            ss = np.random.SeedSequence(entropy=99, spawn_key=(it,))
            g = np.random.Generator(np.random.Philox(ss))
            ref = np.stack([g.choice(n, size=4, replace=False) for _ in range(10)])
            key = ss.generate_state(2, np.uint64)
            k2 = (ctypes.c_uint64 * 2)(int(key[0]), int(key[1]))
            out = np.zeros((10, 4), dtype=np.int64)
            assert lib.hdr_choice4_host(k2, n, 10, out.ctypes.data) == 0
            np.testing.assert_array_equal(out, ref)


@pytest.mark.parametrize("field,value,msg", [
    ("tile", 8, "tile must be >= 16"),
    ("patch", 20, "patch must be odd and >= 3"),
    ("max_levels", 6, "max_levels must be in [1, 5]"),
    ("delta", 3, "delta must be >= 4"),
    ("ssim_window", 10, "ssim_window must be odd and >= 3"),
    ("workers", 3, "iterations must be divisible by workers"),
])
def test_params_validate_native_matches_python(field, value, msg):
    from paper_1504_01441_b200.errors import ConfigError
    p = PipelineParams(**{field: value})
    with pytest.raises(ConfigError, match=msg.replace("[", r"\[").replace("]", r"\]")):
        p.validate()
    buf = ctypes.create_string_buffer(128)
    np_ = p.to_native()
    rc = _native.lib().hdr_params_validate(ctypes.byref(np_), buf, 128)
    assert rc == _native.HDR_ERR_CONFIG
    assert buf.value.decode() == msg


def test_params_default_matches_dataclass():
    p = _native.HdrParams()
    _native.lib().hdr_params_default(ctypes.byref(p))
    ref = PipelineParams().to_native()
    for name, _ in _native.HdrParams._fields_:
        assert getattr(p, name) == getattr(ref, name), name


def test_missing_library_fails_loudly(monkeypatch, tmp_path):
    """No silent fallback: without libhdrb200.so the binding raises."""
    monkeypatch.setattr(_native, "LIB_PATH", str(tmp_path / "absent.so"))
    monkeypatch.setattr(_native, "_lib", None)
    with pytest.raises(RuntimeError, match="no CPU fallback"):
        _native.lib()


def test_no_cuda_fails_loudly(monkeypatch):
    """Without a CUDA device the drop-in raises instead of computing on the CPU."""
    import torch
    from paper_1504_01441_b200 import engine, pipeline
    monkeypatch.setattr(torch.cuda, "is_available", lambda: False)
    img = np.zeros((120, 160, 3), np.float32)
    with pytest.raises(RuntimeError, match="no CPU fallback"):
        pipeline.register_and_fuse(img, img)
    with pytest.raises(RuntimeError, match="no CPU fallback"):
        engine.to_dev(img, torch.float32)


def test_product_package_never_imports_the_oracle():
    """oracle/ is test infrastructure only: no module of the product package
    imports it."""
    pkg = os.path.join(ROOT, "paper_1504_01441_b200")
    for name in os.listdir(pkg):
        if name.endswith(".py"):
            text = open(os.path.join(pkg, name)).read()
            assert "oracle" not in re.findall(r"^\s*(?:from|import)\s+(\w+)", text, flags=re.M), name


def test_options_and_probe_arguments_validated():
    """hdr_set_option rejects unknown names; kernel probes validate their
    family and launch count before touching a context (no GPU work)."""
    lib = _native.lib()
    assert lib.hdr_set_option(b"no_such_option", 1) == _native.HDR_ERR_INVALID
    assert "unknown option" in _native.last_error()
    assert lib.hdr_set_option(None, 1) == _native.HDR_ERR_INVALID
    # null context -> invalid, whatever the other arguments
    assert lib.hdr_ctx_set_kernel_probes(None, 0, None, 0) == _native.HDR_ERR_INVALID
    assert lib.hdr_ctx_set_probes(None, None) == _native.HDR_ERR_INVALID
    assert lib.hdr_ctx_destroy(None) == _native.HDR_OK
