"""Device plumbing: one hdr context (preallocated workspace) per CUDA device,
bound to torch's current stream at every call. Torch is used for device
memory and streams only; all arithmetic happens in libhdrb200.so.
"""

from __future__ import annotations

import ctypes
import threading

import numpy as np
import torch

from . import _native

_lock = threading.Lock()
_engines: dict[int, "Engine"] = {}


def _require_cuda():
    if not torch.cuda.is_available():
        raise RuntimeError("paper_1504_01441_b200 needs a CUDA device (sm_100a); "
                           "there is no CPU fallback")


class Engine:
    """An hdr_ctx sized for images up to (width, height)."""

    def __init__(self, width: int, height: int, device: int):
        self.width, self.height, self.device = width, height, device
        handle = ctypes.c_void_p()
        with torch.cuda.device(device):
            stream = torch.cuda.current_stream(device).cuda_stream
            _native.check(_native.lib().hdr_ctx_create(width, height, ctypes.c_void_p(stream),
                                                       ctypes.byref(handle)), "hdr_ctx_create")
        self.handle = handle

    def bind_stream(self, stream: torch.cuda.Stream | None = None):
        s = stream if stream is not None else torch.cuda.current_stream(self.device)
        _native.check(_native.lib().hdr_ctx_set_stream(self.handle, ctypes.c_void_p(s.cuda_stream)))
        return self.handle

    def sync(self):
        _native.check(_native.lib().hdr_ctx_sync(self.handle), "hdr_ctx_sync")

    def close(self):
        if self.handle:
            _native.lib().hdr_ctx_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def engine(width: int, height: int, device: int | None = None) -> Engine:
    """Shared context for `device` with capacity >= (width, height)."""
    _require_cuda()
    dev = torch.cuda.current_device() if device is None else device
    with _lock:
        e = _engines.get(dev)
        if e is None or e.width < width or e.height < height:
            if e is not None:
                torch.cuda.synchronize(dev)
                w, h = max(width, e.width), max(height, e.height)
                e.close()
            else:
                w, h = width, height
            e = Engine(w, h, dev)
            _engines[dev] = e
        e.bind_stream()
        return e


def engine_for_rows(n_rows: int, device: int | None = None) -> Engine:
    """Shared context whose match-row workspace (one row per 16-px tile of
    its capacity, hdr_max_matches) holds n_rows."""
    side = 16 * int(np.ceil(np.sqrt(max(n_rows, 1)))) + 16
    e = engine(1, 1, device)
    if e.width < side or e.height < side:
        e = engine(max(e.width, side), max(e.height, side), device)
    return e


def device_of(*arrays) -> int:
    for a in arrays:
        if isinstance(a, torch.Tensor) and a.is_cuda:
            return a.device.index
    _require_cuda()
    return torch.cuda.current_device()


def to_dev(x, dtype: torch.dtype, device: int | None = None) -> torch.Tensor:
    """Contiguous CUDA tensor of `dtype` (uploads numpy / host tensors)."""
    _require_cuda()
    dev = torch.cuda.current_device() if device is None else device
    if isinstance(x, torch.Tensor):
        t = x.to(device=f"cuda:{dev}", dtype=dtype)
    else:
        t = torch.from_numpy(np.ascontiguousarray(x)).to(device=f"cuda:{dev}", dtype=dtype)
    return t.contiguous()


def ptr(t: torch.Tensor | None):
    return ctypes.c_void_p(t.data_ptr()) if t is not None else ctypes.c_void_p(0)


def is_torch(*arrays) -> bool:
    return any(isinstance(a, torch.Tensor) for a in arrays)


def out(t: torch.Tensor, as_torch: bool):
    """Return a result in the caller's flavour (numpy in, numpy out)."""
    return t if as_torch else t.cpu().numpy()
