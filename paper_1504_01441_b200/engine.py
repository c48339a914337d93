"""Device plumbing: hdr contexts (preallocated workspaces) for the drop-in
calls. Torch is used for device memory and streams only; all arithmetic
happens in libhdrb200.so.

Re-entrancy (the reference's functions are pure): every
host thread gets its own context per device, so concurrent calls never share
scratch, host state or a graph cache, and a thread only ever resizes (closes)
its own context. Within one thread a context follows torch's current stream;
when a call moves it to another stream, the new stream first waits for the
work already queued on the old one (an event, no host sync), so asynchronous
enqueues on different streams never overlap on the same scratch.
"""

from __future__ import annotations

import ctypes
import threading

import numpy as np
import torch

from . import _native

_tls = threading.local()


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
            self.stream = torch.cuda.current_stream(device)
            _native.check(_native.lib().hdr_ctx_create(width, height,
                                                       ctypes.c_void_p(self.stream.cuda_stream),
                                                       ctypes.byref(handle)), "hdr_ctx_create")
        self.handle = handle

    def bind_stream(self, stream: torch.cuda.Stream | None = None):
        """Queue this context's next work on `stream` (default: torch's
        current stream on the context's device), ordered after everything
        it already queued elsewhere."""
        s = stream if stream is not None else torch.cuda.current_stream(self.device)
        if s.cuda_stream != self.stream.cuda_stream:
            ev = torch.cuda.Event()
            ev.record(self.stream)
            s.wait_event(ev)
            self.stream = s
        _native.check(_native.lib().hdr_ctx_set_stream(self.handle, ctypes.c_void_p(s.cuda_stream)))
        return self.handle

    def drain(self):
        """Wait for every queued use of the workspace (before freeing it)."""
        self.stream.synchronize()

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
    """This thread's context for `device`, with capacity >= (width, height),
    bound to the current stream."""
    _require_cuda()
    dev = torch.cuda.current_device() if device is None else device
    engines = getattr(_tls, "engines", None)
    if engines is None:
        engines = _tls.engines = {}
    e = engines.get(dev)
    if e is None or e.width < width or e.height < height:
        if e is not None:
            e.drain()
            w, h = max(width, e.width), max(height, e.height)
            e.close()
        else:
            w, h = width, height
        e = Engine(w, h, dev)
        engines[dev] = e
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


def to_host(*ts: torch.Tensor):
    """numpy copies of device tensors: each lands by DMA in a pinned block of
    torch's caching host allocator (reused by later calls, so no fresh pages
    to fault in -- a pageable .cpu() of a 5MP pair's outputs ran at ~2 GB/s),
    one synchronisation for all of them."""
    hs = []
    for t in ts:
        if not t.is_cuda:
            hs.append(t)
            continue
        h = torch.empty(t.shape, dtype=t.dtype, pin_memory=True)
        h.copy_(t, non_blocking=True)
        hs.append(h)
    if any(t.is_cuda for t in ts):
        torch.cuda.current_stream(next(t for t in ts if t.is_cuda).device).synchronize()
    return [h.numpy() for h in hs]


def out(t: torch.Tensor, as_torch: bool):
    """Return a result in the caller's flavour (numpy in, numpy out)."""
    return t if as_torch else to_host(t)[0]
