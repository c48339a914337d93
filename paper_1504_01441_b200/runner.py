"""Throughput runner: many pairs in flight over several CUDA streams.

Each stream owns its own hdr context (workspace) so pairs on different
streams never share scratch; every pair is one CUDA-graph replay of the whole
register+merge chain. `run_host` is the end-to-end public path (pinned host
inputs -> H2D -> pair -> D2H of the composite and the verdict words), with
copies of one stream overlapping compute of the others.
"""

from __future__ import annotations

import ctypes

import numpy as np
import torch

from . import _native
from .engine import Engine
from .pipeline import PairBuffers, PipelineParams


class BatchRunner:
    def __init__(self, width: int, height: int, streams: int = 4,
                 params: PipelineParams | None = None, device: int | None = None,
                 graph: bool = True):
        self.device = torch.cuda.current_device() if device is None else device
        self.width, self.height = width, height
        self.params = params or PipelineParams()
        self.params.validate()
        self.native_params = self.params.to_native()
        self.graph = graph
        self.streams = [torch.cuda.Stream(self.device) for _ in range(streams)]
        self.engines = [Engine(width, height, self.device) for _ in range(streams)]
        for e, s in zip(self.engines, self.streams):
            e.bind_stream(s)
        self._staging = None

    # ---------------------------------------------------------- device path
    def enqueue(self, k: int, ref: torch.Tensor, src: torch.Tensor, bufs: PairBuffers):
        """Queue one pair on stream k % S (no host sync)."""
        e = self.engines[k % len(self.engines)]
        fn = (_native.lib().hdr_register_and_fuse_graph if self.graph
              else _native.lib().hdr_register_and_fuse)
        _native.check(fn(e.handle, ctypes.byref(self.native_params), self.width, self.height,
                         ctypes.c_void_p(ref.data_ptr()), ctypes.c_void_p(src.data_ptr()),
                         ctypes.byref(bufs.native)), "register_and_fuse")

    def run_device(self, pairs, outs, start_event=None, stop_event=None):
        """All pairs device-resident; optional events bracket the whole batch
        on the current stream (the streams wait on start, stop waits on all)."""
        cur = torch.cuda.current_stream(self.device)
        if start_event is not None:
            start_event.record(cur)
        for s in self.streams:
            s.wait_stream(cur)
        for k, ((ref, src), bufs) in enumerate(zip(pairs, outs)):
            self.enqueue(k, ref, src, bufs)
        for s in self.streams:
            cur.wait_stream(s)
        if stop_event is not None:
            stop_event.record(cur)

    def set_probes(self, k: int, events):
        """Stage probes (hdr_ctx_set_probes) for the context of stream k."""
        e = self.engines[k % len(self.engines)]
        arr = None
        if events is not None:
            arr = (ctypes.c_void_p * len(events))(*[ev.cuda_event for ev in events])
        _native.check(_native.lib().hdr_ctx_set_probes(e.handle, arr))

    def set_kernel_probes(self, k: int, family: int, events):
        """Kernel probes (hdr_ctx_set_kernel_probes) for the context of stream
        k: events[2j], events[2j+1] bracket launch j of kernel `family`."""
        e = self.engines[k % len(self.engines)]
        arr, n = None, 0
        if events:
            arr = (ctypes.c_void_p * len(events))(*[ev.cuda_event for ev in events])
            n = len(events) // 2
        _native.check(_native.lib().hdr_ctx_set_kernel_probes(e.handle, family, arr, n))

    # ---------------------------------------------------------- host path
    def _ensure_staging(self):
        """Two device slots per compute stream (inputs + outputs), so the
        upload of a stream's next pair and the download of its previous one
        overlap its current pair."""
        if self._staging is None:
            h, w = self.height, self.width
            dev = f"cuda:{self.device}"
            self._staging = [[dict(ref=torch.empty((h, w, 3), dtype=torch.float32, device=dev),
                                   src=torch.empty((h, w, 3), dtype=torch.float32, device=dev),
                                   out=PairBuffers(w, h, self.device),
                                   consumed=None, drained=None)
                              for _ in range(2)] for _ in self.streams]
            self._h2d = torch.cuda.Stream(self.device)
            self._d2h = torch.cuda.Stream(self.device)
        return self._staging

    def run_host(self, host_pairs, host_out, start_event=None, stop_event=None):
        """End to end: pinned host (ref, src) in, composite + info words out.

        host_out[k] = (composite pinned (h, w, 3) f32, info pinned (32,) i32).
        Uploads run back to back on one copy stream (the host link is the
        bottleneck of this path), pairs on the compute streams, downloads on a
        second copy stream; events order each slot's reuse. Returns the H2D /
        D2H byte counts of the batch."""
        st = self._ensure_staging()
        cur = torch.cuda.current_stream(self.device)
        if start_event is not None:
            start_event.record(cur)
        for s in self.streams + [self._h2d, self._d2h]:
            s.wait_stream(cur)
        h2d = d2h = 0
        S = len(self.streams)
        for k, ((href, hsrc), (hcomp, hinfo)) in enumerate(zip(host_pairs, host_out)):
            j = k % S
            slot = st[j][(k // S) % 2]
            cs = self.streams[j]
            with torch.cuda.stream(self._h2d):
                if slot["consumed"] is not None:      # previous pair of this slot read its inputs
                    self._h2d.wait_event(slot["consumed"])
                slot["ref"].copy_(href, non_blocking=True)
                slot["src"].copy_(hsrc, non_blocking=True)
                loaded = torch.cuda.Event()
                loaded.record(self._h2d)
            cs.wait_event(loaded)
            if slot["drained"] is not None:           # previous outputs of this slot downloaded
                cs.wait_event(slot["drained"])
            with torch.cuda.stream(cs):
                self.enqueue(j, slot["ref"], slot["src"], slot["out"])
                done = torch.cuda.Event()
                done.record(cs)
            slot["consumed"] = done
            with torch.cuda.stream(self._d2h):
                self._d2h.wait_event(done)
                hcomp.copy_(slot["out"].composite, non_blocking=True)
                hinfo.copy_(slot["out"].info, non_blocking=True)
                drained = torch.cuda.Event()
                drained.record(self._d2h)
            slot["drained"] = drained
            h2d += href.numel() * 4 + hsrc.numel() * 4
            d2h += hcomp.numel() * 4 + hinfo.numel() * 4
        for s in self.streams + [self._h2d, self._d2h]:
            cur.wait_stream(s)
        if stop_event is not None:
            stop_event.record(cur)
        return h2d, d2h

    def enqueue_raw(self, k: int, ref_raw: torch.Tensor, src_raw: torch.Tensor, bits: int,
                    bufs: PairBuffers, composite_u8: torch.Tensor | None):
        """Queue one pair from raw 8/16-bit device samples on stream k % S
        (hdr_register_and_fuse_raw: decode, pair graph, 8-bit composite)."""
        e = self.engines[k % len(self.engines)]
        channels = 1 if ref_raw.dim() == 2 else ref_raw.shape[2]
        _native.check(_native.lib().hdr_register_and_fuse_raw(
            e.handle, ctypes.byref(self.native_params), self.width, self.height,
            ctypes.c_void_p(ref_raw.data_ptr()), ctypes.c_void_p(src_raw.data_ptr()), channels, bits,
            1 if self.graph else 0, ctypes.byref(bufs.native),
            ctypes.c_void_p(0 if composite_u8 is None else composite_u8.data_ptr())),
            "register_and_fuse_raw")

    def run_host_raw(self, host_pairs, host_out, bits: int = 8):
        """End to end on the file path: pinned raw samples
        in ((h, w, 3) uint8, or int16-viewed uint16), the 8-bit composite
        (save_png's samples) + info words out. Same slot / stream scheme as
        run_host; returns the H2D / D2H byte counts."""
        h, w = self.height, self.width
        dev = f"cuda:{self.device}"
        if bits not in (8, 16):
            raise ValueError("bits must be 8 or 16")
        if getattr(self, "_raw_bits", None) != bits:
            # staging slots typed for this sample width (uint8, or uint16 viewed as int16)
            torch.cuda.synchronize(self.device)
            self._raw_bits = bits
            dt = torch.uint8 if bits == 8 else torch.int16
            self._raw_staging = [[dict(ref=torch.empty((h, w, 3), dtype=dt, device=dev),
                                       src=torch.empty((h, w, 3), dtype=dt, device=dev),
                                       out=PairBuffers(w, h, self.device),
                                       comp8=torch.empty((h, w, 3), dtype=torch.uint8, device=dev),
                                       consumed=None, drained=None)
                                  for _ in range(2)] for _ in self.streams]
            self._ensure_staging()
        st = self._raw_staging
        cur = torch.cuda.current_stream(self.device)
        for s in self.streams + [self._h2d, self._d2h]:
            s.wait_stream(cur)
        h2d = d2h = 0
        S = len(self.streams)
        for k, ((href, hsrc), (hcomp, hinfo)) in enumerate(zip(host_pairs, host_out)):
            j = k % S
            slot = st[j][(k // S) % 2]
            cs = self.streams[j]
            with torch.cuda.stream(self._h2d):
                if slot["consumed"] is not None:
                    self._h2d.wait_event(slot["consumed"])
                slot["ref"].copy_(href, non_blocking=True)
                slot["src"].copy_(hsrc, non_blocking=True)
                loaded = torch.cuda.Event()
                loaded.record(self._h2d)
            cs.wait_event(loaded)
            if slot["drained"] is not None:
                cs.wait_event(slot["drained"])
            with torch.cuda.stream(cs):
                self.enqueue_raw(j, slot["ref"], slot["src"], bits, slot["out"], slot["comp8"])
                done = torch.cuda.Event()
                done.record(cs)
            slot["consumed"] = done
            with torch.cuda.stream(self._d2h):
                self._d2h.wait_event(done)
                hcomp.copy_(slot["comp8"], non_blocking=True)
                hinfo.copy_(slot["out"].info, non_blocking=True)
                drained = torch.cuda.Event()
                drained.record(self._d2h)
            slot["drained"] = drained
            h2d += href.numel() * href.element_size() + hsrc.numel() * hsrc.element_size()
            d2h += hcomp.numel() + hinfo.numel() * 4
        for s in self.streams + [self._h2d, self._d2h]:
            cur.wait_stream(s)
        return h2d, d2h

    def graph_kernels(self) -> int:
        return int(_native.lib().hdr_ctx_graph_kernels(self.engines[0].handle))

    def close(self):
        for e in self.engines:
            e.close()


def verdicts(info: np.ndarray):
    """(registered?, n_weeded_level0) from one pair's info words."""
    return int(info[0]) == _native.HDR_OK, int(info[16])
