"""Per-kernel timing through the C-ABI stage twins (CUDA events on the
context stream), for tuning on the GPU box:

  python scripts/kbench.py [dt|warp|all] [W H]

dt: hdr_dt_filter on 3 f64 planes (sparse like the splat maps) for every
column-path option, with the max difference against the default path.
warp: hdr_warp_image (RGB) with a smooth synthetic flow.
"""
import ctypes
import sys

sys.path.insert(0, ".")
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1504_01441_b200 import _native  # noqa: E402

what = sys.argv[1] if len(sys.argv) > 1 else "all"
W = int(sys.argv[2]) if len(sys.argv) > 2 else 2592
H = int(sys.argv[3]) if len(sys.argv) > 3 else 1944
L = _native.lib()
ctx = ctypes.c_void_p()
stream = torch.cuda.current_stream().cuda_stream
_native.check(L.hdr_ctx_create(W, H, ctypes.c_void_p(stream), ctypes.byref(ctx)))
P = W * H


def timed(fn, reps=10):
    fn()
    torch.cuda.synchronize()
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0.record()
    for _ in range(reps):
        fn()
    t1.record()
    torch.cuda.synchronize()
    return t0.elapsed_time(t1) / reps * 1e3  # us


if what in ("dt", "all"):
    g = torch.rand((H, W), device="cuda", dtype=torch.float32)
    base = torch.zeros((3, H, W), device="cuda", dtype=torch.float64)
    idx = torch.randint(0, P, (P // 4000,), device="cuda")
    for k in range(3):
        base[k].view(-1)[idx] = torch.randn(idx.numel(), device="cuda", dtype=torch.float64)
    base[2].view(-1)[idx] = 1.0
    planes = base.clone()
    ref = None
    for cl, pf in ((1, 1), (1, 0), (0, 1)):
        L.hdr_set_option(b"dt_cluster_columns", cl)
        L.hdr_set_option(b"dt_cols_prefetch", pf)

        def run():
            planes.copy_(base)
            _native.check(L.hdr_dt_filter(ctx, ctypes.c_void_p(g.data_ptr()),
                                          ctypes.c_void_p(planes.data_ptr()), 3, W, H, 400.0, 0.2, 3))
        us = timed(run)
        cp = timed(lambda: planes.copy_(base))
        run()
        torch.cuda.synchronize()
        out = planes.clone()
        if ref is None:
            ref = out
        d = (out - ref).abs().max().item()
        print(f"dt_filter cluster={cl} prefetch={pf}: {us - cp:8.1f} us (3 passes, copy {cp:.1f} excluded)"
              f"  max|diff| vs first = {d:.3e}")
    L.hdr_set_option(b"dt_cluster_columns", 1)
    L.hdr_set_option(b"dt_cols_prefetch", 1)

if what in ("warp", "all"):
    src = torch.rand((H, W, 3), device="cuda", dtype=torch.float32)
    yy, xx = torch.meshgrid(torch.arange(H, device="cuda"), torch.arange(W, device="cuda"), indexing="ij")
    flow = torch.stack([3.5 * torch.sin(yy / 200.0) - 3, 2.0 * torch.cos(xx / 300.0) + 2], -1).float()
    warped = torch.empty_like(src)
    valid = torch.empty((H, W), device="cuda", dtype=torch.uint8)

    def runw():
        _native.check(L.hdr_warp_image(ctx, ctypes.c_void_p(src.data_ptr()), 3, W, H,
                                       ctypes.c_void_p(flow.data_ptr()), ctypes.c_void_p(warped.data_ptr()),
                                       ctypes.c_void_p(valid.data_ptr())))
    us = timed(runw, 20)
    nbytes = P * (8 + 12 + 12 + 1 + 1)
    print(f"warp_image RGB: {us:8.1f} us  {nbytes / us / 1e3:.0f} GB/s algorithmic ({nbytes / 1e6:.1f} MB)")
