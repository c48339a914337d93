"""Time the merge (hdr_fuse: weights, pyramids, collapse) on one 5MP pair's
real stage outputs, for each value of the test hooks given on the command
line (python scripts/fuse_bench.py [W H] [option=v1,v2 ...]).
Prints us per call and the max |diff| against the first variant."""
import ctypes
import itertools
import sys

sys.path.insert(0, ".")
import torch  # noqa: E402

from harness import synth  # noqa: E402
from paper_1504_01441_b200 import _native, pipeline  # noqa: E402

args = [a for a in sys.argv[1:] if "=" not in a]
opts = [a.split("=") for a in sys.argv[1:] if "=" in a]
W = int(args[0]) if args else 2592
H = int(args[1]) if len(args) > 1 else 1944
st = synth.synth_stack(synth.working_spec(W, H), 0)
ref = torch.from_numpy(st.ref).cuda()
res = pipeline.register_and_fuse(ref, torch.from_numpy(st.src).cuda())
warped = res.warped.contiguous()
ssim = res.ssim.float().contiguous()
valid = res.valid.to(torch.uint8).contiguous()
L = _native.lib()
ctx = ctypes.c_void_p()
_native.check(L.hdr_ctx_create(W, H, ctypes.c_void_p(torch.cuda.current_stream().cuda_stream), ctypes.byref(ctx)))
out = torch.empty_like(ref)
P = ctypes.c_void_p


def run():
    _native.check(L.hdr_fuse(ctx, P(ref.data_ptr()), P(warped.data_ptr()), P(ssim.data_ptr()),
                             P(valid.data_ptr()), W, H, 0, P(out.data_ptr())), "fuse")


def timed(fn, reps=20):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps * 1e3


names = [o[0] for o in opts]
first = None
for vals in itertools.product(*[[int(v) for v in o[1].split(",")] for o in opts]):
    for n, v in zip(names, vals):
        _native.check(L.hdr_set_option(n.encode(), v))
    us = timed(run)
    o = out.clone()
    first = o if first is None else first
    print(f"fuse {W}x{H} {dict(zip(names, vals))}: {us:8.1f} us  max|diff| {float((o - first).abs().max()):.3e}"
          f"  vs pipeline composite {float((o - res.composite).abs().max()):.3e}")
