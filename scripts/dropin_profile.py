"""Where the drop-in register_and_fuse(numpy) call spends its time (host wall clock)."""
import sys
import time

sys.path.insert(0, ".")
import numpy as np  # noqa: E402
import torch  # noqa: E402

from harness import synth  # noqa: E402
from paper_1504_01441_b200 import pipeline  # noqa: E402
from paper_1504_01441_b200.engine import to_dev  # noqa: E402

st = synth.synth_stack(synth.working_spec(2592, 1944), 0)
ref, src = st.ref, st.src
pipeline.register_and_fuse(ref, src)
for _ in range(3):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    r = to_dev(ref, torch.float32, 0)
    s = to_dev(src, torch.float32, 0)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    bufs = pipeline.PairBuffers(2592, 1944, 0)
    pipeline.enqueue_pair(r, s, pipeline.PipelineParams(), bufs)
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    outs = {k: getattr(bufs, k) for k in ("composite", "flow", "warped", "valid", "ssim")}
    for k, v in outs.items():
        ta = time.perf_counter()
        x = (v.double() if k == "ssim" else v).cpu().numpy()
        torch.cuda.synchronize()
        print(f"  D2H {k}: {1e3 * (time.perf_counter() - ta):.1f} ms ({x.nbytes / 1e6:.0f} MB)")
    t3 = time.perf_counter()
    tt = time.perf_counter()
    res = pipeline.register_and_fuse(ref, src)
    t4 = time.perf_counter()
    print(f"H2D {1e3 * (t1 - t0):.1f} ms, pair {1e3 * (t2 - t1):.1f} ms, D2H {1e3 * (t3 - t2):.1f} ms; "
          f"register_and_fuse {1e3 * (t4 - tt):.1f} ms")
