"""Run one synthetic pair through register_and_fuse (for ncu captures)."""
import sys
import time

sys.path.insert(0, ".")
import torch  # noqa: E402

from paper_1504_01441_b200 import pipeline  # noqa: E402
from harness import synth  # noqa: E402

w = int(sys.argv[1]) if len(sys.argv) > 1 else 2592
h = int(sys.argv[2]) if len(sys.argv) > 2 else 1944
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 1
st = synth.synth_stack(synth.working_spec(w, h), 0)
ref = torch.from_numpy(st.ref).cuda()
src = torch.from_numpy(st.src).cuda()
for _ in range(reps):
    t = time.perf_counter()
    out = pipeline.register_and_fuse(ref, src)
    torch.cuda.synchronize()
    print(f"pair {w}x{h}: {1e3 * (time.perf_counter() - t):.2f} ms, level_counts={out.level_counts}")
