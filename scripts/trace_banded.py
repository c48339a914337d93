"""Per-launch device times of one banded pair on one rank (scripts/trace_pair.py for banded.py)."""
import ctypes
import sys

sys.path.insert(0, ".")
import torch  # noqa: E402

from harness import synth  # noqa: E402
from paper_1504_01441_b200 import _native  # noqa: E402
from paper_1504_01441_b200.banded import register_and_fuse_banded  # noqa: E402

W = int(sys.argv[1]) if len(sys.argv) > 1 else 4000
H = int(sys.argv[2]) if len(sys.argv) > 2 else 3000
st = synth.synth_stack(synth.working_spec(W, H), 0)
ref, src = torch.from_numpy(st.ref).cuda(), torch.from_numpy(st.src).cuda()
register_and_fuse_banded(ref, src)
torch.cuda.synchronize()
L = _native.lib()
L.hdr_set_option(b"trace", 1)
register_and_fuse_banded(ref, src)
torch.cuda.synchronize()
L.hdr_set_option(b"trace", 0)
buf = ctypes.create_string_buffer(1 << 20)
_native.check(L.hdr_trace_dump(buf, len(buf)))
rows = [l.split("\t") for l in buf.value.decode().splitlines()]
agg = {}
for name, us in rows:
    short = name.split("(")[0].replace("void ", "").replace("hdr::", "")
    a = agg.setdefault(short, [0, 0.0])
    a[0] += 1
    a[1] += float(us)
print(f"{len(rows)} launches, {sum(float(u) for _, u in rows):.1f} us summed")
for k, (n, us) in sorted(agg.items(), key=lambda t: -t[1][1])[:25]:
    print(f"{us:8.1f} us {n:3d}x  {k}")
