"""Per-launch device times of one 5MP pair on the stream path (events around
every launch: hdr_set_option("trace", 1)); the sum over launches is below
the pair latency by the launch gaps the events expose.
python scripts/trace_pair.py [W H] [--all]"""
import ctypes
import sys

sys.path.insert(0, ".")
import torch  # noqa: E402

from harness import synth  # noqa: E402
from paper_1504_01441_b200 import _native  # noqa: E402
from paper_1504_01441_b200.pipeline import PairBuffers  # noqa: E402
from paper_1504_01441_b200.runner import BatchRunner  # noqa: E402

args = [a for a in sys.argv[1:] if not a.startswith("--")]
W = int(args[0]) if args else 2592
H = int(args[1]) if len(args) > 1 else 1944
st = synth.synth_stack(synth.working_spec(W, H), 0)
ref, src = torch.from_numpy(st.ref).cuda(), torch.from_numpy(st.src).cuda()
r = BatchRunner(W, H, streams=1, graph=False)
bufs = PairBuffers(W, H, 0)
L = _native.lib()
for _ in range(2):
    r.enqueue(0, ref, src, bufs)
torch.cuda.synchronize()
L.hdr_set_option(b"trace", 1)
r.enqueue(0, ref, src, bufs)
torch.cuda.synchronize()
L.hdr_set_option(b"trace", 0)
buf = ctypes.create_string_buffer(1 << 20)
_native.check(L.hdr_trace_dump(buf, len(buf)))
rows = [l.split("\t") for l in buf.value.decode().splitlines()]
tot = sum(float(us) for _, us in rows)
agg = {}
for name, us in rows:
    short = name.split("(")[0].replace("void ", "").replace("hdr::", "")
    a = agg.setdefault(short, [0, 0.0])
    a[0] += 1
    a[1] += float(us)
if "--all" in sys.argv:
    for name, us in rows:
        print(f"{float(us):8.1f}  {name.split('(')[0][:70]}")
print(f"{len(rows)} launches, {tot:.1f} us summed")
for k, (n, us) in sorted(agg.items(), key=lambda t: -t[1][1]):
    print(f"{us:8.1f} us {n:3d}x  {k}")
