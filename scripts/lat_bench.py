"""Single-pair device latency of the graph and stream paths without probes,
for each value of hdr options given as name=v1,v2 (python scripts/lat_bench.py [W H] pdl=0,1)."""
import itertools
import statistics
import sys

sys.path.insert(0, ".")
import torch  # noqa: E402

from harness import synth  # noqa: E402
from paper_1504_01441_b200 import _native  # noqa: E402
from paper_1504_01441_b200.pipeline import PairBuffers  # noqa: E402
from paper_1504_01441_b200.runner import BatchRunner  # noqa: E402

args = [a for a in sys.argv[1:] if "=" not in a]
opts = [a.split("=") for a in sys.argv[1:] if "=" in a]
W = int(args[0]) if args else 2592
H = int(args[1]) if len(args) > 1 else 1944
st = synth.synth_stack(synth.working_spec(W, H), 0)
ref, src = torch.from_numpy(st.ref).cuda(), torch.from_numpy(st.src).cuda()
names = [o[0] for o in opts]
for vals in itertools.product(*[[int(v) for v in o[1].split(",")] for o in opts]):
    for n, v in zip(names, vals):
        _native.check(_native.lib().hdr_set_option(n.encode(), v))
    for graph in (True, False):
        r = BatchRunner(W, H, streams=1, graph=graph)
        bufs = PairBuffers(W, H, 0)
        s = r.streams[0]
        ts = []
        for i in range(8):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            e0.record(s)
            r.enqueue(0, ref, src, bufs)
            e1.record(s)
            torch.cuda.synchronize()
            if i >= 2:
                ts.append(e0.elapsed_time(e1))
        print(f"{dict(zip(names, vals))} graph={graph}: pair latency {statistics.median(ts):.3f} ms "
              f"(min {min(ts):.3f})")
        r.close()
