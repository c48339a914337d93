"""One-line summary of the last JSON line of a bench log (value, latency, stage and kernel times)."""
import json
import sys

d = json.loads([ln for ln in open(sys.argv[1]) if ln.startswith("{")][-1])
print("value", round(d["value"], 1), "lat", round(d["pair_latency_ms"], 3),
      {k: round(v, 3) for k, v in d["stage_ms"].items()}, {k: round(v * 1e3, 1) for k, v in d["kernel_ms"].items()})
