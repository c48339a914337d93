"""Hot SASS regions of an ncu report: stall samples per instruction with the
dominant stall reasons, grouped into runs (python scripts/ncu_sass_hot.py rep [top])."""
import csv
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = rows[1]
data = [dict(zip(hdr, r)) for r in rows[2:] if len(r) == len(hdr)]
reasons = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]


def n(x):
    try:
        return float(x)
    except ValueError:
        return 0.0


tot = sum(n(d["Warp Stall Sampling (All Samples)"]) for d in data)
ins = sum(n(d["Instructions Executed"]) for d in data)
agg = {r: sum(n(d[r]) for d in data) for r in reasons}
print(f"samples {tot:.0f}  warp-instructions {ins:.0f}  sass lines {len(data)}")
print("  ".join(f"{r[6:]} {100 * v / tot:.1f}%" for r, v in sorted(agg.items(), key=lambda t: -t[1])[:8]))
idx = sorted(range(len(data)), key=lambda i: -n(data[i]["Warp Stall Sampling (All Samples)"]))[:top]
for i in sorted(idx):
    d = data[i]
    s = n(d["Warp Stall Sampling (All Samples)"])
    rs = sorted(((n(d[r]), r[6:]) for r in reasons), reverse=True)[:2]
    print(f"{i:5d} {100 * s / tot:5.1f}% {d['Source'].strip()[:60]:60s} " + " ".join(f"{r}:{100 * v / max(s, 1):.0f}" for v, r in rs))
