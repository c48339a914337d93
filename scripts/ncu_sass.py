"""Instruction-mix and stall summary by SASS opcode from an ncu report."""
import collections, csv, subprocess, sys
rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 20
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = next(r for r in rows if r and r[0] == "Address")
agg = collections.defaultdict(lambda: [0.0, 0.0])
stalls = collections.defaultdict(float)
skeys = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
for r in rows:
    if len(r) != len(hdr) or r[0] == "Address":
        continue
    d = dict(zip(hdr, r))
    op = d["Source"].strip().split(" ")[0]
    if op.startswith("@"):
        op = d["Source"].strip().split(" ")[1]
    op = op.split(".")[0]
    f = lambda k: float(d.get(k, "0") or 0)
    agg[op][0] += f("Instructions Executed")
    agg[op][1] += f("Warp Stall Sampling (All Samples)")
    for k in skeys:
        stalls[k] += f(k)
ti = sum(v[0] for v in agg.values())
ts = sum(v[1] for v in agg.values())
print(f"warp instructions {ti:.0f}")
for op, (i, s) in sorted(agg.items(), key=lambda x: -x[1][0])[:top]:
    print(f"  {op:10s} inst {100 * i / ti:5.1f}%  stall-samples {100 * s / max(ts, 1):5.1f}%")
st = sum(stalls.values())
print("stall reasons:", ", ".join(f"{k[6:]} {100 * v / st:.0f}%" for k, v in sorted(stalls.items(), key=lambda x: -x[1])[:6]))
