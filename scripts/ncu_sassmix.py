"""Opcode mix (instructions executed) and top stalled SASS lines of an ncu report."""
import csv, subprocess, sys, collections
rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = rows[1]
data = [dict(zip(hdr, r)) for r in rows[2:] if len(r) == len(hdr)]
mix = collections.Counter()
tot = 0
for d in data:
    n = int(d["Instructions Executed"] or 0)
    op = d["Source"].split()
    op = [t for t in op if not t.startswith("@")][0].split(".")[0] if op else "?"
    mix[op] += n
    tot += n
print(f"total warp instructions {tot/1e6:.1f}M")
for op, n in mix.most_common(25):
    print(f"  {op:10s} {n/1e6:8.2f}M {100*n/tot:5.1f}%")
st = sorted(data, key=lambda d: -int(d["Warp Stall Sampling (All Samples)"] or 0))[:15]
print("top stalled:")
for d in st:
    print(f"  {d['Warp Stall Sampling (All Samples)']:>6} {d['Address'][-5:]} {d['Source'].strip()[:70]}")
