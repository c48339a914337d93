"""Warp-stall samples of an ncu report grouped by SASS opcode (where the time goes)."""
import csv, subprocess, sys, collections
rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = rows[1]
data = [dict(zip(hdr, r)) for r in rows[2:] if len(r) == len(hdr)]
by = collections.Counter()
tot = 0
for d in data:
    n = int(d["Warp Stall Sampling (All Samples)"] or 0)
    toks = [t for t in d["Source"].split() if not t.startswith("@")]
    op = toks[0] if toks else "?"
    by[op] += n
    tot += n
print(f"total stall samples {tot}")
for op, n in by.most_common(20):
    print(f"  {op:28s} {n:7d} {100*n/tot:5.1f}%")
