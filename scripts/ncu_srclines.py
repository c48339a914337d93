"""Per-CUDA-source-line instructions and stall samples of one kernel in an
ncu report (python scripts/ncu_srclines.py rep kernel_regex [top])."""
import csv
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass",
                      "-k", f"regex:{kern}", "--launch-count", "1"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
fname = ""
agg = {}
hdr = None
for r in rows:
    if r and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if hdr and r and r[0] and r[0] != "Line No":
        try:
            ins = float(r[7]); st = float(r[4])
        except (ValueError, IndexError):
            continue
        agg[(fname, int(r[0]), r[1][:80])] = (ins, st)
ti = sum(v[0] for v in agg.values()) or 1
ts = sum(v[1] for v in agg.values()) or 1
print(f"warp instructions {ti:.0f}, stall samples {ts:.0f}")
for (f, ln, src), (ins, st) in sorted(agg.items(), key=lambda t: -t[1][0])[:top]:
    print(f"{100 * ins / ti:5.1f}% ins {100 * st / ts:5.1f}% stall  {f}:{ln}  {src.strip()}")
