"""Per-source-line instruction and stall summary from an ncu report (CUDA view)."""
import csv, subprocess, sys
rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = None
data = []
for r in rows:
    if r and r[0] == "Line":
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        data.append(dict(zip(hdr, r)))
if not data:
    print(out[:2000])
    sys.exit()
def num(x):
    try:
        return float(x)
    except ValueError:
        return 0.0
tot_i = sum(num(d.get("Instructions Executed", 0)) for d in data)
tot_s = sum(num(d.get("Warp Stall Sampling (All Samples)", 0)) for d in data)
print(f"total warp instructions {tot_i:.0f}, stall samples {tot_s:.0f}")
data.sort(key=lambda d: -num(d.get("Warp Stall Sampling (All Samples)", 0)))
for d in data[:top]:
    print(f"{num(d['Warp Stall Sampling (All Samples)'])/max(tot_s,1)*100:5.1f}% stall "
          f"{num(d['Instructions Executed'])/max(tot_i,1)*100:5.1f}% inst  L{d['Line']}: {d['Source'].strip()[:90]}")
