"""Summarise an ncu --metrics gpu__time_duration.sum CSV: per-kernel totals."""
import collections, csv, sys
path = sys.argv[1]
pairs = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
rows = list(csv.reader(open(path)))
hdr = None
agg = collections.OrderedDict()
for r in rows:
    if r and r[0] == "ID":
        hdr = r
        continue
    if not hdr or len(r) != len(hdr):
        continue
    d = dict(zip(hdr, r))
    if d["Metric Name"] != "gpu__time_duration.sum":
        continue
    v = float(d["Metric Value"].replace(",", ""))
    u = d["Metric Unit"]
    v = v / 1000 if u in ("ns", "nsecond") else v * 1000 if u in ("ms", "msecond") else v
    name = d["Kernel Name"].split("(")[0].replace("void ", "")[:48]
    a = agg.setdefault(name, [0, 0.0])
    a[0] += 1
    a[1] += v
tot = sum(a[1] for a in agg.values())
print(f"{'us/pair':>9} {'launches':>8} {'share':>6}  kernel")
for n, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{t / pairs:9.1f} {c / pairs:8.1f} {100 * t / tot:5.1f}%  {n}")
print(f"{tot / pairs:9.1f} us per pair total (serialised, cold cache)")
