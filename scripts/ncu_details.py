"""Print the details page of an ncu report as 'section | metric | value unit'."""
import csv, subprocess, sys
rep = sys.argv[1]
want = sys.argv[2:]
out = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = rows[0]
i_sec, i_name, i_unit, i_val = (hdr.index(k) for k in ("Section Name", "Metric Name", "Metric Unit", "Metric Value"))
for r in rows[1:]:
    if len(r) <= i_val or not r[i_name]:
        continue
    if want and not any(w.lower() in r[i_sec].lower() for w in want):
        continue
    print(f"{r[i_sec][:28]:28s} | {r[i_name][:45]:45s} | {r[i_val]} {r[i_unit]}")
