"""Summarise ncu --set full reports into profiles/ (markdown + traffic.json).

usage: python scripts/ncu_summary.py gpurun_out/prof_*.ncu-rep > profiles/ncu_r01_kernels.md
"""
import csv, json, os, subprocess, sys

KEYS = [
    ("gpu__time_duration.sum", "time"),
    ("dram__bytes_read.sum", "dram_read"),
    ("dram__bytes_write.sum", "dram_write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram_%"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm_%"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps_active_%"),
    ("sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active", "fp64_pipe_%"),
    ("launch__registers_per_thread", "regs"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
]

# report name (scripts/ncu_top.sh) -> kernel-probe family (bench.py kernel_bytes)
STAGE_OF = {"dt_rows": "dt_rows", "dt_cols": "dt_cols", "warp": "warp", "ssim": "ssim",
            "weights0": "fuse_weights0", "collapse0": "fuse_collapse0"}


def unit_scale(unit):
    return {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "usecond": 1e-6, "us": 1e-6, "ns": 1e-9, "ms": 1e-3,
            "nsecond": 1e-9, "msecond": 1e-3}.get(unit, 1.0)


def load(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr, units, vals = rows[0], rows[1], rows[2]
    d = {}
    for k, short in KEYS:
        for i, h in enumerate(hdr):
            if h == k:
                try:
                    d[short] = float(vals[i].replace(",", "")) * unit_scale(units[i])
                except ValueError:
                    d[short] = vals[i]
    d["kernel"] = vals[hdr.index("Kernel Name")] if "Kernel Name" in hdr else "?"
    return d


print("| report | kernel | time (us) | DRAM read (MB) | DRAM write (MB) | DRAM % | SM % | warps active % | FP64 pipe % | regs | grid x block |")
print("|---|---|---|---|---|---|---|---|---|---|---|")
traffic = {}
for rep in sys.argv[1:]:
    name = os.path.basename(rep).replace("prof_", "").replace(".ncu-rep", "")
    d = load(rep)
    t = d.get("time", 0) * 1e6
    rd, wr = d.get("dram_read", 0) / 1e6, d.get("dram_write", 0) / 1e6
    print(f"| {name} | `{d['kernel'][:40]}` | {t:.1f} | {rd:.1f} | {wr:.1f} | {d.get('dram_%', 0):.1f} | "
          f"{d.get('sm_%', 0):.1f} | {d.get('warps_active_%', 0):.1f} | {d.get('fp64_pipe_%', 0):.1f} | "
          f"{int(d.get('regs', 0))} | {int(d.get('grid', 0))} x {int(d.get('block', 0))} |")
    st = STAGE_OF.get(name)
    if st:
        traffic.setdefault(st, []).append(d.get("dram_read", 0) + d.get("dram_write", 0))
os.makedirs("profiles", exist_ok=True)
# bytes per launch, averaged over the captured launches of the family
with open("profiles/traffic.json", "w") as f:
    json.dump({k: sum(v) / len(v) for k, v in traffic.items()}, f, indent=1)
