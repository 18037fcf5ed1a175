"""Summarise an ncu report (raw page) per kernel: time, DRAM bytes, throughput, occupancy, top stalls."""
import csv
import subprocess
import sys

rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(raw.splitlines()))
h, units, data = rows[0], rows[1], rows[2:]
col = {c: i for i, c in enumerate(h)}


def g(r, name):
    i = col.get(name)
    if i is None:
        return None
    try:
        return float(r[i].replace(",", ""))
    except ValueError:
        return r[i]


stall_cols = [c for c in h if c.startswith("smsp__pcsamp_warps_issue_stalled_") and not c.endswith("not_issued")]
for r in data:
    name = r[col["Kernel Name"]]
    t = g(r, "gpu__time_duration.sum")
    rd, wr = g(r, "dram__bytes_read.sum"), g(r, "dram__bytes_write.sum")
    tu = units[col["gpu__time_duration.sum"]]
    du = units[col["dram__bytes_read.sum"]]
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(du, 1)
    tscale = {"ns": 1e-9, "us": 1e-6, "usecond": 1e-6, "ms": 1e-3, "msecond": 1e-3, "nsecond": 1e-9}.get(tu, 1e-9)
    secs = t * tscale
    bw = (rd + wr) * scale / secs / 1e9 if secs else 0
    st = sorted(((g(r, c) or 0, c.replace("smsp__pcsamp_warps_issue_stalled_", "")) for c in stall_cols), reverse=True)[:5]
    tot = sum(g(r, c) or 0 for c in stall_cols) or 1
    print(f"{name[:70]}")
    print(f"   time {t} {tu}  dram R {rd} W {wr} {du}  -> {bw:.0f} GB/s  dram% {g(r, 'dram__throughput.avg.pct_of_peak_sustained_elapsed')}"
          f"  occ(warps) {g(r, 'sm__warps_active.avg.pct_of_peak_sustained_active')}%  regs {g(r, 'launch__registers_per_thread')}"
          f"  L2% {g(r, 'lts__throughput.avg.pct_of_peak_sustained_elapsed')}  SM% {g(r, 'sm__throughput.avg.pct_of_peak_sustained_elapsed')}")
    print("   stalls: " + ", ".join(f"{n} {v / tot:.0%}" for v, n in st))
