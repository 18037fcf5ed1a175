"""Per-kernel table from an ncu launch-list CSV (gpu__time_duration + dram bytes)."""
import csv
import sys
from collections import OrderedDict

rows = list(csv.reader(open(sys.argv[1])))
hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
h, data = rows[hi], rows[hi + 1:]
ki, mi, vi, idi = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("ID")
k = OrderedDict()
for r in data:
    k.setdefault((int(r[idi]), r[ki]), {})[r[mi]] = float(r[vi].replace(",", ""))
tot = sum(m["gpu__time_duration.sum"] for (i, n), m in k.items() if "mn::" in n)
print(f"{'id':>4} {'kernel':<62} {'us':>10} {'share':>6} {'DRAM rd GB':>10} {'DRAM wr GB':>10} {'GB/s':>7}")
for (i, n), m in k.items():
    if "mn::" not in n:
        continue
    t = m["gpu__time_duration.sum"]
    rd, wr = m["dram__bytes_read.sum"] / 1e9, m["dram__bytes_write.sum"] / 1e9
    name = n.replace("void ", "").replace("mn::", "")[:62]
    print(f"{i:>4} {name:<62} {t / 1e3:>10.1f} {t / tot:>6.1%} {rd:>10.3f} {wr:>10.3f} {(rd + wr) / (t * 1e-9):>7.0f}")
