"""Registers / stack / shared memory per kernel instantiation of libmeshnbr.so (cuobjdump -res-usage)."""
import re
import subprocess
import sys

lib = sys.argv[1] if len(sys.argv) > 1 else "paper_1604_04689_b200/libmeshnbr.so"
pat = sys.argv[2] if len(sys.argv) > 2 else ""
out = subprocess.run(["cuobjdump", "-res-usage", lib], capture_output=True, text=True).stdout.splitlines()
for i, line in enumerate(out):
    m = re.search(r"Function (\S+):", line)
    if not m or i + 1 >= len(out):
        continue
    name = subprocess.run(["c++filt", m.group(1)], capture_output=True, text=True).stdout.strip()
    name = re.sub(r"\(.*", "", name)
    if pat not in name:
        continue
    r = dict(re.findall(r"(REG|STACK|SHARED|LOCAL):(\d+)", out[i + 1]))
    print(f"{name:60s} reg {r.get('REG')} stack {r.get('STACK')} shared {r.get('SHARED')}")
