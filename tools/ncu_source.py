"""Per-source-line stall samples of one kernel in an ncu report: python tools/ncu_source.py rep regex [launch]"""
import csv
import subprocess
import sys

rep, rx = sys.argv[1], sys.argv[2]
skip = sys.argv[3] if len(sys.argv) > 3 else "0"
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass",
                      "--kernel-name", f"regex:{rx}", "--launch-skip", skip, "--launch-count", "1"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
cur, res, hdr = None, [], None
for r in rows:
    if len(r) == 2 and r[0] == "File Path":
        cur = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if hdr and r and r[0].isdigit():
        d = dict(zip(hdr, r))
        try:
            smp = int(d["Warp Stall Sampling (All Samples)"])
        except (KeyError, ValueError):
            continue
        if smp:
            top = sorted(((int(d[k] or 0), k.replace("stall_", "")) for k in hdr
                          if k.startswith("stall_") and "Not Issued" not in k and (d[k] or "0").isdigit()), reverse=True)[:3]
            res.append((smp, cur, int(r[0]), r[1].strip()[:80], top))
tot = sum(x[0] for x in res) or 1
print("total samples", tot)
for smp, f, ln, src, top in sorted(res, reverse=True)[:25]:
    print(f"{smp / tot:6.1%} {f}:{ln:<4} {src:<80} {' '.join(f'{n}={v}' for v, n in top)}")
