"""Hottest SASS instructions of an ncu report (warp-stall samples), with instruction counts.

    python profiles/sass_hot.py <report.ncu-rep> [top]
"""
import csv
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True,
                     text=True).stdout.splitlines()
rows = list(csv.reader(out[1:]))
h = rows[0]
iS, iE = h.index("Warp Stall Sampling (All Samples)"), h.index("Instructions Executed")
data = [r for r in rows[1:] if len(r) == len(h)]
tot = sum(float(r[iS] or 0) for r in data)
tot_e = sum(float(r[iE] or 0) for r in data)
print(f"samples {tot:.0f}  warp-instructions {tot_e:.3g}")
for r in sorted(data, key=lambda r: -float(r[iS] or 0))[:top]:
    print(f"{r[0]:>6} {float(r[iS] or 0) / tot * 100:5.1f}% exec={r[iE]:>10}  {r[1][:90]}")
