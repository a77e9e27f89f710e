"""Top CUDA source lines of an ncu report by warp-stall samples and instructions executed.

    python tools/ncu_source.py report.ncu-rep [top]
"""
import csv
import io
import os
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
data, fname, h = [], "?", None
for r in csv.reader(io.StringIO(out)):
    if not r:
        continue
    if r[0] == "File Path":
        fname = os.path.basename(r[1])
        continue
    if r[0] == "Line No":
        h = r
        si, ii = h.index("Warp Stall Sampling (All Samples)"), h.index("Instructions Executed")
        continue
    if h is None or len(r) <= max(si, ii) or r[2] != "-":
        continue
    try:
        s, n = float(r[si] or 0), float(r[ii] or 0)
    except ValueError:
        continue
    data.append((s, n, f"{fname}:{r[0]}", r[1].strip()[:100]))
ts = sum(d[0] for d in data) or 1
tn = sum(d[1] for d in data) or 1
print(f"# {rep}: {ts:.0f} stall samples, {tn:.0f} warp instructions")
for s, n, l, t in sorted(data, reverse=True)[:top]:
    print(f"{100 * s / ts:5.1f}% smp {100 * n / tn:5.1f}% ins  {l:<16} {t}")
