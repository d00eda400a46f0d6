"""Stall-reason totals (and top SASS lines per reason) from an ncu report's source page.

    python tools/ncu_stalls.py report.ncu-rep [N]
"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 8
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[1]
idx = {h: i for i, h in enumerate(hdr)}
data = [r for r in rows[2:] if len(r) == len(hdr)]
cols = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
tot = {c: sum(float(r[idx[c]] or 0) for r in data) for c in cols}
allsum = sum(tot.values()) or 1
print("stall reason totals (% of samples):")
for c, v in sorted(tot.items(), key=lambda kv: -kv[1]):
    if v > 0:
        print(f"  {c:24s} {100 * v / allsum:5.1f}%")
for c, v in sorted(tot.items(), key=lambda kv: -kv[1])[:3]:
    print(f"top lines for {c}:")
    for r in sorted(data, key=lambda r: -float(r[idx[c]] or 0))[:n]:
        print(f"   {100 * float(r[idx[c]]) / allsum:5.1f}%  {r[idx['Source']].strip()[:100]}")
