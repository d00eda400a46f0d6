"""Top SASS lines by warp-stall samples from an ncu report (source page).

    python tools/ncu_hot.py report.ncu-rep [N]
"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[1]
idx = {h: i for i, h in enumerate(hdr)}
data = [r for r in rows[2:] if len(r) == len(hdr)]
sc = idx["Warp Stall Sampling (All Samples)"]
tot = sum(float(r[sc] or 0) for r in data) or 1
print(f"{len(data)} SASS lines, {tot:.0f} samples")
for i, r in enumerate(data):
    r.append(i)
for r in sorted(data, key=lambda r: -float(r[sc] or 0))[:n]:
    print(f"{100 * float(r[sc]) / tot:5.1f}%  [{r[-1]:5d}] {r[idx['Source']].strip()[:110]}")
