"""Per-SASS-line instruction counts and stall samples from an ncu report, in address order,
grouped into runs: shows where a kernel's executed instructions and samples go.

    python tools/ncu_lines.py report.ncu-rep [min_share_percent]
"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
thr = float(sys.argv[2]) if len(sys.argv) > 2 else 0.5
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[1]
idx = {h: i for i, h in enumerate(hdr)}
data = [r for r in rows[2:] if len(r) == len(hdr)]
ie = [float(r[idx["Instructions Executed"]] or 0) for r in data]
sm = [float(r[idx["Warp Stall Sampling (All Samples)"]] or 0) for r in data]
tot_i, tot_s = sum(ie) or 1, sum(sm) or 1
print(f"{len(data)} SASS lines, {tot_i:.0f} warp instructions, {tot_s:.0f} samples")
for r, i, s in zip(data, ie, sm):
    if 100 * i / tot_i >= thr or 100 * s / tot_s >= thr:
        print(f"{r[idx['Address']]:>8s} inst {100 * i / tot_i:5.1f}% samp {100 * s / tot_s:5.1f}%  "
              f"{r[idx['Source']].strip()[:80]}")
