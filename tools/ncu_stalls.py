"""Stall-reason totals (and top SASS lines per reason) per kernel from an ncu report's source page.

    python tools/ncu_stalls.py report.ncu-rep [N] [kernel-substring]
"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 8
only = sys.argv[3] if len(sys.argv) > 3 else None
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
sections, cur = [], None
i = 0
while i < len(rows):
    r = rows[i]
    if r and r[0] == "Kernel Name":
        cur = {"name": r[1], "hdr": rows[i + 1], "data": []}
        sections.append(cur)
        i += 2
        continue
    if cur is not None and len(r) == len(cur["hdr"]):
        cur["data"].append(r)
    i += 1
seen = set()
for sec in sections:
    name = sec["name"].split("(")[0]
    if (only and only not in name) or name in seen:
        continue
    seen.add(name)
    hdr, data = sec["hdr"], sec["data"]
    idx = {h: j for j, h in enumerate(hdr)}
    cols = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
    tot = {c: sum(float(r[idx[c]] or 0) for r in data) for c in cols}
    allsum = sum(tot.values()) or 1
    print(f"== {name}: stall reason totals (% of samples)")
    for c, v in sorted(tot.items(), key=lambda kv: -kv[1]):
        if v > 0:
            print(f"  {c:24s} {100 * v / allsum:5.1f}%")
    for c, v in sorted(tot.items(), key=lambda kv: -kv[1])[:3]:
        print(f"  top lines for {c}:")
        for r in sorted(data, key=lambda r: -float(r[idx[c]] or 0))[:n]:
            print(f"   {100 * float(r[idx[c]]) / allsum:5.1f}%  {r[idx['Address']][-5:]} {r[idx['Source']].strip()[:90]}")
