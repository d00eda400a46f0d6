"""Top stall-sampled SASS lines with context from an ncu source CSV (ncu -i rep --page source --csv
--print-source sass > f.csv).   python tools/sass_top.py f.csv [n] [ctx]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
n = int(sys.argv[2]) if len(sys.argv) > 2 else 6
ctx = int(sys.argv[3]) if len(sys.argv) > 3 else 6
hdr = rows[1]
idx = {h: i for i, h in enumerate(hdr)}
data = [r for r in rows[2:] if len(r) == len(hdr)]
samp = [float(r[idx["Warp Stall Sampling (All Samples)"]] or 0) for r in data]
inst = [float(r[idx["Instructions Executed"]] or 0) for r in data]
tot, toti = sum(samp) or 1, sum(inst) or 1
print(f"{len(data)} lines, {toti:.0f} warp inst, {tot:.0f} samples")
for i in sorted(range(len(data)), key=lambda i: -samp[i])[:n]:
    print(f"=== line {i} {100 * samp[i] / tot:.1f}%")
    for j in range(max(0, i - ctx), min(len(data), i + 2)):
        print(f"{j:5d} {100 * samp[j] / tot:5.1f}% {100 * inst[j] / toti:5.2f}%i {data[j][idx['Source']][:100]}")
