"""Per-kernel-class DRAM traffic of one training step, from an ncu capture.

    ncu --profile-from-start off --clock-control none --csv --log-file T.csv \
        --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \
        python tools/profile_step.py --trace trace.json
    python tools/traffic.py T.csv trace.json OUT.json

ncu lists the step's kernels in issue order (one stream); the trace gives the
library's launch scopes in the same order (class, kernels per scope), so each
ncu kernel is attributed to its scope's class.  OUT.json holds, per class, the
DRAM bytes (read + write) per launch scope -- the unit bench.py's roofline uses.
"""
import collections
import csv
import json
import sys


def load_ncu(path):
    rows = list(csv.reader(open(path)))
    hdr, kern = None, collections.OrderedDict()
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if not hdr or len(r) != len(hdr):
            continue
        d = dict(zip(hdr, r))
        k = kern.setdefault(int(d["ID"]), {"name": d["Kernel Name"]})
        v = float(d["Metric Value"].replace(",", ""))
        unit = d.get("Metric Unit", "")
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1, "usecond": 1e3,
                 "msecond": 1e6}.get(unit, 1)
        k[d["Metric Name"]] = v * scale
    return [kern[i] for i in sorted(kern)]


def main(ncu_csv, trace_json, out_json):
    kernels = load_ncu(ncu_csv)
    trace = json.load(open(trace_json))
    expanded = [(cls, si) for si, (cls, n) in enumerate(trace) for _ in range(n)]
    if len(expanded) != len(kernels):
        raise SystemExit(f"trace has {len(expanded)} kernels, ncu captured {len(kernels)}")
    agg = collections.defaultdict(lambda: {"scopes": set(), "kernels": 0, "dram_bytes": 0.0, "ncu_ns": 0.0})
    for (cls, si), k in zip(expanded, kernels):
        a = agg[cls]
        a["scopes"].add(si)
        a["kernels"] += 1
        a["dram_bytes"] += k.get("dram__bytes_read.sum", 0) + k.get("dram__bytes_write.sum", 0)
        a["ncu_ns"] += k.get("gpu__time_duration.sum", 0)
    out = {}
    for cls, a in agg.items():
        n = len(a["scopes"])
        out[cls] = {"launches": n, "kernels": a["kernels"], "dram_bytes_per_launch": a["dram_bytes"] / n,
                    "ncu_us_per_launch": a["ncu_ns"] / n / 1e3,
                    "dram_GBps_cold": a["dram_bytes"] / max(a["ncu_ns"], 1)}
    json.dump({"source": f"ncu dram__bytes_read.sum + dram__bytes_write.sum over one step ({ncu_csv})",
               "classes": out}, open(out_json, "w"), indent=1)
    for cls, v in sorted(out.items(), key=lambda kv: -kv[1]["ncu_us_per_launch"] * kv[1]["launches"]):
        print(f"{cls:14s} scopes {v['launches']:4d} {v['dram_bytes_per_launch']/1e6:9.2f} MB/launch "
              f"{v['ncu_us_per_launch']:8.1f} us/launch (cold)  {v['dram_GBps_cold']:7.1f} GB/s")


if __name__ == "__main__":
    main(*sys.argv[1:4])
