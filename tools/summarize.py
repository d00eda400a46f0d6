"""Summaries of gpurun_out artefacts: bench JSON line, ncu launch list (one step)."""
import collections
import csv
import json
import sys


def bench(path):
    d = json.loads(open(path).read().strip().splitlines()[-1])
    print(f"value {d['value']:.0f} tok/s  ms/step {d['ms_per_step']:.3f}  model TFLOP/s {d['model_tflops']:.1f}  "
          f"e2e {d['e2e']['value']:.0f}  clocks {d['clocks']}")
    for k, v in sorted(d['kernels'].items(), key=lambda kv: -kv[1]['ms_per_step']):
        print(f"  {k:14s} {v['ms_per_step']:7.3f} ms {v['share']*100:5.1f}% {v['achieved']:8.1f} {v['unit']:7s} "
              f"frac {v['frac']:.2f} launches {v['launches_per_step']:.0f}")


def launches(path, top=30):
    rows = list(csv.reader(open(path)))
    hdr, data = None, []
    for r in rows:
        if r and r[0] == 'ID':
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            data.append(dict(zip(hdr, r)))
    agg = collections.defaultdict(lambda: [0, 0.0])
    for d in data:
        name = d['Kernel Name'].replace('(anonymous namespace)::', '')[:80]
        agg[name][0] += 1
        agg[name][1] += float(d['Metric Value'])
    tot = sum(v[1] for v in agg.values())
    print(f"{len(data)} launches, total {tot/1e3:.1f} us (ncu, serialised)")
    for k, v in sorted(agg.items(), key=lambda kv: -kv[1][1])[:top]:
        print(f"  {v[1]/1e3:9.1f} us {100*v[1]/tot:5.1f}% n={v[0]:4d} avg {v[1]/1e3/v[0]:7.1f} {k}")


if __name__ == "__main__":
    import signal
    signal.signal(signal.SIGPIPE, signal.SIG_DFL)
    for p in sys.argv[1:]:
        (bench if p.endswith('.log') or p.endswith('.json') else launches)(p)
