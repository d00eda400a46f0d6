"""Summarise an NNT_PARITY_LOG file (one JSON line per gpu_util.close call): per test and
tolerance, the largest norm-wise and element-wise error as a fraction of its bound.

    python tools/parity_summary.py gpurun_out/parity.jsonl > profiles/r2_parity_log_summary.txt
"""
import collections
import json
import sys


def main(path):
    rows = [json.loads(l) for l in open(path)]
    worst = collections.defaultdict(lambda: [0.0, 0.0, 0])
    for r in rows:
        test = r["test"].split("[")[0]
        k = (test, r["tol"])
        w = worst[k]
        w[0] = max(w[0], r["rel"] / r["tol"])
        if r["max_tol"] not in (None, float("inf")) and r["max_tol"] < 1e300:
            w[1] = max(w[1], r["rel_max"] / r["max_tol"])
        w[2] += 1
    print(f"{len(rows)} comparisons; columns: max(norm rel / tol), max(elementwise rel / max_tol), count, test, tol")
    for (test, tol), (a, b, n) in sorted(worst.items()):
        print(f"{a:8.3f} {b:8.3f} {n:5d}  {test}  tol={tol:g}")


if __name__ == "__main__":
    main(sys.argv[1])
