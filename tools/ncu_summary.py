"""One-paragraph summaries of ncu --set full reports: duration, clocks, DRAM / L2 / L1<-L2 traffic,
tensor-pipe activity, issue activity and the top stall reasons.

    python tools/ncu_summary.py report.ncu-rep [...]
"""
import csv
import io
import subprocess
import sys

KEYS = [("gpu__time_duration.sum", "duration us"), ("sm__cycles_elapsed.avg.per_second", "SM GHz"),
        ("dram__bytes_read.sum", "DRAM read MB"), ("dram__bytes_write.sum", "DRAM write MB"),
        ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "DRAM % of peak"),
        ("lts__throughput.avg.pct_of_peak_sustained_elapsed", "L2 % of peak"),
        ("l1tex__m_xbar2l1tex_read_bytes.sum", "L2->SM read GB"),
        ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed", "tensor pipe % elapsed"),
        ("sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active", "XU (MUFU) % active"),
        ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue % active"),
        ("sm__warps_active.avg.pct_of_peak_sustained_active", "occupancy % active")]


def main():
    for rep in sys.argv[1:]:
        out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
        rows = list(csv.reader(io.StringIO(out)))
        if len(rows) < 3:
            print(rep, ": no data")
            continue
        h, units, v = rows[0], rows[1], rows[2]
        d, u = dict(zip(h, v)), dict(zip(h, units))
        name = d.get("Kernel Name", "?")[:90]
        print(f"== {rep.split('/')[-1]}: {name}")
        for k, label in KEYS:
            if k in d:
                print(f"   {label:24s} {d[k]:>14s} {u.get(k, '')}")
        st = subprocess.run([sys.executable, __file__.replace("ncu_summary.py", "ncu_stalls.py"), rep, "3"],
                            capture_output=True, text=True).stdout.splitlines()
        print("   " + "\n   ".join(l for l in st[1:6]))


if __name__ == "__main__":
    main()
