"""Compact text summary of an ncu --set full report (development tool):
duration, DRAM bytes, issue / pipe utilisation, occupancy and the stall
reasons per issued instruction of every profiled kernel.
usage: python tools/dev/ncu_summary.py REPORT.ncu-rep [--name-filter k_join]"""
import csv
import io
import subprocess
import sys

WANT = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "dram read"),
    ("dram__bytes_write.sum", "dram write"),
    ("sm__inst_issued.avg.pct_of_peak_sustained_active", "issue slots busy %"),
    ("sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active", "FP64 pipe %"),
    ("sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active", "FMA pipe %"),
    ("sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active", "ALU pipe %"),
    ("sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "LSU pipe %"),
    ("sm__warps_active.avg.per_cycle_active", "warps active / SM"),
    ("launch__registers_per_thread", "registers"),
    ("smsp__inst_executed.sum", "warp instructions"),
]


def main():
    rep = sys.argv[1]
    filt = sys.argv[sys.argv.index("--name-filter") + 1] if "--name-filter" in sys.argv else ""
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    head, units, data = rows[0], rows[1], rows[2:]
    col = {n: i for i, n in enumerate(head)}
    for r in data:
        name = r[col["Kernel Name"]]
        if filt not in name:
            continue
        print(name[:110])
        for key, label in WANT:
            if key in col:
                print(f"  {label:22s} {r[col[key]]:>18s} {units[col[key]]}")
        stalls = []
        for n, i in col.items():
            if n.startswith("smsp__average_warps_issue_stalled_") and n.endswith("_per_issue_active.ratio"):
                try:
                    v = float(r[i].replace(",", ""))
                except ValueError:
                    continue
                if v >= 0.05:
                    stalls.append((v, n[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]))
        print("  stalls per issued instruction: " + ", ".join(f"{k} {v:.2f}" for v, k in sorted(stalls, reverse=True)))


if __name__ == "__main__":
    main()
