#!/usr/bin/env python3
"""Summarise an .ncu-rep (raw page) into the handful of metrics we track."""
import csv
import subprocess
import sys

WANT = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "launch__grid_size", "launch__occupancy_limit_registers",
        "sm__inst_executed.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "smsp__thread_inst_executed_per_inst_executed.ratio", "lts__t_bytes.sum",
        "smsp__average_warp_latency_per_inst_issued.ratio"]
STALL = "smsp__average_warps_issue_stalled_"


def main(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    h, units = rows[0], rows[1]
    for r in rows[2:]:
        name = r[h.index("Kernel Name")]
        print("==", name[:90])
        for w in WANT:
            if w in h:
                print(f"  {w:62s} {r[h.index(w)]:>16s} {units[h.index(w)]}")
        stalls = [(float(r[i]), h[i][len(STALL):].replace("_per_issue_active.ratio", ""))
                  for i in range(len(h)) if h[i].startswith(STALL) and
                  h[i].endswith("_per_issue_active.ratio") and r[i] not in ("", "0")]
        stalls.sort(reverse=True)
        print("  stalls/issue:", ", ".join(f"{n}={v:.2f}" for v, n in stalls[:7]))


if __name__ == "__main__":
    for p in sys.argv[1:]:
        main(p)
