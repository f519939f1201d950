"""Print selected raw metrics from an ncu report: tools/ncu_metrics.py rep.ncu-rep [substr ...]"""
import csv
import subprocess
import sys

rep = sys.argv[1]
want = sys.argv[2:] or ["gpu__time_duration.sum", "dram__throughput.avg.pct_of_peak_sustained_elapsed",
                        "sm__warps_active.avg.pct_of_peak_sustained_active", "stalled_barrier_per_issue_active",
                        "stalled_long_scoreboard_per_issue_active", "stalled_short_scoreboard_per_issue_active",
                        "stalled_wait_per_issue_active", "stalled_lg_throttle_per_issue_active",
                        "launch__occupancy_limit", "launch__registers_per_thread",
                        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "smsp__inst_executed.sum",
                        "dram__bytes_read.sum", "dram__bytes_write.sum", "sm__pipe_tensor_cycles_active.avg.pct"]
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
h = rows[0]
for row in rows[2:]:
    print("---", row[h.index("Kernel Name")][:60])
    for i, n in enumerate(h):
        if any(w in n for w in want) and "pcsamp" not in n:
            print(f"  {n:86s} {row[i]}")
