"""Summarise a full ncu capture of the Burgers Leja kernel (tools/prof_burgers.sh) in a few lines."""
import csv
import sys

details, raw, label = sys.argv[1], sys.argv[2], sys.argv[3]
keys = ["Duration", "DRAM Throughput", "Registers Per Thread", "Grid Size", "Theoretical Occupancy",
        "Achieved Occupancy", "Issue Slots Busy", "L2 Hit Rate"]
rows = list(csv.reader(open(details)))
h = {k: i for i, k in enumerate(rows[0])}
print(f"[{label}]")
name = None
for r in rows[1:]:
    name = r[h["Kernel Name"]]
    if r[h["Metric Name"]] in keys:
        print(f"  {r[h['Metric Name']]}: {r[h['Metric Value']]} {r[h['Metric Unit']]}")
print(f"  kernel: {name}")
rr = list(csv.reader(open(raw)))
for k in ["dram__bytes_read.sum", "dram__bytes_write.sum",
          "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio",
          "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
          "smsp__inst_executed.sum"]:
    if k in rr[0]:
        i = rr[0].index(k)
        print(f"  {k}: {rr[2][i]} {rr[1][i]}")
