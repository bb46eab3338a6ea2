"""Key lines of an ncu `--page details --csv` export.  usage: python tools/ncu_details_summary.py f.csv"""
import csv
import sys

KEEP = ("GPU Speed Of Light Throughput", "Memory Workload Analysis", "Occupancy", "Launch Statistics",
        "Scheduler Statistics", "Warp State Statistics", "Compute Workload Analysis")
NAMES = ("Duration", "DRAM Throughput", "Memory Throughput", "L1/TEX Cache Throughput",
         "L2 Cache Throughput", "Compute (SM) Throughput", "Executed Ipc Active", "Issue Slots Busy",
         "L2 Hit Rate", "L1/TEX Hit Rate", "Mem Busy", "Max Bandwidth", "Eligible Warps Per Scheduler",
         "No Eligible", "Achieved Active Warps Per SM", "Theoretical Occupancy", "Registers Per Thread",
         "Dynamic Shared Memory Per Block", "Grid Size", "Block Size", "Warp Cycles Per Issued Instruction",
         "Block Limit Registers", "Block Limit Shared Mem")
rows = list(csv.reader(open(sys.argv[1])))
h = rows[0]
iS, iM, iU, iV = (h.index(x) for x in ("Section Name", "Metric Name", "Metric Unit", "Metric Value"))
print(rows[1][h.index("Kernel Name")])
for r in rows[1:]:
    if len(r) > iV and r[iS] in KEEP and r[iM] in NAMES:
        print(f"  {r[iM]:40s} {r[iV]:>14s} {r[iU]}")
