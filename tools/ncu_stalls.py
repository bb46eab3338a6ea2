"""Warp-stall breakdown and pipe utilisation of one kernel from an ncu `--page raw --csv` export.
usage: python tools/ncu_stalls.py raw.csv"""
import csv
import sys

KEYS = ["gpu__time_duration.sum", "smsp__inst_executed.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__warps_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active"]
rows = list(csv.reader(open(sys.argv[1])))
hdr = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
H, U, V = rows[hdr], rows[hdr + 1], rows[hdr + 2]
d = {h: (x, u) for h, u, x in zip(H, U, V)}
print(d.get("Kernel Name", ("?",))[0])
for k in KEYS:
    if k in d:
        print(f"  {k:80s} {d[k][0]} {d[k][1]}")
st = []
for h, (val, _) in d.items():
    if "warps_issue_stalled" in h and h.endswith("per_issue_active.ratio") and "not_issued" not in h:
        try:
            st.append((float(val.replace(",", "")), h))
        except ValueError:
            pass
print("  warp stall cycles per issued instruction:")
for x, h in sorted(st, reverse=True)[:14]:
    name = h.replace("smsp__average_warps_issue_stalled_", "").replace("_per_issue_active.ratio", "")
    print(f"    {x:7.3f} {name}")
