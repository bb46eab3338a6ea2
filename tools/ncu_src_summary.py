"""Per-source-line summary of an ncu `--page source --csv --print-source cuda,sass` export:
stall samples and executed warp instructions per CUDA line (top N).
usage: python tools/ncu_src_summary.py prof_source.csv [top]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
agg = {}
hdr = None
for r in rows:
    if r and r[0] == "Line No":
        hdr = r
        iW, iI = hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Instructions Executed")
        continue
    if hdr is None or not r or not r[0].isdigit():
        continue
    try:
        agg[int(r[0])] = (int(r[iW] or 0), int(r[iI] or 0), r[1][:90])
    except ValueError:
        pass
tw = sum(v[0] for v in agg.values()) or 1
ti = sum(v[1] for v in agg.values()) or 1
print(f"total stall samples {tw}, warp instructions {ti:.4e}")
for ln, (w, i, s) in sorted(agg.items(), key=lambda x: -x[1][0])[:top]:
    print(f"{100*w/tw:5.1f}% smp {100*i/ti:5.1f}% ins  L{ln:<5d} {s}")
