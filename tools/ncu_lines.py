"""Summarise an ncu report's source page per CUDA source line (stall samples, instructions).
usage: python tools/ncu_lines.py report.ncu-rep [top]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = None
agg = {}
for r in rows:
    if len(r) > 5 and r[0] == "Line No":
        hdr = r
        iW = hdr.index("Warp Stall Sampling (All Samples)")
        iI = hdr.index("Instructions Executed")
        continue
    if hdr is None or len(r) != len(hdr) or not r[0]:
        continue
    try:
        agg[int(r[0])] = (int(r[iW] or 0), int(r[iI] or 0), r[1][:100])
    except ValueError:
        pass
tw = sum(v[0] for v in agg.values()) or 1
ti = sum(v[1] for v in agg.values()) or 1
print(f"total stall samples {tw}, instructions {ti}")
for ln, (w, i, s) in sorted(agg.items(), key=lambda x: -x[1][0])[:top]:
    print(f"{100*w/tw:5.1f}% smp {100*i/ti:5.1f}% ins  L{ln:<5d} {s}")


def ranges(agg, spans):
    """Aggregate (samples, instructions) over named line ranges."""
    tw = sum(v[0] for v in agg.values()) or 1
    ti = sum(v[1] for v in agg.values()) or 1
    for name, (a, b) in spans.items():
        w = sum(v[0] for k, v in agg.items() if a <= k <= b)
        i = sum(v[1] for k, v in agg.items() if a <= k <= b)
        print(f"{name:24s} {100*w/tw:5.1f}% smp {100*i/ti:5.1f}% ins  ({i:.3e})")
