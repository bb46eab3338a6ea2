"""SASS opcode histogram (executed warp instructions) of an ncu source-page CSV export.
usage: python tools/ncu_sass_hist.py prof_source.csv [top]"""
import collections
import csv
import re
import sys

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
hdr = None
cnt = collections.Counter()
tot = 0
for r in rows:
    if r and r[0] == "Line No":
        hdr = r
        iI = hdr.index("Instructions Executed")
        continue
    if hdr is None or len(r) <= iI:
        continue
    if r[0] == "" and r[2].startswith("0x"):
        m = re.match(r"(@!?U?P\w+\s+)?([A-Z0-9_]+)", r[3].strip())
        if not m:
            continue
        try:
            n = int(r[iI] or 0)
        except ValueError:
            continue
        cnt[m.group(2)] += n
        tot += n
print("total", tot)
for op, n in cnt.most_common(top):
    print(f"{op:12s} {n:12d} {100 * n / tot:5.1f}%")
