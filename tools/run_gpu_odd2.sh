#!/bin/bash
set -x
mkdir -p gpurun_out
python -c "from paper_2404_02844_b200 import build; build.build()" || exit 1
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "wide or odd or paper_tmd or shape or large" 2>&1 | tail -5
timeout 600 python bench.py --config paper_tmd --steps 50 --warmup 5 --no-cpu --no-ttt > gpurun_out/paper_tmd_bench2.json 2> gpurun_out/paper_tmd_bench2.err; tail -3 gpurun_out/paper_tmd_bench2.err
cat gpurun_out/paper_tmd_bench2.json
timeout 600 python bench.py --config large --steps 50 --warmup 5 --no-cpu --no-ttt > gpurun_out/large_bench2.json 2>&1
cat gpurun_out/large_bench2.json | tail -1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/paper_tmd_launches.csv python bench.py --config paper_tmd --steps 3 --warmup 3 --no-cpu --no-ttt --no-e2e > /dev/null 2>&1
python - <<'PY'
import csv, collections
rows = list(csv.reader(open("gpurun_out/paper_tmd_launches.csv")))
h = None; agg = collections.defaultdict(list)
for r in rows:
    if "Kernel Name" in r: h = r; continue
    if h and len(r) == len(h):
        d = dict(zip(h, r))
        agg[d["Kernel Name"][:60]].append(float(d["Metric Value"]))
for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
    print(f"{k:60s} n={len(v):3d} avg={sum(v)/len(v)/1e3:9.1f} us")
PY
