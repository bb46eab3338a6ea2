#!/bin/bash
mkdir -p gpurun_out
python -c "from paper_2404_02844_b200 import build; build.build()" || exit 1
timeout 1500 python -m pytest tests -m gpu -x -q -p no:warnings 2>&1 | tail -3
for r in 1 2 3; do
  timeout 600 python bench.py --steps 200 --warmup 10 --no-cpu --no-ttt --no-e2e 2>/dev/null | tail -1 > gpurun_out/cache$r.json
  python -c "
import json; d=json.load(open('gpurun_out/cache$r.json')); print('run $r', round(d['ms_per_step'],4), round(d['loop_ms_per_step'],4), d['value'])"
done
timeout 900 python bench.py > gpurun_out/bench_cache.json 2> gpurun_out/bench_cache.err; tail -1 gpurun_out/bench_cache.json | cut -c1-400
