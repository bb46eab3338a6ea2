#!/bin/bash
# FISTA split kernel with the tensor-copy tile: GPU tests + time-to-tol A/B (QDT_TMA_TILE=1/0)
mkdir -p gpurun_out
python -c "from paper_2404_02844_b200 import build; build.build()" || exit 1
timeout 1200 python -m pytest tests -m gpu -x -q -p no:warnings 2>&1 | tail -2
for v in 1 0 1 0; do
  QDT_TMA_TILE=$v timeout 600 python bench.py --no-cpu --no-e2e 2>/dev/null | tail -1 > gpurun_out/tp2_$v.json
  python -c "
import json; d=json.load(open('gpurun_out/tp2_$v.json')); t=d['time_to_tol']['modes']['SQS-FISTA']; print('tma_tile=$v', round(d['ms_per_step'],4), 'bwd', round(d['kernels']['bwd_step']['avg_ms'],4), {r:(x['iters'], round(x['seconds'],3), round(x['loop_ms_per_iter'],4)) for r,x in t.items()})"
done
