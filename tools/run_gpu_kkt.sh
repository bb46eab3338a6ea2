#!/bin/bash
mkdir -p gpurun_out
python -c "from paper_2404_02844_b200 import build; build.build()" || exit 1
for ke in 1 16; do
  timeout 600 python bench.py --steps 200 --warmup 10 --no-cpu --no-ttt --kkt-every $ke 2>/dev/null | tail -1 > gpurun_out/kkt$ke.json
  python -c "
import json; d=json.load(open('gpurun_out/kkt$ke.json')); k=d['kernels']; print('kkt_every $ke', round(d['ms_per_step'],4), 'bwd', round(k['bwd_step']['avg_ms'],4), 'fwd', round(k['fwd_partial']['avg_ms'],4), 'e2e', d['e2e']['value'])"
done
