#!/bin/bash
mkdir -p gpurun_out
python -c "from paper_2404_02844_b200 import build; build.build()" || exit 1
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -p no:warnings -k "newton" 2>&1 | tail -3
for c in medium large megascale; do
  timeout 900 python tools/newton_vs_fista.py --config $c > gpurun_out/newton_$c.json 2>&1; tail -1 gpurun_out/newton_$c.json | cut -c1-1500
done
echo "== clamp A/B"
for v in "" _clamp; do
  QDT_LIB=$PWD/paper_2404_02844_b200/libqdt$v.so timeout 600 python bench.py --steps 100 --warmup 5 --no-cpu --no-ttt --no-e2e 2>/dev/null | tail -1 > gpurun_out/ab2$v.json
  python -c "
import json; d=json.load(open('gpurun_out/ab2$v.json')); k=d['kernels']; print('${v:-default}', round(d['ms_per_step'],4), 'bwd', round(k['bwd_step']['avg_ms'],4), 'fwd', round(k['fwd_partial']['avg_ms'],4))"
done
