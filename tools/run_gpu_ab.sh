#!/bin/bash
# A/B of in-tree library variants (QDT_LIB): quick parity subset + Megascale / paper-shape kernel times
mkdir -p gpurun_out
L=paper_2404_02844_b200
for v in "" _nomin _noxn _both; do
  lib=$PWD/$L/libqdt$v.so
  echo "== variant ${v:-default}"
  QDT_LIB=$lib timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -p no:warnings -k "tiny or medium or fista or wide_sweep_parity or megascale" 2>&1 | tail -1
  for c in megascale paper_tmd; do
    QDT_LIB=$lib timeout 600 python bench.py --config $c --steps 100 --warmup 5 --no-cpu --no-ttt --no-e2e 2>/dev/null | tail -1 > gpurun_out/ab_${c}${v}.json
    python -c "
import json; d=json.load(open('gpurun_out/ab_${c}${v}.json')); k=d['kernels']; print('$c', round(d['ms_per_step'],4), 'bwd', round(k['bwd_step']['avg_ms'],4), 'fwd', round(k['fwd_partial']['avg_ms'],4))"
  done
done
