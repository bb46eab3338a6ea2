#!/bin/bash
# forward DMMA: two accumulator chains (default) vs one chain (QDT_FWD_ONECHAIN build)
mkdir -p gpurun_out
L=paper_2404_02844_b200
python -c "from paper_2404_02844_b200 import build; build.build()" || exit 1
timeout 1200 python -m pytest tests -m gpu -x -q -p no:warnings 2>&1 | tail -2
for r in 1 2; do for v in "" _onechain; do
  for c in megascale medium large; do
    QDT_LIB=$PWD/$L/libqdt$v.so timeout 600 python bench.py --config $c --steps 200 --warmup 10 --no-cpu --no-ttt --no-e2e 2>/dev/null | tail -1 > gpurun_out/fwd2_${c}${v}.json
    python -c "
import json; d=json.load(open('gpurun_out/fwd2_${c}${v}.json')); k=d['kernels']; print('${v:-twochain}', '$c', round(d['ms_per_step'],4), 'bwd', round(k['bwd_step']['avg_ms'],4), 'fwd', round(k['fwd_partial']['avg_ms'],4))"
  done
done; done
