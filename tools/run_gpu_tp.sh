#!/bin/bash
# tensor-map Theta tile at the conflict-free pitch (QDT_TMA_TILE=1, default) vs contiguous copy (0)
mkdir -p gpurun_out
python -c "from paper_2404_02844_b200 import build; build.build()" || exit 1
timeout 1200 python -m pytest tests -m gpu -x -q -p no:warnings 2>&1 | tail -2
for r in 1 2; do for v in 1 0; do
  for c in megascale medium; do
    QDT_TMA_TILE=$v timeout 600 python bench.py --config $c --steps 200 --warmup 10 --no-cpu --no-ttt --no-e2e 2>/dev/null | tail -1 > gpurun_out/tp${v}_${c}.json
    python -c "
import json; d=json.load(open('gpurun_out/tp${v}_${c}.json')); k=d['kernels']; print('tma_tile=$v', '$c', round(d['ms_per_step'],4), 'bwd', round(k['bwd_step']['avg_ms'],4), 'fwd', round(k['fwd_partial']['avg_ms'],4))"
  done
done; done
CMD="python bench.py --steps 4 --warmup 3 --no-cpu --no-e2e --no-ttt"
timeout 900 ncu -f --set full --clock-control none -k regex:k_bwd_mma -s 4 -c 1 -o /tmp/prof_tp $CMD > gpurun_out/ncu_tp.log 2>&1; tail -1 gpurun_out/ncu_tp.log
ncu -i /tmp/prof_tp.ncu-rep --page raw --csv > gpurun_out/prof_tp_raw.csv 2>&1
ncu -i /tmp/prof_tp.ncu-rep --page details --csv > gpurun_out/prof_tp_details.csv 2>&1
