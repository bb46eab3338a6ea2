#!/bin/bash
# A/B: padded Theta-tile pitch (QDT_TH_TMA) vs default
mkdir -p gpurun_out
L=paper_2404_02844_b200
python -c "from paper_2404_02844_b200 import build; build.build()" || exit 1
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -p no:warnings 2>&1 | tail -2
QDT_LIB=$PWD/$L/libqdt_tma.so timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -p no:warnings 2>&1 | tail -2
QDT_SPLITN=1 QDT_LIB=$PWD/$L/libqdt_tma.so timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -p no:warnings -k "fista_sweep or tiny or medium" 2>&1 | tail -1
for v in "" _tma "" _tma; do
  lib=$PWD/$L/libqdt$v.so
  for c in megascale medium; do
    QDT_LIB=$lib timeout 600 python bench.py --config $c --steps 200 --warmup 10 --no-cpu --no-ttt --no-e2e 2>/dev/null | tail -1 > gpurun_out/ab4_${c}${v}.json
    python -c "
import json; d=json.load(open('gpurun_out/ab4_${c}${v}.json')); k=d['kernels']; print('${v:-default}', '$c', round(d['ms_per_step'],4), 'bwd', round(k['bwd_step']['avg_ms'],4), 'fwd', round(k['fwd_partial']['avg_ms'],4))"
  done
done
CMD="python bench.py --steps 4 --warmup 3 --no-cpu --no-e2e --no-ttt"
QDT_LIB=$PWD/$L/libqdt_tma.so timeout 900 ncu -f --set full --clock-control none -k regex:k_bwd_mma -s 4 -c 1 -o /tmp/prof_tma $CMD > gpurun_out/ncu_tma.log 2>&1; tail -1 gpurun_out/ncu_tma.log
ncu -i /tmp/prof_tma.ncu-rep --page raw --csv > gpurun_out/prof_tma_raw.csv 2>&1
ncu -i /tmp/prof_tma.ncu-rep --page details --csv > gpurun_out/prof_tma_details.csv 2>&1
