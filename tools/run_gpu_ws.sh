#!/bin/bash
# warm-started Michelot + mask-free forward: all GPU tests, Megascale and paper-shape bench, fidelity
mkdir -p gpurun_out
python -c "from paper_2404_02844_b200 import build; build.build()" || exit 1
timeout 1500 python -m pytest tests -m gpu -x -q -p no:warnings 2>&1 | tail -4
timeout 600 python bench.py --steps 200 --warmup 10 --no-cpu --no-ttt --no-e2e 2>/dev/null | tail -1 > gpurun_out/ws_mega.json; python -c "
import json; d=json.load(open('gpurun_out/ws_mega.json')); print('mega', d['ms_per_step'], d['kernels'])"
timeout 600 python bench.py --config paper_tmd --steps 100 --warmup 5 --no-cpu --no-ttt --no-e2e 2>/dev/null | tail -1 > gpurun_out/ws_tmd.json; python -c "
import json; d=json.load(open('gpurun_out/ws_tmd.json')); print('tmd', d['ms_per_step'], d['kernels'])"
timeout 900 python tools/paper_tmd_fidelity.py --D 1076 --tols 1e-6,1e-7,1e-8 > gpurun_out/fid1076b.json 2>&1; tail -1 gpurun_out/fid1076b.json
timeout 900 python tools/paper_tmd_fidelity.py --D 1076 --tols 1e-8 --smooth > gpurun_out/fid1076b_smooth.json 2>&1; tail -1 gpurun_out/fid1076b_smooth.json
