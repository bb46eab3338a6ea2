#!/bin/bash
set -x
mkdir -p gpurun_out
python -c "from paper_2404_02844_b200 import build; build.build()" || exit 1
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "wide or odd or paper_tmd or shape or early" 2>&1 | tail -5
timeout 600 python bench.py --config paper_tmd --steps 50 --warmup 5 --no-cpu --no-ttt > gpurun_out/paper_tmd_bench3.json 2> gpurun_out/paper_tmd_bench3.err; tail -3 gpurun_out/paper_tmd_bench3.err
cat gpurun_out/paper_tmd_bench3.json
QDT_WIDE_PLAIN=1 timeout 600 python bench.py --config paper_tmd --steps 50 --warmup 5 --no-cpu --no-ttt --no-e2e 2>&1 | tail -1
timeout 900 python tools/paper_tmd_fidelity.py --D 1076 --tols 1e-6,1e-7,1e-8 > gpurun_out/fid1076.json 2>&1; cat gpurun_out/fid1076.json
