#!/bin/bash
# odd-N wide path + paper workload: targeted GPU tests, paper-shape bench, fidelity report
set -x
mkdir -p gpurun_out
python -c "from paper_2404_02844_b200 import build; build.build()" || exit 1
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "wide or odd or paper_tmd or shape" 2>&1 | tail -15
timeout 600 python bench.py --config paper_tmd --steps 50 --warmup 5 --no-cpu --no-ttt > gpurun_out/paper_tmd_bench.json 2> gpurun_out/paper_tmd_bench.err; tail -3 gpurun_out/paper_tmd_bench.err
cat gpurun_out/paper_tmd_bench.json
timeout 900 python tools/paper_tmd_fidelity.py --D 300 --tols 1e-3,1e-4,1e-5 > gpurun_out/fid300.json 2>&1; cat gpurun_out/fid300.json
timeout 900 python tools/paper_tmd_fidelity.py --D 1076 --tols 1e-3,1e-4 > gpurun_out/fid1076.json 2>&1; cat gpurun_out/fid1076.json
