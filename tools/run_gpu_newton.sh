#!/bin/bash
mkdir -p gpurun_out
python -c "from paper_2404_02844_b200 import build; build.build()" || exit 1
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -p no:warnings -k "newton" 2>&1 | tail -30
