mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_wide.py -q -x -p no:warnings -k "not stress_shaped" > gpurun_out/wide.log 2>&1; echo "rc=$?" >> gpurun_out/wide.log
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -p no:warnings -k "wide or odd or shape or paper_tmd or stress_cut or large" > gpurun_out/wide2.log 2>&1; echo "rc=$?" >> gpurun_out/wide2.log
