mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_round2.py tests/test_gpu_virtual.py -q -x -p no:warnings -k "tiny or early or edge or shape or resume or banded or binding or small or virtual or bb_step" > gpurun_out/tiny_tests.log 2>&1; echo "rc=$?" >> gpurun_out/tiny_tests.log
timeout 900 python bench.py --config tiny --steps 2000 --warmup 5 --no-cpu --no-ttt > gpurun_out/bench_tiny.json 2> gpurun_out/bench_tiny.err
