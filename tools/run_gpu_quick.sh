# quick GPU check: parity tests + bench (no ncu)
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x --durations=8 -p no:warnings > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py --no-cpu --no-ttt > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?" >> gpurun_out/bench.err
