mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -p no:warnings --durations=5 > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
timeout 900 python bench.py --no-ttt > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err
timeout 600 python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1; echo "rc=$?" >> gpurun_out/smoke.log
