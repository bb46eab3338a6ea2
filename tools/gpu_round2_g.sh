mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -p no:warnings --durations=5 > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
bash tools/gpu_sanitize.sh
