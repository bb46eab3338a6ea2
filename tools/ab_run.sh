mkdir -p gpurun_out
timeout 300 python tools/ab_config.py megascale 16,200 scal_mb > gpurun_out/ab_mega.jsonl 2>>gpurun_out/ab_err.log
timeout 300 python tools/ab_config.py medium 16,200 medium >> gpurun_out/ab_mega.jsonl 2>>gpurun_out/ab_err.log
timeout 300 python tools/small_ab.py > gpurun_out/small_ab.jsonl 2>&1
timeout 2400 python -m pytest tests -m gpu -x -q -p no:warnings --durations=5 > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
