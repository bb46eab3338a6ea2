# tests + bench + ncu of bwd/fwd (one gpurun call)
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x -p no:warnings > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
CMD="python bench.py --steps 4 --warmup 3 --no-cpu --no-e2e"
timeout 600 python bench.py --no-cpu --no-e2e > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?" >> gpurun_out/bench.err
timeout 300 $CMD > gpurun_out/plain_small.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_bwd -s 6 -c 1 -o gpurun_out/prof_bwd $CMD > gpurun_out/ncu_bwd.log 2>&1; echo "ncu bwd rc=$?" >> gpurun_out/ncu_bwd.log
