mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x -p no:warnings -k "fista or tiny or medium" > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
for m in 0 2; do
QDT_SPLITN=$m timeout 600 python bench.py --no-cpu --no-e2e --steps 20 > gpurun_out/bench_split$m.json 2>> gpurun_out/bench.err
done
