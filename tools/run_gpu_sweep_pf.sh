mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -q -x -p no:warnings > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
for pf in 0 148 296 592; do
QDT_PF_AHEAD=$pf timeout 300 python bench.py --no-cpu --no-e2e --steps 50 > gpurun_out/bench_pf$pf.json 2>> gpurun_out/bench.err
done
