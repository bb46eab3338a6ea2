mkdir -p gpurun_out
for dbg in 0 1 2 3; do
QDT_DEBUG_BWD=$dbg timeout 300 python bench.py --no-cpu --no-e2e --steps 30 > gpurun_out/bench_dbg$dbg.json 2>> gpurun_out/bench.err
done
