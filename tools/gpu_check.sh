# GPU round trip (run under gpurun from the repo root): host facts, smoke, GPU tests, bench.
#   TESTS="..."   pytest selection (default: tests -m gpu)
#   BENCH="..."   bench.py arguments (empty: skip the bench)
mkdir -p gpurun_out
{ nproc; grep -m1 "model name" /proc/cpuinfo; free -g | head -2;
  nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv; } > gpurun_out/host.txt 2>&1
timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout ${PYTEST_TIMEOUT:-2400} python -m pytest ${TESTS:-tests -m gpu} -q --durations=15 -p no:warnings \
  > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
if [ -n "$BENCH" ]; then
  timeout 900 python bench.py $BENCH > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?" >> gpurun_out/bench.err
fi
