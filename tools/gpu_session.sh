# One GPU round trip: smoke, GPU tests (TESTS, empty = skip), bench (BENCH, empty = skip),
# ncu launch list + one --set full capture (NCU=1; CFG/KERNEL/TAG as in gpu_profile.sh) with the
# source page (per-line stall samples).
mkdir -p gpurun_out
{ nproc; nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv; } > gpurun_out/host.txt 2>&1
timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
if [ -n "$TESTS" ]; then
  timeout ${PYTEST_TIMEOUT:-2400} python -m pytest $TESTS -q --durations=10 -p no:warnings \
    > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
fi
if [ -n "$BENCH" ]; then
  timeout 900 python bench.py $BENCH > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?" >> gpurun_out/bench.err
fi
if [ -n "$NCU" ]; then
  bash tools/gpu_profile.sh
  TAG=${TAG:-${CFG:-megascale}}
  ncu -i /tmp/prof_$TAG.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/${TAG}_source.csv 2>&1
  python tools/ncu_src_summary.py gpurun_out/${TAG}_source.csv 40 > gpurun_out/${TAG}_src_summary.txt 2>&1
  python tools/ncu_details_summary.py gpurun_out/${TAG}_details.csv > gpurun_out/${TAG}_summary.txt 2>&1
  grep -i "stall\|warp state" gpurun_out/${TAG}_details.csv | head -60 > gpurun_out/${TAG}_stalls.txt
  rm -f gpurun_out/${TAG}_source.csv
fi
