# round-1 re-entry: tests + smoke + bench + fp64 peak + ncu launch list + ncu full (k_bwd)
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > gpurun_out/gpu.txt 2>&1
timeout 60 ./tools/fp64_peak > gpurun_out/fp64_peak.json 2>&1
timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 1200 python -m pytest tests -m gpu -q -x --durations=15 -p no:warnings > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?" >> gpurun_out/bench.err
CMD="python bench.py --steps 4 --warmup 3 --no-cpu --no-e2e"
timeout 300 $CMD > gpurun_out/plain_small.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_list.log 2>&1; echo "ncu list rc=$?" >> gpurun_out/ncu_list.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_bwd -s 6 -c 1 -o gpurun_out/prof_bwd $CMD > gpurun_out/ncu_bwd.log 2>&1; echo "ncu bwd rc=$?" >> gpurun_out/ncu_bwd.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_fwd -s 6 -c 1 -o gpurun_out/prof_fwd $CMD > gpurun_out/ncu_fwd.log 2>&1; echo "ncu fwd rc=$?" >> gpurun_out/ncu_fwd.log
