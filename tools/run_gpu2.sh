# full GPU check + bench + ncu evidence (one gpurun call)
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q --durations=8 -p no:warnings > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?" >> gpurun_out/bench.err
CMD="python bench.py --steps 4 --warmup 3 --no-cpu --no-e2e"
timeout 300 $CMD > gpurun_out/plain_small.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_list.log 2>&1; echo "ncu list rc=$?" >> gpurun_out/ncu_list.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_bwd -s 6 -c 1 -o gpurun_out/prof_bwd $CMD > gpurun_out/ncu_bwd.log 2>&1; echo "ncu bwd rc=$?" >> gpurun_out/ncu_bwd.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_fwd -s 6 -c 1 -o gpurun_out/prof_fwd $CMD > gpurun_out/ncu_fwd.log 2>&1; echo "ncu fwd rc=$?" >> gpurun_out/ncu_fwd.log
