# full check: smoke, all GPU tests, default bench (+ cpu baseline + time-to-tol), launch list, ncu of bwd/fwd
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > gpurun_out/gpu.txt 2>&1
timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 1500 python -m pytest tests -m gpu -q --durations=10 -p no:warnings > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?" >> gpurun_out/bench.err
CMD="python bench.py --steps 4 --warmup 3 --no-cpu --no-e2e --no-ttt"
timeout 300 $CMD > gpurun_out/plain_small.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 300 --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_list.log 2>&1; echo "ncu list rc=$?" >> gpurun_out/ncu_list.log
for k in bwd_mma fwd_mma; do
  timeout 900 ncu -f --set full --clock-control none --import-source on -k regex:k_$k -s 4 -c 1 -o /tmp/prof_$k $CMD > gpurun_out/ncu_$k.log 2>&1; echo "ncu $k rc=$?" >> gpurun_out/ncu_$k.log
  ncu -i /tmp/prof_$k.ncu-rep --page raw --csv > gpurun_out/prof_${k}_raw.csv 2>&1
  ncu -i /tmp/prof_$k.ncu-rep --page details --csv > gpurun_out/prof_${k}_details.csv 2>&1
  ncu -i /tmp/prof_$k.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/prof_${k}_source.csv 2>&1
done
# the paper's shape (M = 1 210 581, N = 151): bench line, fidelity report, ncu of the NB = 19 step
timeout 900 python bench.py --config paper_tmd --steps 100 --warmup 5 --no-cpu --no-ttt > gpurun_out/bench_paper_tmd.json 2> gpurun_out/bench_paper_tmd.err
timeout 900 python tools/paper_tmd_fidelity.py --D 1076 --gamma 1e-5 --tols 1e-6,1e-7,1e-8 > gpurun_out/fid1076.json 2>&1
timeout 900 python tools/paper_tmd_fidelity.py --D 1076 --gamma 1e-5 --tols 1e-8 --smooth > gpurun_out/fid1076_smooth.json 2>&1
CMD2="python bench.py --config paper_tmd --steps 4 --warmup 3 --no-cpu --no-e2e --no-ttt"
timeout 900 ncu -f --set full --clock-control none --import-source on -k regex:k_bwd_mma -s 4 -c 1 -o /tmp/prof_bwd_tmd $CMD2 > gpurun_out/ncu_bwd_tmd.log 2>&1; echo "ncu rc=$?" >> gpurun_out/ncu_bwd_tmd.log
ncu -i /tmp/prof_bwd_tmd.ncu-rep --page raw --csv > gpurun_out/prof_bwd_tmd_raw.csv 2>&1
ncu -i /tmp/prof_bwd_tmd.ncu-rep --page details --csv > gpurun_out/prof_bwd_tmd_details.csv 2>&1
