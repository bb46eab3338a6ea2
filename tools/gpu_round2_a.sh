mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_virtual.py -q -x -p no:warnings --durations=5 > gpurun_out/virtual.log 2>&1; echo "rc=$?" >> gpurun_out/virtual.log
timeout 900 python bench.py --config stress --steps 50 --warmup 3 --no-cpu --no-ttt > gpurun_out/bench_stress.json 2> gpurun_out/bench_stress.err; echo "rc=$?" >> gpurun_out/bench_stress.err
CFG=stress_cut KERNEL=k_wstep TAG=wstep_cut STEPS=4 NLAUNCH=100 timeout 1500 bash tools/gpu_profile.sh
ncu -i /tmp/prof_wstep_cut.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/wstep_cut_source.csv 2>&1
