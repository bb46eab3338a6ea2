mkdir -p gpurun_out
for c in tiny medium; do
  timeout 900 python bench.py --config $c --steps 200 --warmup 5 --no-cpu --no-ttt > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err
done
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -p no:warnings -k "tiny or early or smoke or edge or shape" > gpurun_out/tiny_tests.log 2>&1; echo "rc=$?" >> gpurun_out/tiny_tests.log
CFG=megascale KERNEL=k_bwd_mma TAG=mega STEPS=4 NLAUNCH=300 timeout 1500 bash tools/gpu_profile.sh
CFG=stress_cut KERNEL=k_wstep TAG=wstep_cut STEPS=4 NLAUNCH=100 timeout 1500 bash tools/gpu_profile.sh
CFG=large KERNEL=k_grad_wide TAG=large STEPS=4 NLAUNCH=200 timeout 1500 bash tools/gpu_profile.sh
