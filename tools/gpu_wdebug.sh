mkdir -p gpurun_out
for c in stress_cut large stress; do
QDT_WDEBUG=1 timeout 900 python bench.py --config $c --steps 16 --warmup 3 --no-cpu --no-ttt --no-e2e > gpurun_out/wdbg_$c.json 2> gpurun_out/wdbg_$c.err
done
CFG=stress_cut KERNEL=k_wstep TAG=wstep_cut2 STEPS=4 NLAUNCH=100 timeout 1500 bash tools/gpu_profile.sh
ncu -i /tmp/prof_wstep_cut2.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/wstep_cut2_source.csv 2>&1
