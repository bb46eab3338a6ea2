mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_wide.py tests/test_gpu_virtual.py -q -x -p no:warnings > gpurun_out/wide.log 2>&1; echo "rc=$?" >> gpurun_out/wide.log
for c in stress_cut stress; do
QDT_WIDE=new QDT_LIB=paper_2404_02844_b200/libqdt_wprof.so timeout 900 python bench.py --config $c --steps 16 --warmup 3 --no-cpu --no-ttt --no-e2e > gpurun_out/wprof_$c.json 2> gpurun_out/wprof_$c.err
done
timeout 900 python bench.py --config stress --steps 20 --warmup 3 --no-cpu --no-ttt --no-e2e > gpurun_out/bench_stress.json 2> gpurun_out/bench_stress.err
