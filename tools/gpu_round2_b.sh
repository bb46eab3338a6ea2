mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_wide.py tests/test_gpu_virtual.py -q -x -p no:warnings -k "not stress_shaped" > gpurun_out/wide.log 2>&1; echo "rc=$?" >> gpurun_out/wide.log
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_round2.py -q -x -p no:warnings -k "wide or odd or shape or paper_tmd or stress_cut or large or banded or resume" > gpurun_out/wide2.log 2>&1; echo "rc=$?" >> gpurun_out/wide2.log
for c in stress_cut large; do
timeout 900 python bench.py --config $c --steps 100 --warmup 3 --no-cpu --no-ttt --no-e2e > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; echo "rc=$?" >> gpurun_out/bench_$c.err
done
timeout 900 python bench.py --config stress --steps 20 --warmup 3 --no-cpu --no-ttt --no-e2e > gpurun_out/bench_stress.json 2> gpurun_out/bench_stress.err; echo "rc=$?" >> gpurun_out/bench_stress.err
