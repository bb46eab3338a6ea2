mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_round2.py tests/test_gpu_parity.py -q -x -p no:warnings -k "bb" > gpurun_out/bb.log 2>&1; echo "rc=$?" >> gpurun_out/bb.log
timeout 2400 python -m pytest tests -m gpu -q -p no:warnings --durations=5 --deselect tests/test_gpu_round2.py::test_large_200_iterations > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
for c in large stress_cut; do
QDT_WIDE=new timeout 900 python bench.py --config $c --steps 100 --warmup 3 --no-cpu --no-ttt --no-e2e > gpurun_out/benchnew_$c.json 2> gpurun_out/benchnew_$c.err
done
