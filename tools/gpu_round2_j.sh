mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_round2.py -q -x -p no:warnings -k "tiny or early or edge or shape or resume or banded or binding" > gpurun_out/tiny_tests.log 2>&1; echo "rc=$?" >> gpurun_out/tiny_tests.log
for c in tiny megascale; do
  timeout 900 python bench.py --config $c --steps 200 --warmup 5 --no-cpu --no-ttt > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err
done
