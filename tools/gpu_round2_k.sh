mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -x -p no:warnings --durations=5 > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
for c in medium megascale paper_tmd; do
  timeout 900 python bench.py --config $c --steps 200 --warmup 5 --no-cpu --no-ttt > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err
  QDT_PDL=0 timeout 900 python bench.py --config $c --steps 200 --warmup 5 --no-cpu --no-ttt --no-e2e > gpurun_out/bench_${c}_nopdl.json 2> gpurun_out/bench_${c}_nopdl.err
done
