mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; echo "rc=$?" >> gpurun_out/bench_default.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_reference.json 2> gpurun_out/bench_reference.err
for c in tiny medium large stress_cut paper_tmd; do
  timeout 900 python bench.py --config $c --steps 200 --warmup 5 --no-cpu --no-ttt > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err
done
timeout 1500 python bench.py --config stress --steps 200 --warmup 3 --no-cpu --no-ttt > gpurun_out/bench_stress.json 2> gpurun_out/bench_stress.err
