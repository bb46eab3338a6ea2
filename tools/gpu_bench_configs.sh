# bench lines of several configurations (run under gpurun): CONFIGS="large stress ..." STEPS=...
mkdir -p gpurun_out
for c in ${CONFIGS:-megascale large stress_cut paper_tmd stress}; do
  timeout ${BTIMEOUT:-900} python bench.py --config $c --steps ${STEPS:-200} --warmup 5 ${BARGS:---no-cpu --no-ttt} \
    > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; echo "rc=$?" >> gpurun_out/bench_$c.err
done
if [ -n "$TESTS" ]; then
  timeout 2400 python -m pytest $TESTS -q -p no:warnings --durations=10 > gpurun_out/pytest_extra.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_extra.log
fi
