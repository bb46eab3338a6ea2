# compute-sanitizer memcheck / racecheck / synccheck over tools/sanitize_cases.py (run under gpurun)
mkdir -p gpurun_out/sanitize
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for tool in memcheck racecheck synccheck; do
  for c in tiny_sweep tiny_fista tiny_small tiny_bbls medium_split wide_two_kernel wide_fused; do
    timeout 900 compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize_cases.py $c \
      > gpurun_out/sanitize/${tool}_$c.log 2>&1; echo "rc=$?" >> gpurun_out/sanitize/${tool}_$c.log
  done
done
grep -H "ERROR SUMMARY\|RACECHECK SUMMARY\|rc=" gpurun_out/sanitize/*.log > gpurun_out/sanitize/summary.txt
