# Final-state evidence of a round (run under gpurun): GPU tests, every bench line, the reference arm,
# ncu launch list + --set full captures (Megascale k_bwd_mma, Medium k_coop_solve, Tiny k_small_dense).
mkdir -p gpurun_out/final
O=gpurun_out/final
{ nproc; nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv; } > $O/host.txt 2>&1
timeout 300 python __graft_entry__.py smoke > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
timeout 900 python bench.py > $O/bench_megascale.json 2> $O/bench_megascale.err; echo "rc=$?" >> $O/bench_megascale.err
for c in tiny medium large stress_cut paper_tmd; do
  timeout 600 python bench.py --config $c --steps 200 --warmup 5 --no-cpu --no-ttt > $O/bench_$c.json 2> $O/bench_$c.err; echo "rc=$?" >> $O/bench_$c.err
done
timeout 900 python bench.py --config stress --steps 8 --warmup 3 --no-cpu --no-ttt > $O/bench_stress.json 2> $O/bench_stress.err; echo "rc=$?" >> $O/bench_stress.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > $O/bench_reference.json 2> $O/bench_reference.err; echo "rc=$?" >> $O/bench_reference.err
CMD="python bench.py --config megascale --steps 4 --warmup 3 --no-cpu --no-e2e --no-ttt"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/mega_launches.csv $CMD > $O/mega_ncu_list.log 2>&1
timeout 1200 ncu -f --set full --clock-control none --import-source on -k regex:k_bwd_mma -s 4 -c 1 -o /tmp/prof_mega $CMD > $O/mega_ncu.log 2>&1
ncu -i /tmp/prof_mega.ncu-rep --page details --csv > $O/mega_details.csv 2>&1
ncu -i /tmp/prof_mega.ncu-rep --page raw --csv > $O/mega_raw.csv 2>&1
python tools/ncu_details_summary.py $O/mega_details.csv > $O/ncu_mega_bwd_summary.txt 2>&1
CMDM="python tools/ab_config.py medium 50"
timeout 900 ncu -f --set full --clock-control none --import-source on -k regex:k_coop_solve -c 1 -o /tmp/prof_med $CMDM > $O/med_ncu.log 2>&1
ncu -i /tmp/prof_med.ncu-rep --page details --csv > $O/med_details.csv 2>&1
python tools/ncu_details_summary.py $O/med_details.csv > $O/ncu_medium_coop_summary.txt 2>&1
timeout 600 ncu -f --set full --clock-control none --import-source on -k regex:k_small_dense -c 1 -o /tmp/prof_tiny python tools/small_prof.py 200 > $O/tiny_ncu.log 2>&1
ncu -i /tmp/prof_tiny.ncu-rep --page details --csv > $O/tiny_details.csv 2>&1
python tools/ncu_details_summary.py $O/tiny_details.csv > $O/ncu_tiny_small_dense_summary.txt 2>&1
timeout 2400 python -m pytest tests -m gpu -q -p no:warnings --durations=10 > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
