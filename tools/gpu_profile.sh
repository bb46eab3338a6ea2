# ncu pass of one bench configuration (run under gpurun after the same command exited 0 alone):
# launch list (gpu__time_duration per launch) + one `--set full` capture of kernel $KERNEL.
#   CFG (default megascale), KERNEL (regex, default k_bwd_mma), TAG (output prefix)
mkdir -p gpurun_out
CFG=${CFG:-megascale}; KERNEL=${KERNEL:-k_bwd_mma}; TAG=${TAG:-$CFG}
CMD="python bench.py --config $CFG --steps ${STEPS:-4} --warmup 3 --no-cpu --no-e2e --no-ttt"
timeout 600 $CMD > gpurun_out/${TAG}_alone.log 2>&1 || { echo "bench failed" >> gpurun_out/${TAG}_alone.log; exit 1; }
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c ${NLAUNCH:-400} --csv \
  --log-file gpurun_out/${TAG}_launches.csv $CMD > gpurun_out/${TAG}_ncu_list.log 2>&1
timeout 1200 ncu -f --set full --clock-control none --import-source on -k regex:$KERNEL -s ${SKIP:-4} -c 1 \
  -o /tmp/prof_$TAG $CMD > gpurun_out/${TAG}_ncu.log 2>&1; echo "ncu rc=$?" >> gpurun_out/${TAG}_ncu.log
ncu -i /tmp/prof_$TAG.ncu-rep --page raw --csv > gpurun_out/${TAG}_raw.csv 2>&1
ncu -i /tmp/prof_$TAG.ncu-rep --page details --csv > gpurun_out/${TAG}_details.csv 2>&1
