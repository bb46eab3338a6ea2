mkdir -p gpurun_out
rm -f gpurun_out/ab_wide.jsonl
timeout 300 python tools/ab_config.py stress_cut 16,100 cut_tkhoist >> gpurun_out/ab_wide.jsonl 2>>gpurun_out/ab_err.log
QDT_WIDE=new timeout 300 python tools/ab_config.py large 16,100 large_wstep_tkhoist >> gpurun_out/ab_wide.jsonl 2>>gpurun_out/ab_err.log
timeout 1200 python -m pytest tests/test_gpu_wide.py -x -q -p no:warnings > gpurun_out/pytest_wide.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_wide.log
