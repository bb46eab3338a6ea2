# A/B of the integer-key bounds in the fused wide step (build_variant library wik), run under gpurun;
# also re-checks the NB >= 17 sweep epilogue (key identities) at the default library.
mkdir -p gpurun_out/ab3
O=gpurun_out/ab3
P=$PWD/paper_2404_02844_b200
for rep in 1 2; do
for v in base wik; do
  L=$P/libqdt_$v.so; [ $v = base ] && L=$P/libqdt.so
  QDT_LIB=$L timeout 600 python tools/ab_config.py stress_cut 16,64 $v >> $O/ab_stress_cut.jsonl 2>> $O/ab.err
  QDT_LIB=$L AB_ACCEL=1 timeout 600 python tools/ab_config.py stress_cut 16,64 fista_$v >> $O/ab_stress_cut.jsonl 2>> $O/ab.err
done
done
QDT_LIB=$P/libqdt_wik.so timeout 1500 python -m pytest tests/test_gpu_wide.py tests/test_gpu_virtual.py tests/test_gpu_parity.py -m gpu -q -x -p no:warnings -k "wide or stress or virtual or shape" > $O/pytest_wik.log 2>&1
timeout 900 python -m pytest tests -m gpu -q -x -p no:warnings -k "paper_tmd or odd or long_axis or fista_sweep or one_step or projection" > $O/pytest_main_nb17.log 2>&1
QDT_LIB=$P/libqdt_wik.so timeout 900 python bench.py --config stress --steps 8 --warmup 3 --no-cpu --no-ttt > $O/bench_stress_wik.json 2> $O/bench_stress_wik.err
